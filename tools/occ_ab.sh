# Narrow kernel: CTAs per SM (RFD_SMALL_OCC) vs cfg 1-4 graph timings and the cfg-4 trace.
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
for o in 0 1 2 3; do
  echo "occ $o"
  if [ $o = 0 ]; then unset RFD_SMALL_OCC; else export RFD_SMALL_OCC=$o; fi
  python tools/graph_small.py 2>&1 | tail -4
  RFD_SMALL_TRACE=1 python tools/small_trace.py 4 2>&1 | tail -1
done
