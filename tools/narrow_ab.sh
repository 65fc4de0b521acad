python -c "from paper_2302_00942_b200 import build; build.build()" >/dev/null 2>&1
for c in 1 2 4 3; do
  for nv in 1 0; do
    echo "cfg $c RFD_NARROW=$nv"; RFD_NARROW=$nv timeout 300 python tools/cfg4_paths.py $c 2>&1 | grep "^d=[134]:"
  done
done
