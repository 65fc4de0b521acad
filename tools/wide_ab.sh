# Narrow kernel CTA size A/B: abtest/old vs abtest/new (graph timings, cfg-5 points by d), then GPU tests.
for r in 1 2; do for v in old new; do
  echo "== $v"; python tools/graph_small.py abtest/$v/librfd.so 2>&1 | tail -4
  python tools/cfg4_paths.py 5 abtest/$v/librfd.so 2>&1 | tail -6 | head -3
done; done
RFD_SMALL_TRACE=1 python tools/small_trace.py 4 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
