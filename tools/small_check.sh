# Narrow-kernel change check: GPU tests of the small configs, graph timings, cfg-4 trace.
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/small_tests.log 2>&1; echo tests rc $?
tail -2 gpurun_out/small_tests.log
python tools/graph_small.py 2>&1 | tail -4
RFD_SMALL_TRACE=1 python tools/small_trace.py 4 2>&1 | tail -1
