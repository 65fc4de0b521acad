# Round-2 first check: build, quick parity, full GPU suite, barycenter trace,
# short bench.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -s -k "config_parity" > gpurun_out/quick_parity.log 2>&1; rc=$?; echo quick rc $rc
if [ $rc -ne 0 ]; then tail -30 gpurun_out/quick_parity.log; exit 1; fi
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
timeout 300 python tools/bary_trace.py > gpurun_out/bary_trace.log 2>&1; echo trace rc $?
timeout 300 python tools/bary_trace.py --floor 0.2 > gpurun_out/bary_trace_floor.log 2>&1; echo trace2 rc $?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo bench rc $?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -15; cat gpurun_out/bary_trace.log | tail -12; tail -c 1500 gpurun_out/bench.log
