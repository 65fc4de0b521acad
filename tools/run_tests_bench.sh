# GPU suite + full default bench (parity, eps-graph, cpu baseline, e2e).
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -s -k "config_parity" > gpurun_out/quick_parity.log 2>&1; rc=$?; echo quick rc $rc
if [ $rc -ne 0 ]; then tail -30 gpurun_out/quick_parity.log; exit 1; fi
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv 2>&1 &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
kill $SMI
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -15; grep -E "sharded|barycenter" gpurun_out/gpu_tests.log | head -20; tail -c 600 gpurun_out/bench.log
