# Quick GPU check: small parity first (short timeout: a hang dies fast), then the
# full GPU suite, then a short bench (no cpu baseline / e2e).
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -s -k "config_parity" > gpurun_out/quick_parity.log 2>&1; rc=$?; echo quick rc $rc
if [ $rc -ne 0 ]; then tail -30 gpurun_out/quick_parity.log; exit 1; fi
timeout 900 python -m pytest tests -m gpu -x -q -s > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/bench.log 2>&1; echo bench rc $?
tail -3 gpurun_out/gpu_tests.log; tail -c 3000 gpurun_out/bench.log
