timeout 900 python -X faulthandler -m pytest tests/test_gpu_parity.py -q -s -x > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_tc.log 2>&1; echo bench rc $?
C="python tools/profile_step.py"
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_tc_kernel" -c 1 -o gpurun_out/tc $C > gpurun_out/ncu_tc.log 2>&1; echo ncu rc $?
