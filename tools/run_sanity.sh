# Session-start check on a fresh box: build, GPU tests, smoke, default bench.
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
tail -c 600 gpurun_out/bench.log
