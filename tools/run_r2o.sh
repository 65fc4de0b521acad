mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "barycenter" 2>&1 | grep -E "barycenter|passed|failed|Error|assert" | tail -30
