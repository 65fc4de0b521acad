python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity or narrow or batched or graph or spectrum_batched or back_to_back" 2>&1 | tail -2
timeout 300 python tools/graph_small.py
