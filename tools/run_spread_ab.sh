python -c "from paper_2302_00942_b200 import build; build.build()" >/dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -m gpu -s -k "spread or gfi or degenerate or config5 or determin" 2>&1 | grep -E "passed|failed|FAILED|spread|G'|Error" | head -30
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash tools/ab_run.sh 2>&1 | grep -o "^[^ ]*\|'rfd_nufft_spread': [0-9.]*" | paste - -
