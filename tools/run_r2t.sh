python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity or reparam or nonsym or spectrum_matches" 2>&1 | tail -2
for i in 1 2; do timeout 120 python tools/ab_time.py --reps 10 2>&1 | tail -1 | grep -o '"rfd_core_[a-z]*": [0-9.]*'; done
