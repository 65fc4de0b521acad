mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity or narrow or batched or graph or host" 2>&1 | tail -2
timeout 120 python tools/trace_small.py 2>&1 | grep "small" | sort -u | tail -8
for c in 1 2 4 3; do timeout 120 python tools/ab_time.py --reps 20 --cfg $c --integrates 10 2>&1 | tail -1 | grep -o '"rfd_integrate_small": [0-9.]*'; done
