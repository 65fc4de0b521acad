# Step-level change check: GPU tests, one gfi timeline, the bench step (no side legs).
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/step_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/step_tests.log
python tools/gfi_timeline.py 2>&1 | tail -40
for i in 1 2; do
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-configs --no-parity 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step ms', j['ms_per_step'], 'integrate', j['integrate']['ms_per_call'], 'frac', j['roofline']['frac'])"
done
