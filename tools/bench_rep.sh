# The bench step (no side legs) several times on one box: run-to-run spread.
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
for i in 1 2 3 4 5; do
timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-configs --no-parity 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step ms', round(j['ms_per_step'],4), 'integrate', round(j['integrate']['ms_per_call'],4), 'frac', round(j['roofline']['frac'],4))"
done
