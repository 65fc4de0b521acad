python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
for i in 1 2 3 4; do
timeout 900 python bench.py --no-cpu-baseline --no-configs --no-parity --no-e2e --step-times > gpurun_out/bt_$i.log 2>&1
grep '^{' gpurun_out/bt_$i.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('run', $i, j['ms_per_step'], j['integrate']['ms_per_call'])"
grep "step ms" gpurun_out/bt_$i.log
done
