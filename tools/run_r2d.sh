mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -s -k "config_parity or narrow or batched or profiler" > gpurun_out/quick.log 2>&1; rc=$?; echo quick rc $rc
tail -15 gpurun_out/quick.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
timeout 900 python bench.py --no-cpu-baseline --no-parity > gpurun_out/bench.log 2>&1; echo bench rc $?
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests.log | tail -15
python - <<'PY'
import json
l = [x for x in open('gpurun_out/bench.log') if x.startswith('{')][-1]
j = json.loads(l)
for k, v in j['configs'].items(): print(k, {kk: round(vv, 3) if isinstance(vv, float) else vv for kk, vv in v.items()})
print(j['ms_per_step'], j['e2e']['ms_per_step'])
PY
