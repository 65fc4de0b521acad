# A/B of an env-selected kernel variant: parity (config tests) + short bench per value.
#   bash tools/run_ab.sh VAR "v1 v2 ..."
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
for v in $2; do
  export $1=$v
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity or ragged or column" > gpurun_out/ab_tests_$v.log 2>&1; echo "$1=$v tests rc $?"; tail -1 gpurun_out/ab_tests_$v.log
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/ab_bench_$v.log 2>&1; echo "$1=$v bench rc $?"
  python - "$v" <<'PY'
import json, sys
line = [l for l in open("gpurun_out/ab_bench_%s.log" % sys.argv[1]) if l.startswith("{")][-1]
b = json.loads(line)
print("  step ms %.3f" % b["ms_per_step"], "integrate ms %.3f" % b["integrate"]["ms_per_call"],
      {k: round(v["ms_per_launch"], 4) for k, v in b["kernels"].items() if v["ms_per_launch"] > 0.05})
PY
done
