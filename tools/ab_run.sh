# A/B: per-kernel times of the regular build vs abtest variants (alternating, 2 rounds each)
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
for r in 1 2; do
  for lib in paper_2302_00942_b200/lib/librfd.so abtest/*/librfd.so; do
    timeout 300 python tools/ab_time.py --lib $lib --reps 10 --integrates 3 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); print(j['lib'], {k: round(v, 4) for k, v in j['ms'].items() if v > 0.015})"
  done
done
