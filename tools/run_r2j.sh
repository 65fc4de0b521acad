python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 120 python tools/trace_small.py 2>&1 | grep -E "small|last|phase-1 end" | tail -12
