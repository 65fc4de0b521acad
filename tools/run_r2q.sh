python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 300 python tools/bary_fused_check.py 0.1 30
timeout 300 python tools/bary_fused_check.py 0.5 30
timeout 300 python tools/bary_fused_check.py 0.1 16
