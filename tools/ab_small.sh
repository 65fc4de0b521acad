# A/B of the narrow-field / small-config integrate (graph replay, cfgs 1-4) for the regular build vs abtest/*
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
for r in 1 2; do for lib in paper_2302_00942_b200/lib/librfd.so abtest/*/librfd.so; do echo $lib; timeout 300 python tools/graph_small.py $lib 2>&1 | tr '\n' ' '; echo; done; done
