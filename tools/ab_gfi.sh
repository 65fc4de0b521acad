# A/B of the cfg-5 gfi step (and pass 1 alone) for the regular build vs abtest/*
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
for r in 1 2; do for lib in paper_2302_00942_b200/lib/librfd.so abtest/*/librfd.so; do echo $lib; timeout 300 python tools/gfi_timing.py $lib | tail -1; done; done
bash tools/ab_run.sh 2>&1 | grep -o "^[^ ]*\|'rfd_pass1_tc': [0-9.]*\|'rfd_core_dgemm': [0-9.]*" | paste - - -
