# A/B of core-GEMM variants (tools/build_variant.py NAME FLAGS k_core.cu first):
# per-launch GEMM time and the cfg-5 gfi step, regular build vs abtest/*.
bash tools/ab_run.sh 2>&1 | grep -o "^[^ ]*\|'rfd_core_dgemm': [0-9.]*" | paste - -
for r in 1 2; do for lib in paper_2302_00942_b200/lib/librfd.so abtest/*/librfd.so; do echo $lib; timeout 300 python tools/gfi_timing.py $lib | tail -1; done; done
