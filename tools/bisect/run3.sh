for v in old new old new; do
  cp tools/bisect/p1_$v.cu paper_2302_00942_b200/csrc/k_pass1_tc.cu
  python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build_$v.log 2>&1 || { echo build $v failed; continue; }
  echo "$v: $(timeout 120 python tools/profile_wide.py 16 20 | grep pass1)"
done
