for v in ${VARS:-1 2 3 4}; do
  cp tools/bisect/v$v.cu paper_2302_00942_b200/csrc/k_pass2_tc.cu
  python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build_$v.log 2>&1 || { echo build $v failed; continue; }
  echo "variant $v: $(timeout 300 python -m pytest tests/test_gpu_parity.py -q -k 'ragged' 2>&1 | tail -1)"
done
