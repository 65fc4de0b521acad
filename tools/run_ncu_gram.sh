# ncu --set full of the Gram kernel (one cfg-5 plan + integrate).
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
C="python tools/profile_step.py"
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${1:-gram_tc_kernel}" -c 1 -o gpurun_out/${2:-gram} $C > gpurun_out/ncu_gram.log 2>&1; echo ncu rc $?
tail -5 gpurun_out/ncu_gram.log
