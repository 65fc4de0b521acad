# One ncu --set full capture of the spread kernel (cfg 5 step) -> gpurun_out/nufft_spread_imma.ncu-rep
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 300 python tools/profile_step.py > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:nufft_spread -c 1 -o gpurun_out/nufft_spread_imma -f python tools/profile_step.py > gpurun_out/nufft_ncu.log 2>&1; tail -1 gpurun_out/nufft_ncu.log
