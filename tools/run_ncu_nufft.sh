#!/bin/bash
# Spread-grid Gram kernels (k_nufft.cu): timings, then one ncu --set full of
# the spread kernel.  Writes gpurun_out/nufft_*.
set -x
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python tools/nufft_check.py 262144 > gpurun_out/nufft_check.log 2>&1
timeout 300 python tools/profile_step.py > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nufft_spread -c 1 \
  -o gpurun_out/nufft_spread -f python tools/profile_step.py > gpurun_out/nufft_ncu.log 2>&1
ncu -i gpurun_out/nufft_spread.ncu-rep --page details --csv > gpurun_out/nufft_spread_details.csv 2>/dev/null
ncu -i gpurun_out/nufft_spread.ncu-rep --page source --csv > gpurun_out/nufft_spread_source.csv 2>/dev/null
tail -25 gpurun_out/nufft_check.log
