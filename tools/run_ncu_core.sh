#!/bin/bash
# Core GEMM (k_core.cu): one ncu --set full capture of a doubling-step launch.
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 300 python tools/profile_step.py > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm -s 10 -c 1 \
  -o gpurun_out/core_gemm -f python tools/profile_step.py > gpurun_out/core_ncu.log 2>&1
ncu -i gpurun_out/core_gemm.ncu-rep --page details --csv > gpurun_out/core_gemm_details.csv 2>/dev/null
ncu -i gpurun_out/core_gemm.ncu-rep --page source --csv > gpurun_out/core_gemm_source.csv 2>/dev/null
tail -3 gpurun_out/core_ncu.log
