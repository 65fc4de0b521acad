mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 120 python tools/ab_time.py --reps 10 > gpurun_out/ab_now.json 2>&1; echo ab rc $?
C="python tools/profile_step.py"
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pass1_tc|pass2_tc" -c 2 -o gpurun_out/passes $C > gpurun_out/ncu_passes.log 2>&1; echo ncu rc $?
python tools/ncu_lines.py gpurun_out/passes.ncu-rep 40 > gpurun_out/passes_lines.txt 2>&1
python tools/ncu_summary.py gpurun_out/passes.ncu-rep > gpurun_out/passes_summary.txt 2>&1
python tools/ncu_sass.py gpurun_out/passes.ncu-rep > gpurun_out/passes_sass.txt 2>&1
cat gpurun_out/ab_now.json; head -60 gpurun_out/passes_summary.txt
