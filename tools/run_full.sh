# Full round measurement: GPU tests, smoke, default bench (cpu_baseline + e2e +
# parity), reference arm, ncu launch list of the bench command, ncu --set full
# of the top kernels (cfg 5 step: spread, grid Gram, passes; the narrow-field kernel at cfg 4; the fused
# barycenter), source-level stall summaries.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/gpu_tests.log 2>&1; echo tests rc $?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv 2>&1 &
SMI=$!
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
kill $SMI
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc $?
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-configs --no-parity"
timeout 600 $C > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launches.log 2>&1; echo launches rc $?
C2="python tools/profile_step.py"
timeout 300 $C2 > gpurun_out/plain2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"nufft_spread|gram_pair_kernel|pass1_tc|pass2_tc" -c 4 -o gpurun_out/full $C2 > gpurun_out/ncu_full.log 2>&1; echo full rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"dgemm" -c 1 -o gpurun_out/full2 $C2 > gpurun_out/ncu_full2.log 2>&1; echo full2 rc $?
C3="python tools/profile_step.py --cfg 4"
timeout 300 $C3 > gpurun_out/plain3.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"integrate_small" -c 1 -o gpurun_out/full3 $C3 > gpurun_out/ncu_full3.log 2>&1; echo full3 rc $?
C4="python tools/bary_fused_check.py 0.5 30"
timeout 300 $C4 > gpurun_out/plain4.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bary_fused" -c 1 -o gpurun_out/full4 $C4 > gpurun_out/ncu_full4.log 2>&1; echo full4 rc $?
for f in full full2 full3 full4; do [ -f gpurun_out/$f.ncu-rep ] && python tools/ncu_lines.py gpurun_out/$f.ncu-rep 30 > gpurun_out/${f}_lines.txt 2>&1; done
