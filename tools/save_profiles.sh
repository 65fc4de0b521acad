# Copy the judged evidence of a tools/run_full.sh run into profiles/ under a tag.
#   bash tools/save_profiles.sh r01_xxx
T=$1
grep '^{' gpurun_out/bench.log | tail -1 > profiles/${T}_bench.json
grep '^{' gpurun_out/bench_ref.log | tail -1 > profiles/${T}_bench_reference.json
tail -3 gpurun_out/gpu_tests.log > profiles/${T}_gpu_tests.txt
cp gpurun_out/smoke.log profiles/${T}_smoke.txt
cp gpurun_out/launches.csv profiles/${T}_launches.csv
python tools/ncu_launches.py gpurun_out/launches.csv > profiles/${T}_launches.txt
{ echo "# ncu --set full --clock-control none, tools/profile_step.py (cfg5 plan + integrate), tag $T"; python tools/ncu_summary.py gpurun_out/full.ncu-rep; [ -f gpurun_out/full2.ncu-rep ] && python tools/ncu_summary.py gpurun_out/full2.ncu-rep; } > profiles/${T}_ncu_full.txt
python tools/ncu_traffic.py gpurun_out/full.ncu-rep $( [ -f gpurun_out/full2.ncu-rep ] && echo gpurun_out/full2.ncu-rep ) > profiles/traffic.json
cp profiles/traffic.json profiles/${T}_traffic.json
