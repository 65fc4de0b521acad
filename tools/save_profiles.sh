# Copy the judged evidence of a tools/run_full.sh run into profiles/ under a tag.
#   bash tools/save_profiles.sh r02_xxx
T=$1
grep '^{' gpurun_out/bench.log | tail -1 > profiles/${T}_bench.json
grep '^{' gpurun_out/bench_ref.log | tail -1 > profiles/${T}_bench_reference.json
cp gpurun_out/gpu_tests.log profiles/${T}_gpu_tests.txt
cp gpurun_out/smoke.log profiles/${T}_smoke.txt
cp gpurun_out/launches.csv profiles/${T}_launches.csv
python tools/ncu_launches.py gpurun_out/launches.csv > profiles/${T}_launches.txt
{ echo "# ncu --set full --clock-control none: tools/profile_step.py (cfg5 plan + integrate), tools/profile_step.py --cfg 4 (narrow-field kernel), tools/bary_fused_check.py (fused barycenter); tag $T"
  for f in full full2 full3 full4; do [ -f gpurun_out/$f.ncu-rep ] && python tools/ncu_summary.py gpurun_out/$f.ncu-rep; done; } > profiles/${T}_ncu_full.txt
{ for f in full full2 full3 full4; do [ -f gpurun_out/${f}_lines.txt ] && { echo "## $f"; cat gpurun_out/${f}_lines.txt; }; done; } > profiles/${T}_ncu_source_lines.txt
python tools/ncu_traffic.py gpurun_out/full.ncu-rep $( [ -f gpurun_out/full2.ncu-rep ] && echo gpurun_out/full2.ncu-rep ) > profiles/traffic.json
cp profiles/traffic.json profiles/${T}_traffic.json
python tools/sass_histogram.py > profiles/${T}_sass_histogram.txt
