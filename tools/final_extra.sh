# Extra evidence after the full run: the new GPU tests and a step timeline.
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -k "overflow or bounding_box or scan_variants or gfi_one_shot" 2>&1 | tail -3
python tools/gfi_timeline.py > /dev/null 2>&1; cp gpurun_out/timeline.txt gpurun_out/timeline_final.txt; tail -40 gpurun_out/timeline_final.txt | head -5
