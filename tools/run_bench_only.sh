mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv 2>&1 &
SMI=$!
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
kill $SMI
tail -c 400 gpurun_out/bench.log
