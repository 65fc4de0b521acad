# Bench line (default args) + ncu launch list of a short bench, round-1 artefacts.
mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/clocks.csv 2>&1 &
SMI=$!
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc $?
kill $SMI
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launches.log 2>&1; echo launches rc $?
tail -c 2500 gpurun_out/bench.log
