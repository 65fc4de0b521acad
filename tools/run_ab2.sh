mkdir -p gpurun_out
python -c "from paper_2302_00942_b200 import build; build.build()" > gpurun_out/build.log 2>&1
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity or ragged" > gpurun_out/quick.log 2>&1; echo quick rc $?
RFD_P2_PW=8 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config_parity or ragged or multi_column or batched" > gpurun_out/quick8.log 2>&1; echo quick8 rc $?
for i in 1 2 3; do
  timeout 120 python tools/ab_time.py --reps 10 > gpurun_out/ab_new_$i.json 2>&1
  RFD_P2_PW=8 timeout 120 python tools/ab_time.py --reps 10 > gpurun_out/ab_pw8_$i.json 2>&1
  timeout 120 python tools/ab_time.py --reps 10 --lib abtest/librfd_old.so > gpurun_out/ab_old_$i.json 2>&1
done
for c in 3 4; do
  timeout 120 python tools/ab_time.py --reps 20 --cfg $c --integrates 5 > gpurun_out/ab_c${c}_16.json 2>&1
  RFD_P2_PW=8 timeout 120 python tools/ab_time.py --reps 20 --cfg $c --integrates 5 > gpurun_out/ab_c${c}_8.json 2>&1
done
tail -3 gpurun_out/quick.log gpurun_out/quick8.log
for f in gpurun_out/ab_*.json; do echo $f; python -c "
import json,sys; j=json.loads(open('$f').read().strip().split('\n')[-1]); print({k: round(v,4) for k,v in j['ms'].items() if k in ('rfd_gram_tc','rfd_pass1_tc','rfd_pass2_tc','rfd_bbox','rfd_pack_points')})"; done
