python -c "from paper_2302_00942_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python -c "
import sys, os; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2302_00942_b200 import rfd
from workloads import barycenter_inputs
xb, ab, musb = barycenter_inputs(18944)
pb = rfd.Plan(torch.from_numpy(xb).cuda(), 0.01, 0.5, 30, 5)
mb = torch.from_numpy(musb.astype(np.float32)).cuda(); abd = torch.from_numpy(ab.astype(np.float32)).cuda()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for mode in ('1', '0'):
    os.environ['RFD_BARY_FUSED'] = mode
    ts = []
    for it in (2, 22):
        pb.barycenter(mb, abd, [1/3]*3, it); torch.cuda.synchronize()
        e0.record(); pb.barycenter(mb, abd, [1/3]*3, it); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print('fused' if mode == '1' else 'unfused', 'ms/iter %.4f' % ((ts[1]-ts[0])/20), 'total 22 it %.3f ms' % ts[1])
"
