"""Time the cfg-5 Gram kernel in its diagnostic modes (RFD_GRAM_MODE 0/1/2).

    python tools/gram_modes.py   (spawns one process per mode)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
from paper_2302_00942_b200 import rfd
from workloads import make_config
p, x, F = make_config(%d)
xd = torch.from_numpy(x).cuda()
lib = rfd.load_library()
for rep in range(4):
    rfd.profile_enable(True)
    try:
        plan = rfd.Plan(xd, p["eps"], p["lam"], p["m"], p["seed"])
        plan.close()
    except rfd.RFDError:
        pass  # diagnostic modes produce a meaningless G
    torch.cuda.synchronize()
    prof = rfd.profile_read()
print({k: v for k, v in prof.items() if "gram" in k})
'''
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for mode in [int(a) for a in (sys.argv[2].split(',') if len(sys.argv) > 2 else '0,1,2'.split(','))]:
    env = dict(os.environ, RFD_GRAM_MODE=str(mode))
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, cfg)], env=env, capture_output=True, text=True)
    print("mode", mode, r.stdout.strip()[-400:], r.stderr.strip()[-400:])
