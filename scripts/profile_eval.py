"""One warm-up + one profiled evaluation of a BASELINE config (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2412_04595_b200 import Plan
from synth import config_system, CONFIGS
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
n_eval = int(sys.argv[2]) if len(sys.argv) > 2 else 2
xyz, q, L = config_system(name)
pl = Plan(len(q), L, CONFIGS[name].tol, validate=False, window=os.environ.get("SOG_WINDOW", "gs"))
xd, qd = torch.from_numpy(xyz).cuda(), torch.from_numpy(q).cuda()
for _ in range(n_eval):
    pl.eval(xd, qd)
torch.cuda.synchronize()
print("ok", pl.describe()["Ix"])
