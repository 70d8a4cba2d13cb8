"""One device-resident multiply of a named workload (profiling driver, not the bench).
  python tools/one_multiply.py rmat18 [det|nodet]   |  cfg1 / cfg2 / cfg3 / cfg4"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S

what = sys.argv[1]
det = (sys.argv[2] if len(sys.argv) > 2 else "det") == "det"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if what.startswith("rmat"):
    sc = int(what[4:])
    mats = [S.rmat(sc, 16, seed=sc)] * 2
else:
    mats = list(S.config_matrices(int(what[3:])))
dev = [m.to_device() for m in mats]
o = sg.SpgemmOptions(deterministic=det)
for _ in range(reps):
    if len(dev) == 3:
        a, p, r = dev
        dm1, _ = sg.multiply_device(a, p, options=o)
        dm1.free()
    else:
        dm, out = sg.multiply_device(dev[0], dev[1], options=o)
        dm.free()
torch.cuda.synchronize()
print("ok")
