"""Minimal driver for ncu: N device-resident multiplies of one config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mats = [m.to_device() for m in S.config_matrices(cfg)]
for _ in range(reps):
    if cfg == 4:
        a, p, r = mats
        dm, _ = sg.multiply_device(a, p)
        dm.free()
    else:
        dm, _ = sg.multiply_device(mats[0], mats[1])
        dm.free()
torch.cuda.synchronize()
print("done")
