"""Numeric-phase time of one config under each numeric preset (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mats = S.config_matrices(cfg)
a = mats[0].to_device(); b = mats[1].to_device()
for num in sys.argv[2:] or ["num_2x", "num_1x"]:
    opts = sg.SpgemmOptions(num_preset=num)
    dm, out = sg.multiply_device(a, b, opts); dm.free()
    ts = []
    for _ in range(3):
        dm, out = sg.multiply_device(a, b, opts)
        torch.cuda.synchronize(); ts.append(out.timings.numeric); dm.free()
    print(f"cfg{cfg} {num}: numeric ms {[round(t * 1e3, 2) for t in ts]}", flush=True)
