"""Per-run wall times of device-resident multiplies + pool stats (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gc
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mats = [m.to_device() for m in S.config_matrices(cfg)]
ctx = sg.get_context()
gc.disable() if "--nogc" in sys.argv else None
for i in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dm, out = sg.multiply_device(mats[0], mats[1])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dm.free()
    r, u = ctx.pool_stats()
    tm = out.timings
    print(f"{i:2d} {1e3*(t1-t0):8.3f} ms  reserved {r/1e9:6.2f} GB used {u/1e9:6.2f} GB  "
          + " ".join(f"{k}={getattr(tm,k)*1e3:.2f}" for k in ("setup","sym_binning","symbolic","num_binning","rpt_alloc","numeric")))
