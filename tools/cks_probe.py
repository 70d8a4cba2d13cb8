"""Time the device checksum of a large C (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
sc = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d = S.rmat(sc, 16, seed=sc).to_device()
dm, out = sg.multiply_device(d, d)
ctx = sg.get_context()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    v, h = dm.checksum(0, 0)
    print("checksum ms", round((time.perf_counter() - t0) * 1e3, 2), dm.nnz)
ctx.set_profiling(True); dm.checksum(0, 0); ctx.set_profiling(False); print(ctx.profile_summary())
dm.free()
