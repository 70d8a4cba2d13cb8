"""Per-call latency of multiply_device on tiny and config-1 inputs, with a cProfile
split of the Python side (diagnostic)."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
tiny = S.poisson2d_5pt(8).to_device()
c1 = S.poisson2d_5pt(1024).to_device()
def loop(m, k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        dm, out = sg.multiply_device(m, m); dm.free()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
for m, name in ((tiny, "tiny 64 rows"), (c1, "config 1")):
    loop(m, 5)
    print(f"{name}: {loop(m, 50):.3f} ms/call")
pr = cProfile.Profile(); pr.enable(); loop(tiny, 200); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(14); print(s.getvalue()[:3500])
