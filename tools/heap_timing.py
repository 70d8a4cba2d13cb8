"""Config-3 style timing of the numeric heap tier: deterministic (ordered) vs
deterministic=False (fp64 atomics). Dev aid, not the bench."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
a = S.rmat(scale, 16, seed=scale).to_device()
for det in (False, True):
    o = sg.SpgemmOptions(deterministic=det)
    dm, out = sg.multiply_device(a, a, options=o); dm.free()
    torch.cuda.synchronize()
    ts = []
    for i in range(2):
        t0 = time.perf_counter()
        dm, out = sg.multiply_device(a, a, options=o)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0); dm.free()
    t = min(ts)
    print(f"rmat{scale} deterministic={det}: {t*1e3:.1f} ms GFLOPS {2*out.stats.total_nprod/t/1e9:.1f} " +
          " ".join(f"{k}={getattr(out.timings,k)*1e3:.2f}" for k in ("setup","symbolic","numeric")), flush=True)
