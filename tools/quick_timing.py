"""Quick device-resident timing of multiply on configs 1/2/4 (dev aid, not the bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S

cfgs = [int(x) for x in sys.argv[1:]] or [1, 2]
for cfg in cfgs:
    mats = S.config_matrices(cfg)
    a = mats[0].to_device(); b = mats[1].to_device()
    for i in range(3):
        dm, out = sg.multiply_device(a, b); dm.free()
    torch.cuda.synchronize()
    ts = []
    for i in range(5):
        t0 = time.perf_counter()
        dm, out = sg.multiply_device(a, b)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0); dm.free()
    t = min(ts)
    print(f"  runs ms: {[round(x*1e3, 3) for x in ts]}")
    print(f"cfg{cfg}: wall {t*1e3:.3f} ms  GFLOPS {2*out.stats.total_nprod/t/1e9:.1f}  steps(ms) " +
          " ".join(f"{k}={getattr(out.timings,k)*1e3:.3f}" for k in ("setup","sym_binning","symbolic","num_binning","rpt_alloc","numeric")), flush=True)
