"""Host time per pipeline call in a back-to-back loop (diagnostic)."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
mats = [m.to_device() for m in S.config_matrices(int(sys.argv[1]) if len(sys.argv) > 1 else 2)]
acc = collections.defaultdict(float)
def step():
    t = time.perf_counter
    t0 = t(); p = sg.SpgemmPipeline(mats[0], mats[1]); t1 = t(); acc["create"] += t1 - t0
    for name in ("setup", "symbolic_binning", "run_symbolic", "numeric_binning", "finalize_rpt", "run_numeric"):
        a = t(); getattr(p, name)(); acc[name] += t() - a
    a = t(); rep = p._finish_report(); acc["finish"] += t() - a
    a = t(); dm = p._take(); p.close(); dm.free(); acc["close+free"] += t() - a
for _ in range(3): step()
acc.clear()
n = 20
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(n): step()
torch.cuda.synchronize(); tot = (time.perf_counter() - t0) / n * 1e3
print(f"per step {tot:.3f} ms: " + " ".join(f"{k}={v / n * 1e3:.3f}" for k, v in acc.items()))
