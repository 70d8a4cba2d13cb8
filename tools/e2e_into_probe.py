"""multiply_into (row blocks, overlapped downloads) vs separate calls, interleaved
rounds, median ms per call (diagnostic)."""
import os, sys, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200.api import CsrMatrix
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
h = S.config_matrices(cfg)[0]
pin = lambda x: torch.from_numpy(x).pin_memory()
pr, pc, pv = pin(h.rpt), pin(h.col), pin(h.val)
a = CsrMatrix(h.rows, h.cols, pr.numpy(), pc.numpy(), pv.numpy())
nnz = sg.forecast_nnz(a, a, per_row=False).total_nnz
orpt = torch.empty(a.rows + 1, dtype=torch.int64).pin_memory()
ocol = torch.empty(nnz, dtype=torch.int32).pin_memory()
oval = torch.empty(nnz, dtype=torch.float64).pin_memory()
def separate():
    p = sg.SpgemmPipeline(a, a); dm, out = p.run_device(); p.close()
    dm.download_into(orpt.numpy(), ocol.numpy(), oval.numpy()); dm.free()
def into(parts):
    return lambda: sg.multiply_into(a, a, orpt.numpy(), ocol.numpy(), oval.numpy(), parts=parts)
if os.environ.get("PRE_DEVICE"):
    d = h.to_device()
    for _ in range(20):
        dm, out = sg.multiply_device(d, d); dm.free()
    torch.cuda.synchronize()
    print("pool after device runs:", sg.get_context().pool_stats())
modes = {"separate": separate, "into1": into(1), "into2": into(2), "into4": into(4), "into8": into(8)}
res = {k: [] for k in modes}
for f in modes.values():
    f(); f()
for r in range(4):
    for k, f in modes.items():
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter(); f(); res[k].append((time.perf_counter() - t0) * 1e3)
print("pool:", sg.get_context().pool_stats())
for k, v in res.items():
    print(f"{k:9s} median {statistics.median(v):7.2f} ms  min {min(v):7.2f}  max {max(v):7.2f}")
for name, f in (("into8 back-to-back", into(8)), ("separate back-to-back", separate), ("into8 b2b again", into(8))):
    for _ in range(3):
        f()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(12):
        f()
    torch.cuda.synchronize(); print(f"{name}: {(time.perf_counter() - t0) / 12 * 1e3:.2f} ms/call")
