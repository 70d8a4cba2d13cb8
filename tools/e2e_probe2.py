"""Per-step e2e timings, pipelined (download_async) vs synchronous (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200.api import CsrMatrix
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ah = S.config_matrices(cfg)[0]
pr = torch.from_numpy(ah.rpt).pin_memory(); pc = torch.from_numpy(ah.col).pin_memory(); pv = torch.from_numpy(ah.val).pin_memory()
a = CsrMatrix(ah.rows, ah.cols, pr.numpy(), pc.numpy(), pv.numpy())
p = sg.SpgemmPipeline(a, a); dm, o = p.run_device(); p.close(); nnz = dm.nnz; dm.free()
orr = torch.empty(a.rows + 1, dtype=torch.int64).pin_memory(); oc = torch.empty(nnz, dtype=torch.int32).pin_memory(); ov = torch.empty(nnz, dtype=torch.float64).pin_memory()
ctx = sg.get_context()
T = time.perf_counter
for mode in ("sync", "async", "sync", "async"):
    ts = []
    t00 = T()
    for it in range(8):
        t0 = T()
        p = sg.SpgemmPipeline(a, a); dm, o = p.run_device(); p.close()
        if mode == "async":
            dm.download_async(orr.numpy(), oc.numpy(), ov.numpy(), release=True)
        else:
            dm.download_into(orr.numpy(), oc.numpy(), ov.numpy())
        dm.free()
        ts.append(round(1e3 * (T() - t0), 2))
    ctx.wait_downloads(); torch.cuda.synchronize()
    tot = 1e3 * (T() - t00) / 8
    print(mode, ts, "mean incl. wait %.2f ms" % tot, "pool", [x >> 20 for x in ctx.pool_stats()])
