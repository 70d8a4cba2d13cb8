"""Break down the synchronous e2e step of config 2 (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200.api import CsrMatrix
ah = S.config_matrices(2)[0]
pr = torch.from_numpy(ah.rpt).pin_memory(); pc = torch.from_numpy(ah.col).pin_memory(); pv = torch.from_numpy(ah.val).pin_memory()
a = CsrMatrix(ah.rows, ah.cols, pr.numpy(), pc.numpy(), pv.numpy())
p = sg.SpgemmPipeline(a, a); dm, o = p.run_device(); p.close(); nnz = dm.nnz; dm.free()
orr = torch.empty(a.rows + 1, dtype=torch.int64).pin_memory(); oc = torch.empty(nnz, dtype=torch.int32).pin_memory(); ov = torch.empty(nnz, dtype=torch.float64).pin_memory()
T = time.perf_counter
for it in range(10):
    t0 = T(); p = sg.SpgemmPipeline(a, a); t1 = T(); dm, o = p.run_device(); p.close(); t2 = T()
    dm.download_into(orr.numpy(), oc.numpy(), ov.numpy()); t3 = T(); dm.free(); torch.cuda.synchronize(); t4 = T()
    print(f"create {1e3*(t1-t0):.1f} run {1e3*(t2-t1):.1f} d2h {1e3*(t3-t2):.1f} ({3.07/(t3-t2):.1f} GB/s) free {1e3*(t4-t3):.1f}")
