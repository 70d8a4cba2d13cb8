"""Config 4 RAP chain step timing and pipelined-download probe (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200.api import CsrMatrix
a, p, r = [m.to_device() for m in S.config_matrices(4)]
T = time.perf_counter
def sync(): torch.cuda.synchronize()
class _V:
    def __init__(self, ptr, n, t): self.__cuda_array_interface__ = {"shape": (n,), "typestr": t, "data": (ptr, False), "version": 3}
for it in range(4):
    sync(); t0 = T()
    dm1, o1 = sg.multiply_device(a, p); sync(); t1 = T()
    ap = CsrMatrix(dm1.rows, dm1.cols, torch.as_tensor(_V(dm1.ptrs[0], dm1.rows + 1, "<i8"), device="cuda"),
                   torch.as_tensor(_V(dm1.ptrs[1], dm1.nnz, "<i4"), device="cuda"),
                   torch.as_tensor(_V(dm1.ptrs[2], dm1.nnz, "<f8"), device="cuda")); sync(); t2 = T()
    dm2, o2 = sg.multiply_device(r, ap); sync(); t3 = T()
    dm2.free(); dm1.free(); sync(); t4 = T()
    print(f"AP {1e3*(t1-t0):.2f} wrap {1e3*(t2-t1):.2f} RAP {1e3*(t3-t2):.2f} free {1e3*(t4-t3):.2f}", o2.timings.__dict__)
# pipelined download on config 1
a1 = S.config_matrices(1)[0]
pr = torch.from_numpy(a1.rpt).pin_memory(); pc = torch.from_numpy(a1.col).pin_memory(); pv = torch.from_numpy(a1.val).pin_memory()
ah = CsrMatrix(a1.rows, a1.cols, pr.numpy(), pc.numpy(), pv.numpy())
dm, o = sg.multiply_device(ah, ah); nnz = dm.nnz; dm.free()
orr = torch.empty(a1.rows + 1, dtype=torch.int64).pin_memory(); oc = torch.empty(nnz, dtype=torch.int32).pin_memory(); ov = torch.empty(nnz, dtype=torch.float64).pin_memory()
ctx = sg.get_context()
for mode in ("async", "sync", "async"):
    ts = []
    for it in range(6):
        t0 = T()
        dm, o = sg.multiply_device(ah, ah)
        if mode == "async":
            dm.download_async(orr.numpy(), oc.numpy(), ov.numpy(), release=True)
        else:
            dm.download_into(orr.numpy(), oc.numpy(), ov.numpy())
        dm.free()
        ts.append(1e3 * (T() - t0))
    ctx.wait_downloads()
    print(mode, [round(x, 2) for x in ts], "pool", ctx.pool_stats())
