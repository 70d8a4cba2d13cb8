"""Dissect the e2e step (host buffers in, host C out) and the sampler effect (diagnostic)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
from paper_2206_07244_b200.api import CsrMatrix
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
a_host = S.config_matrices(cfg)[0]
pr = torch.from_numpy(a_host.rpt).pin_memory(); pc = torch.from_numpy(a_host.col).pin_memory(); pv = torch.from_numpy(a_host.val).pin_memory()
a = CsrMatrix(a_host.rows, a_host.cols, pr.numpy(), pc.numpy(), pv.numpy())
print("pinned?", pr.is_pinned(), a.rpt.ctypes.data == pr.data_ptr())
p = sg.SpgemmPipeline(a, a); dm, out = p.run_device(); p.close(); nnz = dm.nnz; dm.free()
orpt = torch.empty(a.rows + 1, dtype=torch.int64).pin_memory(); ocol = torch.empty(nnz, dtype=torch.int32).pin_memory(); oval = torch.empty(nnz, dtype=torch.float64).pin_memory()
T = time.perf_counter
acc = {}
def add(k, v): acc[k] = acc.get(k, 0) + v
for it in range(8):
    t0 = T(); p = sg.SpgemmPipeline(a, a); t1 = T()
    dm, out = p.run_device(); t2 = T()
    p.close(); t3 = T()
    dm.download_into(orpt.numpy(), ocol.numpy(), oval.numpy()); t4 = T()
    dm.free(); t5 = T()
    if it >= 3:
        add("create(H2D)", t1 - t0); add("run", t2 - t1); add("close", t3 - t2); add("D2H", t4 - t3); add("free", t5 - t4)
print({k: round(v / 5 * 1e3, 3) for k, v in acc.items()})
mats = [a_host.to_device()]
def loop(k=20):
    torch.cuda.synchronize(); t0 = T()
    for _ in range(k):
        dm, out = sg.multiply_device(mats[0], mats[0]); dm.free()
    torch.cuda.synchronize(); return (T() - t0) / k * 1e3
for _ in range(3): loop(2)
print("device loop plain %.3f" % loop())
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = threading.Event(); n = [0]
def run():
    while not stop.is_set():
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); pynvml.nvmlDeviceGetCurrentClocksEventReasons(h); n[0] += 1
        stop.wait(0.2)
th = threading.Thread(target=run, daemon=True); th.start()
print("device loop + nvml thread %.3f (%d samples)" % (loop(), n[0])); stop.set(); th.join()
print("device loop plain %.3f" % loop())
t0 = T(); [pynvml.nvmlDeviceGetCurrentClocksEventReasons(h) for _ in range(20)]; print("nvml reasons call %.3f ms" % ((T() - t0) / 20 * 1e3))
t0 = T(); [pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM) for _ in range(20)]; print("nvml clock call %.3f ms" % ((T() - t0) / 20 * 1e3))
