"""Which part of the bench harness slows the timed loop? (diagnostic)"""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
mats = [m.to_device() for m in S.config_matrices(2)]
ctx = sg.get_context()
def loop(k):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        dm, out = sg.multiply_device(mats[0], mats[1]); dm.free()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
for _ in range(3): loop(1)
print("plain            %.3f ms" % loop(10))
ctx.set_profiling(True); print("profiling on     %.3f ms" % loop(10)); ctx.set_profiling(False); ctx.profile_summary()
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", "50"], stdout=subprocess.DEVNULL)
time.sleep(0.5); print("nvidia-smi -lms50 %.3f ms" % loop(10)); p.terminate(); p.wait()
print("plain again      %.3f ms" % loop(10))
