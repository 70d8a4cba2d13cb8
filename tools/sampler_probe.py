"""Perturbation of the timed loop by clock samplers (diagnostic)."""
import os, sys, time, subprocess, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
mats = [m.to_device() for m in S.config_matrices(2)]
def loop(k=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k):
        dm, out = sg.multiply_device(mats[0], mats[1]); dm.free()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
for _ in range(5): loop(1)
print("plain              %.3f ms" % loop())
print("plain              %.3f ms" % loop())
for period in (50, 200, 1000):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader", "-lms", str(period)], stdout=subprocess.DEVNULL)
    time.sleep(0.5); r = loop(); p.terminate(); p.wait()
    print(f"nvidia-smi {period:4d}ms  %.3f ms" % r)
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
for period in (0.05, 0.2):
    stop = threading.Event(); samples = []
    def run():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
            stop.wait(period)
    th = threading.Thread(target=run, daemon=True); th.start(); time.sleep(0.2)
    r = loop(); stop.set(); th.join()
    print(f"nvml {period*1e3:4.0f}ms         %.3f ms  ({len(samples)} samples, {samples[-1]})" % r)
print("plain              %.3f ms" % loop())
