import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
cfg = int(sys.argv[1])
a = S.config_matrices(cfg)[0]
print("iso", bench.run_e2e(sg, torch, a, 8, 0))
d = a.to_device()
for _ in range(20):
    dm, o = sg.multiply_device(d, d); dm.free()
torch.cuda.synchronize()
print("after device passes", bench.run_e2e(sg, torch, a, 8, 0))
ctx = sg.get_context()
ctx.set_profiling(True)
for _ in range(10):
    dm, o = sg.multiply_device(d, d); dm.free()
ctx.set_profiling(False)
print(ctx.profile_summary())
print("after profiled pass", bench.run_e2e(sg, torch, a, 8, 0))
c = bench.ClockSampler(0); c.start(); time.sleep(0.5); c.stop()
print("after sampler", bench.run_e2e(sg, torch, a, 8, 0))
