"""Tiled vs untiled timing at one R-MAT scale (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S, tiled as T
sc = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d = S.rmat(sc, 16, seed=sc).to_device()
nprod, tot = sg.compute_nprod(d, d)
wins = T.split_columns(d)
def t(f, n=2):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
def untiled():
    dm, out = sg.multiply_device(d, d); dm.free()
print("untiled ms", t(untiled))
for budget in (10**13, 12 * 10**9, 4 * 10**9):
    rep = [None]
    def f():
        rep[0] = T.stream_multiply(d, d, nprod=nprod, b_windows=wins, budget=budget)
    ms = t(f)
    print(f"budget {budget:.0e}: tiles {rep[0].tiles} ms {ms:.1f} tile nprod {[f'{x:.2e}' for x in rep[0].tile_nprod[:6]]}")
    for i in range(len(rep[0].tile_nprod)):
        pass
# per-tile timing for budget 12e9
bounds = T.row_blocks(nprod, 12 * 10**9)
for i in range(len(bounds) - 1):
    a_blk = T._slice_rows_dev(d, bounds[i], bounds[i + 1])
    def g():
        dm, out = sg.multiply_device(a_blk, d); dm.free()
    print("block", bounds[i], bounds[i + 1], "ms", round(t(g), 1))
