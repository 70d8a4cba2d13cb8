"""Break down one streamed tile (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S, tiled as T
sc = int(sys.argv[1]) if len(sys.argv) > 1 else 20
d = S.rmat(sc, 16, seed=sc).to_device()
T_ = time.perf_counter
def sync(): torch.cuda.synchronize()
for it in range(3):
    sync(); t0 = T_()
    a_blk = T._slice_rows_dev(d, 0, d.rows); sync(); t1 = T_()
    dm, out = sg.multiply_device(a_blk, d); sync(); t2 = T_()
    v, h = dm.checksum(0, 0); sync(); t3 = T_()
    dm.free(); sync(); t4 = T_()
    print(f"slice {1e3*(t1-t0):.1f} multiply {1e3*(t2-t1):.1f} checksum {1e3*(t3-t2):.1f} free {1e3*(t4-t3):.1f}")
for it in range(2):
    sync(); t0 = T_()
    dm, out = sg.multiply_device(d, d); sync(); t1 = T_()
    dm.free(); sync(); t2 = T_()
    print(f"untiled multiply {1e3*(t1-t0):.1f} free {1e3*(t2-t1):.1f}")
