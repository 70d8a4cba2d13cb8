"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family once -- thread, group, spec, block and heap tiers, scan and binning
(one and several row-block tiles), multiply_into with several blocks, forecast (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2206_07244_b200 as sg
from paper_2206_07244_b200 import synthetic as S
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import random_csr, spill_pair

cases = [(S.poisson2d_5pt(64),) * 2, (S.random_values(S.stencil3d_27pt(16), 1),) * 2,
         (S.random_values(S.rmat(11, 16, seed=3), 2),) * 2, spill_pair(21000, 4),
         (random_csr(300, 200, 0.05, 1), random_csr(200, 400, 0.04, 2))]
for a, b in cases:
    out = sg.multiply(a, b)
    n = out.c.nnz()
    rpt, col, val = np.zeros(a.rows + 1, np.int64), np.zeros(n, np.int32), np.zeros(n)
    m, _ = sg.multiply_into(a, b, rpt, col, val, parts=3)
    assert m == n and np.array_equal(rpt, out.c.rpt) and np.array_equal(col, out.c.col)
    f = sg.forecast_nnz(a, b)
    assert f.total_nnz == n
cfg = sg.preset(1, sg.kDefaultNumPreset)
for m in (5000, 2 * 1024 * 2048 + 7):
    sg.run_binning(np.random.default_rng(m).integers(0, 3000, size=m), cfg)
print("sanitize workload done")
