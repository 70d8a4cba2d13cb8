"""csr_from_coo on the device (reference csr.cpp:12-72):
triples in input order -> CSR with sorted columns and duplicates summed in input
order (the first duplicate's value as is, then +=), checked against a direct
restatement of the reference's loop and against the host ingestion path."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MTX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mtx")


def _reference_csr_from_coo(rows, cols, r, c, v):
    """csr.cpp:12-72 restated (test oracle): bucket by row in input order, stable
    sort each row by column, fold duplicates left to right (first value as is)."""
    buckets = [[] for _ in range(rows)]
    for i in range(len(r)):
        buckets[int(r[i])].append((int(c[i]), float(v[i])))
    rpt, col, val = [0], [], []
    for b in buckets:
        b.sort(key=lambda t: t[0])  # stable
        for cc, vv in b:
            if len(col) > rpt[-1] and col[-1] == cc:
                val[-1] = val[-1] + vv
            else:
                col.append(cc)
                val.append(vv)
        rpt.append(len(col))
    return np.array(rpt, np.int64), np.array(col, np.int32), np.array(val, np.float64)


def _bitwise(dm, rpt, col, val):
    got = dm.download()
    return (np.array_equal(got.rpt, rpt) and np.array_equal(got.col, col)
            and np.array_equal(got.val.view(np.int64), val.view(np.int64)))


@pytest.mark.parametrize("n,rows,cols,seed", [(0, 5, 7, 0), (1, 1, 1, 1), (5000, 60, 40, 2), (30000, 3000, 17, 3),
                                              (40000, 7, 5000, 4)])
def test_small_cases_match_reference_loop(sg, n, rows, cols, seed):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, rows, n)
    c = rng.integers(0, cols, n)
    v = rng.uniform(-1, 1, n)
    v[rng.random(n) < 0.05] = -0.0   # a -0.0 first duplicate stays -0.0 (no +0.0 start)
    v[rng.random(n) < 0.05] = 0.0
    dm = sg.csr_from_coo_device(rows, cols, r, c, v)
    assert _bitwise(dm, *_reference_csr_from_coo(rows, cols, r, c, v))
    dm.free()


def test_large_input_matches_host_path(sg):
    from paper_2206_07244_b200.synthetic import csr_from_coo
    rng = np.random.default_rng(7)
    n, rows, cols = 3_000_000, 200_000, 150_000
    r = rng.integers(0, rows, n)
    c = rng.integers(0, cols, n)
    v = rng.uniform(0.5, 1.5, n)  # no signed zeros: the numpy host path starts its sums from +0.0
    dm = sg.csr_from_coo_device(rows, cols, r, c, v)
    h = csr_from_coo(rows, cols, r, c, v)
    assert _bitwise(dm, h.rpt, h.col, h.val)
    dm.free()


def test_device_triples_and_errors(sg):
    import torch
    r = torch.tensor([2, 0, 2, 1, 0], dtype=torch.int64, device="cuda")
    c = torch.tensor([1, 3, 1, 0, 3], dtype=torch.int64, device="cuda")
    v = torch.tensor([1.5, 2.0, 0.25, -1.0, 4.0], dtype=torch.float64, device="cuda")
    dm = sg.csr_from_coo_device(3, 4, r, c, v)
    assert _bitwise(dm, np.array([0, 1, 2, 3]), np.array([3, 0, 1], np.int32), np.array([6.0, -1.0, 1.75]))
    dm.free()
    with pytest.raises(IndexError, match=r"entry \(2, 9\) outside 3x4 shape"):
        sg.csr_from_coo_device(3, 4, np.array([0, 2]), np.array([1, 9]), np.array([1.0, 2.0]))
    with pytest.raises(sg.InvalidArgument):
        sg.csr_from_coo_device(-1, 4, np.zeros(0), np.zeros(0), np.zeros(0))


@pytest.mark.parametrize("name", ["identity3.mtx", "rect2x3.mtx", "sym3.mtx"])
def test_matrix_market_on_device(sg, name):
    from paper_2206_07244_b200.matrix_market import read_matrix_market_csr, read_matrix_market_device
    host = read_matrix_market_csr(os.path.join(MTX, name))
    dm = read_matrix_market_device(os.path.join(MTX, name))
    assert _bitwise(dm, host.rpt, host.col, host.val)
    dm.free()
