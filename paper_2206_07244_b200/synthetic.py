"""Synthetic inputs for the BASELINE.json configs (synthetic.hpp analogue, numpy).

All generators are deterministic functions of their arguments (no libstdc++
distributions), so the CPU checkers and the GPU see identical matrices:

* ``poisson2d_5pt(n)``        config 1: 2D 5-point Laplacian (diag 4, off -1)
* ``stencil3d_27pt(n)``       config 2: 3D 27-point box stencil (diag 26, off -1)
* ``poisson3d_7pt(n)``        config 4's A: 3D 7-point Poisson (diag 6, off -1)
* ``trilinear_prolongation``  config 4's P (64^3 -> 128^3); R = P^T via ``transpose``
* ``rmat(scale, ef)``         configs 3/5: R-MAT (a,b,c,d)=(.57,.19,.19,.05), duplicates summed
* ``random_values(m, seed)``  replaces values by U[-1,1) from splitmix64(seed ^ (row<<32|col))

Grids use natural ordering (x fastest) with Dirichlet truncation (no wrap).
"""
from __future__ import annotations

import numpy as np

try:
    from .api import CsrMatrix, InvalidArgument
except ImportError:
    # Loaded by file path, outside the package (bench.py --impl reference builds
    # the reference arm's inputs this way): no package import, so the sm_100a
    # library is never loaded into the reference's process. A host-only record
    # with the fields the checkers and the reference binding read.
    class InvalidArgument(ValueError):
        pass

    class CsrMatrix:  # noqa: D101 -- host arrays only
        def __init__(self, rows, cols, rpt, col, val):
            self.rows, self.cols = int(rows), int(cols)
            self.rpt = np.ascontiguousarray(rpt, np.int64)
            self.col = np.ascontiguousarray(col, np.int32)
            self.val = np.ascontiguousarray(val, np.float64)

        def to_host(self):
            return self

        def nnz(self) -> int:
            return int(self.rpt[self.rows]) if self.rows >= 0 else 0


def identity_csr(n: int) -> CsrMatrix:
    """synthetic.cpp:20-36."""
    return CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n))


def csr_from_coo(rows: int, cols: int, r, c, v) -> CsrMatrix:
    """csr.cpp:12-72: triples -> CSR, duplicates summed in input order, columns sorted."""
    r = np.asarray(r, np.int64)
    c = np.asarray(c, np.int64)
    v = np.asarray(v, np.float64)
    if rows < 0 or cols < 0:
        raise InvalidArgument("csr_from_coo: negative matrix shape")
    if r.size and (r.min() < 0 or r.max() >= rows or c.min() < 0 or c.max() >= cols):
        raise IndexError("csr_from_coo: entry outside the declared shape")
    key = r * max(cols, 1) + c
    order = np.argsort(key, kind="stable")
    ks = key[order]
    first = np.ones(ks.size, bool)
    first[1:] = ks[1:] != ks[:-1]
    uniq = ks[first]
    slot = np.cumsum(first) - 1
    vals = np.zeros(uniq.size, np.float64)
    np.add.at(vals, slot, v[order])  # sequential, in input order within a key
    ur = uniq // max(cols, 1)
    uc = uniq % max(cols, 1)
    rpt = np.zeros(rows + 1, np.int64)
    np.add.at(rpt, ur + 1, 1)
    np.cumsum(rpt, out=rpt)
    return CsrMatrix(rows, cols, rpt, uc.astype(np.int32), vals)


def transpose(m: CsrMatrix) -> CsrMatrix:
    m = m.to_host()
    rows = np.repeat(np.arange(m.rows, dtype=np.int64), np.diff(m.rpt))
    order = np.lexsort((rows, m.col.astype(np.int64)))
    col_t = rows[order].astype(np.int32)
    val_t = m.val[order]
    rpt = np.zeros(m.cols + 1, np.int64)
    np.add.at(rpt, m.col.astype(np.int64) + 1, 1)
    np.cumsum(rpt, out=rpt)
    return CsrMatrix(m.cols, m.rows, rpt, col_t, val_t)


def _stencil(shape, offsets, diag, off):
    """Box/star stencil on a grid (natural order, x fastest), Dirichlet truncation."""
    dims = len(shape)
    n = int(np.prod(shape))
    idx = np.arange(n, dtype=np.int64)
    coords = []
    rem = idx
    for d in range(dims):
        coords.append(rem % shape[d])
        rem = rem // shape[d]
    strides = [int(np.prod(shape[:d])) for d in range(dims)]
    offsets = sorted(offsets, key=lambda o: sum(o[d] * strides[d] for d in range(dims)))
    cols, valid = [], []
    for o in offsets:
        ok = np.ones(n, bool)
        lin = idx.copy()
        for d in range(dims):
            cd = coords[d] + o[d]
            ok &= (cd >= 0) & (cd < shape[d])
            lin += o[d] * strides[d]
        cols.append(lin)
        valid.append(ok)
    cols = np.stack(cols, 1)
    valid = np.stack(valid, 1)
    vals = np.where(np.all(np.array(offsets) == 0, axis=1)[None, :], float(diag), float(off))
    vals = np.broadcast_to(vals, cols.shape)
    counts = valid.sum(1)
    rpt = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=rpt[1:])
    return CsrMatrix(n, n, rpt, cols[valid].astype(np.int32), np.ascontiguousarray(vals[valid]))


def poisson2d_5pt(n: int = 1024) -> CsrMatrix:
    offs = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)]
    return _stencil((n, n), offs, 4.0, -1.0)


def stencil3d_27pt(n: int = 128) -> CsrMatrix:
    offs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    return _stencil((n, n, n), offs, 26.0, -1.0)


def poisson3d_7pt(n: int = 128) -> CsrMatrix:
    offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    return _stencil((n, n, n), offs, 6.0, -1.0)


def trilinear_prolongation(nc: int = 64, nf: int = 128) -> CsrMatrix:
    """P: nf^3 x nc^3. 1-D rule: even i -> i/2 (weight 1); odd i -> (i-1)/2 and (i+1)/2
    (weight 1/2 each), dropping an out-of-range top index. Tensor product (<= 8 per row)."""
    i = np.arange(nf)
    lo = np.where(i % 2 == 0, i // 2, (i - 1) // 2)
    hi = np.where(i % 2 == 0, -1, (i + 1) // 2)
    hi = np.where(hi >= nc, -1, hi)
    w_lo = np.where(i % 2 == 0, 1.0, 0.5)
    c1 = np.stack([lo, hi], 1)            # (nf, 2)
    w1 = np.stack([w_lo, np.where(hi >= 0, 0.5, 0.0)], 1)
    ok1 = c1 >= 0
    # tensor product over (z, y, x) with x fastest
    cz, cy, cx = c1[:, None, None, :, None, None], c1[None, :, None, None, :, None], c1[None, None, :, None, None, :]
    wz, wy, wx = w1[:, None, None, :, None, None], w1[None, :, None, None, :, None], w1[None, None, :, None, None, :]
    oz, oy, ox = ok1[:, None, None, :, None, None], ok1[None, :, None, None, :, None], ok1[None, None, :, None, None, :]
    col = cx + nc * cy + nc * nc * cz
    w = wx * wy * wz
    ok = ox & oy & oz
    col = col.reshape(nf ** 3, 8)
    w = w.reshape(nf ** 3, 8)
    ok = ok.reshape(nf ** 3, 8)
    col = np.where(ok, col, np.iinfo(np.int64).max)
    order = np.argsort(col, axis=1, kind="stable")
    col = np.take_along_axis(col, order, 1)
    w = np.take_along_axis(w, order, 1)
    ok = np.take_along_axis(ok, order, 1)
    counts = ok.sum(1)
    rpt = np.zeros(nf ** 3 + 1, np.int64)
    np.cumsum(counts, out=rpt[1:])
    return CsrMatrix(nf ** 3, nc ** 3, rpt, col[ok].astype(np.int32), w[ok])


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    z = x
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def random_values(m: CsrMatrix, seed: int = 0) -> CsrMatrix:
    """Values U[-1,1) (53-bit) from splitmix64(seed ^ (row<<32 | col)); same pattern."""
    m = m.to_host()
    rows = np.repeat(np.arange(m.rows, dtype=np.uint64), np.diff(m.rpt))
    key = (rows << np.uint64(32)) | m.col.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = _splitmix64(key ^ np.uint64(seed))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return CsrMatrix(m.rows, m.cols, m.rpt, m.col, 2.0 * u - 1.0)


def rmat(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, seed: int = 20) -> CsrMatrix:
    """R-MAT graph: E = ef * 2^scale directed draws, duplicates summed (value = count),
    self-loops kept, no noise and no vertex permutation."""
    n = 1 << scale
    e = edge_factor * n
    rng = np.random.Generator(np.random.PCG64(seed))
    src = np.zeros(e, np.int64)
    dst = np.zeros(e, np.int64)
    ab, abc = a + b, a + b + c
    chunk = 1 << 22
    for s0 in range(0, e, chunk):
        s1 = min(e, s0 + chunk)
        rs = np.zeros(s1 - s0, np.int64)
        rd = np.zeros(s1 - s0, np.int64)
        for lvl in range(scale):
            u = rng.random(s1 - s0)
            bit = np.int64(1) << np.int64(scale - 1 - lvl)
            down = u >= ab            # quadrants c, d -> source bit set
            right = ((u >= a) & (u < ab)) | (u >= abc)  # quadrants b, d -> dest bit set
            rs += np.where(down, bit, 0)
            rd += np.where(right, bit, 0)
        src[s0:s1] = rs
        dst[s0:s1] = rd
    key = src * n + dst
    key.sort()
    first = np.ones(key.size, bool)
    first[1:] = key[1:] != key[:-1]
    starts = np.nonzero(first)[0]
    uniq = key[starts]
    counts = np.diff(np.append(starts, key.size)).astype(np.float64)
    ur = uniq // n
    rpt = np.zeros(n + 1, np.int64)
    np.add.at(rpt, ur + 1, 1)
    np.cumsum(rpt, out=rpt)
    return CsrMatrix(n, n, rpt, (uniq % n).astype(np.int32), counts)


def config_matrices(config: int, small: bool = False):
    """(A, B[, ...]) for BASELINE.json configs 1-4 (1-based). small=True gives a
    reduced-size instance of the same shape family for parity tests."""
    if config == 1:
        a = poisson2d_5pt(64 if small else 1024)
        return a, a
    if config == 2:
        a = stencil3d_27pt(16 if small else 128)
        return a, a
    if config == 3:
        a = rmat(10 if small else 20, 16)
        return a, a
    if config == 4:
        nf = 16 if small else 128
        a = poisson3d_7pt(nf)
        p = trilinear_prolongation(nf // 2, nf)
        return a, p, transpose(p)
    raise InvalidArgument(f"unknown config {config}")
