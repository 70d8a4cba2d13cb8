"""Tiled, streamed SpGEMM for products whose C does not fit HBM (BASELINE config 5,
SURVEY.md §8(e) "Config 5 feasibility").

R-MAT scale 24 gives nprod = 1.0e12 and a TB-scale C, so C cannot be materialised
on one -- or eight -- B200s. The product is computed in TILES and streamed:

* columns: B is split into windows of 2^20 columns (``split_columns``). A window of
  C = A.B[:, window] has at most 2^20 columns, so every heap-tier row of the tile
  fits the 128 KB shared-memory bitmap of kernels_heap.cuh in ONE pass (a wider B
  would otherwise be re-walked once per window inside the kernel);
* rows: A's rows are cut into blocks of bounded nprod, so a tile's C (<= 12 B per
  product) fits the memory budget.

Every tile is one ordinary ``multiply_device`` (the full OpSparse pipeline on the
device); its C is reduced to a checksum on the device and released ("C streamed,
not materialised"). The sum of the tiles' nprod is exactly the product's nprod,
so GFLOPS = 2 * nprod / time is the same metric as for a materialised C.

Checksums per tile: nnz, sum of values (fp64), and sum over entries of
(global column + 1) * (global row + 1) mod 2^64 -- structure and values of the
streamed C can be compared against an untiled run (tests/test_tiled_gpu.py).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .api import CsrMatrix, compute_nprod, get_context, multiply_device

WINDOW = 1 << 20


def _torch():
    import torch
    return torch


def _as_tensors(m: CsrMatrix):
    torch = _torch()
    r, c, v = m.rpt, m.col, m.val
    if not (torch.is_tensor(r) and r.is_cuda):
        raise ValueError("tiled SpGEMM expects device-resident operands (CsrMatrix.to_device())")
    return r, c, v


def split_columns(b: CsrMatrix, window: int = WINDOW) -> List[CsrMatrix]:
    """B[:, w*window:(w+1)*window] for every window w, columns re-based to 0, as device
    CSR matrices. Rows keep their order and each row's columns stay sorted."""
    torch = _torch()
    rpt, col, val = _as_tensors(b)
    nwin = max(1, (b.cols + window - 1) // window)
    if nwin == 1:
        return [b]
    dev = col.device
    rows = torch.repeat_interleave(torch.arange(b.rows, device=dev, dtype=torch.int64), rpt[1:] - rpt[:-1])
    wid = (col.to(torch.int64) // window)
    out = []
    for w in range(nwin):
        sel = wid == w
        r_w = rows[sel]
        counts = torch.bincount(r_w, minlength=b.rows)
        rpt_w = torch.zeros(b.rows + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=rpt_w[1:])
        col_w = (col[sel].to(torch.int64) - w * window).to(torch.int32)
        width = min(window, b.cols - w * window)
        out.append(CsrMatrix(b.rows, width, rpt_w, col_w.contiguous(), val[sel].contiguous()))
    return out


def row_blocks(nprod: np.ndarray, budget: int) -> List[int]:
    """Contiguous row blocks of at most ``budget`` products each (a single row
    above the budget forms its own block). Returns the block boundaries."""
    nprod = np.asarray(nprod, np.int64)
    cs = np.cumsum(nprod)
    total = int(cs[-1]) if cs.size else 0
    bounds = [0]
    base = 0  # products before the current block
    while bounds[-1] < nprod.size and total - base > budget:
        # first row whose inclusive prefix exceeds base + budget ends the block
        i = int(np.searchsorted(cs, base + budget, side="right"))
        i = max(i, bounds[-1] + 1)  # a row above the budget: a block of its own
        bounds.append(i)
        base = int(cs[i - 1])
    if bounds[-1] < nprod.size:
        bounds.append(int(nprod.size))
    return bounds


def _slice_rows_dev(m: CsrMatrix, r0: int, r1: int) -> CsrMatrix:
    rpt, col, val = _as_tensors(m)
    p0, p1 = int(rpt[r0]), int(rpt[r1])
    return CsrMatrix(r1 - r0, m.cols, rpt[r0:r1 + 1] - p0, col[p0:p1], val[p0:p1])


@dataclass
class StreamReport:
    total_nprod: int = 0
    nnz: int = 0
    val_sum: float = 0.0
    pattern_hash: int = 0
    tiles: int = 0
    spilled_rows: int = 0
    kernel_launches: int = 0  # summed over the tiles' contexts (each worker thread has its own)
    tile_nprod: List[int] = field(default_factory=list)


def _tile_checksum(dm, row0: int, col0: int):
    return dm.checksum(row0, col0) if dm.nnz else (0.0, 0)


def stream_multiply(a: CsrMatrix, b: CsrMatrix, rows: Optional[range] = None, nprod: Optional[np.ndarray] = None,
                    budget: int = 4_000_000_000, window: int = WINDOW, b_windows: Optional[List[CsrMatrix]] = None,
                    device: Optional[int] = None, options=None, workers: int = 1) -> StreamReport:
    """C = A[rows].B computed tile by tile (row blocks x column windows) and
    streamed into checksums. A row block holds at most ``budget`` products over
    all windows, so no tile's C exceeds 12 * budget bytes. ``nprod`` (per row of
    A, from K1) and ``b_windows`` can be passed in to share them across calls.

    ``workers`` > 1 runs that many tiles at once, each on its own host thread
    and context (streams): the SMs a tile leaves idle while its heaviest rows
    finish (R-MAT hubs) are taken by the next tile."""
    if nprod is None:
        nprod, _ = compute_nprod(a, b, device=device)
    nprod = np.asarray(nprod, np.int64)
    r_lo, r_hi = (0, a.rows) if rows is None else (rows.start, rows.stop)
    wins = b_windows if b_windows is not None else split_columns(b, window)
    bounds = row_blocks(nprod[r_lo:r_hi], max(1, budget))
    tiles = []
    for i in range(len(bounds) - 1):
        r0, r1 = r_lo + bounds[i], r_lo + bounds[i + 1]
        if r1 > r0:
            tiles.extend((r0, r1, w) for w in range(len(wins)))

    def run_tile(t):
        r0, r1, w = t
        if device is not None:
            _torch().cuda.set_device(device)
        ctx = get_context(device)
        l0 = ctx.kernel_launches
        dm, out = multiply_device(_slice_rows_dev(a, r0, r1), wins[w], options, device=device)
        try:
            s, h = _tile_checksum(dm, r0, w * window)
            return out.stats.total_nprod, out.stats.nnz_of_product, s, h, out.spilled_rows, ctx.kernel_launches - l0
        finally:
            dm.free()

    if workers > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=workers) as ex:
            results = list(ex.map(run_tile, tiles))
    else:
        results = [run_tile(t) for t in tiles]
    rep = StreamReport()
    for np_t, nnz_t, s, h, spilled, nl in results:
        rep.kernel_launches += nl
        rep.total_nprod += np_t
        rep.tile_nprod.append(np_t)
        rep.nnz += nnz_t
        rep.val_sum += s
        rep.pattern_hash = (rep.pattern_hash + h) & ((1 << 64) - 1)
        rep.spilled_rows += spilled
        rep.tiles += 1
    return rep


def checksum_of(c: CsrMatrix) -> StreamReport:
    """The same checksums for a materialised (host) C -- the test-side comparison."""
    c = c.to_host()
    rows = np.repeat(np.arange(c.rows, dtype=np.uint64) + np.uint64(1), np.diff(c.rpt))
    h = int(np.sum((c.col.astype(np.uint64) + np.uint64(1)) * rows, dtype=np.uint64))
    return StreamReport(nnz=int(c.nnz()), val_sum=float(np.sum(c.val)), pattern_hash=h, tiles=1)
