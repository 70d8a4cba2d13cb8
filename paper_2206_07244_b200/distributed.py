"""Multi-GPU SpGEMM: row-block data parallelism.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch on the GPU box;
gloo in the CPU tests). The only exchange is the replication of B:

1. rank 0 broadcasts B (rpt, col, val) -- one ``ncclBroadcast`` per array, B.rpt
   first (its length sizes the receive buffers);
2. every rank computes per-row nprod with kernel K1 (identical on all ranks)
   and derives the same nprod-prefix balanced split deterministically -- no
   collective needed for the partition;
3. each rank multiplies its contiguous row block A[r0:r1, :] by B independently;
4. row pointers are stitched from the per-rank nnz totals (one all-gather of G
   int64 values); C stays distributed unless the caller asks for it on one rank
   (``gather_csr``: point-to-point transfers of each slice's arrays to that rank,
   assembled into one host CSR -- SURVEY.md §8(f) item 4).

``forecast_distributed`` is the symbolic-only variant (§8(f) item 4): the same
broadcast and split, every rank counting its block's nnz(C) without allocating
C, the totals combined with one all-reduce -- sizing a TB-scale product (config
5) before committing memory to it.

The local multiply / nprod functions default to the B200 library; the CPU tests
inject the oracle to exercise the partition/broadcast/stitch logic with gloo.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np

from .api import CsrMatrix


def nprod_split(nprod, parts: int) -> List[int]:
    """Contiguous row blocks balanced by the nprod prefix sum: rank g takes the rows
    whose exclusive prefix lies in [g*T/G, (g+1)*T/G). Rows never split. Returns
    parts+1 boundaries (bounds[0] = 0, bounds[-1] = M)."""
    nprod = np.asarray(nprod, np.int64)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    excl = np.concatenate([[0], np.cumsum(nprod)[:-1]]) if nprod.size else np.zeros(0, np.int64)
    total = int(nprod.sum())
    bounds = [0]
    for g in range(1, parts):
        target = (g * total) // parts if total else 0
        bounds.append(int(np.searchsorted(excl, target, side="left")) if total else (g * nprod.size) // parts)
    bounds.append(int(nprod.size))
    for g in range(1, len(bounds)):  # monotone even for degenerate inputs
        bounds[g] = max(bounds[g], bounds[g - 1])
    return bounds


def slice_rows(m: CsrMatrix, r0: int, r1: int) -> CsrMatrix:
    """Rows [r0, r1) of m as a CSR matrix (col/val are zero-copy views)."""
    p0, p1 = int(m.rpt[r0]), int(m.rpt[r1])
    return CsrMatrix(r1 - r0, m.cols, m.rpt[r0:r1 + 1] - p0, m.col[p0:p1], m.val[p0:p1])


def stitch(slices: List[CsrMatrix], cols: int) -> CsrMatrix:
    """Concatenate row-block results: each slice's rpt is offset by the nnz of the
    slices before it (the host side of kernel K8)."""
    hosts = [s.to_host() for s in slices]
    offsets = np.cumsum([0] + [s.nnz() for s in hosts])
    rpt = np.concatenate([np.zeros(1, np.int64)] + [h.rpt[1:] + off for h, off in zip(hosts, offsets[:-1])])
    col = np.concatenate([h.col for h in hosts]) if hosts else np.zeros(0, np.int32)
    val = np.concatenate([h.val for h in hosts]) if hosts else np.zeros(0)
    return CsrMatrix(int(rpt.size - 1), cols, rpt, col, val)


def _dist():
    import torch.distributed as dist
    return dist


def broadcast_csr(m: Optional[CsrMatrix], src: int = 0, device=None, group=None) -> CsrMatrix:
    """Replicate a CSR matrix from rank `src` to every rank (B.rpt length first)."""
    import torch
    dist = _dist()
    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    if rank == src:
        shape = torch.tensor([m.rows, m.cols, m.nnz()], dtype=torch.int64, device=dev)
    else:
        shape = torch.zeros(3, dtype=torch.int64, device=dev)
    dist.broadcast(shape, src, group=group)
    rows, cols, nnz = (int(x) for x in shape.tolist())
    if rank == src:
        src_m = m if (m.on_device and dev.type == "cuda") else None
        if src_m is None:
            h = m.to_host()
            rpt = torch.from_numpy(np.ascontiguousarray(h.rpt)).to(dev)
            col = torch.from_numpy(np.ascontiguousarray(h.col)).to(dev)
            val = torch.from_numpy(np.ascontiguousarray(h.val)).to(dev)
        else:
            rpt, col, val = src_m.rpt, src_m.col, src_m.val
    else:
        rpt = torch.empty(rows + 1, dtype=torch.int64, device=dev)
        col = torch.empty(nnz, dtype=torch.int32, device=dev)
        val = torch.empty(nnz, dtype=torch.float64, device=dev)
    for t in (rpt, col, val):
        if t.numel():
            dist.broadcast(t, src, group=group)
    if dev.type == "cuda":
        return CsrMatrix(rows, cols, rpt, col, val)
    return CsrMatrix(rows, cols, rpt.numpy(), col.numpy(), val.numpy())


@dataclass
class DistributedResult:
    c_local: CsrMatrix          # this rank's row block of C (local row pointers)
    row_bounds: List[int]       # global row split
    nnz_offsets: List[int]      # global C offset of every rank's block (stitched row pointers)
    total_nprod: int
    c: Optional[CsrMatrix] = None  # the stitched C, on `gather_to` only


def multiply_distributed(a: Optional[CsrMatrix], b: Optional[CsrMatrix], *, same: bool = False, src: int = 0,
                         device=None, group=None, gather_to: Optional[int] = None,
                         local_multiply: Optional[Callable] = None,
                         local_nprod: Optional[Callable] = None) -> DistributedResult:
    """C = A*B row-partitioned over the ranks of `group`. A and B need only exist on
    rank `src`; with same=True (C = A*A) only B is broadcast and A is taken from it."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if local_multiply is None or local_nprod is None:
        from . import api as sg
        dev_index = None if device is None else (device.index if hasattr(device, "index") else int(str(device).split(":")[-1]))
        if local_multiply is None:
            def local_multiply(x, y):  # noqa: E306
                dm, out = sg.multiply_device(x, y, device=dev_index)
                c = dm.download()
                dm.free()
                return c
        if local_nprod is None:
            def local_nprod(x, y):  # noqa: E306
                return sg.compute_nprod(x, y, device=dev_index)[0]
    B = broadcast_csr(b if rank == src else None, src, device, group)
    A = B if same else broadcast_csr(a if rank == src else None, src, device, group)
    nprod = np.asarray(local_nprod(A, B), np.int64)
    bounds = nprod_split(nprod, world)
    r0, r1 = bounds[rank], bounds[rank + 1]
    c_loc = local_multiply(slice_rows(A, r0, r1), B)
    c_loc = c_loc if isinstance(c_loc, CsrMatrix) else CsrMatrix(c_loc.rows, c_loc.cols, c_loc.rpt, c_loc.col, c_loc.val)
    nnzs = [None] * world
    dist.all_gather_object(nnzs, int(c_loc.nnz()), group=group)
    offsets = [int(x) for x in np.concatenate([[0], np.cumsum(nnzs)[:-1]])]
    res = DistributedResult(c_loc, bounds, offsets, int(nprod.sum()))
    if gather_to is not None:
        res.c = gather_csr(c_loc, gather_to, device=device, group=group)
    return res


def gather_csr(c_local: CsrMatrix, dst: int = 0, device=None, group=None) -> Optional[CsrMatrix]:
    """Assemble the ranks' row blocks of C (in rank order) into one host CSR on rank
    ``dst`` (None elsewhere). The block sizes travel in one all-gather; every other
    rank then sends its rpt/col/val with point-to-point transfers (NCCL from HBM on
    the GPU box, gloo on CPU), received one block at a time so ``dst`` needs device
    room for the largest block only. Row pointers are rebased by the nnz offsets."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    mine = torch.tensor([c_local.rows, c_local.nnz()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(2, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, mine, group=group)
    sizes = [(int(t[0]), int(t[1])) for t in sizes]

    def tensors(m: CsrMatrix):
        if m.on_device and dev.type == "cuda":
            return m.rpt, m.col, m.val
        h = m.to_host()
        return tuple(torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (h.rpt, h.col, h.val))

    if rank != dst:
        for t in tensors(c_local):
            if t.numel():
                dist.send(t.contiguous(), dst, group=group)
        return None
    rows = sum(r for r, _ in sizes)
    nnz = sum(n for _, n in sizes)
    rpt = np.empty(rows + 1, np.int64)
    col = np.empty(nnz, np.int32)
    val = np.empty(nnz, np.float64)
    rpt[0] = 0
    r0 = off = 0
    for g, (rg, ng) in enumerate(sizes):
        if g == rank:
            h = c_local.to_host()
            brpt, bcol, bval = np.asarray(h.rpt), np.asarray(h.col), np.asarray(h.val)
        else:
            ts = [torch.empty(rg + 1, dtype=torch.int64, device=dev), torch.empty(ng, dtype=torch.int32, device=dev),
                  torch.empty(ng, dtype=torch.float64, device=dev)]
            for t in ts:
                if t.numel():
                    dist.recv(t, g, group=group)
            brpt, bcol, bval = (t.cpu().numpy() for t in ts)
        rpt[r0 + 1:r0 + rg + 1] = brpt[1:] + off
        col[off:off + ng] = bcol
        val[off:off + ng] = bval
        r0 += rg
        off += ng
    return CsrMatrix(rows, c_local.cols, rpt, col, val)


@dataclass
class DistributedForecast:
    total_nnz: int              # nnz(C) of the whole product (all-reduced)
    total_nprod: int
    local_nnz: int              # this rank's block
    row_bounds: List[int]
    row_nnz: Optional[np.ndarray] = None  # this rank's rows' nnz(C(i,:))


def forecast_distributed(a: Optional[CsrMatrix], b: Optional[CsrMatrix], *, same: bool = False, src: int = 0,
                         device=None, group=None, local_forecast: Optional[Callable] = None,
                         local_nprod: Optional[Callable] = None) -> DistributedForecast:
    """nnz(C) of C = A*B without computing C, row-partitioned like
    multiply_distributed. ``local_forecast(A_block, B)`` returns the block's per-row
    nnz(C) (default: the B200 library's forecast_nnz)."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev_index = None if device is None else (device.index if hasattr(device, "index") else int(str(device).split(":")[-1]))
    if local_forecast is None or local_nprod is None:
        from . import api as sg
        if local_forecast is None:
            def local_forecast(x, y):  # noqa: E306
                return sg.forecast_nnz(x, y, device=dev_index).row_nnz
        if local_nprod is None:
            def local_nprod(x, y):  # noqa: E306
                return sg.compute_nprod(x, y, device=dev_index)[0]
    B = broadcast_csr(b if rank == src else None, src, device, group)
    A = B if same else broadcast_csr(a if rank == src else None, src, device, group)
    nprod = np.asarray(local_nprod(A, B), np.int64)
    bounds = nprod_split(nprod, world)
    r0, r1 = bounds[rank], bounds[rank + 1]
    rows = np.asarray(local_forecast(slice_rows(A, r0, r1), B), np.int64) if r1 > r0 else np.zeros(0, np.int64)
    local = int(rows.sum())
    dev = torch.device("cpu") if device is None else torch.device(device)
    t = torch.tensor([local], dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    return DistributedForecast(int(t.item()), int(nprod.sum()), local, bounds, rows)


# ---------------------------------------------------------------------------
# Streamed, row-partitioned C = B*B with the broadcast inside the step (config
# 5 strong scaling, SURVEY.md §8(e) "Collective" and "Timing" rows).
@dataclass
class PendingCsr:
    """A broadcast CSR matrix whose arrays may still be in flight."""
    m: CsrMatrix
    works: dict

    def wait(self, *names: str) -> None:
        for n in names:
            w = self.works.pop(n, None)
            if w is not None:
                w.wait()  # NCCL: the current CUDA stream waits (no host block); gloo: blocks


def broadcast_csr_async(m: Optional[CsrMatrix], src: int = 0, device=None, group=None) -> PendingCsr:
    """broadcast_csr with the three array broadcasts issued asynchronously, B.rpt
    first, then B.col, then B.val (one NCCL stream, in that order): K1 needs only
    rpt and col, so B.val's transfer overlaps it (and the row split)."""
    import torch
    dist = _dist()
    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    if rank == src:
        shape = torch.tensor([m.rows, m.cols, m.nnz()], dtype=torch.int64, device=dev)
    else:
        shape = torch.zeros(3, dtype=torch.int64, device=dev)
    dist.broadcast(shape, src, group=group)
    rows, cols, nnz = (int(x) for x in shape.tolist())
    if rank == src:
        if m.on_device and dev.type == "cuda":
            rpt, col, val = m.rpt, m.col, m.val
        else:
            h = m.to_host()
            rpt, col, val = (torch.from_numpy(np.ascontiguousarray(x)).to(dev) for x in (h.rpt, h.col, h.val))
    else:
        rpt = torch.empty(rows + 1, dtype=torch.int64, device=dev)
        col = torch.empty(nnz, dtype=torch.int32, device=dev)
        val = torch.empty(nnz, dtype=torch.float64, device=dev)
    works = {}
    for name, t in (("rpt", rpt), ("col", col), ("val", val)):
        works[name] = dist.broadcast(t, src, group=group, async_op=True) if t.numel() else None
    if dev.type == "cuda":
        out = CsrMatrix(rows, cols, rpt, col, val)
    else:
        out = CsrMatrix(rows, cols, rpt.numpy(), col.numpy(), val.numpy())
    return PendingCsr(out, works)


@dataclass
class StreamedResult:
    row_bounds: List[int]
    total_nprod: int          # of the whole product (every rank's K1 sees all of it)
    local: object             # this rank's tiles' report (tiled.StreamReport or the injected equivalent)


def stream_square_distributed(b: Optional[CsrMatrix], *, src: int = 0, device=None, group=None,
                              local_nprod: Optional[Callable] = None,
                              local_stream: Optional[Callable] = None) -> StreamedResult:
    """One step of the config-5 strong-scaling workload, C = B*B with B on rank
    `src` only: B is broadcast (rpt, col, val in flight together); each rank runs
    K1 as soon as rpt and col have landed -- B.val's transfer overlaps it -- and
    derives the same nprod-balanced row split; then its row block is streamed
    through row-block x column-window tiles (tiled.stream_multiply). No further
    collective: the caller reduces the checksums and the max time."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if local_nprod is None:
        from . import api as sg
        dev_index = None if device is None else (device.index if hasattr(device, "index") else int(str(device).split(":")[-1]))

        def local_nprod(x, y):  # noqa: E306
            return sg.compute_nprod(x, y, device=dev_index)[0]
    if local_stream is None:
        raise ValueError("local_stream(B, rows, nprod) is required")
    pend = broadcast_csr_async(b if rank == src else None, src, device, group)
    B = pend.m
    pend.wait("rpt", "col")
    nprod = np.asarray(local_nprod(B, B), np.int64)   # K1 while B.val is still arriving
    bounds = nprod_split(nprod, world)
    pend.wait("val")
    rep = local_stream(B, range(bounds[rank], bounds[rank + 1]), nprod)
    return StreamedResult(bounds, int(nprod.sum()), rep)
