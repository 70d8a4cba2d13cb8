"""CPU, world_size 2 (gloo on 127.0.0.1): the multi-GPU logic of SURVEY.md §8(e) --
B broadcast, deterministic nprod-balanced row split, per-rank block products,
row-pointer stitching -- checked bitwise against the single-shot oracle product.
The per-rank multiply is the oracle here (no GPU in the CPU suite); on the B200 box
the same code runs the sm_100a library over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from helpers import random_csr


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2206_07244_b200.distributed import multiply_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case == "square":
            a = random_csr(700, 700, 0.02, 5) if rank == 0 else None
            b, same = a, True
        else:
            a = random_csr(333, 250, 0.04, 6) if rank == 0 else None
            b = random_csr(250, 410, 0.03, 7) if rank == 0 else None
            same = False
        res = multiply_distributed(a, b, same=same, gather_to=0,
                                   local_multiply=O.spgemm, local_nprod=lambda x, y: O.compute_nprod(x, y)[0])
        out = dict(rank=rank, bounds=res.row_bounds, offsets=res.nnz_offsets, nnz=int(res.c_local.nnz()),
                   total_nprod=res.total_nprod)
        if rank == 0:
            exp = O.spgemm(a, b)
            c = res.c
            out["same_pattern"] = bool(np.array_equal(c.rpt, exp.rpt) and np.array_equal(c.col, exp.col))
            out["bitwise"] = bool(np.array_equal(c.val.view(np.int64), exp.val.view(np.int64)))
            nprod, total = O.compute_nprod(a, b)
            out["exp_total_nprod"] = total
            b0, b1, b2 = res.row_bounds
            out["halves"] = (int(nprod[b0:b1].sum()), int(nprod[b1:b2].sum()))
        q.put(out)
    finally:
        dist.destroy_process_group()


def _worker_forecast(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2206_07244_b200.distributed import forecast_distributed
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = random_csr(500, 500, 0.03, 9) if rank == 0 else None
        f = forecast_distributed(a, a, same=True,
                                 local_forecast=lambda x, y: np.diff(np.asarray(O.spgemm(x, y).rpt)),
                                 local_nprod=lambda x, y: O.compute_nprod(x, y)[0])
        out = dict(rank=rank, total=f.total_nnz, local=f.local_nnz, bounds=f.row_bounds,
                   rows=f.row_nnz.tolist(), nprod=f.total_nprod)
        if rank == 0:
            exp = O.spgemm(a, a)
            out["exp_rows"] = np.diff(np.asarray(exp.rpt)).tolist()
            out["exp_nprod"] = O.compute_nprod(a, a)[1]
        q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_forecast():
    """forecast_distributed: the per-rank symbolic counts add up to the single-shot C."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_forecast, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=120) for _ in procs), key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = outs
    assert r0["bounds"] == r1["bounds"]
    assert r0["rows"] + r1["rows"] == r0["exp_rows"]
    assert r0["total"] == r1["total"] == sum(r0["exp_rows"]) == r0["local"] + r1["local"]
    assert r0["nprod"] == r0["exp_nprod"]


@pytest.mark.parametrize("case", ["square", "rect"])
def test_two_rank_gloo_matches_single_shot(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda d: d["rank"])
    r0, r1 = outs
    assert r0["bounds"] == r1["bounds"]                  # same split derived independently
    assert r0["offsets"] == r1["offsets"] == [0, r0["nnz"]]
    assert r0["same_pattern"] and r0["bitwise"]
    assert r0["total_nprod"] == r0["exp_total_nprod"]
    lo, hi = r0["halves"]
    assert abs(lo - hi) <= max(lo, hi) * 0.05 + 400     # balanced by nprod


def test_nprod_split_properties():
    from paper_2206_07244_b200.distributed import nprod_split
    rng = np.random.default_rng(0)
    nprod = rng.integers(0, 1000, 10_000)
    for parts in (1, 2, 3, 8):
        b = nprod_split(nprod, parts)
        assert b[0] == 0 and b[-1] == nprod.size and len(b) == parts + 1
        assert all(x <= y for x, y in zip(b, b[1:]))
        sums = [nprod[b[g]:b[g + 1]].sum() for g in range(parts)]
        assert max(sums) - min(sums) <= 2 * nprod.max() + 1
    assert nprod_split(np.zeros(5, np.int64), 2) == [0, 2, 5]
    assert nprod_split(np.zeros(0, np.int64), 3) == [0, 0, 0, 0]


def test_stitch_offsets():
    from paper_2206_07244_b200.api import CsrMatrix
    from paper_2206_07244_b200.distributed import slice_rows, stitch
    a = random_csr(50, 40, 0.1, 3)
    parts = [slice_rows(a, 0, 17), slice_rows(a, 17, 17), slice_rows(a, 17, 50)]
    s = stitch(parts, a.cols)
    assert isinstance(s, CsrMatrix) and s == a


def _worker_streamed(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from oracle import oracle as O
    from paper_2206_07244_b200 import synthetic as S
    from paper_2206_07244_b200.distributed import slice_rows, stream_square_distributed
    from paper_2206_07244_b200.tiled import checksum_of
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = S.random_values(S.rmat(9, 16, seed=9), 4) if rank == 0 else None

        def local_stream(B, rows, nprod):  # the per-rank tiles, checked with the oracle on CPU
            from paper_2206_07244_b200.api import CsrMatrix
            c = O.spgemm(slice_rows(B, rows.start, rows.stop), B)
            c = CsrMatrix(c.rows, c.cols, c.rpt, c.col, c.val)
            cs = checksum_of(c)
            # global row numbers in the pattern hash, as tiled.stream_multiply reports them
            rr = np.repeat(np.arange(c.rows, dtype=np.uint64) + np.uint64(rows.start + 1), np.diff(c.rpt))
            cs.pattern_hash = int(np.sum((c.col.astype(np.uint64) + np.uint64(1)) * rr, dtype=np.uint64))
            return cs

        res = stream_square_distributed(b, local_nprod=lambda x, y: O.compute_nprod(x, y)[0],
                                        local_stream=local_stream)
        t = torch.tensor([res.local.nnz, res.local.pattern_hash & ((1 << 62) - 1)], dtype=torch.int64)
        parts = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, t)
        out = dict(rank=rank, bounds=res.row_bounds, total=res.total_nprod, nnz=[int(p[0]) for p in parts],
                   hashes=[int(p[1]) for p in parts], hash_full=res.local.pattern_hash, vsum=res.local.val_sum)
        if rank == 0:
            from paper_2206_07244_b200.api import CsrMatrix
            exp = O.spgemm(b, b)
            full = checksum_of(CsrMatrix(exp.rows, exp.cols, exp.rpt, exp.col, exp.val))
            out["exp_nnz"], out["exp_hash"], out["exp_vsum"] = full.nnz, full.pattern_hash, full.val_sum
            out["exp_total"] = O.compute_nprod(b, b)[1]
        q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_streamed_square_with_async_broadcast():
    """stream_square_distributed (bench.py's multi-GPU step): B broadcast with rpt/col/val
    in flight together, K1 after rpt+col, the nprod split, each rank's row block --
    the ranks' checksums add up to the single-shot product's."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_streamed, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=180) for _ in procs), key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = outs
    assert r0["bounds"] == r1["bounds"]
    assert r0["total"] == r1["total"] == r0["exp_total"]
    assert sum(r0["nnz"]) == r0["exp_nnz"]
    assert (r0["hash_full"] + r1["hash_full"]) % (1 << 64) == r0["exp_hash"]
    assert abs(r0["vsum"] + r1["vsum"] - r0["exp_vsum"]) <= 1e-9 * max(1.0, abs(r0["exp_vsum"]))
