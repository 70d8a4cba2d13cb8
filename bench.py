#!/usr/bin/env python
"""bench.py -- SpGEMM GFLOPS (2*nprod/time) on B200, BASELINE.json's metric.

Default workload (N=1): BASELINE.json configs[1], C = A*A with A the 3-D 27-point
stencil on a 128^3 grid (2.1M rows, 55.7M nnz, nprod 1.489e9). One *step* = one
full SpGEMM (setup, binning, symbolic, row_ptr scan + C allocation, numeric) with
A resident in HBM; C is freed (stream-ordered) after each step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1|2|3|4]
  python bench.py --impl reference ...   # the reference CPU pipeline (oracle/_ref)

N>1 (torchrun, one process per GPU, NCCL): weak scaling. The global matrix is
the 27-point stencil on 128 x 128 x (128*N); rank 0 builds it and broadcasts it
(B = A) over NVLink once; every rank computes nprod (K1) and the deterministic
nprod-prefix row split itself, then multiplies its row block.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpGEMM GFLOPS (2*nprod/time)"
UNIT = "GFLOPS"
CONFIG_NAMES = {
    1: "C=A*A 2D 5-pt Poisson 1024^2",
    2: "C=A*A 3D 27-pt stencil 128^3",
    3: "C=A*A R-MAT scale 20 ef 16",
    4: "RAP: A*P then R*(AP), 3D 7-pt Poisson 128^3, trilinear P",
    5: "C=A*A R-MAT scale 24 ef 16, row blocks x 2^20-column windows, C streamed to checksums",
}


def csr_bytes(rows, nnz):
    """8*(rows+1) + 4*nnz + 8*nnz."""
    return 8 * (rows + 1) + 12 * nnz


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# -------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled in-process through NVML every 200 ms
    during the timed region (nvidia-smi polling contends with the CUDA driver
    and perturbs a ms-scale step loop; tools/sampler_probe.py measures it)."""

    REASONS = {  # NVML clocks-event-reason bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index=0, period=0.2):
        self.index, self.period = index, period
        self.samples = []
        self._stop = threading.Event()
        self.ok = False

    def _sample(self):
        import pynvml
        self.samples.append((time.time(), pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM),
                             pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)))

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return

        def run():
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(self.period)
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()

    def stop(self):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()  # always at least one sample at the end of the region

    def summary(self, t0, t1):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        inwin = [x for x in self.samples if t0 - 0.25 <= x[0] <= t1 + 0.25] or self.samples
        reasons = sorted({n for _, _, bits in inwin for n, b in self.REASONS.items() if bits & b})
        return {"sm_mhz": statistics.median(c for _, c, _ in inwin), "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(inwin), "source": "nvml"}


# -------------------------------------------------------- CPU baseline
def cpu_baseline(a, rows_frac=1.0, runs=2):
    """The reference CPU pipeline (oracle/_ref, all host threads) on a bounded sample."""
    from oracle import oracle as O
    CsrMatrix = type(a)
    m = a.to_host()
    if rows_frac < 1.0:
        r0 = int(m.rows * (0.5 - rows_frac / 2))
        r1 = r0 + int(m.rows * rows_frac)
        rpt = m.rpt[r0:r1 + 1] - m.rpt[r0]
        sample = CsrMatrix(r1 - r0, m.cols, rpt, m.col[m.rpt[r0]:m.rpt[r1]], m.val[m.rpt[r0]:m.rpt[r1]])
        desc = f"rows [{r0},{r1}) of A times A"
    else:
        sample, desc = m, "the full product"
    cores = os.cpu_count() or 1
    if O.ref_available():
        _, info = O.ref_multiply(sample, m)  # warm-up
        ts = []
        for _ in range(runs):
            t0 = time.perf_counter()
            _, info = O.ref_multiply(sample, m)
            ts.append(time.perf_counter() - t0)
        t = sum(ts) / len(ts)
        return {"value": 2 * info["total_nprod"] / t / 1e9, "unit": UNIT, "cores": info["workers"] or cores,
                "kind": "reference", "cpu": cpu_model(), "host_threads": cores,
                "sample": f"oracle/_ref spgemm::multiply (workers={info['workers']}) on {desc}, "
                          f"1 warm-up + {runs} timed, mean {t:.3f} s"}
    # C restatement (single thread) on a smaller sample
    t0 = time.perf_counter()
    O.spgemm(sample, m)
    t = time.perf_counter() - t0
    _, nprod = O.compute_nprod(sample, m)
    return {"value": 2 * nprod / t / 1e9, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"oracle/spgemm_oracle.c (1 thread) on {desc}, 1 run {t:.3f} s"}


# ---------------------------------------------------------- workloads
def build_workload(cfg):
    from paper_2206_07244_b200 import synthetic as S
    mats = S.config_matrices(cfg)
    return list(mats)


def stencil_weak(n_ranks):
    from paper_2206_07244_b200 import synthetic as S
    offs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    return S._stencil((128, 128, 128 * n_ranks), offs, 26.0, -1.0)


def launch_bytes(sg, torch, a, b, device, device_tensors):
    """Algorithmic bytes of one product C = A*B (A + B + C, each
    8*(rows+1) + 12*nnz) and their split over the per-bin launches: a launch
    for symbolic bin j (tag "s<j>") or numeric bin j ("n<j>") is charged its
    rows' A bytes, their C bytes (numeric, and the speculative numeric of the
    symbolic phase) or their 8-byte counts (symbolic), plus B's bytes times the
    rows' share of the product's nprod (B is gathered per product)."""
    import numpy as np
    nprod, total = sg.compute_nprod(a, b, device=device)
    dm, out = sg.multiply_device(a, b, device=device)
    crpt = torch.as_tensor(device_tensors(dm)[0]).cpu().numpy() if dm.rows >= 0 else None
    dm.free()
    arpt = a.rpt.cpu().numpy() if hasattr(a.rpt, "cpu") else np.asarray(a.rpt)
    nnza = np.diff(arpt)
    nnzc = np.diff(crpt)
    bbytes = csr_bytes(b.rows, b.nnz())
    step = csr_bytes(a.rows, int(nnza.sum())) + bbytes + csr_bytes(a.rows, int(nnzc.sum()))
    sym = np.asarray(sg.symbolic_preset("sym_1.2x").upper[:-1])
    num = np.asarray(sg.numeric_preset("num_2x").upper[:-1])
    sbin = np.searchsorted(sym, nprod, side="left")
    nbin = np.searchsorted(num, nnzc, side="left")
    share = nprod.astype(np.float64) / max(total, 1) * bbytes
    out_b = {}
    for j in range(8):
        m = sbin == j
        if m.any():
            base = float((16 + 12 * nnza[m]).sum() + share[m].sum())
            out_b[f"s{j}"] = base + 8.0 * int(m.sum())                       # symbolic: the row counts
            out_b[f"s{j}+c"] = base + float((16 + 12 * nnzc[m]).sum())      # speculative numeric: C rows
        m = nbin == j
        if m.any():
            out_b[f"n{j}"] = float((16 + 12 * nnza[m]).sum() + share[m].sum() + (16 + 12 * nnzc[m]).sum())
    return step, out_b


# ---------------------------------------------------------------- main
def cpu_model() -> str:
    """The host CPU (state the core count and CPU model)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_synthetic():
    """paper_2206_07244_b200/synthetic.py loaded by file path: the reference arm
    builds the same matrices without importing the package (so the sm_100a
    library is never loaded into its process)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_spgemm_synthetic_host",
                                                  os.path.join(ROOT, "paper_2206_07244_b200", "synthetic.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def run_reference(args):
    """The reference's own CPU pipeline (oracle/_ref: the unmodified proj/core
    compiled in place) through its public spgemm::multiply, with every host
    thread, on this arm's workload: the full product for configs 1, 2 and 4 (4 =
    A*P then R*(AP), both on the host), a bounded row sample for configs 3 and 5,
    whose C does not fit host memory."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    S = host_synthetic()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    workload = CONFIG_NAMES[args.config]
    if args.config == 5:
        mats = [S.rmat(args.rmat_scale, 16, seed=args.rmat_scale)] * 2
    else:
        mats = list(S.config_matrices(args.config))
    a = mats[0]
    frac = {1: 1.0, 2: 1.0, 3: 0.02, 4: 1.0, 5: 0.0005 if args.rmat_scale >= 24 else 0.0002}[args.config]
    r0 = int(a.rows * (0.5 - frac / 2)) if frac < 1 else 0
    r1 = r0 + int(a.rows * frac) if frac < 1 else a.rows
    if frac < 1:
        rpt = a.rpt[r0:r1 + 1] - a.rpt[r0]
        sample = S.CsrMatrix(r1 - r0, a.cols, rpt, a.col[a.rpt[r0]:a.rpt[r1]], a.val[a.rpt[r0]:a.rpt[r1]])
        desc = f"rows [{r0},{r1}) of A times B (C does not fit host memory)"
    else:
        sample = a
        desc = "the full product" + (" chain A*P then R*(AP)" if args.config == 4 else "")
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return

    def step():
        if args.config == 4:
            _, p, r = mats
            ap, i1 = O.ref_multiply(a, p)
            _, i2 = O.ref_multiply(r, ap)
            return i1["total_nprod"] + i2["total_nprod"], i1["workers"]
        _, info = O.ref_multiply(sample, mats[1])
        return info["total_nprod"], info["workers"]

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    nprod = 0
    workers = 0
    for _ in range(args.steps):
        n, workers = step()
        nprod += n
    t = time.perf_counter() - t0
    value = 2 * nprod / t / 1e9
    cores = os.cpu_count() or 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "nprod_per_step": nprod // args.steps,
                   **({"sample_rows": [r0, r1]} if frac < 1 else {})},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers or cores, "kind": "reference",
                         "cpu": cpu_model(), "host_threads": cores,
                         "sample": f"oracle/_ref spgemm::multiply (workers={workers}) on {desc}, "
                                   f"{args.warmup} warm-up + {args.steps} timed steps"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=None, choices=[1, 2, 3, 4, 5],
                    help="default: 2 (the headline) on one GPU; 5 (strong scaling) on N > 1")
    ap.add_argument("--rmat-scale", type=int, default=None,
                    help="config 5's R-MAT scale (24 = BASELINE; default 24 on one GPU, 22 for the N > 1 scaling run)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config is None:
        args.config = 5 if world_env > 1 else 2
    if args.rmat_scale is None:
        args.rmat_scale = 22 if world_env > 1 else 24
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 5:
        return run_config5(args)

    import torch
    import paper_2206_07244_b200 as sg
    from paper_2206_07244_b200.api import CsrMatrix

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; SPGEMM_DIST_BACKEND=gloo lets several ranks share one GPU
    # to exercise the N>1 code path on a single-GPU box (timings then meaningless)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("SPGEMM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    ctx = sg.get_context(local)
    peak, peak_kind = load_peaks()

    # ------------------------------------------------------------ operands
    bcast_s = None
    if world == 1:
        mats = build_workload(args.config)
        host_ops = mats
        dev = [m.to_device(local) for m in mats]
        pairs = [(dev[0], dev[1])] if args.config != 4 else None
        workload = CONFIG_NAMES[args.config]
    else:
        if args.config != 2:
            raise SystemExit("multi-GPU bench runs the weak-scaled 27-point stencil (config 2)")
        from paper_2206_07244_b200.distributed import broadcast_csr, nprod_split, slice_rows
        g = stencil_weak(world) if rank == 0 else None
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        B = broadcast_csr(g.to_device(local) if rank == 0 else None, 0, torch.device("cuda", local))
        torch.cuda.synchronize()
        bcast_s = time.perf_counter() - t0
        nprod, _ = sg.compute_nprod(B, B, device=local)   # K1 on every rank: identical split, no collective
        bounds = nprod_split(nprod, world)
        A_loc = slice_rows(B, bounds[rank], bounds[rank + 1])
        pairs = [(A_loc, B)]
        host_ops = None
        workload = f"C=A*A 3D 27-pt stencil 128x128x{128 * world} (weak: 128^3 rows/GPU), nprod-balanced row blocks"

    def one_step():
        if pairs is not None:
            tot = 0
            for a, b in pairs:
                dm, out = sg.multiply_device(a, b, device=local)
                tot += out.stats.total_nprod
                dm.free()
            return tot
        # RAP chain: AP stays on device and feeds R*(AP)
        a, p, r = dev
        dm1, o1 = sg.multiply_device(a, p, device=local)
        ap = CsrMatrix(dm1.rows, dm1.cols, *device_tensors(dm1))
        dm2, o2 = sg.multiply_device(r, ap, device=local)
        dm2.free()
        dm1.free()
        return o1.stats.total_nprod + o2.stats.total_nprod

    def device_tensors(dm):
        # zero-copy torch views of a DeviceMatrix (CUDA array interface)
        class _V:
            def __init__(self, ptr, n, typestr):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                                 "version": 3}
        r = torch.as_tensor(_V(dm.ptrs[0], dm.rows + 1, "<i8"), device="cuda")
        c = torch.as_tensor(_V(dm.ptrs[1], dm.nnz, "<i4"), device="cuda") if dm.nnz else \
            torch.zeros(0, dtype=torch.int32, device="cuda")
        v = torch.as_tensor(_V(dm.ptrs[2], dm.nnz, "<f8"), device="cuda") if dm.nnz else \
            torch.zeros(0, dtype=torch.float64, device="cuda")
        return r, c, v

    # ------------------------------------------------------------- warm-up
    # W untimed steps, then more (untimed, at most ~3 s) until two consecutive
    # steps agree within 5%: a fresh box's first seconds (pool growth, clocks,
    # lazy module loading) must not leak into the timed region.
    for _ in range(max(3, args.warmup)):
        nprod_step = one_step()
    torch.cuda.synchronize()
    t_end = time.perf_counter() + 3.0
    prev = None
    while time.perf_counter() < t_end:
        t0 = time.perf_counter()
        one_step()
        torch.cuda.synchronize()
        cur = time.perf_counter() - t0
        if prev is not None and abs(cur - prev) <= 0.05 * prev:
            break
        prev = cur
    if dist:
        dist.barrier()

    # ------------------------------------------------------------- timed
    # Pass 1 (value): K steps bracketed by barrier + synchronize, CUDA events on
    # the library's stream. Pass 2 (roofline): the same K steps again with every
    # kernel bracketed by events on its own stream (per-kernel device time), so
    # the per-launch events cannot perturb pass 1.
    import gc
    stream = torch.cuda.ExternalStream(ctx.stream)
    clocks = ClockSampler(local)

    def timed_pass(profile):
        if profile:
            ctx.profile_summary()  # clear
            ctx.set_profiling(True)
        launches0 = ctx.kernel_launches
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        gc.disable()
        tw0 = time.time()
        ev0.record(stream)
        tot = 0
        dbg = os.environ.get("SPGEMM_BENCH_DEBUG")
        for _ in range(args.steps):
            ts = time.perf_counter()
            tot += one_step()
            if dbg:
                print(f"step {1e3 * (time.perf_counter() - ts):.3f} ms", file=sys.stderr)
        ev1.record(stream)
        torch.cuda.synchronize()
        tw1 = time.time()
        gc.enable()
        if dist:
            dist.barrier()
        kern = None
        if profile:
            ctx.set_profiling(False)
            kern = ctx.profile_summary()
        return ev0.elapsed_time(ev1), tot, ctx.kernel_launches - launches0, kern, tw0, tw1

    if rank == 0:
        clocks.start()
    t_ms, total_nprod, launches, _, tw0, tw1 = timed_pass(False)
    if rank == 0:
        clocks.stop()
    t_prof_ms, _, _, kernels, _, _ = timed_pass(True)
    t_max = t_ms
    nprod_all = total_nprod
    if dist:
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
        nn = torch.tensor([total_nprod], dtype=torch.int64, device="cuda")
        dist.all_reduce(nn)
        nprod_all = int(nn.item())
    value = 2 * nprod_all / (t_max * 1e-3) / 1e9
    ms_per_step = t_max / args.steps

    # ------------------------------------------------------------ roofline
    # Algorithmic bytes of one SpGEMM: A + B + C compulsory bytes.
    def unit_bytes():
        if pairs is not None:
            out = 0
            for a, b in pairs:
                c_rows, c_nnz = a.rows, None
                out += csr_bytes(a.rows, a.nnz()) + csr_bytes(b.rows, b.nnz())
            return out
        return None

    roof = None
    step_roof = None
    if rank == 0 and kernels:
        # the dominant launch record: "<kernel>#s<bin>" / "#n<bin>" (phase, bin)
        name, (n_launch, ms_total) = max(kernels.items(), key=lambda kv: kv[1][1])
        avg_s = ms_total / n_launch * 1e-3
        prods = pairs if pairs is not None else [(dev[0], dev[1]), None]
        tag_bytes = {}   # per step, summed over the step's products
        step_bytes = 0
        for pr in prods:
            if pr is None:  # RAP: R * (AP), AP from the chain's first product
                a, p, r = dev
                dm1, _ = sg.multiply_device(a, p, device=local)
                pr = (r, CsrMatrix(dm1.rows, dm1.cols, *device_tensors(dm1)))
                b_keep = dm1
            else:
                b_keep = None
            sb, tb = launch_bytes(sg, torch, pr[0], pr[1], local, device_tensors)
            step_bytes += sb
            for k, v in tb.items():
                tag_bytes[k] = tag_bytes.get(k, 0) + v
            if b_keep is not None:
                b_keep.free()
        tag = name.rsplit("#", 1)[1] if "#" in name else None
        if tag and tag[0] == "s" and "spec" in name:
            tag += "+c"
        launches_per_step = max(1, n_launch // args.steps)
        if tag in tag_bytes:
            kernel_bytes = tag_bytes[tag] / launches_per_step
            attribution = (f"rows of {'symbolic' if tag[0] == 's' else 'numeric'} bin {tag[1:2]}: their A rows"
                           f"{' and C rows' if tag[0] == 'n' or 'spec' in name else ' and counts'}, plus B's "
                           f"bytes times the rows' share of nprod")
        else:
            kernel_bytes = step_bytes
            attribution = "whole step (kernel not bound to a bin)"
        achieved = kernel_bytes / avg_s / 1e9
        traffic = None
        prof_path = os.path.join(ROOT, "profiles", f"ncu_config{args.config}_summary.json")
        if os.path.exists(prof_path):
            with open(prof_path) as f:
                prof = json.load(f)
            k = prof.get("kernels", {}).get(name.split("#")[0])
            if k:
                traffic = k.get("dram_bytes_per_launch")
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                "algorithmic_bytes_per_launch": kernel_bytes, "bytes_attribution": attribution,
                "avg_launch_ms": avg_s * 1e3,
                "share_of_step": ms_total / t_prof_ms, "profiled_pass_ms_per_step": t_prof_ms / args.steps,
                "profiled_pass": "second timed pass with per-launch events; bins serialised on one stream so each launch is timed alone"}
        step_roof = {"bytes_per_step": step_bytes, "achieved": step_bytes / (ms_per_step * 1e-3) / 1e9,
                     "frac": step_bytes / (ms_per_step * 1e-3) / 1e9 / peak}

    # ----------------------------------------------------------------- e2e
    e2e = None
    if rank == 0 and host_ops is not None and args.config in (1, 2):
        e2e = run_e2e(sg, torch, host_ops[0], max(8, args.e2e_steps or args.steps // 2), local)
    elif rank == 0:
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "note": "e2e measured on configs 1-2 (config 3's C is 116.7 GB; config 4 chains on device)"}

    # ------------------------------------------------------------ baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            frac = {1: 1.0, 2: 1.0, 3: 0.02, 4: 1.0}[args.config]
            cpu = cpu_baseline(host_ops[0], rows_frac=frac)
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable", "sample": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "nprod_per_step": nprod_all // args.steps,
                       "l2": "inputs larger than L2 (A is 0.67 GB vs 126 MB L2)" if args.config == 2 else
                       "L2 not flushed between steps",
                       "parallelism": f"row-block dp{world}" if world > 1 else "single GPU",
                       "b_broadcast_s": bcast_s},
            "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "kernels_ms": {k: round(v[1], 4) for k, v in sorted(kernels.items(), key=lambda kv: -kv[1][1])},
            "clocks": clocks.summary(tw0, tw1),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_config5(args):
    """BASELINE config 5: R-MAT, C = A*A with a TB-scale C, row
    partitioned across the ranks -- strong scaling (the product is fixed). Rank 0
    holds A (= B). One step, timed from the broadcast's start to the last tile
    (SURVEY §8(e) "Timing"): B is broadcast over NCCL with rpt, col and val in
    flight together; every rank runs K1 as soon as rpt and col have landed
    (B.val still arriving) and derives the same nprod-balanced row split; its
    rows are streamed through row-block x 2^20-column-window tiles
    (paper_2206_07244_b200/tiled.py), each tile a full device pipeline whose C is
    reduced to checksums and freed. Max time over ranks; GFLOPS counts the whole
    product's 2*nprod. The ranks' checksums are combined and reported."""
    import torch
    import paper_2206_07244_b200 as sg
    from paper_2206_07244_b200 import synthetic as S
    from paper_2206_07244_b200 import tiled as T
    from paper_2206_07244_b200.distributed import stream_square_distributed

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("SPGEMM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    ctx = sg.get_context(local)
    t0 = time.perf_counter()
    a_host = S.rmat(args.rmat_scale, 16, seed=args.rmat_scale) if rank == 0 else None
    gen_s = time.perf_counter() - t0
    a_dev = a_host.to_device(local) if rank == 0 else None
    budget = int(os.environ.get("SPGEMM_TILE_BUDGET", 12_000_000_000))
    workers = int(os.environ.get("SPGEMM_TILE_WORKERS", 3))  # measured best at scale 22 (1: 4.2 s, 3: 3.5 s)
    bcast = "on" if world > 1 else "none (one GPU)"

    def local_stream(B, rows, nprod):
        return T.stream_multiply(B, B, rows=rows, nprod=nprod, b_windows=T.split_columns(B), budget=budget,
                                 device=local, workers=workers)

    def step():
        l0 = ctx.kernel_launches
        if dist:
            res = stream_square_distributed(a_dev if rank == 0 else None, device=dev, local_stream=local_stream)
            rep, total = res.local, res.total_nprod
        else:
            nprod, total = sg.compute_nprod(a_dev, a_dev, device=local)
            rep = local_stream(a_dev, range(0, a_dev.rows), nprod)
        return rep, total, ctx.kernel_launches - l0

    for _ in range(max(3, args.warmup)):
        step()
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    if rank == 0:
        clocks.start()
    tw0 = time.time()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    launches = 0
    nprod_done = 0
    local_nprod = 0
    for _ in range(args.steps):
        rep, total, nl = step()
        nprod_done += total
        local_nprod += rep.total_nprod
        launches += nl + rep.kernel_launches
    ev1.record(stream)
    torch.cuda.synchronize()
    tw1 = time.time()
    if rank == 0:
        clocks.stop()
    t_ms = ev0.elapsed_time(ev1)
    nnz_all, vsum, phash = rep.nnz, rep.val_sum, rep.pattern_hash
    per_rank_ms = [t_ms]
    if dist:
        dist.barrier()
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        gathered = [torch.zeros(1, dtype=torch.float64, device="cuda") for _ in range(world)]
        dist.all_gather(gathered, tt)
        per_rank_ms = [float(g.item()) for g in gathered]
        t_ms = max(per_rank_ms)
        nn = torch.tensor([rep.nnz, local_nprod, launches], dtype=torch.int64, device="cuda")
        dist.all_reduce(nn)
        nnz_all, local_sum, launches = (int(x) for x in nn.tolist())
        assert local_sum == nprod_done, "the ranks' row blocks must cover the product exactly"
        vs = torch.tensor([vsum], dtype=torch.float64, device="cuda")
        dist.all_reduce(vs)
        vsum = float(vs.item())
        hh = torch.tensor([phash & ((1 << 62) - 1)], dtype=torch.int64, device="cuda")
        dist.all_reduce(hh)
        phash = int(hh.item())
    if rank == 0:
        value = 2 * nprod_done / (t_ms * 1e-3) / 1e9
        ms = t_ms / args.steps
        step_bytes = 2 * csr_bytes(a_host.rows, a_host.nnz()) + csr_bytes(a_host.rows, nnz_all)
        peak, peak_kind = load_peaks()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[5].replace("scale 24", f"scale {args.rmat_scale}"),
                       "rmat_scale": args.rmat_scale,
                       "nprod_per_step": nprod_done // args.steps, "nnz_c": nnz_all, "window_cols": T.WINDOW,
                       "tile_budget_nprod": budget, "tile_workers": workers,
                       "parallelism": f"row-block dp{world}", "b_broadcast": bcast,
                       "timed": "broadcast start (N>1) to the last tile of every rank, max over ranks",
                       "l2": "inputs larger than L2", "generate_s": round(gen_s, 1),
                       "per_rank_ms_per_step": [round(x / args.steps, 2) for x in per_rank_ms],
                       "note": ("strong scaling at R-MAT scale %d (scale 24 = BASELINE config 5: "
                                "bench.py --config 5 --rmat-scale 24)" % args.rmat_scale)
                       if args.rmat_scale != 24 else "BASELINE config 5"},
            "roofline": None,
            "step_roofline": {"bytes_per_step": step_bytes, "achieved": step_bytes / (ms * 1e-3) / 1e9,
                              "frac": step_bytes / (ms * 1e-3) / 1e9 / peak, "peak": peak, "peak_source": peak_kind},
            "cpu_baseline": None,
            "e2e": {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                    "note": "C is TB-scale: streamed to checksums on the device, never copied to the host"},
            "checksums": {"nnz": nnz_all, "val_sum": vsum, "pattern_hash_mod_2^62": phash & ((1 << 62) - 1)},
            "gpu_launches": launches,
            "clocks": clocks.summary(tw0, tw1),
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                line["cpu_baseline"] = cpu_baseline(a_host, rows_frac=0.0005, runs=1)
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable",
                                        "sample": str(e)}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_e2e(sg, torch, a_host, min_steps, device):
    """Same metric through the public API with host buffers: each step copies A from
    pinned host memory (B aliases A), multiplies, and reads C back into pinned host
    buffers -- one synchronous `multiply_into` call per step (`value`; inside it, row
    blocks' C downloads overlap the next blocks' kernels). Reported alongside: the same
    as separate calls (`separate_calls_value`: run_device, then download_into) and the
    pipelined mode of an application issuing independent products back to back
    (`pipelined_value`: step i's C download via DeviceMatrix.download_async on the
    context's copy lane overlaps step i+1's upload and kernels, at most two
    products in flight; the timed region ends when every download has landed)."""
    from paper_2206_07244_b200.api import CsrMatrix
    pr = torch.from_numpy(a_host.rpt).pin_memory()
    pc = torch.from_numpy(a_host.col).pin_memory()
    pv = torch.from_numpy(a_host.val).pin_memory()
    a = CsrMatrix(a_host.rows, a_host.cols, pr.numpy(), pc.numpy(), pv.numpy())
    h2d = pr.numel() * 8 + pc.numel() * 4 + pv.numel() * 8
    p = sg.SpgemmPipeline(a, a, device=device)
    dm, out = p.run_device()
    p.close()
    nnz = dm.nnz
    dm.free()
    orpt = torch.empty(a.rows + 1, dtype=torch.int64).pin_memory()
    ocol = torch.empty(nnz, dtype=torch.int32).pin_memory()
    oval = torch.empty(nnz, dtype=torch.float64).pin_memory()
    d2h = orpt.numel() * 8 + ocol.numel() * 4 + oval.numel() * 8
    ctx = sg.get_context(device)

    issued = [0]

    def step_pipelined():
        p = sg.SpgemmPipeline(a, a, device=device)
        dm, out = p.run_device()
        p.close()
        dm.download_async(orpt.numpy(), ocol.numpy(), oval.numpy(), release=True)
        dm.free()
        issued[0] += 1
        if issued[0] % 2 == 0:  # double buffering: at most two products in flight
            ctx.wait_downloads()
        return out.stats.total_nprod

    def step_into():
        n, out = sg.multiply_into(a, a, orpt.numpy(), ocol.numpy(), oval.numpy(), device=device,
                                  parts=int(os.environ.get("SPGEMM_INTO_PARTS", 0)))
        return out.stats.total_nprod

    def step_sync():
        t0 = time.perf_counter()
        p = sg.SpgemmPipeline(a, a, device=device)
        dm, out = p.run_device()
        p.close()
        t1 = time.perf_counter()
        dm.download_into(orpt.numpy(), ocol.numpy(), oval.numpy())
        dm.free()
        if os.environ.get("SPGEMM_BENCH_DEBUG"):
            print(f"e2e sync run {1e3 * (t1 - t0):.2f} ms d2h {1e3 * (time.perf_counter() - t1):.2f} ms",
                  file=sys.stderr)
        return out.stats.total_nprod

    dbg = os.environ.get("SPGEMM_BENCH_DEBUG")

    def timed(step, steps):
        import gc
        for _ in range(3):  # warm-up: the pool grows to hold the products in flight
            step()
        ctx.wait_downloads()
        torch.cuda.synchronize()
        if steps is None:  # at least ~1 s of timed work, so a one-off stall cannot dominate
            t1 = time.perf_counter()
            step()
            ctx.wait_downloads()
            steps = int(min(400, max(min_steps, 1.0 / max(time.perf_counter() - t1, 1e-4))))
        gc.collect()
        gc.disable()  # as in the device-timed region: no collector pauses inside the timing
        t0 = time.perf_counter()
        nprod = 0
        for _ in range(steps):
            ts = time.perf_counter()
            nprod += step()
            if dbg:
                print(f"e2e step {1e3 * (time.perf_counter() - ts):.3f} ms", file=sys.stderr)
        tw = time.perf_counter()
        ctx.wait_downloads()
        torch.cuda.synchronize()
        if dbg:
            print(f"e2e final wait {1e3 * (time.perf_counter() - tw):.3f} ms", file=sys.stderr)
        gc.enable()
        return nprod, time.perf_counter() - t0, steps

    nprod, t, steps = timed(step_into, None)
    nprod_s, t_s, _ = timed(step_sync, steps)
    nprod_p, t_p, _ = timed(step_pipelined, steps)
    return {"value": 2 * nprod / t / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "steps": steps, "ms_per_step": t / steps * 1e3,
            "mode": "one synchronous multiply_into call per step (host A in, host C out; row blocks' C "
                    "downloads overlap the next blocks' kernels)",
            "separate_calls_value": 2 * nprod_s / t_s / 1e9, "separate_calls_ms_per_step": t_s / steps * 1e3,
            "pipelined_value": 2 * nprod_p / t_p / 1e9, "pipelined_ms_per_step": t_p / steps * 1e3}


if __name__ == "__main__":
    main()
