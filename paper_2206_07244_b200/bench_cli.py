"""spgemm-bench on the B200 (reference: tools/spgemm_bench_main.cpp, core/src/bench.cpp)
-- SURVEY.md §8(f) "next" row 1: the reference's benchmark CLI surface over the GPU path.

  python -m paper_2206_07244_b200.bench_cli --matrix A.mtx [--b B.mtx] [--repeat 10] [--csv out.csv]
  python -m paper_2206_07244_b200.bench_cli --random 10000,10000,0.001 --seed 1 --verify

Same flags, output (print_report / stats_line), 14-field CSV schema and exit codes
(0 ok, 1 usage, 2 I/O or parse, 3 verify failed) as the reference. ``run_benchmark``
times 1 warm-up + ``--repeat`` full ``multiply`` calls (host in, host out, wall clock
around each whole call, as bench.cpp:46-96) and reports the mean CUDA-event step
timings. Differences, by necessity:

* ``--threads`` sets ``SpgemmOptions.workers`` (reported only: the GPU has no pool);
* ``--random`` draws from numpy's PCG64 (the reference's libstdc++ binomial/uniform
  distributions are not portable): each row gets Binomial(cols, density) distinct
  columns with values U[-1, 1);
* ``--verify`` checks against an independent CPU product written here (expand,
  stable sort by (row, col), per-entry sums) with the reference's 1e-10 tolerance;
  products above 2e8 intermediate products are skipped unless --force-verify
  (the reference skips its known-slow matrices the same way).
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from dataclasses import dataclass, field

import numpy as np

from . import api
from .matrix_market import ParseError, read_matrix_market_csr

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_VERIFY_FAILED = 0, 1, 2, 3
VERIFY_TOLERANCE = 1e-10  # bench.hpp:44
VERIFY_LIMIT_NPROD = 200_000_000
SLOW_VERIFY = ("delaunay_n24", "cage15", "wb-edu", "cop20k_A", "hood", "pwtk", "pdb1HYS")
CSV_HEADER = "name,rows,nnz_a,nprod,nnz_c,cr,t_setup,t_symbin,t_sym,t_rpt,t_numbin,t_num,t_total,gflops"


@dataclass
class BenchReport:
    """bench.hpp:12-24."""
    name: str = ""
    rows: int = 0
    nnz_a: int = 0
    nprod: int = 0
    nnz_c: int = 0
    cr: float = 0.0
    steps: api.StepTimings = field(default_factory=api.StepTimings)
    mean_total: float = 0.0
    gflops: float = 0.0
    repeats: int = 0
    workers: int = 0


def run_benchmark(name, a, b, options: api.SpgemmOptions, repeats=10, warmup=True, on_run=None):
    """bench.cpp:46-96: 1 warm-up (validated) + repeats timed multiplies."""
    if repeats < 1:
        raise api.InvalidArgument("run_benchmark: repeats must be >= 1")
    if warmup:
        t0 = time.perf_counter()
        warm = api.multiply(a, b, options)
        secs = time.perf_counter() - t0
        if on_run:
            on_run(0, True, secs)
        rep = api.validate_csr(warm.c)
        if not rep.ok():
            raise RuntimeError("spgemm produced an invalid matrix:\n" + rep.to_string())
    keys = ("setup", "sym_binning", "symbolic", "rpt_alloc", "num_binning", "numeric", "cleanup", "total")
    sums = dict.fromkeys(keys, 0.0)
    wall = 0.0
    last = None
    for r in range(repeats):
        t0 = time.perf_counter()
        last = api.multiply(a, b, options)
        secs = time.perf_counter() - t0
        if on_run:
            on_run(r + 1, False, secs)
        wall += secs
        for k in keys:
            sums[k] += getattr(last.timings, k)
    report = BenchReport(name=name, rows=last.stats.rows, nnz_a=last.stats.nnz, nprod=last.stats.total_nprod,
                         nnz_c=last.stats.nnz_of_product, cr=last.stats.cr,
                         steps=api.StepTimings(**{k: v / repeats for k, v in sums.items()}),
                         mean_total=wall / repeats, repeats=repeats, workers=last.workers)
    report.gflops = 2.0 * report.nprod / report.mean_total / 1e9 if report.mean_total > 0 else 0.0
    return report, last


def csv_row(r: BenchReport) -> str:
    """bench.cpp:127-143."""
    s = r.steps
    return ",".join([r.name, str(r.rows), str(r.nnz_a), str(r.nprod), str(r.nnz_c), f"{r.cr:.2f}",
                     f"{s.setup:.6f}", f"{s.sym_binning:.6f}", f"{s.symbolic:.6f}", f"{s.rpt_alloc:.6f}",
                     f"{s.num_binning:.6f}", f"{s.numeric:.6f}", f"{r.mean_total:.6f}", f"{r.gflops:.6f}"])


def stats_line(r: BenchReport) -> str:
    """bench.cpp:145-148."""
    return f"{r.name}: {r.rows}, {r.nnz_a}, {r.nprod}, {r.nnz_c}, {r.cr:.2f}"


def print_report(r: BenchReport, out=sys.stdout) -> None:
    """bench.cpp:150-169."""
    s = r.steps
    out.write(f"matrix:        {r.name}\nrows:          {r.rows}\nnnz(A):        {r.nnz_a}\n"
              f"n_prod:        {r.nprod}\nnnz(C):        {r.nnz_c}\nCR:            {r.cr:.2f}\n"
              f"workers:       {r.workers}\nrepeats:       {r.repeats} (+1 warmup)\n"
              f"mean total:    {r.mean_total:.6f} s\ngflops:        {r.gflops:.6f}\nstep means (s):\n"
              f"  setup        {s.setup:.6f}\n  sym binning  {s.sym_binning:.6f}\n"
              f"  symbolic     {s.symbolic:.6f}\n  rpt/alloc    {s.rpt_alloc:.6f}\n"
              f"  num binning  {s.num_binning:.6f}\n  numeric      {s.numeric:.6f}\n"
              f"  cleanup      {s.cleanup:.6f}\n")


def append_csv(path: str, r: BenchReport) -> None:
    """spgemm_bench_main.cpp:50-62: header once, one record per call."""
    need_header = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a") as f:
        if need_header:
            f.write(CSV_HEADER + "\n")
        f.write(csv_row(r) + "\n")


def random_csr(rows: int, cols: int, density: float, seed: int) -> api.CsrMatrix:
    """Binomial(cols, density) distinct sorted columns per row, values U[-1,1) (PCG64)."""
    if rows < 0 or cols < 0 or not 0.0 <= density <= 1.0:
        raise api.InvalidArgument("random_csr: bad shape or density")
    rng = np.random.Generator(np.random.PCG64(seed))
    counts = rng.binomial(cols, density, size=rows) if cols > 0 else np.zeros(rows, np.int64)
    rpt = np.zeros(rows + 1, np.int64)
    np.cumsum(counts, out=rpt[1:])
    col = np.empty(int(rpt[-1]), np.int32)
    for i in range(rows):
        if counts[i]:
            col[rpt[i]:rpt[i + 1]] = np.sort(rng.choice(cols, size=int(counts[i]), replace=False))
    val = rng.uniform(-1.0, 1.0, size=col.size)
    return api.CsrMatrix(rows, cols, rpt, col, val)


def cpu_product(a: api.CsrMatrix, b: api.CsrMatrix) -> api.CsrMatrix:
    """Independent CPU product for --verify: expand the products, stable-sort by
    (row, col), sum each entry's products."""
    a, b = a.to_host(), b.to_host()
    alen = np.diff(a.rpt)
    arow = np.repeat(np.arange(a.rows, dtype=np.int64), alen)
    blen = np.diff(b.rpt)[a.col]
    prow = np.repeat(arow, blen)
    starts = np.repeat(b.rpt[a.col], blen)
    offs = np.arange(int(blen.sum()), dtype=np.int64) - np.repeat(np.cumsum(blen) - blen, blen)
    bidx = starts + offs
    pcol = b.col[bidx].astype(np.int64)
    pval = np.repeat(a.val, blen) * b.val[bidx]
    key = prow * max(b.cols, 1) + pcol
    order = np.argsort(key, kind="stable")
    ks = key[order]
    first = np.ones(ks.size, bool)
    first[1:] = ks[1:] != ks[:-1]
    starts_u = np.nonzero(first)[0]
    vals = np.add.reduceat(pval[order], starts_u) if ks.size else np.zeros(0)
    uniq = ks[first]
    rows = uniq // max(b.cols, 1)
    rpt = np.zeros(a.rows + 1, np.int64)
    np.add.at(rpt, rows + 1, 1)
    np.cumsum(rpt, out=rpt)
    return api.CsrMatrix(a.rows, b.cols, rpt, (uniq % max(b.cols, 1)).astype(np.int32), vals)


def verify(a, b, c, tol=VERIFY_TOLERANCE):
    """bench.cpp:98-125: (PASS?, detail)."""
    exp = cpu_product(a, b)
    if not api.same_pattern(exp, c):
        return False, f"output pattern differs from the reference product (nnz {c.nnz()} vs {exp.nnz()})"
    err = api.max_relative_error(exp, c)
    if err > tol:
        return False, f"max relative value error {err:.6f} exceeds {tol:.6f}"
    return True, f"max relative value error {err:.6f}"


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (CLI11 convention of the reference)
        self.print_usage(sys.stderr)
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def main(argv=None) -> int:
    p = _Parser(description="B200 two-phase SpGEMM benchmark (computes A*A, or A*B with --b)")
    p.add_argument("--matrix", default="", help="Matrix Market file for A")
    p.add_argument("--b", default="", help="Matrix Market file for B (default: B = A)")
    p.add_argument("--sym-range", default="1.2x", choices=["1x", "1.2x", "1.5x"])
    p.add_argument("--num-range", default="2x", choices=["1x", "1.5x", "2x", "3x"])
    p.add_argument("--threads", type=int, default=0, help="reported as workers (GPU run)")
    p.add_argument("--repeat", type=int, default=10)
    p.add_argument("--verify", action="store_true")
    p.add_argument("--force-verify", action="store_true")
    p.add_argument("--stats-only", action="store_true")
    p.add_argument("--csv", default="")
    p.add_argument("--no-overlap", action="store_true")
    p.add_argument("--deterministic", dest="deterministic", action="store_true", default=True)
    p.add_argument("--no-deterministic", dest="deterministic", action="store_false")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--random", default="", help="rows,cols,density (alternative to --matrix)")
    p.add_argument("--device", type=int, default=0)
    try:
        args = p.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code in (0, None) else EXIT_USAGE
    if bool(args.matrix) == bool(args.random):
        sys.stderr.write("error: exactly one of --matrix or --random is required\n")
        return EXIT_USAGE
    if args.repeat < 1:
        sys.stderr.write("error: --repeat must be positive\n")
        return EXIT_USAGE
    spec = None
    if args.random:
        try:
            r, c, d = args.random.split(",")
            spec = (int(r), int(c), float(d))
            if spec[0] < 0 or spec[1] < 0 or not 0.0 <= spec[2] <= 1.0:
                raise ValueError
        except ValueError:
            sys.stderr.write("error: --random expects rows,cols,density (density in [0,1])\n")
            return EXIT_USAGE
    try:
        if args.matrix:
            a = read_matrix_market_csr(args.matrix)
            name = os.path.splitext(os.path.basename(args.matrix))[0]
        else:
            a = random_csr(spec[0], spec[1], spec[2], args.seed)
            name = f"random_{spec[0]}x{spec[1]}"
        b = read_matrix_market_csr(args.b) if args.b else a
        opts = api.SpgemmOptions(sym_preset="sym_" + args.sym_range, num_preset="num_" + args.num_range,
                                 workers=args.threads, overlap=not args.no_overlap,
                                 deterministic=args.deterministic)
        on_run = None if args.stats_only else (
            lambda run, warm, secs: print(f"run {run}{' (warmup)' if warm else ''}: {secs:g} s"))
        a_dev = a.to_device(args.device)
        b_dev = a_dev if b is a else b.to_device(args.device)
        report, out = run_benchmark(name, a_dev, b_dev, opts, repeats=1 if args.stats_only else args.repeat,
                                    warmup=not args.stats_only, on_run=on_run)
        if args.stats_only:
            print(stats_line(report))
        else:
            print_report(report)
        if args.csv:
            append_csv(args.csv, report)
        if args.verify or args.force_verify:
            if (name in SLOW_VERIFY or report.nprod > VERIFY_LIMIT_NPROD) and not args.force_verify:
                print(f"verify: SKIP ({name} is slow under the CPU check; use --force-verify)")
            else:
                ok, detail = verify(a, b, out.c)
                print(f"verify: {'PASS' if ok else 'FAIL'} ({detail})")
                if not ok:
                    return EXIT_VERIFY_FAILED
        return EXIT_OK
    except (ParseError, api.InvalidArgument, OSError, ValueError) as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
