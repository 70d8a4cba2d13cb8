"""Python mirror of the reference's SpGEMM API (proj/core/include/spgemm), over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API so the
parity tests read like the reference's own tests:

=====================================  ============================================
reference (file:line)                  here
=====================================  ============================================
``CsrMatrix`` (csr.hpp:45-63)           :class:`CsrMatrix` (numpy on host, or torch CUDA tensors)
``SpgemmOptions`` (pipeline.hpp:78-91)  :class:`SpgemmOptions`
``SpgemmPipeline`` (pipeline.hpp:119)   :class:`SpgemmPipeline` (step API + ``run``)
``multiply`` (pipeline.hpp:170-173)     :func:`multiply` / :func:`multiply_device`
``preset``/``classify`` (binning.hpp)   :func:`preset`, :func:`classify`, :func:`preset_names`
``make_execution_plan`` (pipeline.cpp:64-87)  :func:`make_execution_plan`
``run_binning`` (binning.cpp:281-313)   :func:`run_binning` (runs the device kernels)
``build_rpt`` (pipeline.hpp:114-115)    :func:`build_rpt` (device scan)
``compute_nprod`` (reference.hpp:15)    :func:`compute_nprod` (device kernel K1)
=====================================  ============================================

Exceptions: ``std::invalid_argument`` -> :class:`InvalidArgument` (a ``ValueError``),
``std::logic_error`` -> :class:`LogicError`, ``std::overflow_error`` -> ``OverflowError``,
``std::bad_alloc`` -> ``MemoryError``. All compute runs in the sm_100a library.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as _c

# ----------------------------------------------------------------- constants
kNumBins = _c.NUM_BINS
kNoUpperBound = _c.NO_UPPER_BOUND
kDefaultSymPreset = "sym_1.2x"
kDefaultNumPreset = "num_2x"
kDefaultChunkRows = 4096
kMaxSymbolicTableSize = 24575
kMaxNumericTableSize = 8191
kSymbolicSpillThreshold = kMaxSymbolicTableSize * 4 // 5
kEmptySlot = -1
SYMBOLIC, NUMERIC = 0, 1


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class LogicError(RuntimeError):
    """std::logic_error."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the library."""


class NoDevice(RuntimeError):
    """No sm_100 GPU visible."""


def _check(status: int) -> None:
    if status == _c.OK:
        return
    msg = _c.last_error()
    if status == _c.INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == _c.LOGIC_ERROR:
        raise LogicError(msg)
    if status == _c.OVERFLOW:
        raise OverflowError(msg)
    if status == _c.OUT_OF_MEMORY:
        raise MemoryError(msg)
    if status == _c.NO_DEVICE:
        raise NoDevice(msg)
    raise CudaError(msg)


# ------------------------------------------------------------------- context
class Context:
    """One (host thread, device) context: streams, events, pinned scratch."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(_c.lib.spgemm_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)

    def close(self):
        if self.handle:
            _c.lib.spgemm_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def num_sms(self) -> int:
        return _c.lib.spgemm_ctx_num_sms(self.handle)

    @property
    def kernel_launches(self) -> int:
        return _c.lib.spgemm_ctx_kernel_launches(self.handle)

    @property
    def stream(self) -> int:
        return _c.lib.spgemm_ctx_stream(self.handle) or 0

    def wait_downloads(self):
        """Wait for every DeviceMatrix.download_async issued on this context."""
        _check(_c.lib.spgemm_ctx_wait_downloads(self.handle))

    def synchronize(self):
        _check(_c.lib.spgemm_ctx_synchronize(self.handle))

    def set_profiling(self, on: bool):
        """Bracket every kernel launch with CUDA events on its own stream."""
        _c.lib.spgemm_ctx_set_profiling(self.handle, int(bool(on)))

    def pool_stats(self):
        """(reserved, used) bytes of the device's stream-ordered memory pool."""
        r, u = C.c_uint64(), C.c_uint64()
        _check(_c.lib.spgemm_ctx_pool_stats(self.handle, C.byref(r), C.byref(u)))
        return r.value, u.value

    def trim(self, keep_bytes: int = 0) -> None:
        """Return cached scratch and pooled HBM beyond keep_bytes to the driver."""
        _check(_c.lib.spgemm_ctx_trim(self.handle, int(keep_bytes)))

    def profile_summary(self) -> dict:
        """{kernel name: (launches, total ms)} since the last call (synchronises)."""
        buf = (_c.KernelTime * 64)()
        n = _c.lib.spgemm_ctx_profile_summary(self.handle, buf, 64)
        return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms)) for i in range(n)}


_tls = threading.local()


def get_context(device: Optional[int] = None) -> Context:
    if device is None:
        device = 0
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    ctx = cache.get(device)
    if ctx is None:
        ctx = cache[device] = Context(device)
    return ctx


# --------------------------------------------------------------- containers
def _is_torch_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


class CsrMatrix:
    """csr.hpp:45-63. rpt int64[rows+1], col int32[nnz], val float64[nnz].

    Arrays may be numpy (host) or torch CUDA tensors (device-resident operands,
    borrowed by the library without a copy).
    """

    def __init__(self, rows: int = 0, cols: int = 0, rpt=None, col=None, val=None):
        self.rows = int(rows)
        self.cols = int(cols)
        if rpt is None:
            rpt = np.zeros(self.rows + 1, np.int64)
        if col is None:
            col = np.zeros(0, np.int32)
        if val is None:
            val = np.zeros(0, np.float64)
        self.on_device = _is_torch_cuda(rpt)
        if self.on_device:
            import torch
            self.rpt = rpt.to(torch.int64).contiguous()
            self.col = col.to(torch.int32).contiguous()
            self.val = val.to(torch.float64).contiguous()
        else:
            self.rpt = np.ascontiguousarray(rpt, np.int64)
            self.col = np.ascontiguousarray(col, np.int32)
            self.val = np.ascontiguousarray(val, np.float64)

    def nnz(self) -> int:
        if self.on_device:
            return int(self.rpt[-1].item()) if self.rpt.numel() else 0
        return int(self.rpt[-1]) if self.rpt.size else 0

    def row_nnz(self, i: int) -> int:
        return int(self.rpt[i + 1] - self.rpt[i])

    def row_cols(self, i: int):
        return self.col[int(self.rpt[i]):int(self.rpt[i + 1])]

    def row_vals(self, i: int):
        return self.val[int(self.rpt[i]):int(self.rpt[i + 1])]

    def to_host(self) -> "CsrMatrix":
        if not self.on_device:
            return self
        return CsrMatrix(self.rows, self.cols, self.rpt.cpu().numpy(), self.col.cpu().numpy(),
                         self.val.cpu().numpy())

    def to_device(self, device: int = 0) -> "CsrMatrix":
        import torch
        if self.on_device:
            return self
        d = torch.device("cuda", device)
        return CsrMatrix(self.rows, self.cols, torch.from_numpy(self.rpt).to(d), torch.from_numpy(self.col).to(d),
                         torch.from_numpy(self.val).to(d))

    def __eq__(self, other) -> bool:
        if not isinstance(other, CsrMatrix):
            return NotImplemented
        a, b = self.to_host(), other.to_host()
        return (a.rows == b.rows and a.cols == b.cols and np.array_equal(a.rpt, b.rpt)
                and np.array_equal(a.col, b.col) and np.array_equal(a.val, b.val))

    def __repr__(self) -> str:
        return f"CsrMatrix({self.rows}x{self.cols}, nnz={self.nnz()}, {'device' if self.on_device else 'host'})"

    def _view(self) -> _c.CsrView:
        if self.on_device:
            if self.rpt.numel() != self.rows + 1:
                raise InvalidArgument("rpt length is not rows+1")
            return _c.CsrView(self.rows, self.cols, self.rpt.data_ptr(), self.col.data_ptr() or None,
                              self.val.data_ptr() or None, 1)
        if self.rpt.size != self.rows + 1:
            raise InvalidArgument("rpt length is not rows+1")
        return _c.CsrView(self.rows, self.cols, self.rpt.ctypes.data, self.col.ctypes.data,
                          self.val.ctypes.data, 0)


def same_pattern(a: CsrMatrix, b: CsrMatrix) -> bool:
    """csr.hpp:105-107."""
    a, b = a.to_host(), b.to_host()
    return a.rows == b.rows and a.cols == b.cols and np.array_equal(a.rpt, b.rpt) and np.array_equal(a.col, b.col)


def max_relative_error(a: CsrMatrix, b: CsrMatrix) -> float:
    """csr.cpp:169-181: max |x-y| / max(|x|,|y|,1); patterns must match."""
    if not same_pattern(a, b):
        raise InvalidArgument("max_relative_error: patterns differ")
    x, y = a.to_host().val, b.to_host().val
    if x.size == 0:
        return 0.0
    denom = np.maximum(np.maximum(np.abs(x), np.abs(y)), 1.0)
    return float(np.max(np.abs(x - y) / denom))


@dataclass
class Violation:
    row: int
    message: str


@dataclass
class ValidationReport:
    violations: List[Violation] = field(default_factory=list)

    def ok(self) -> bool:
        return not self.violations

    def to_string(self) -> str:
        return "".join((f"row {v.row}: " if v.row >= 0 else "") + v.message + "\n" for v in self.violations)


def validate_csr(m: CsrMatrix) -> ValidationReport:
    """csr.cpp:98-151 (vectorised; reports the same violation kinds)."""
    m = m.to_host()
    rep = ValidationReport()
    add = lambda r, s: rep.violations.append(Violation(int(r), s))  # noqa: E731
    if m.rows < 0 or m.cols < 0:
        add(-1, "negative matrix shape")
        return rep
    if m.rpt.size != m.rows + 1:
        add(-1, "rpt length is not rows+1")
        return rep
    if m.rpt[0] != 0:
        add(-1, "rpt[0] is not 0")
    d = np.diff(m.rpt)
    for i in np.nonzero(d < 0)[0]:
        add(i, f"non-monotone rpt at row {i}")
    if m.rpt[-1] != m.col.size:
        add(-1, "rpt[rows] does not equal len(col)")
    if m.col.size != m.val.size:
        add(-1, "len(col) does not equal len(val)")
    if m.col.size and (d >= 0).all() and m.rpt[-1] == m.col.size:
        row_of = np.repeat(np.arange(m.rows), d)
        bad = np.nonzero((m.col < 0) | (m.col >= m.cols))[0]
        for p in bad:
            add(row_of[p], f"column index {m.col[p]} out of range")
        same_row = row_of[1:] == row_of[:-1]
        dup = np.nonzero(same_row & (m.col[1:] == m.col[:-1]))[0]
        for p in dup:
            add(row_of[p + 1], f"duplicate column {m.col[p + 1]}")
        uns = np.nonzero(same_row & (m.col[1:] < m.col[:-1]))[0]
        for p in uns:
            add(row_of[p + 1], f"unsorted columns ({m.col[p]} before {m.col[p + 1]})")
    return rep


# ----------------------------------------------------------------- binning
@dataclass
class BinConfig:
    """binning.hpp:29-34."""
    phase: int = SYMBOLIC
    upper: List[int] = field(default_factory=lambda: [0] * kNumBins)
    table_size: List[int] = field(default_factory=lambda: [0] * kNumBins)
    preset_name: str = ""

    def _c(self) -> _c.BinConfig:
        c = _c.BinConfig()
        c.phase = self.phase
        for j in range(kNumBins):
            c.upper[j] = int(self.upper[j])
            c.table_size[j] = int(self.table_size[j])
        c.preset_name = self.preset_name.encode()[:15]
        return c

    @staticmethod
    def _from(c: _c.BinConfig) -> "BinConfig":
        return BinConfig(int(c.phase), list(c.upper), list(c.table_size), c.preset_name.decode())


def preset(phase: int, name: str) -> BinConfig:
    """binning.cpp:33-66; InvalidArgument for unknown names."""
    c = _c.BinConfig()
    _check(_c.lib.spgemm_preset(int(phase), name.encode(), C.byref(c)))
    return BinConfig._from(c)


def symbolic_preset(name: str) -> BinConfig:
    return preset(SYMBOLIC, name)


def numeric_preset(name: str) -> BinConfig:
    return preset(NUMERIC, name)


def preset_names(phase: int) -> List[str]:
    if phase == SYMBOLIC:
        return ["sym_1x", "sym_1.2x", "sym_1.5x"]
    return ["num_1x", "num_1.5x", "num_2x", "num_3x"]


def classify(value: int, config: BinConfig) -> int:
    """binning.cpp:75-82."""
    c = config._c()
    return int(_c.lib.spgemm_classify(int(value), C.byref(c)))


@dataclass
class BinStrategy:
    bin: int
    metric_lo: int
    metric_hi: int
    table_size: int
    tier: str  # "fixed" | "heap"
    spill_threshold: int
    launch_rank: int


@dataclass
class ExecutionPlan:
    """pipeline.hpp:31-39."""
    phase: int
    config: BinConfig
    strategies: List[BinStrategy]
    _order: List[int]

    def launch_order(self) -> List[int]:
        return list(self._order)

    @staticmethod
    def _from(p: _c.Plan) -> "ExecutionPlan":
        st = [BinStrategy(int(s.bin), int(s.metric_lo), int(s.metric_hi), int(s.table_size),
                          "fixed" if s.tier == 0 else "heap", int(s.spill_threshold), int(s.launch_rank))
              for s in p.strategies]
        return ExecutionPlan(int(p.phase), BinConfig._from(p.config), st, list(p.launch_order))


def make_execution_plan(config: BinConfig) -> ExecutionPlan:
    """pipeline.cpp:64-87."""
    c = config._c()
    p = _c.Plan()
    _check(_c.lib.spgemm_make_plan(C.byref(c), C.byref(p)))
    return ExecutionPlan._from(p)


@dataclass
class BinningResult:
    """binning.hpp:90-102 (bins as a host int64 array)."""
    bins: np.ndarray
    bin_size: List[int]
    bin_offset: List[int]
    max_metric: int
    total_metric: int
    fast_path: bool

    def segment(self, j: int) -> np.ndarray:
        return self.bins[self.bin_offset[j]:self.bin_offset[j] + self.bin_size[j]]


def run_binning(metric, config: BinConfig, deterministic: bool = True, device: Optional[int] = None) -> BinningResult:
    """binning.cpp:281-313 on the GPU (pass 1, offsets, stable scatter / fast path)."""
    m = np.ascontiguousarray(metric, np.int64)
    bins = np.empty(m.size, np.int64)
    info = _c.BinningInfo()
    c = config._c()
    ctx = get_context(device)
    _check(_c.lib.spgemm_run_binning(ctx.handle, m.ctypes.data, m.size, C.byref(c), int(deterministic),
                                     bins.ctypes.data, C.byref(info)))
    return BinningResult(bins, list(info.bin_size), list(info.bin_offset), int(info.max_metric),
                         int(info.total_metric), bool(info.fast_path))


def build_rpt(rpt_region: np.ndarray, device: Optional[int] = None) -> int:
    """pipeline.cpp:104-107: in-place exclusive sum (device scan); returns the total."""
    if rpt_region.dtype != np.int64 or not rpt_region.flags.c_contiguous:
        raise InvalidArgument("build_rpt needs a contiguous int64 array")
    total = C.c_int64()
    _check(_c.lib.spgemm_build_rpt(get_context(device).handle, rpt_region.ctypes.data, rpt_region.size,
                                   C.byref(total)))
    return int(total.value)


def compute_nprod(a: CsrMatrix, b: CsrMatrix, out: Optional[np.ndarray] = None, device: Optional[int] = None):
    """reference.cpp:37-55 on the device (kernel K1). Returns (out, total)."""
    if a.cols != b.rows:
        raise InvalidArgument("compute_nprod: a.cols != b.rows")
    if out is None:
        out = np.empty(a.rows, np.int64)
    if out.size != a.rows:
        raise InvalidArgument("compute_nprod: out length != a.rows")
    total = C.c_int64()
    va, vb = a._view(), b._view()
    if a.on_device or b.on_device:
        _order_device_operands(get_context(device), a, b)
    _check(_c.lib.spgemm_compute_nprod(get_context(device).handle, C.byref(va), C.byref(vb), out.ctypes.data,
                                       C.byref(total)))
    return out, int(total.value)


# ----------------------------------------------------------------- pipeline
@dataclass
class AllocStats:
    """pipeline.hpp:45-50 (filled after the run)."""
    metadata_calls: int = 0
    metadata_bytes: int = 0
    output_calls: int = 0
    output_bytes: int = 0


@dataclass
class SpgemmOptions:
    """pipeline.hpp:78-91."""
    sym_preset: str = kDefaultSymPreset
    num_preset: str = kDefaultNumPreset
    workers: int = 0
    overlap: bool = True
    deterministic: bool = True
    chunk_rows: int = kDefaultChunkRows
    hash_scale: int = 107
    alloc_stats: Optional[AllocStats] = None
    sym_launch_order: Optional[Sequence[int]] = None
    num_launch_order: Optional[Sequence[int]] = None
    # deterministic=True (default): every row, heap tier included, folds in the
    # reference's order (bitwise); deterministic=False lets heap-tier rows
    # accumulate with fp64 atomics (1e-12). B200 extension: ordered_heap forces
    # the ordered heap tier even with deterministic=False.
    ordered_heap: bool = False

    def _c(self) -> _c.Options:
        o = _c.Options()
        _c.lib.spgemm_options_default(C.byref(o))
        o.sym_preset = self.sym_preset.encode()[:15]
        o.num_preset = self.num_preset.encode()[:15]
        o.workers = int(self.workers)
        o.overlap = int(bool(self.overlap))
        o.deterministic = int(bool(self.deterministic))
        o.chunk_rows = int(self.chunk_rows)
        o.hash_scale = int(self.hash_scale)
        o.ordered_heap = int(bool(self.ordered_heap))
        if self.sym_launch_order is not None:
            if len(self.sym_launch_order) != kNumBins:
                raise InvalidArgument("launch order must be a permutation of the bin indices")
            o.has_sym_launch_order = 1
            for j, v in enumerate(self.sym_launch_order):
                o.sym_launch_order[j] = int(v)
        if self.num_launch_order is not None:
            if len(self.num_launch_order) != kNumBins:
                raise InvalidArgument("launch order must be a permutation of the bin indices")
            o.has_num_launch_order = 1
            for j, v in enumerate(self.num_launch_order):
                o.num_launch_order[j] = int(v)
        return o


@dataclass
class StepTimings:
    """pipeline.hpp:93-102 (seconds, CUDA-event measured)."""
    setup: float = 0.0
    sym_binning: float = 0.0
    symbolic: float = 0.0
    rpt_alloc: float = 0.0
    num_binning: float = 0.0
    numeric: float = 0.0
    cleanup: float = 0.0
    total: float = 0.0


@dataclass
class MatrixStats:
    """reference.hpp:23-31."""
    rows: int = 0
    nnz: int = 0
    nnz_per_row_mean: float = 0.0
    max_nnz_per_row: int = 0
    total_nprod: int = 0
    nnz_of_product: int = 0
    cr: float = 0.0


@dataclass
class SpgemmOutput:
    """pipeline.hpp:104-110."""
    c: CsrMatrix
    stats: MatrixStats
    timings: StepTimings
    spilled_rows: int = 0
    workers: int = 0


def _output_from(rep: _c.Report, c: CsrMatrix, options: Optional[SpgemmOptions]) -> SpgemmOutput:
    t = rep.timings
    timings = StepTimings(t.setup, t.sym_binning, t.symbolic, t.rpt_alloc, t.num_binning, t.numeric, t.cleanup,
                          t.total)
    stats = MatrixStats(rep.rows, rep.nnz, rep.nnz_per_row_mean, rep.max_nnz_per_row, rep.total_nprod,
                        rep.nnz_of_product, rep.cr)
    if options is not None and options.alloc_stats is not None:
        s = options.alloc_stats
        s.metadata_calls += rep.metadata_calls
        s.metadata_bytes += rep.metadata_bytes
        s.output_calls += rep.output_calls
        s.output_bytes += rep.output_bytes
    return SpgemmOutput(c, stats, timings, int(rep.spilled_rows), int(rep.workers))


class DeviceMatrix:
    """A result C kept in HBM (spgemm_matrix). Free with :meth:`free` (or GC)."""

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
        _c.lib.spgemm_matrix_shape(handle, C.byref(r), C.byref(c), C.byref(n))
        self.rows, self.cols, self.nnz = r.value, c.value, n.value
        pr, pc, pv = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _c.lib.spgemm_matrix_device_ptrs(handle, C.byref(pr), C.byref(pc), C.byref(pv))
        self.ptrs = (pr.value, pc.value, pv.value)

    def download_into(self, rpt: np.ndarray, col: np.ndarray, val: np.ndarray) -> None:
        """D2H of C into caller buffers (pinned buffers give full PCIe/C2C bandwidth)."""
        if rpt.size < self.rows + 1 or col.size < self.nnz or val.size < self.nnz:
            raise InvalidArgument("download_into: buffers too small")
        _check(_c.lib.spgemm_matrix_download(self.ctx.handle, self.handle, rpt.ctypes.data,
                                             col.ctypes.data if self.nnz else None,
                                             val.ctypes.data if self.nnz else None))

    def download_async(self, rpt: np.ndarray, col: np.ndarray, val: np.ndarray, release: bool = True) -> None:
        """Stream-ordered D2H of C on the context's copy lane (returns at once; the copy
        overlaps whatever is queued next). Buffers (pinned for full speed) are valid after
        Context.wait_downloads(). release=True frees C's device buffers behind the copy."""
        if rpt.size < self.rows + 1 or col.size < self.nnz or val.size < self.nnz:
            raise InvalidArgument("download_async: buffers too small")
        _check(_c.lib.spgemm_matrix_download_async(self.ctx.handle, self.handle, rpt.ctypes.data,
                                                   col.ctypes.data if self.nnz else None,
                                                   val.ctypes.data if self.nnz else None, int(bool(release))))

    def checksum(self, row_offset: int = 0, col_offset: int = 0):
        """(sum of values, sum of (col+col_offset+1)*(row+row_offset+1) mod 2^64) on the device."""
        v = C.c_double()
        h = C.c_uint64()
        _check(_c.lib.spgemm_matrix_checksum(self.ctx.handle, self.handle, int(row_offset), int(col_offset),
                                             C.byref(v), C.byref(h)))
        return v.value, h.value

    def as_operand(self) -> CsrMatrix:
        """C as a device-resident operand of the next product (zero copy; the
        reference's chained --b / RAP flow without the host round trip). The
        returned CsrMatrix keeps this DeviceMatrix alive; its tensors are valid
        until :meth:`free`."""
        import torch
        v = _c.CsrView()
        _check(_c.lib.spgemm_matrix_as_operand(self.handle, C.byref(v)))
        dev = torch.device("cuda", self.ctx.device)

        def wrap(ptr, n, typestr, dtype):
            if n == 0 or not ptr:
                return torch.zeros(0, dtype=dtype, device=dev)
            cai = type("_Cai", (), {"__cuda_array_interface__": {"shape": (n,), "typestr": typestr,
                                                                  "data": (ptr, False), "version": 3}})()
            return torch.as_tensor(cai, device=dev)

        m = CsrMatrix(self.rows, self.cols, wrap(v.rpt, self.rows + 1, "<i8", torch.int64),
                      wrap(v.col, self.nnz, "<i4", torch.int32), wrap(v.val, self.nnz, "<f8", torch.float64))
        m._owner = self  # the buffers belong to this DeviceMatrix
        return m

    def download(self) -> CsrMatrix:
        rpt = np.empty(self.rows + 1, np.int64)
        col = np.empty(self.nnz, np.int32)
        val = np.empty(self.nnz, np.float64)
        self.download_into(rpt, col, val)
        return CsrMatrix(self.rows, self.cols, rpt, col, val)

    def free(self):
        if self.handle:
            _c.lib.spgemm_matrix_free(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass


def _order_device_operands(ctx: "Context", *ms: CsrMatrix) -> None:
    """Device operands must live on the context's device, and the product is
    ordered after the work torch has queued on its current stream there (the
    producer of the tensors): an event on that stream, waited on by the
    context's stream -- no host synchronisation."""
    import torch
    for m in ms:
        if m.on_device:
            for t in (m.rpt, m.col, m.val):
                if t.device.index != ctx.device:
                    raise InvalidArgument(f"device operand on cuda:{t.device.index}, context on cuda:{ctx.device}")
    stream = torch.cuda.current_stream(ctx.device)
    _check(_c.lib.spgemm_ctx_wait_stream(ctx.handle, C.c_void_p(stream.cuda_stream or None)))


class SpgemmPipeline:
    """pipeline.hpp:119-168: six-step two-phase SpGEMM, drivable one step at a time."""

    def __init__(self, a: CsrMatrix, b: CsrMatrix, options: Optional[SpgemmOptions] = None,
                 device: Optional[int] = None):
        self._options = options if options is not None else SpgemmOptions()
        self._ctx = get_context(device)
        self._a, self._b = a, b  # borrowed: keep alive for the pipeline's lifetime
        self._rows = a.rows
        self._cols = b.cols
        self._va, self._vb = a._view(), b._view()
        if a.on_device or b.on_device:
            _order_device_operands(self._ctx, a, b)
        if (not a.on_device and not b.on_device and a is not b and a.rpt is b.rpt):
            self._vb = self._va
        h = C.c_void_p()
        _check(_c.lib.spgemm_pipeline_create(self._ctx.handle, C.byref(self._va), C.byref(self._vb),
                                             C.byref(self._options._c()), C.byref(h)))
        self._h = h

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def close(self):
        if getattr(self, "_h", None):
            _c.lib.spgemm_pipeline_destroy(self._h)
            self._h = None

    def setup(self):
        _check(_c.lib.spgemm_pipeline_setup(self._h))

    def symbolic_binning(self):
        _check(_c.lib.spgemm_pipeline_symbolic_binning(self._h))

    def run_symbolic(self):
        _check(_c.lib.spgemm_pipeline_run_symbolic(self._h))

    def numeric_binning(self):
        _check(_c.lib.spgemm_pipeline_numeric_binning(self._h))

    def finalize_rpt(self) -> int:
        t = C.c_int64()
        _check(_c.lib.spgemm_pipeline_finalize_rpt(self._h, C.byref(t)))
        return int(t.value)

    def run_numeric(self):
        _check(_c.lib.spgemm_pipeline_run_numeric(self._h))

    def _finish_report(self) -> _c.Report:
        rep = _c.Report()
        _check(_c.lib.spgemm_pipeline_finish(self._h, C.byref(rep)))
        return rep

    def _take(self) -> DeviceMatrix:
        m = C.c_void_p()
        _check(_c.lib.spgemm_pipeline_take_result(self._h, C.byref(m)))
        return DeviceMatrix(m, self._ctx)

    def finish(self) -> SpgemmOutput:
        rep = self._finish_report()
        dm = self._take()
        c = dm.download()
        dm.free()
        return _output_from(rep, c, self._options)

    def run(self) -> SpgemmOutput:
        rep = _c.Report()
        _check(_c.lib.spgemm_pipeline_run(self._h, C.byref(rep)))
        dm = self._take()
        c = dm.download()
        dm.free()
        return _output_from(rep, c, self._options)

    def run_device(self):
        """run() keeping C in HBM: returns (DeviceMatrix, SpgemmOutput without c)."""
        rep = _c.Report()
        _check(_c.lib.spgemm_pipeline_run(self._h, C.byref(rep)))
        dm = self._take()
        return dm, _output_from(rep, None, self._options)

    def rpt_region(self) -> np.ndarray:
        out = np.empty(self._rows, np.int64)
        _check(_c.lib.spgemm_pipeline_rpt_region(self._h, out.ctypes.data if out.size else None))
        return out

    def binning(self) -> BinningResult:
        info = _c.BinningInfo()
        bins = np.empty(self._rows, np.int64)
        _check(_c.lib.spgemm_pipeline_binning(self._h, C.byref(info), bins.ctypes.data if bins.size else None))
        return BinningResult(bins, list(info.bin_size), list(info.bin_offset), int(info.max_metric),
                             int(info.total_metric), bool(info.fast_path))

    def _plan(self, phase) -> ExecutionPlan:
        p = _c.Plan()
        _check(_c.lib.spgemm_pipeline_plan(self._h, phase, C.byref(p)))
        return ExecutionPlan._from(p)

    def symbolic_plan(self) -> ExecutionPlan:
        return self._plan(SYMBOLIC)

    def numeric_plan(self) -> ExecutionPlan:
        return self._plan(NUMERIC)


def multiply(a: CsrMatrix, b: CsrMatrix, options: Optional[SpgemmOptions] = None,
             device: Optional[int] = None) -> SpgemmOutput:
    """pipeline.hpp:170-173: C = A*B on the GPU, C returned on the host."""
    p = SpgemmPipeline(a, b, options, device)
    try:
        return p.run()
    finally:
        p.close()


def multiply_multi(a: CsrMatrix, b: CsrMatrix, options: Optional[SpgemmOptions] = None,
                   devices: Sequence[int] = (0,)) -> SpgemmOutput:
    """SURVEY.md §8(e) inside one process (C ABI spgemm_multiply_multi): A's rows split
    by the nprod prefix sum over `devices` (an index may repeat: one fresh context per
    entry), every block multiplied by all of B on its own host thread, C stitched on the
    host. `row_bounds` of the split is attached to the returned SpgemmOutput."""
    devices = list(devices)
    if not devices:
        raise InvalidArgument("multiply_multi: no devices")
    ctxs = [Context(d) for d in devices]
    n = len(ctxs)
    handles = (C.c_void_p * n)(*[c.handle for c in ctxs])
    slices = (C.c_void_p * n)()
    bounds = (C.c_int64 * (n + 1))()
    rep = _c.Report()
    va, vb = a._view(), b._view()
    opts = options._c() if options is not None else None
    try:
        _check(_c.lib.spgemm_multiply_multi(handles, n, C.byref(va), C.byref(vb),
                                            C.byref(opts) if opts is not None else None, slices, bounds,
                                            C.byref(rep)))
        nnz = int(rep.nnz_of_product)
        rpt = np.empty(a.rows + 1, np.int64)
        col = np.empty(nnz, np.int32)
        val = np.empty(nnz, np.float64)
        try:
            _check(_c.lib.spgemm_matrices_download_stitched(handles, slices, n, rpt.ctypes.data,
                                                            col.ctypes.data if nnz else None,
                                                            val.ctypes.data if nnz else None))
        finally:
            for h in slices:
                if h:
                    _c.lib.spgemm_matrix_free(h)
    finally:
        for c in ctxs:
            c.close()
    out = _output_from(rep, CsrMatrix(a.rows, b.cols, rpt, col, val), options)
    out.row_bounds = [int(x) for x in bounds]
    return out


def multiply_into(a: CsrMatrix, b: CsrMatrix, rpt: np.ndarray, col: np.ndarray, val: np.ndarray,
                  options: Optional[SpgemmOptions] = None, device: Optional[int] = None, parts: int = 0):
    """C = A*B from host operands into caller buffers (C ABI spgemm_multiply_into):
    rpt int64[a.rows + 1], col int32 / val float64 of capacity >= nnz(C) (size them with
    forecast_nnz or a previous product; pinned buffers run at full PCIe speed). A's rows
    go in `parts` nprod-balanced blocks (0: by size) and each block's C is downloaded
    while the next block is multiplied. Returns (nnz, SpgemmOutput without c)."""
    if a.on_device or b.on_device:
        raise InvalidArgument("multiply_into: operands must be host-resident")
    if rpt.dtype != np.int64 or col.dtype != np.int32 or val.dtype != np.float64:
        raise InvalidArgument("multiply_into: rpt int64, col int32, val float64")
    if rpt.size < a.rows + 1 or not (rpt.flags.c_contiguous and col.flags.c_contiguous and val.flags.c_contiguous):
        raise InvalidArgument("multiply_into: rpt needs a.rows + 1 entries; contiguous buffers")
    cap = min(col.size, val.size)
    va, vb = a._view(), b._view()
    if a is not b and a.rpt is b.rpt:
        vb = va
    nnz = C.c_int64()
    rep = _c.Report()
    opts = options._c() if options is not None else None
    _check(_c.lib.spgemm_multiply_into(get_context(device).handle, C.byref(va), C.byref(vb),
                                       C.byref(opts) if opts is not None else None, int(parts), rpt.ctypes.data,
                                       cap, col.ctypes.data if cap else None, val.ctypes.data if cap else None,
                                       C.byref(nnz), C.byref(rep)))
    return int(nnz.value), _output_from(rep, None, options)


@dataclass
class NnzForecast:
    """Symbolic-only sizing of C = A*B."""
    rows: int
    total_nnz: int
    total_nprod: int
    row_nnz: Optional[np.ndarray] = None      # nnz(C(i,:)) per row, when asked for
    row_bounds: Optional[List[int]] = None    # the row split (forecast_nnz_multi)

    @property
    def cr(self) -> float:
        """Compression ratio nprod / nnz(C) (pipeline.hpp SpgemmStats::cr)."""
        return self.total_nprod / self.total_nnz if self.total_nnz else 0.0

    @property
    def c_bytes(self) -> int:
        """Bytes C will take as CSR (int64 rpt, int32 col, fp64 val)."""
        return 8 * (self.rows + 1) + 12 * self.total_nnz


def forecast_nnz(a: CsrMatrix, b: CsrMatrix, options: Optional[SpgemmOptions] = None,
                 device: Optional[int] = None, per_row: bool = True) -> NnzForecast:
    """nnz(C) without computing or allocating C (C ABI spgemm_forecast_nnz): the
    reference's setup + symbolic_binning + run_symbolic + row_ptr region
    (pipeline.cpp:152-239) in one call, O(rows) device memory."""
    if a.cols != b.rows:
        raise InvalidArgument("forecast_nnz: a.cols != b.rows")
    rows = np.empty(a.rows, np.int64) if per_row else None
    tn, tp = C.c_int64(), C.c_int64()
    va, vb = a._view(), b._view()
    opts = options._c() if options is not None else None
    _check(_c.lib.spgemm_forecast_nnz(get_context(device).handle, C.byref(va), C.byref(vb),
                                      C.byref(opts) if opts is not None else None,
                                      rows.ctypes.data if per_row and a.rows else None, C.byref(tn), C.byref(tp)))
    return NnzForecast(a.rows, int(tn.value), int(tp.value), rows)


def forecast_nnz_multi(a: CsrMatrix, b: CsrMatrix, options: Optional[SpgemmOptions] = None,
                       devices: Sequence[int] = (0,), per_row: bool = True) -> NnzForecast:
    """forecast_nnz over several devices in one process (spgemm_forecast_nnz_multi):
    the nprod-balanced row split of multiply_multi, each block counted on its own
    device and host thread."""
    devices = list(devices)
    if not devices:
        raise InvalidArgument("forecast_nnz_multi: no devices")
    if a.cols != b.rows:
        raise InvalidArgument("forecast_nnz_multi: a.cols != b.rows")
    ctxs = [Context(d) for d in devices]
    n = len(ctxs)
    handles = (C.c_void_p * n)(*[c.handle for c in ctxs])
    bounds = (C.c_int64 * (n + 1))()
    rows = np.empty(a.rows, np.int64) if per_row else None
    tn, tp = C.c_int64(), C.c_int64()
    va, vb = a._view(), b._view()
    opts = options._c() if options is not None else None
    try:
        _check(_c.lib.spgemm_forecast_nnz_multi(handles, n, C.byref(va), C.byref(vb),
                                                C.byref(opts) if opts is not None else None,
                                                rows.ctypes.data if per_row and a.rows else None, bounds,
                                                C.byref(tn), C.byref(tp)))
    finally:
        for c in ctxs:
            c.close()
    return NnzForecast(a.rows, int(tn.value), int(tp.value), rows, [int(x) for x in bounds])


def csr_from_coo_device(rows: int, cols: int, row, col, val, device: Optional[int] = None) -> "DeviceMatrix":
    """csr.cpp:12-72 (csr_from_coo) on the device: triples in input order (numpy
    arrays or torch CUDA tensors) -> a device CSR with each row's columns sorted
    and duplicates summed in input order. Raises IndexError for an entry outside
    the shape and InvalidArgument for a bad shape, like the reference."""
    ctx = get_context(device)
    if _is_torch_cuda(row):
        import torch
        r, c, v = (t.contiguous() for t in (row.to(torch.int64), col.to(torch.int64), val.to(torch.float64)))
        ptrs, on_dev, keep = (r.data_ptr(), c.data_ptr(), v.data_ptr()), 1, (r, c, v)
        _order_device_operands(ctx)
    else:
        r = np.ascontiguousarray(row, np.int64)
        c = np.ascontiguousarray(col, np.int64)
        v = np.ascontiguousarray(val, np.float64)
        if not (r.size == c.size == v.size):
            raise InvalidArgument("csr_from_coo: row/col/val lengths differ")
        ptrs, on_dev, keep = (r.ctypes.data, c.ctypes.data, v.ctypes.data), 0, (r, c, v)
    n = int(keep[0].numel() if on_dev else keep[0].size)
    h = C.c_void_p()
    st = _c.lib.spgemm_csr_from_coo(ctx.handle, int(rows), int(cols), n, *(p if n else None for p in ptrs), on_dev,
                                    C.byref(h))
    if st != _c.OK and "outside" in _c.last_error():
        raise IndexError(_c.last_error())
    _check(st)
    return DeviceMatrix(h, ctx)


def multiply_device(a: CsrMatrix, b: CsrMatrix, options: Optional[SpgemmOptions] = None,
                    device: Optional[int] = None):
    """C = A*B with C left in HBM. Returns (DeviceMatrix, SpgemmOutput with c=None)."""
    p = SpgemmPipeline(a, b, options, device)
    try:
        return p.run_device()
    finally:
        p.close()
