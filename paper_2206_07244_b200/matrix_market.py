"""Matrix Market ingestion (reference: core/include/spgemm/matrix_market.hpp,
core/src/matrix_market.cpp:65-193) -- SURVEY.md §8(f) "next" row 3.

Same contract as the reference: ASCII ``coordinate`` files with ``real``,
``integer`` or ``pattern`` fields (pattern values are 1.0) and ``general`` or
``symmetric`` symmetry (off-diagonal entries mirrored, an entry above the
diagonal is an error); banner keywords case-insensitive; ``%`` comments and
blank lines skipped; 1-based indices converted to 0-based; the declared entry
count must match; every violation raises ``ParseError`` with the 1-based line
number when one is known. ``read_matrix_market_csr`` builds the CSR with the
reference's ``csr_from_coo`` semantics (duplicates summed in input order,
columns sorted).

The body is parsed in bulk with numpy (one tokenisation of the whole file);
only when that fails or the token count is off is the file re-scanned line by
line to report the offending line exactly as the reference does.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .api import CsrMatrix

INDEX_MAX = 2**31 - 1  # csr.hpp index_t


class ParseError(RuntimeError):
    """matrix_market.hpp:11-22: malformed input, with the 1-based line when known."""

    def __init__(self, what: str, line: int = 0):
        super().__init__(f"{what} (line {line})" if line > 0 else what)
        self.line = line


@dataclass
class CooEntries:
    """csr.hpp CooEntries: shape + triples (0-based), in file order (mirrors appended)."""
    rows: int
    cols: int
    row: np.ndarray
    col: np.ndarray
    value: np.ndarray

    def __len__(self) -> int:
        return int(self.row.size)


def _lines(text: str):
    """(line number, stripped content) of non-blank lines."""
    for no, raw in enumerate(text.split("\n"), start=1):
        s = raw.strip(" \t\r")
        if s:
            yield no, s


def _header(text: str):
    it = _lines(text)
    try:
        no, banner = next(it)
    except StopIteration:
        raise ParseError("empty file") from None
    parts = banner.lower().split()
    parts += [""] * (5 - len(parts))
    tag, obj, fmt, field, symmetry = parts[:5]
    if tag != "%%matrixmarket":
        raise ParseError("missing %%MatrixMarket banner", no)
    if obj != "matrix":
        raise ParseError(f"unsupported object '{obj}' (only 'matrix')", no)
    if fmt != "coordinate":
        raise ParseError(f"unsupported format '{fmt}' (only 'coordinate')", no)
    if field not in ("real", "integer", "pattern"):
        raise ParseError(f"unsupported field '{field}' (real, integer, or pattern)", no)
    if symmetry not in ("general", "symmetric"):
        raise ParseError(f"unsupported symmetry '{symmetry}' (general or symmetric)", no)
    for no, s in it:
        if s.startswith("%"):
            continue
        toks = s.split()
        names = ("row count", "column count", "entry count")
        vals = []
        for k, name in enumerate(names):
            if k >= len(toks):
                raise ParseError(f"expected {name}", no)
            try:
                vals.append(int(toks[k]))
            except ValueError:
                raise ParseError(f"expected {name}", no) from None
        if len(toks) > 3:
            raise ParseError("trailing characters after entry", no)
        rows, cols, declared = vals
        if rows < 0 or cols < 0 or declared < 0:
            raise ParseError("negative size field", no)
        if rows > INDEX_MAX or cols > INDEX_MAX:
            raise ParseError("matrix dimensions exceed 32-bit index range", no)
        return field, symmetry, rows, cols, declared, no, it
    raise ParseError("missing size line")


def _slow_body(it, field, symmetry, rows, cols, declared):
    """Line-by-line parse: exact ParseError lines (matrix_market.cpp:155-191)."""
    r_out, c_out, v_out = [], [], []
    seen = 0
    ncol = 2 if field == "pattern" else 3
    for no, s in it:
        if s.startswith("%"):
            continue
        if seen == declared:
            raise ParseError(f"more entries than the declared {declared}", no)
        toks = s.split()
        try:
            r1 = int(toks[0])
        except (ValueError, IndexError):
            raise ParseError("expected row index", no) from None
        try:
            c1 = int(toks[1])
        except (ValueError, IndexError):
            raise ParseError("expected column index", no) from None
        v = 1.0
        if field != "pattern":
            try:
                v = float(toks[2])
            except (ValueError, IndexError):
                raise ParseError("expected numeric value", no) from None
        if len(toks) > ncol:
            raise ParseError("trailing characters after entry", no)
        if r1 < 1 or r1 > rows or c1 < 1 or c1 > cols:
            raise ParseError(f"entry ({r1}, {c1}) outside declared {rows}x{cols} bounds", no)
        r, c = r1 - 1, c1 - 1
        if symmetry == "symmetric" and c > r:
            raise ParseError("entry above the diagonal in a symmetric file", no)
        r_out.append(r)
        c_out.append(c)
        v_out.append(v)
        if symmetry == "symmetric" and r != c:
            r_out.append(c)
            c_out.append(r)
            v_out.append(v)
        seen += 1
    if seen != declared:
        raise ParseError(f"file declares {declared} entries but has {seen}")
    return (np.asarray(r_out, np.int64), np.asarray(c_out, np.int64), np.asarray(v_out, np.float64))


def parse_matrix_market(text: str) -> CooEntries:
    """matrix_market.cpp:65-193 on an in-memory buffer."""
    field, symmetry, rows, cols, declared, size_line, it = _header(text)
    ncol = 2 if field == "pattern" else 3
    # bulk path: everything after the size line, comments dropped
    body = [s for _, s in it if not s.startswith("%")]
    fast = None
    if body and all(len(s.split()) == ncol for s in (body[0], body[-1])):
        try:
            toks = np.array(" ".join(body).split())
            if toks.size == ncol * len(body) and len(body) == declared:
                t = toks.reshape(len(body), ncol)
                r1 = t[:, 0].astype(np.int64)
                c1 = t[:, 1].astype(np.int64)
                v = t[:, 2].astype(np.float64) if ncol == 3 else np.ones(len(body))
                ok = (r1 >= 1) & (r1 <= rows) & (c1 >= 1) & (c1 <= cols)
                if symmetry == "symmetric":
                    ok &= c1 <= r1
                if ok.all():
                    fast = (r1 - 1, c1 - 1, v)
        except ValueError:
            fast = None
    if fast is None and not (declared == 0 and not body):
        _, _, _, _, _, _, it2 = _header(text)
        r, c, v = _slow_body(it2, field, symmetry, rows, cols, declared)
        return CooEntries(rows, cols, r, c, v)
    if fast is None:
        z = np.zeros(0, np.int64)
        return CooEntries(rows, cols, z, z.copy(), np.zeros(0))
    r, c, v = fast
    if symmetry == "symmetric":
        # each entry followed by its mirror (off-diagonal only), file order kept
        off = r != c
        n = r.size + int(off.sum())
        pos = np.arange(r.size) + np.concatenate([[0], np.cumsum(off)[:-1]])
        R = np.empty(n, np.int64)
        C = np.empty(n, np.int64)
        V = np.empty(n, np.float64)
        R[pos], C[pos], V[pos] = r, c, v
        mpos = pos[off] + 1
        R[mpos], C[mpos], V[mpos] = c[off], r[off], v[off]
        r, c, v = R, C, V
    return CooEntries(rows, cols, r, c, v)


def read_matrix_market(path: str) -> CooEntries:
    """matrix_market.cpp read_matrix_market: the file's text, then parse."""
    try:
        with open(path, "rb") as f:
            text = f.read().decode("utf-8", errors="replace")
    except OSError:
        raise ParseError(f"cannot open '{path}'") from None
    return parse_matrix_market(text)


def read_matrix_market_csr(path: str) -> CsrMatrix:
    """matrix_market.hpp:37-39: csr_from_coo(read_matrix_market(path))."""
    from .synthetic import csr_from_coo
    coo = read_matrix_market(path)
    return csr_from_coo(coo.rows, coo.cols, coo.row, coo.col, coo.value)


def read_matrix_market_device(path: str, device=None):
    """read_matrix_market_csr with the CSR assembled on the device: the file is
    parsed on the host (text I/O), the triples are sorted, folded (duplicates
    summed in input order) and compacted by the sm_100a kernels
    (api.csr_from_coo_device). Returns a DeviceMatrix."""
    from .api import csr_from_coo_device
    coo = read_matrix_market(path)
    return csr_from_coo_device(coo.rows, coo.cols, coo.row, coo.col, coo.value, device=device)
