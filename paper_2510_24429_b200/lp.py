"""Host-side LP container in the reference's layout.

`LinearProgram` mirrors ``cclp::LinearProgram`` (proj/include/cclp/lp.hpp:37-64)
restricted to what the PDHG path reads: CSC ``A`` with int32 indices and fp64
values (types.hpp:25-31), objective ``c``, row activity bounds and column
bounds with IEEE +-inf for absent bounds (types.hpp:35).
"""
from __future__ import annotations

import dataclasses

import numpy as np

INF = float("inf")


@dataclasses.dataclass
class LinearProgram:
    m: int
    n: int
    colptr: np.ndarray  # int32[n+1]
    rowind: np.ndarray  # int32[nnz], ascending within each column
    val: np.ndarray  # float64[nnz]
    c: np.ndarray  # float64[n]
    row_lower: np.ndarray  # float64[m]
    row_upper: np.ndarray  # float64[m]
    col_lower: np.ndarray  # float64[n]
    col_upper: np.ndarray  # float64[n]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.colptr[-1])

    def all_rows_equality(self) -> bool:
        """lp.cpp:22-27 with row_is_equality (lp.hpp:68-70)."""
        rl, ru = self.row_lower, self.row_upper
        return bool(np.all((rl == ru) & np.isfinite(rl)))

    def representative_rhs(self) -> np.ndarray:
        """lp.cpp:29-39: upper bound when finite, else lower, else 0."""
        b = np.where(np.isfinite(self.row_upper), self.row_upper,
                     np.where(np.isfinite(self.row_lower), self.row_lower, 0.0))
        return b.astype(np.float64)

    def validate(self) -> None:
        """lp.cpp:49-86 (vectorised)."""
        def check(ok, what):
            if not ok:
                raise ValueError("invalid LP: " + what)
        check(self.colptr.shape == (self.n + 1,), "colptr length != ncols+1")
        check(self.c.shape == (self.n,), "objective length != ncols")
        check(self.row_lower.shape == (self.m,) and self.row_upper.shape == (self.m,),
              "row bound length != nrows")
        check(self.col_lower.shape == (self.n,) and self.col_upper.shape == (self.n,),
              "column bound length != ncols")
        check(bool(np.all(self.col_lower <= self.col_upper)), "crossed column bounds")
        check(not bool(np.any(np.isnan(self.c))), "NaN objective coefficient")
        check(bool(np.all(self.row_lower <= self.row_upper)), "crossed activity bounds")
        cp = self.colptr.astype(np.int64)
        check(cp[0] == 0 and bool(np.all(np.diff(cp) >= 0)), "decreasing column offsets")
        nnz = int(cp[-1])
        check(self.rowind.shape == (nnz,) and self.val.shape == (nnz,), "nnz mismatch")
        if nnz:
            check(int(self.rowind.min()) >= 0 and int(self.rowind.max()) < self.m,
                  "row index out of range")
            same_col = np.repeat(np.arange(self.n), np.diff(cp))
            inc = np.diff(self.rowind.astype(np.int64))
            check(bool(np.all((inc > 0) | (np.diff(same_col) != 0))),
                  "unsorted or duplicate row indices")
            check(bool(np.all(self.val != 0.0)), "explicit zero stored")
            check(not bool(np.any(np.isnan(self.val))), "NaN matrix entry")

    def dense(self) -> np.ndarray:
        D = np.zeros((self.m, self.n))
        cols = np.repeat(np.arange(self.n), np.diff(self.colptr.astype(np.int64)))
        D[self.rowind, cols] = self.val
        return D


def csc_from_triplets(m: int, n: int, rows, cols, vals):
    """make_sparse (kernels.cpp:20-27): sort by (col,row), sum duplicates in
    insertion order, prune exact zeros, compress."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((rows, cols))  # stable: duplicates keep insertion order
    rows, cols, vals = rows[order], cols[order], vals[order]
    key = cols * max(m, 1) + rows
    if key.size:
        start = np.concatenate(([True], key[1:] != key[:-1]))
        if not start.all():
            grp = np.cumsum(start) - 1
            summed = np.zeros(int(grp[-1]) + 1)
            for k in range(vals.size):  # duplicates are rare; keep exact order
                summed[grp[k]] += vals[k]
            rows, cols, vals = rows[start], cols[start], summed
    keep = vals != 0.0
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    colptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(colptr, cols + 1, 1)
    colptr = np.cumsum(colptr)
    return colptr.astype(np.int32), rows.astype(np.int32), vals


def to_standard_form(lp: LinearProgram, maximize: bool = False) -> LinearProgram:
    """Restatement of to_standard_form (standard_form.cpp:23-104): one slack
    column (+1) per non-equality row, b pinned to a finite side, slack bounds
    [b-ru, b-rl]; a max objective is negated."""
    m, n = lp.m, lp.n
    rl, ru = lp.row_lower, lp.row_upper
    is_eq = (rl == ru) & np.isfinite(rl)
    if np.any(~np.isfinite(rl) & ~np.isfinite(ru)):
        raise ValueError("to_standard_form: free row")
    slack_rows = np.nonzero(~is_eq)[0]
    ns = slack_rows.size
    n_std = n + ns
    b = np.where(np.isfinite(ru), ru, rl)
    c = np.zeros(n_std)
    c[:n] = -lp.c if maximize else lp.c
    cl = np.zeros(n_std)
    cu = np.zeros(n_std)
    cl[:n], cu[:n] = lp.col_lower, lp.col_upper
    sb = b[slack_rows]
    cl[n:] = np.where(np.isfinite(ru[slack_rows]), 0.0, -INF)
    cu[n:] = np.where(np.isfinite(rl[slack_rows]), sb - rl[slack_rows], INF)
    # Slack columns are appended after the structural ones; each has one +1.
    colptr = np.concatenate([lp.colptr.astype(np.int64),
                             lp.colptr[-1] + np.arange(1, ns + 1, dtype=np.int64)])
    rowind = np.concatenate([lp.rowind, slack_rows.astype(np.int32)])
    val = np.concatenate([lp.val, np.ones(ns)])
    return LinearProgram(m, n_std, colptr.astype(np.int32), rowind.astype(np.int32), val, c,
                         b.astype(np.float64).copy(), b.astype(np.float64).copy(), cl, cu,
                         name=lp.name)


# ---- binary CSC ingest -----------------------------------
# A flat file the engine maps and uploads directly (cclp_cu_create_from_file):
#   bytes 0-7   magic b"CCLPCSC1"
#   bytes 8-31  int32 m, int32 n, int64 nnz, int64 reserved (0)
#   then, each starting on an 8-byte boundary: colptr int32[n+1], rowind
#   int32[nnz], val f64[nnz], c f64[n], row_lower f64[m], row_upper f64[m],
#   col_lower f64[n], col_upper f64[n]
CSCB_MAGIC = b"CCLPCSC1"


def _cscb_layout(m: int, n: int, nnz: int):
    out, off = [], 32
    for name, dt, cnt in (("colptr", np.int32, n + 1), ("rowind", np.int32, nnz),
                          ("val", np.float64, nnz), ("c", np.float64, n),
                          ("row_lower", np.float64, m), ("row_upper", np.float64, m),
                          ("col_lower", np.float64, n), ("col_upper", np.float64, n)):
        out.append((name, dt, cnt, off))
        off += cnt * np.dtype(dt).itemsize
        off = (off + 7) // 8 * 8
    return out, off


def write_cscb(lp: LinearProgram, path: str) -> None:
    layout, total = _cscb_layout(lp.m, lp.n, lp.nnz)
    with open(path, "wb") as f:
        f.write(CSCB_MAGIC + np.array([lp.m, lp.n], np.int32).tobytes() +
                np.array([lp.nnz, 0], np.int64).tobytes())
        for name, dt, cnt, off in layout:
            f.seek(off)
            f.write(np.ascontiguousarray(getattr(lp, name), dt).tobytes())
        f.truncate(total)


def read_cscb(path: str) -> LinearProgram:
    """Memory-mapped view of a .cscb file (no copy until touched)."""
    with open(path, "rb") as f:
        head = f.read(32)
    if head[:8] != CSCB_MAGIC:
        raise ValueError(f"{path}: not a CCLPCSC1 file")
    m, n = np.frombuffer(head[8:16], np.int32)
    nnz = int(np.frombuffer(head[16:24], np.int64)[0])
    layout, _ = _cscb_layout(int(m), int(n), nnz)
    arrs = {name: np.memmap(path, dtype=dt, mode="r", offset=off, shape=(cnt,))
            for name, dt, cnt, off in layout}
    return LinearProgram(int(m), int(n), **arrs, name=path)
