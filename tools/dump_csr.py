"""Dumps CSR(A) and CSR(A^T) of a config for tools/spmv_bench (dev tool)."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from paper_2510_24429_b200 import lpgen  # noqa: E402

cfg, out = sys.argv[1], sys.argv[2]
lp = lpgen.make_config(cfg)
A = sp.csc_matrix((lp.val, lp.rowind, lp.colptr), shape=(lp.m, lp.n))
R = A.tocsr()
R.sort_indices()
rng = np.random.default_rng(0)
for tag, M, ncols in (("a", R, lp.n), ("t", A, lp.m)):
    # CSR of A is R; CSR of A^T has ptr=colptr, idx=rowind (the CSC of A)
    ptr = M.indptr.astype(np.int32)
    idx = M.indices.astype(np.int32)
    val = M.data.astype(np.float64)
    rows = len(ptr) - 1
    np.array([rows, ncols, len(idx)], np.int64).tofile(f"{out}_{tag}.meta")
    ptr.tofile(f"{out}_{tag}.ptr")
    idx.tofile(f"{out}_{tag}.idx")
    val.tofile(f"{out}_{tag}.val")
    rng.standard_normal(ncols).tofile(f"{out}_{tag}.x")
