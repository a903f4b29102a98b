"""CPU, world_size 2 over gloo: the sharded iteration's data decomposition
 - each rank owns an nnz-balanced row block of A and column
block of A' (cclp_cu_partition, the split the engine uses), computes its rows
of A x and A'y completely and all-gathers y and x slices once per half-step -
reproduces the single-process pdhg_step (pdhg.cpp:118-143) bit for bit. Runs
a numpy restatement of the step, no GPU."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_24429_b200 import lpgen
from paper_2510_24429_b200.pdhg import partition

ITERS = 60


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    lp = lpgen.random_equality_lp(300, 1200, 6, seed=4)[0]
    A = sp.csc_matrix((lp.val, lp.rowind, lp.colptr), shape=(lp.m, lp.n))
    return lp, A.tocsr(), A.T.tocsr()


def _step_single(lp, Ar, At, tau, sigma, iters):
    """Reference step order: x+ = clamp(x - tau(c - aty)); ax+ = A x+;
    y+ = y + sigma(b - (2 ax+ - ax)); aty+ = A' y+."""
    x = np.clip(np.zeros(lp.n), lp.col_lower, lp.col_upper)
    y = np.zeros(lp.m)
    ax, aty = Ar @ x, At @ y
    for _ in range(iters):
        xn = np.minimum(np.maximum(x - tau * (lp.c - aty), lp.col_lower), lp.col_upper)
        axn = Ar @ xn
        yn = y + sigma * (lp.row_lower - (2.0 * axn - ax))
        atyn = At @ yn
        x, y, ax, aty = xn, yn, axn, atyn
    return x, y


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lp, Ar, At = _problem()
    rb = partition(Ar.indptr.astype(np.int32), world)
    cb = partition(lp.colptr, world)
    r0, r1, c0, c1 = rb[rank], rb[rank + 1], cb[rank], cb[rank + 1]
    A_loc = Ar[r0:r1]          # my rows of A (full column range)
    At_loc = At[c0:c1]         # my rows of A' = my columns of A
    tau, sigma = 0.05, 0.05
    c, l, u = lp.c[c0:c1], lp.col_lower[c0:c1], lp.col_upper[c0:c1]
    b = lp.row_lower[r0:r1]

    def allgather(local, bounds, total):
        counts = np.diff(bounds)
        pad = int(counts.max())
        buf = torch.zeros(pad, dtype=torch.float64)
        buf[:local.size] = torch.from_numpy(local)
        parts = [torch.zeros(pad, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, buf)
        full = np.empty(total)
        for q in range(world):
            full[bounds[q]:bounds[q + 1]] = parts[q].numpy()[:counts[q]]
        return full

    x_loc = np.clip(np.zeros(c1 - c0), l, u)
    y_loc = np.zeros(r1 - r0)
    x_full = allgather(x_loc, cb, lp.n)
    y_full = allgather(y_loc, rb, lp.m)
    ax_loc, aty_loc = A_loc @ x_full, At_loc @ y_full
    for _ in range(ITERS):
        xn = np.minimum(np.maximum(x_loc - tau * (c - aty_loc), l), u)
        x_full = allgather(xn, cb, lp.n)
        axn = A_loc @ x_full
        yn = y_loc + sigma * (b - (2.0 * axn - ax_loc))
        y_full = allgather(yn, rb, lp.m)
        atyn = At_loc @ y_full
        x_loc, y_loc, ax_loc, aty_loc = xn, yn, axn, atyn
    if rank == 0:
        out.put((allgather(x_loc, cb, lp.n), allgather(y_loc, rb, lp.m), rb.tolist(), cb.tolist()))
    else:
        allgather(x_loc, cb, lp.n)
        allgather(y_loc, rb, lp.m)
    dist.destroy_process_group()


def test_partition_covers_and_balances():
    lp, Ar, _ = _problem()
    for P in (1, 2, 3, 8):
        b = partition(lp.colptr, P)
        assert b[0] == 0 and b[-1] == lp.n and np.all(np.diff(b) >= 0)
        w = lp.colptr[b[1:]] - lp.colptr[b[:-1]] + 4 * np.diff(b)
        assert w.max() <= (lp.nnz + 4 * lp.n) / P + lp.colptr.max()  # within one row of ideal


def test_two_rank_gloo_iterates_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    x2, y2, rb, cb = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lp, Ar, At = _problem()
    x1, y1 = _step_single(lp, Ar, At, 0.05, 0.05, ITERS)
    assert 0 < rb[1] < lp.m and 0 < cb[1] < lp.n
    assert np.array_equal(x1, x2)
    assert np.array_equal(y1, y2)


# ---- the distributed setup (csrc/sharded.cuh dist_setup), restated --------
def _repro_consts(M, N):
    import math
    if not (M > 0.0) or not (M <= 1.7e308) or N <= 0:
        return None
    k = 1
    while (1 << k) <= N:
        k += 1
    _, e = math.frexp(M)
    E1 = e + k
    E2 = E1 - 53 + k
    E3 = E2 - 53 + k
    return [math.ldexp(1.5, E1), math.ldexp(1.5, E2), math.ldexp(1.5, E3)]


def _levels(t, T):
    S, rem = [], t.copy()
    for lv in range(3):
        x = (T[lv] + rem) - T[lv]
        rem = rem - x
        S.append(float(np.sum(x)))  # exact in any order
    return np.array(S)


def _rsum(terms, N, reduce_max=None, reduce_sum=None):
    """k_repro_max + k_repro_sum + repro_final; the reducers combine ranks."""
    M = float(np.max(np.abs(terms))) if terms.size else 0.0
    if reduce_max is not None:
        M = reduce_max(M)
    T = _repro_consts(M, N)
    S = _levels(terms, T) if terms.size else np.zeros(3)
    if reduce_sum is not None:
        S = reduce_sum(S)
    return (S[0] + S[1]) + S[2]


def _pow2_sqrt(v):
    return np.exp2(np.round(0.5 * np.log2(v)))


def _setup(Ar_loc, At_loc, b, c, r_of, s_of, gather_r, gather_s, N_m, N_n, rmax_all, rsum_all, any_all,
           v0, gather_v, gather_w, iters=12, passes=10):
    """Ruiz (scaling.cpp:46-90) over gathered scales, then the power
    iteration (pdhg.cpp:46-65) with reproducible norms; single process when
    the gathers are identities."""
    r, s = r_of.copy(), s_of.copy()
    Ab, Atb = abs(Ar_loc), abs(At_loc)
    for _ in range(passes):
        rf, sf = gather_r(r), gather_s(s)
        rowmax = np.array([np.max((Ab[i].data * r[i]) * sf[Ab[i].indices]) if Ab[i].nnz else 0.0
                           for i in range(Ab.shape[0])])
        colmax = np.array([np.max((Atb[j].data * rf[Atb[j].indices]) * s[j]) if Atb[j].nnz else 0.0
                           for j in range(Atb.shape[0])])
        bad = lambda v: np.any((v != 0) & ((v < 0.5) | (v >= 2.0)))  # noqa: E731
        if not any_all(bool(bad(rowmax) or bad(colmax))):
            break
        r = np.where(rowmax > 0, r / _pow2_sqrt(np.where(rowmax > 0, rowmax, 1.0)), r)
        s = np.where(colmax > 0, s / _pow2_sqrt(np.where(colmax > 0, colmax, 1.0)), s)
    rf, sf = gather_r(r), gather_s(s)
    As = Ar_loc.multiply(r[:, None]).multiply(sf[None, :]).tocsr()
    Ats = At_loc.multiply(s[:, None]).multiply(rf[None, :]).tocsr()
    v = v0 / np.sqrt(_rsum(v0 * v0, N_n, rmax_all, rsum_all))
    lam = 0.0
    for _ in range(iters):
        w = As @ gather_v(v)
        u = Ats @ gather_w(w)
        nu = np.sqrt(_rsum(u * u, N_n, rmax_all, rsum_all))
        lam = _rsum(v * u, N_n, rmax_all, rsum_all)
        v = u / nu
    bn = np.sqrt(_rsum(b * b, N_m, rmax_all, rsum_all))
    cn = np.sqrt(_rsum(c * c, N_n, rmax_all, rsum_all))
    return r, s, np.sqrt(max(lam, 0.0)), bn, cn


def _setup_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lp, Ar, At = _problem()
    rb = partition(Ar.indptr.astype(np.int32), world)
    cb = partition(lp.colptr, world)
    r0, r1, c0, c1 = rb[rank], rb[rank + 1], cb[rank], cb[rank + 1]

    def gather(bounds, total):
        counts = np.diff(bounds)
        pad = int(counts.max())

        def g(local):
            buf = torch.zeros(pad, dtype=torch.float64)
            buf[:local.size] = torch.from_numpy(local)
            parts = [torch.zeros(pad, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, buf)
            full = np.empty(total)
            for q in range(world):
                full[bounds[q]:bounds[q + 1]] = parts[q].numpy()[:counts[q]]
            return full
        return g

    def rmax(v):
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def rsum(S):
        t = torch.from_numpy(np.asarray(S, dtype=np.float64).copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)  # exact level sums: any order
        return t.numpy()

    def anyall(b):
        return rmax(1.0 if b else 0.0) > 0.0

    v0 = np.random.default_rng(11).standard_normal(lp.n)
    r, s, nrm, bn, cn = _setup(Ar[r0:r1], At[c0:c1], lp.row_lower[r0:r1], lp.c[c0:c1], np.ones(r1 - r0),
                               np.ones(c1 - c0), gather(rb, lp.m), gather(cb, lp.n), lp.m, lp.n, rmax, rsum,
                               anyall, v0[c0:c1], gather(cb, lp.n), gather(rb, lp.m))
    rf, sf = gather(rb, lp.m)(r), gather(cb, lp.n)(s)
    if rank == 0:
        out.put((rf, sf, nrm, bn, cn))
    dist.destroy_process_group()


def test_two_rank_gloo_distributed_setup_is_bit_identical():
    """World size 2: Ruiz over all-gathered scales and the power iteration with
    max / sum all-reduces of the reproducible level sums give the single
    process's scale factors, ||A||, ||b|| and ||c|| bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_setup_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    r2, s2, n2, bn2, cn2 = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lp, Ar, At = _problem()
    ident = lambda v: v  # noqa: E731
    v0 = np.random.default_rng(11).standard_normal(lp.n)
    r1, s1, n1, bn1, cn1 = _setup(Ar, At, lp.row_lower, lp.c, np.ones(lp.m), np.ones(lp.n), ident, ident, lp.m,
                                  lp.n, None, None, lambda b: b, v0, ident, ident)
    assert np.array_equal(r1, r2) and np.array_equal(s1, s2)
    assert not np.all(r1 == 1.0)
    assert n1 == n2 and bn1 == bn2 and cn1 == cn2
