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
