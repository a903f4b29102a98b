// Row-block sharded PDHG: A is partitioned by rows and A^T
// (the reference's CSC) by columns into P nnz-balanced blocks; shard p owns
// rows [rb[p], rb[p+1]) of A (-> ax, y, b, r and their sums) and columns
// [cb[p], cb[p+1]) (-> aty, x, c, l, u, s, sums and next-x candidates).
// Every shard computes its rows of A x and of A^T y completely, so there is
// no cross-shard summation and the iterates are bit-identical to one device
// (same lanes-per-row G and long-row segments, which depend on the full
// matrix only). Per iteration:
//
//   rows half on every shard (k_spmv_rows over the padded full x, k_dual)
//   all-gather y              (each shard's slice into every full y)
//   cols half on every shard (k_spmv_cols over the padded full y, k_primal)
//   all-gather report sums    (22 doubles per shard)
//   k_finalize_shard: every shard reduces the P sums in shard order and takes
//                     the identical decisions; k_select_x: the chosen next
//                     iterate's slice into the shard's region of the full x
//   all-gather x
//
// Full vectors are stored padded: shard q's slice sits at q * S (S = the
// largest slice), so each all-gather is one in-place collective with equal
// counts; the local CSR column (row) indices are remapped into that padded
// space once at setup. Transport: NCCL (one process per GPU, ncclAllGather
// in place on the engine stream, captured into the CUDA graph with the
// kernels) or, for development and tests on one GPU, P shards in one process
// exchanging by device copies - the same kernels and the same launch order.
//
// The one-time setup (Ruiz, ||A||, step sizes) runs redundantly on every
// rank on the full matrix with the single-device kernels, so every rank
// starts from identical scaled data; the iteration is what scales. The time
// limit is checked on the host between batches so all shards stop together.
#pragma once

#include <dlfcn.h>
#include <nccl.h>  // types only: the library is resolved with dlopen at run time

#include <memory>

namespace cclp_cu {

// The same split as k_partition: part b starts at the first row i with
// ptr[i] + alpha * i >= (ptr[rows] + alpha * rows) * b / parts.
void host_partition(const int* ptr, int rows, int parts, long long alpha, int* bounds) {
  const long long total = static_cast<long long>(ptr[rows]) + alpha * rows;
  for (int b = 0; b <= parts; ++b) {
    if (b == parts) {
      bounds[b] = rows;
      continue;
    }
    const long long target = total * b / parts;
    int lo = 0, hi = rows;
    while (lo < hi) {
      const int mid = lo + (hi - lo) / 2;
      if (static_cast<long long>(ptr[mid]) + alpha * mid >= target) hi = mid; else lo = mid + 1;
    }
    bounds[b] = lo;
  }
}

__global__ void k_slice_ptr(const int* __restrict__ ptr, int r0, int rows, int* __restrict__ out) {
  const int base = ptr[r0];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= rows; i += gridDim.x * blockDim.x)
    out[i] = ptr[r0 + i] - base;
}

// idx -> owner * S + (idx - bounds[owner]) (the padded full-vector index),
// values copied alongside.
__global__ void k_slice_remap(const int* __restrict__ idx, const double* __restrict__ v1,
                              const double* __restrict__ v2, long long cnt,
                              const int* __restrict__ bounds, int P, int S, int* __restrict__ idx_out,
                              double* __restrict__ o1, double* __restrict__ o2) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < cnt;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = idx[q];
    int o = 0;
    while (o + 1 < P && bounds[o + 1] <= j) ++o;
    idx_out[q] = o * S + (j - bounds[o]);
    o1[q] = v1[q];
    o2[q] = v2[q];
  }
}

// ---- NCCL, resolved at run time (the library loads without NCCL) ----------
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = "libnccl.so.2 not found";
      return a;
    }
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.GetErrorString;
    if (!a.ok) a.err = "libnccl.so.2 lacks the needed symbols";
    return a;
  }();
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(CCLP_CU_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// ---- shard slicing ------------------------------------------------------------
void Context::shard_from(Context& F, int rank, int P, const std::vector<int>& rb,
                         const std::vector<int>& cb, cudaStream_t shared) {
  device = F.device;
  stream = shared;
  own_stream = false;
  CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ev_snap, cudaEventDisableTiming));
  CK(cudaEventCreate(&ev_a));
  CK(cudaEventCreate(&ev_b));
  phase_t0 = std::chrono::steady_clock::now();
  shard_rank = rank;
  shard_count = P;
  r0 = rb[rank];
  c0 = cb[rank];
  m = rb[rank + 1] - r0;
  n = cb[rank + 1] - c0;
  Sm = Sn = 0;
  for (int q = 0; q < P; ++q) {
    Sm = std::max(Sm, rb[q + 1] - rb[q]);
    Sn = std::max(Sn, cb[q + 1] - cb[q]);
  }
  // the full matrix's lanes-per-row (the per-row summation order)
  Grow = F.Grow;
  Gcol = F.Gcol;
  exact = F.exact;
  b_norm = F.b_norm;
  c_norm = F.c_norm;
  norm_est = F.norm_est;
  omega = F.omega;
  tau = F.tau;
  sigma = F.sigma;
  equality = F.equality;
  int* d_rb = alloc<int>(P + 1);
  int* d_cb = alloc<int>(P + 1);
  CK(cudaMemcpyAsync(d_rb, rb.data(), sizeof(int) * (P + 1), cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(d_cb, cb.data(), sizeof(int) * (P + 1), cudaMemcpyHostToDevice, stream));
  auto slice = [&](const int* fptr, const int* fidx, const double* fval, const double* fsval, int first,
                   int rows, const int* d_bounds, int S, int*& ptr_out, int*& idx_out,
                   double*& val_out, double*& sval_out) -> long long {
    int pe[2];
    CK(cudaMemcpyAsync(&pe[0], fptr + first, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(&pe[1], fptr + first + rows, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    const long long cnt = static_cast<long long>(pe[1]) - pe[0];
    ptr_out = alloc<int>(rows + 1);
    idx_out = alloc<int>(cnt);
    val_out = alloc<double>(cnt);
    sval_out = alloc<double>(cnt);
    k_slice_ptr<<<blocks_for(rows + 1), kBlock, 0, stream>>>(fptr, first, rows, ptr_out);
    if (cnt > 0)
      k_slice_remap<<<blocks_for(cnt), kBlock, 0, stream>>>(fidx + pe[0], fval + pe[0], fsval + pe[0], cnt,
                                                             d_bounds, P, S, idx_out, val_out, sval_out);
    CKL("shard slice");
    return cnt;
  };
  const long long nnz_a = slice(F.rowptr, F.colind, F.val_csr, F.sval_csr, r0, m, d_cb, Sn, rowptr, colind,
                                val_csr, sval_csr);
  const long long nnz_at = slice(F.colptr, F.rowind, F.val_csc, F.sval_csc, c0, n, d_rb, Sm, colptr, rowind,
                                 val_csc, sval_csc);
  nnz = std::max(nnz_a, nnz_at);
  auto vec = [&](const double* src, int off, int len) {
    double* d = alloc<double>(len);
    if (len > 0)
      CK(cudaMemcpyAsync(d, src + off, sizeof(double) * len, cudaMemcpyDeviceToDevice, stream));
    return d;
  };
  c = vec(F.c, c0, n);
  l = vec(F.l, c0, n);
  u = vec(F.u, c0, n);
  s = vec(F.s, c0, n);
  b = vec(F.b, r0, m);
  r = vec(F.r, r0, m);
  x_full = alloc<double>(static_cast<size_t>(P) * Sn);
  y_full = alloc<double>(static_cast<size_t>(P) * Sm);
  xpart = alloc<double>(static_cast<size_t>(P) * (kRowParts + kColParts));
  vparts = alloc<double>(kRowParts + kColParts);
  CK(cudaMemsetAsync(x_full, 0, sizeof(double) * std::max<size_t>(1, size_t(P) * Sn), stream));
  CK(cudaMemsetAsync(y_full, 0, sizeof(double) * std::max<size_t>(1, size_t(P) * Sm), stream));
  CK(cudaMemsetAsync(xpart, 0, sizeof(double) * P * (kRowParts + kColParts), stream));
  release(d_rb);
  release(d_cb);
  partition();  // setup-kernel grids, the local SpMV plans and their tuned geometry
}

// ---- the sharded solve ---------------------------------------------------------
struct Sharded {
  int P = 1, rank = 0, nranks = 1, device = 0;
  int m = 0, n = 0;  // global
  std::unique_ptr<Context> full;                 // full matrix: setup (replicated per rank)
  std::vector<std::unique_ptr<Context>> shards;  // this process's shards
  std::vector<int> rb, cb;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  cudaGraphExec_t graph = nullptr;
  int graph_k = 0;
  long long launches = 0;
  double *vx_full = nullptr, *vy_full = nullptr, *vz_full = nullptr, *vparts_full = nullptr;
  bool begun = false;

  ~Sharded() {
    if (graph) cudaGraphExecDestroy(graph);
    shards.clear();
    if (full) {
      full->release(vx_full);
      full->release(vy_full);
      full->release(vz_full);
      full->release(vparts_full);
    }
    full.reset();
    if (comm) nccl().CommDestroy(comm);
  }

  Context& s0() { return *shards[0]; }

  // In-place all-gather of a padded full buffer (count doubles per shard).
  void allgather(double* Context::*buf, size_t count) {
    if (comm != nullptr) {
      double* b = s0().*buf;
      nck(nccl().AllGather(b + static_cast<size_t>(rank) * count, b, count, ncclDouble, comm, stream),
          "ncclAllGather");
      return;
    }
    for (int q = 0; q < P; ++q)
      for (int t = 0; t < P; ++t)
        if (t != q)
          CK(cudaMemcpyAsync(shards[t].get()->*buf + static_cast<size_t>(q) * count,
                             shards[q].get()->*buf + static_cast<size_t>(q) * count, sizeof(double) * count,
                             cudaMemcpyDeviceToDevice, stream));
  }

  void create(const cclp_cu_lp* lp, int dev, int local_shards, int rk, int nr, const ncclUniqueId* id) {
    device = dev;
    rank = rk;
    nranks = nr;
    P = (nr > 1 || id != nullptr) ? nr : local_shards;
    m = lp->m;
    n = lp->n;
    if (P < 1) throw std::invalid_argument("sharded: need at least one shard");
    if (nr > 1 && local_shards != 1)
      throw std::invalid_argument("sharded: one shard per process with NCCL");
    full = std::make_unique<Context>();
    full->device = dev;
    full->upload(lp);
    stream = full->stream;
    // nnz-balanced row blocks of A (CSR built on the device) and of A^T
    // (the caller's CSC): the same split on every rank
    std::vector<int> rowptr_h(static_cast<size_t>(m) + 1);
    CK(cudaMemcpy(rowptr_h.data(), full->rowptr, sizeof(int) * (m + 1), cudaMemcpyDeviceToHost));
    rb.assign(P + 1, 0);
    cb.assign(P + 1, 0);
    host_partition(rowptr_h.data(), m, P, 4, rb.data());
    host_partition(lp->colptr, n, P, 4, cb.data());
    if (id != nullptr) {  // NCCL transport (also with one rank: exercises the collective path)
      if (local_shards != 1) throw std::invalid_argument("sharded: one shard per process with NCCL");
      if (!nccl().ok) throw Error(CCLP_CU_ENCCL, nccl().err);
      nck(nccl().CommInitRank(&comm, nr, *id, rk), "ncclCommInitRank");
    }
  }

  void build_shards(const cclp_cu_config& cfg) {
    if (graph) {
      cudaGraphExecDestroy(graph);
      graph = nullptr;
    }
    shards.clear();
    full->exact = cfg.exact_spmv != 0;
    k_stamp<<<1, 1, 0, stream>>>(full->t0);
    CKL("stamp");
    full->setup(cfg);
    const int first = comm != nullptr ? rank : 0;
    const int count = comm != nullptr ? 1 : P;
    for (int q = first; q < first + count; ++q) {
      auto sh = std::make_unique<Context>();
      sh->shard_from(*full, q, P, rb, cb, stream);
      k_stamp<<<1, 1, 0, stream>>>(sh->t0);
      CKL("stamp");
      shards.push_back(std::move(sh));
    }
  }

  void launch_round(bool init) {
    for (auto& s : shards) s->launch_rows_half(init);
    allgather(&Context::y_full, static_cast<size_t>(s0().Sm));
    for (auto& s : shards) s->launch_cols_half(init);
    allgather(&Context::xpart, kRowParts + kColParts);
    for (auto& s : shards) {
      k_finalize_shard<<<1, kEpiBlock, 0, stream>>>(s->params, s->xpart, P, init ? 1 : 0);
      k_select_x<<<blocks_for(s->n), kBlock, 0, stream>>>(
          s->params, s->x_full + static_cast<size_t>(s->shard_rank) * s->Sn);
    }
    CKL("shard finalize");
    allgather(&Context::x_full, static_cast<size_t>(s0().Sn));
    launches += static_cast<long long>(shards.size()) * (kKernelsPerIteration + 2);
  }

  void begin(const cclp_cu_config& cfg, const cclp_cu_tolerances& tol, const double* thr, int nthr) {
    build_shards(cfg);
    for (auto& s : shards) s->init_state(cfg, tol, thr, nthr, false);
    allgather(&Context::x_full, static_cast<size_t>(s0().Sn));
    launch_round(true);
    CK(cudaStreamSynchronize(stream));
    begun = true;
  }

  void build_graph(int k) {
    if (graph && graph_k == k) return;
    if (graph) {
      cudaGraphExecDestroy(graph);
      graph = nullptr;
    }
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    const long long before = launches;
    for (int i = 0; i < k; ++i) launch_round(false);
    launches = before;
    CK(cudaStreamEndCapture(stream, &g));
    CK(cudaGraphInstantiate(&graph, g, 0));
    cudaGraphDestroy(g);
    graph_k = k;
  }

  void run_batch(int k) {
    build_graph(k);
    CK(cudaGraphLaunch(graph, stream));
    launches += static_cast<long long>(k) * shards.size() * (kKernelsPerIteration + 2);
  }

  void fetch_ctrl(Ctrl* st) { s0().fetch_ctrl(st); }

  void clear_halt() {
    const int zero[2] = {0, 0};
    for (auto& s : shards) {
      CK(cudaMemcpyAsync(&s->ctrl->halt, &zero[0], sizeof(int), cudaMemcpyHostToDevice, stream));
      CK(cudaMemcpyAsync(&s->ctrl->snap_pending, &zero[1], sizeof(int), cudaMemcpyHostToDevice, stream));
    }
    CK(cudaStreamSynchronize(stream));
  }

  // Full unscaled x, y, z of a view into host arrays, plus the view's report
  // sums reduced over shards in shard order (for a report to recompute).
  void assemble_view(int view, const Ctrl& st, double* x, double* y, double* z, double* sums) {
    const int Sm = s0().Sm, Sn = s0().Sn;
    if (!vx_full) {
      vx_full = full->alloc<double>(static_cast<size_t>(P) * Sn);
      vy_full = full->alloc<double>(static_cast<size_t>(P) * Sm);
      vz_full = full->alloc<double>(static_cast<size_t>(P) * Sn);
      vparts_full = full->alloc<double>(static_cast<size_t>(P) * (kRowParts + kColParts));
    }
    constexpr int W = kRowParts + kColParts;
    for (auto& s : shards) {
      s->extract_view(view, st, true);
      const int q = s->shard_rank;
      CK(cudaMemcpyAsync(vx_full + static_cast<size_t>(q) * Sn, s->vx, sizeof(double) * s->n,
                         cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(vz_full + static_cast<size_t>(q) * Sn, s->vz, sizeof(double) * s->n,
                         cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(vy_full + static_cast<size_t>(q) * Sm, s->vy, sizeof(double) * s->m,
                         cudaMemcpyDeviceToDevice, stream));
      CK(cudaMemcpyAsync(vparts_full + q * W, s->vparts, sizeof(double) * W, cudaMemcpyDeviceToDevice,
                         stream));
    }
    if (comm != nullptr) {  // every rank ends with the full vectors
      nck(nccl().AllGather(vx_full + static_cast<size_t>(rank) * Sn, vx_full, Sn, ncclDouble, comm, stream),
          "ncclAllGather");
      nck(nccl().AllGather(vz_full + static_cast<size_t>(rank) * Sn, vz_full, Sn, ncclDouble, comm, stream),
          "ncclAllGather");
      nck(nccl().AllGather(vy_full + static_cast<size_t>(rank) * Sm, vy_full, Sm, ncclDouble, comm, stream),
          "ncclAllGather");
      nck(nccl().AllGather(vparts_full + rank * W, vparts_full, W, ncclDouble, comm, stream),
          "ncclAllGather");
    }
    for (int q = 0; q < P; ++q) {
      const int nq = cb[q + 1] - cb[q], mq = rb[q + 1] - rb[q];
      if (nq > 0) {
        CK(cudaMemcpyAsync(x + cb[q], vx_full + static_cast<size_t>(q) * Sn, sizeof(double) * nq,
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(z + cb[q], vz_full + static_cast<size_t>(q) * Sn, sizeof(double) * nq,
                           cudaMemcpyDeviceToHost, stream));
      }
      if (mq > 0)
        CK(cudaMemcpyAsync(y + rb[q], vy_full + static_cast<size_t>(q) * Sm, sizeof(double) * mq,
                           cudaMemcpyDeviceToHost, stream));
    }
    std::vector<double> parts(static_cast<size_t>(P) * W);
    CK(cudaMemcpyAsync(parts.data(), vparts_full, sizeof(double) * parts.size(), cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
    for (int f = 0; f < W; ++f) {
      const bool is_row = f < kRowParts;
      const int k = is_row ? f : f - kRowParts;
      const bool is_max = is_row ? ((kRowMaxMask >> k) & 1u) : ((kColMaxMask >> k) & 1u);
      double a = 0.0;
      for (int q = 0; q < P; ++q) {
        const double v = parts[q * W + f];
        a = is_max ? ((a < v) ? v : a) : a + v;
      }
      sums[f] = a;
    }
  }
};

// ResidualReport from the reduced sums (pdhg.cpp:211-219), host side: the
// same operations as make_report.
void host_make_report(const double* rowv, const double* colv, double bn, double cn, double* rep) {
  rep[kRpNorm2] = std::sqrt(rowv[0]);
  rep[kRdNorm2] = std::sqrt(colv[0]);
  rep[kRpInf] = (rowv[1] < colv[2]) ? colv[2] : rowv[1];
  rep[kRdInf] = colv[1];
  rep[kCompl] = colv[3];
  rep[kPobj] = colv[5];
  rep[kDobj] = rowv[2] + colv[4];
  rep[kGap] = std::fabs(rep[kPobj] - rep[kDobj]);
  rep[kRelP] = rep[kRpNorm2] / (1.0 + bn);
  rep[kRelD] = rep[kRdNorm2] / (1.0 + cn);
  rep[kRelGap] = rep[kGap] / (1.0 + std::fabs(rep[kPobj]) + std::fabs(rep[kDobj]));
  double mx = rep[kRelP];
  if (mx < rep[kRelD]) mx = rep[kRelD];
  if (mx < rep[kRelGap]) mx = rep[kRelGap];
  rep[kMaxResid] = mx;
}

}  // namespace cclp_cu
