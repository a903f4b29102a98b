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
// Each shard is built from the caller's host CSC and holds only its slices
// (rows of A, columns of A^T). The one-time setup is distributed: Ruiz passes
// all-gather the row/column maxima's scale factors, the power iteration runs
// its two products over the shards, and every setup sum (||b||, ||c||, omega's
// norms, ||u||, v.u) is a partition-free reproducible sum (repro_consts,
// setup_kernels.cuh), so scale factors, ||A||, tau and sigma are the same
// doubles as on one device. The time limit and cancel are agreed on the host
// between batches so all shards stop together.
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

// Halo exchange: dst[idx[i]] = src[idx[i]] (one peer's region, same device),
// and the pack / unpack of the NCCL send / receive buffers.
__global__ void k_halo_copy(const double* __restrict__ src, double* __restrict__ dst,
                            const int* __restrict__ idx, int cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
    const int j = idx[i];
    dst[j] = src[j];
  }
}
__global__ void k_halo_pack(const double* __restrict__ src, const int* __restrict__ idx, int cnt,
                            double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) out[i] = src[idx[i]];
}
__global__ void k_halo_unpack(const double* __restrict__ in, const int* __restrict__ idx, int cnt,
                              double* __restrict__ dst) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) dst[idx[i]] = in[i];
}
// flags[col] = 1 for every column referenced by rows [r0, r1) of a CSR
__global__ void k_mark_cols(const int* __restrict__ ptr, const int* __restrict__ idx, int r0, int r1,
                            unsigned char* __restrict__ flags) {
  const long long b = ptr[r0], e = ptr[r1];
  for (long long q = b + blockIdx.x * (long long)blockDim.x + threadIdx.x; q < e;
       q += (long long)gridDim.x * blockDim.x)
    flags[idx[q]] = 1;
}

// ---- NCCL, resolved at run time (the library loads without NCCL) ----------
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
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
    a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.GetErrorString && a.Send &&
           a.Recv && a.GroupStart && a.GroupEnd;
    if (!a.ok) a.err = "libnccl.so.2 lacks the needed symbols";
    return a;
  }();
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(CCLP_CU_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

// ---- shard slicing (from the caller's host CSC: no device copy of the full LP)
// idx -> owner * S + (idx - bounds[owner]) in place (the padded full-vector index)
__global__ void k_remap_idx(int* __restrict__ idx, long long cnt, const int* __restrict__ bounds, int P, int S) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < cnt;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = idx[q];
    int o = 0;
    while (o + 1 < P && bounds[o + 1] <= j) ++o;
    idx[q] = o * S + (j - bounds[o]);
  }
}

// Runs body(t, lo, hi) on T host threads over [0, len).
template <class F>
void host_parallel(long long len, F&& body) {
  const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
  const long long per = (len + T - 1) / T;
  std::vector<std::thread> th;
  for (int t = 1; t < T; ++t)
    th.emplace_back([&, t] { body(t, std::min(len, t * per), std::min(len, (t + 1) * per)); });
  body(0, 0, std::min(len, per));
  for (auto& x : th) x.join();
}

// The entries of rows [rlo, rhi) of the host CSC, still column-major (rows
// ascend within a column, so each column's part is one binary-searched run):
// cptr[n + 1], local row indices, values.
void host_row_slice(const cclp_cu_lp* lp, int rlo, int rhi, std::vector<int>& cptr, std::vector<int>& ridx,
                    std::vector<double>& val) {
  const int n = lp->n;
  std::vector<int> lo(n), hi(n);
  cptr.assign(static_cast<size_t>(n) + 1, 0);
  host_parallel(n, [&](int, long long a, long long b) {
    for (long long j = a; j < b; ++j) {
      const int* first = lp->rowind + lp->colptr[j];
      const int* last = lp->rowind + lp->colptr[j + 1];
      lo[j] = static_cast<int>(std::lower_bound(first, last, rlo) - lp->rowind);
      hi[j] = static_cast<int>(std::lower_bound(first, last, rhi) - lp->rowind);
    }
  });
  for (int j = 0; j < n; ++j) cptr[j + 1] = cptr[j] + (hi[j] - lo[j]);
  ridx.resize(cptr[n]);
  val.resize(cptr[n]);
  host_parallel(n, [&](int, long long a, long long b) {
    for (long long j = a; j < b; ++j)
      for (int q = lo[j], o = cptr[j]; q < hi[j]; ++q, ++o) {
        ridx[o] = lp->rowind[q] - rlo;
        val[o] = lp->val[q];
      }
  });
}

void Context::shard_from_host(const cclp_cu_lp* lp, int rank, int P, const std::vector<int>& rb,
                              const std::vector<int>& cb, cudaStream_t shared, const std::vector<int>& panel_G) {
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
  // the full matrix's lanes-per-row (the per-row summation order), from the
  // global shape alone
  const long long gnnz = lp->colptr[lp->n];
  Grow = pick_group(gnnz, lp->m);
  Gcol = pick_group(gnnz, lp->n);
  equality = true;
  int* d_rb = alloc<int>(P + 1);
  int* d_cb = alloc<int>(P + 1);
  CK(cudaMemcpyAsync(d_rb, rb.data(), sizeof(int) * (P + 1), cudaMemcpyHostToDevice, stream));
  CK(cudaMemcpyAsync(d_cb, cb.data(), sizeof(int) * (P + 1), cudaMemcpyHostToDevice, stream));
  // rows [r0, r0 + m) of A as CSR (global columns -> padded x space)
  long long nnz_a = 0;
  {
    std::vector<int> cptr, ridx;
    std::vector<double> v;
    host_row_slice(lp, r0, r0 + m, cptr, ridx, v);
    nnz_a = static_cast<long long>(ridx.size());
    int* d_cptr = alloc<int>(cptr.size());
    int* d_ridx = alloc<int>(ridx.size());
    double* d_val = alloc<double>(v.size());
    h2d(d_cptr, cptr.data(), sizeof(int) * cptr.size());
    h2d(d_ridx, ridx.data(), sizeof(int) * ridx.size());
    h2d(d_val, v.data(), sizeof(double) * v.size());
    build_csr_from(d_cptr, d_ridx, d_val, lp->n, nnz_a);  // synchronizes
    release(d_cptr);
    release(d_ridx);
    release(d_val);
    if (nnz_a > 0) k_remap_idx<<<blocks_for(nnz_a), kBlock, 0, stream>>>(colind, nnz_a, d_cb, P, Sn);
    CKL("shard rows");
  }
  // columns [c0, c0 + n) of A (the caller's CSC, global rows -> padded y space)
  const long long b0 = lp->colptr[c0];
  const long long nnz_at = static_cast<long long>(lp->colptr[c0 + n]) - b0;
  {
    std::vector<int> cp(static_cast<size_t>(n) + 1);
    for (int j = 0; j <= n; ++j) cp[j] = static_cast<int>(lp->colptr[c0 + j] - b0);
    colptr = alloc<int>(n + 1);
    rowind = alloc<int>(nnz_at);
    val_csc = alloc<double>(nnz_at);
    h2d(colptr, cp.data(), sizeof(int) * (n + 1));
    h2d(rowind, lp->rowind + b0, sizeof(int) * nnz_at);
    h2d(val_csc, lp->val + b0, sizeof(double) * nnz_at);
    if (nnz_at > 0) k_remap_idx<<<blocks_for(nnz_at), kBlock, 0, stream>>>(rowind, nnz_at, d_rb, P, Sm);
    CKL("shard cols");
  }
  nnz = std::max(nnz_a, nnz_at);
  nnz_rows_slice = nnz_a;
  nnz_cols_slice = nnz_at;
  auto vec = [&](const double* src, int len) {
    double* d = alloc<double>(len);
    if (len > 0) h2d(d, src, sizeof(double) * len);
    return d;
  };
  c = vec(lp->c + c0, n);
  l = vec(lp->col_lower + c0, n);
  u = vec(lp->col_upper + c0, n);
  b = vec(lp->row_lower + r0, m);
  s = alloc<double>(n);
  r = alloc<double>(m);
  // the buffers peers write into: plain cudaMalloc when they are shared with
  // other processes over CUDA IPC (pool memory cannot be exported)
  auto xalloc = [&](size_t count) -> double* {
    if (!ipc_buffers) return alloc<double>(count);
    void* q = nullptr;
    CK(cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(double)));
    ipc_owned.push_back(q);
    return static_cast<double*>(q);
  };
  x_full = xalloc(static_cast<size_t>(P) * Sn);
  y_full = xalloc(static_cast<size_t>(P) * Sm);
  xpart = xalloc(static_cast<size_t>(P) * (kRowParts + kColParts));
  push_flags = reinterpret_cast<unsigned long long*>(xalloc(3 * kMaxPushShards));
  push_counter = alloc<unsigned>(2);
  CK(cudaMemsetAsync(push_flags, 0, sizeof(unsigned long long) * 3 * kMaxPushShards, stream));
  CK(cudaMemsetAsync(push_counter, 0, sizeof(unsigned) * 2, stream));
  vparts = alloc<double>(kRowParts + kColParts);
  CK(cudaMemsetAsync(x_full, 0, sizeof(double) * std::max<size_t>(1, size_t(P) * Sn), stream));
  CK(cudaMemsetAsync(y_full, 0, sizeof(double) * std::max<size_t>(1, size_t(P) * Sm), stream));
  CK(cudaMemsetAsync(xpart, 0, sizeof(double) * P * (kRowParts + kColParts), stream));
  CK(cudaStreamSynchronize(stream));
  release(d_rb);
  release(d_cb);
  panel_gn = lp->n;  // column panels on the full matrix's column space
  panel_cb = cb;
  panel_G_hint = panel_G;
  partition();  // setup-kernel grids, the local SpMV plans and their tuned geometry
}

// Per-panel lanes-per-row of the full matrix from the host CSC (build_panels'
// layout: K panels of W original columns), so a shard's panel sums equal the
// single device's bit for bit.
std::vector<int> host_panel_groups(const cclp_cu_lp* lp) {
  long long pb = static_cast<long long>(Context::kPanelBytes);
  if (const char* e = dev_knob("CCLP_CU_PANEL_BYTES")) pb = std::max(64LL, std::atoll(e));  // tests
  const long long gn = lp->n;
  const long long K = (gn * 8 + pb - 1) / pb;
  std::vector<int> G;
  if (K < 3) return G;
  const long long W = (gn + K - 1) / K;
  for (long long k = 0; k < K; ++k) {
    const long long lo = std::min(k * W, gn), hi = std::min((k + 1) * W, gn);
    G.push_back(pick_group(static_cast<long long>(lp->colptr[hi]) - lp->colptr[lo], lp->m));
  }
  return G;
}

// ---- the sharded solve ---------------------------------------------------------
struct Sharded {
  int P = 1, rank = 0, nranks = 1, device = 0;
  int m = 0, n = 0;  // global
  std::unique_ptr<Context> full;                 // no matrix: stream + coordinator scratch
  bool equality = true;                          // all rows equality (run_pdhg's precondition)
  long long gnnz = 0;                            // nonzeros of the full matrix
  std::vector<int> panel_G;                      // the full matrix's per-panel lanes-per-row
  std::vector<double> h_v0;                      // power-iteration start vector (full n)
  unsigned long long v0_seed = ~0ull;
  std::vector<std::unique_ptr<Context>> shards;  // this process's shards
  std::vector<int> rb, cb;
  ncclComm_t comm = nullptr;
  // host-callback coordination (no NCCL): handle exchange, barriers and the
  // result gathers go through the caller's all-gather; the iteration uses the
  // push transport over CUDA IPC
  bool have_hcomm = false;
  cclp_cu_host_comm hcomm{};
  bool multi() const { return comm != nullptr || have_hcomm; }
  cudaStream_t stream = nullptr;
  cudaGraphExec_t graph = nullptr;
  int graph_k = 0;
  long long launches = 0;
  double *vx_full = nullptr, *vy_full = nullptr, *vz_full = nullptr, *vparts_full = nullptr;
  bool begun = false;
  bool halo_built = false;
  std::atomic<int> abort_req{0};  // cclp_cu_sharded_request_cancel

  // Halo exchange of one side (x for the row SpMV, y for the column SpMV):
  // need[p][q] = the sorted local offsets (in shard q's slice) of the entries
  // shard p's SpMV gathers from shard q. Used instead of the all-gather when
  // it moves under half the data (structured LPs: C4 needs only the
  // neighbouring stage); every rank derives every list from the full matrix,
  // so the send side needs no extra round of communication.
  struct Halo {
    bool on = false;
    long long volume = 0;
    std::vector<std::vector<int*>> need;  // [p][q] device lists (empty when q == p)
    std::vector<std::vector<int>> cnt;    // [p][q]
    double* sendbuf = nullptr;
    double* recvbuf = nullptr;
  } halo_x, halo_y;

  // The lists come from the caller's host CSC, which every rank holds: no
  // device copy of the full matrix and no extra communication.
  void build_halo(Halo& h, bool x_side, const cclp_cu_lp* lp) {
    const long long S = x_side ? s0().Sn : s0().Sm;
    const long long allgather = static_cast<long long>(P) * (P - 1) * S;
    h.need.assign(P, std::vector<int*>(P, nullptr));
    h.cnt.assign(P, std::vector<int>(P, 0));
    h.volume = 0;
    h.on = false;
    if (P < 2 || P > 64) return;
    std::vector<int> rown(static_cast<size_t>(m)), coln(static_cast<size_t>(n));
    for (int q = 0; q < P; ++q) {
      for (int i = rb[q]; i < rb[q + 1]; ++i) rown[i] = q;
      for (int j = cb[q]; j < cb[q + 1]; ++j) coln[j] = q;
    }
    std::vector<std::vector<std::vector<int>>> lists(P, std::vector<std::vector<int>>(P));
    if (x_side) {
      // shard p's rows gather x_j (column j, owner q) when a row of p has an entry in column j
      std::vector<unsigned long long> mask(static_cast<size_t>(n), 0ull);
      host_parallel(n, [&](int, long long a, long long b) {
        for (long long j = a; j < b; ++j)
          for (int q = lp->colptr[j]; q < lp->colptr[j + 1]; ++q) mask[j] |= 1ull << rown[lp->rowind[q]];
      });
      for (int j = 0; j < n; ++j) {
        const int q = coln[j];
        for (unsigned long long mk = mask[j] & ~(1ull << q); mk; mk &= mk - 1)
          lists[__builtin_ctzll(mk)][q].push_back(j - cb[q]);
      }
    } else {
      // shard p's columns gather y_i (row i, owner q) when a column of p has an entry in row i
      std::vector<unsigned long long> mask(static_cast<size_t>(m), 0ull);
      host_parallel(n, [&](int, long long a, long long b) {
        for (long long j = a; j < b; ++j) {
          const unsigned long long bit = 1ull << coln[j];
          for (int q = lp->colptr[j]; q < lp->colptr[j + 1]; ++q)
            __atomic_fetch_or(&mask[lp->rowind[q]], bit, __ATOMIC_RELAXED);
        }
      });
      for (int i = 0; i < m; ++i) {
        const int q = rown[i];
        for (unsigned long long mk = mask[i] & ~(1ull << q); mk; mk &= mk - 1)
          lists[__builtin_ctzll(mk)][q].push_back(i - rb[q]);
      }
    }
    for (int p = 0; p < P; ++p)
      for (int q = 0; q < P; ++q) {
        h.cnt[p][q] = static_cast<int>(lists[p][q].size());
        h.volume += h.cnt[p][q];
      }
    h.on = h.volume * 2 < allgather;
    if (!h.on) return;
    for (int p = 0; p < P; ++p)
      for (int q = 0; q < P; ++q)
        if (q != p && h.cnt[p][q] > 0) {
          h.need[p][q] = full->alloc<int>(h.cnt[p][q]);
          CK(cudaMemcpyAsync(h.need[p][q], lists[p][q].data(), sizeof(int) * h.cnt[p][q],
                             cudaMemcpyHostToDevice, stream));
        }
    if (comm != nullptr) {
      long long ns = 0, nr = 0;
      for (int q = 0; q < P; ++q) {
        ns += h.cnt[q][rank];
        nr += h.cnt[rank][q];
      }
      h.sendbuf = full->alloc<double>(std::max(1LL, ns));
      h.recvbuf = full->alloc<double>(std::max(1LL, nr));
    }
    CK(cudaStreamSynchronize(stream));
  }

  void release_halo(Halo& h) {
    for (auto& row : h.need)
      for (int* q : row) full->release(q);
    full->release(h.sendbuf);
    full->release(h.recvbuf);
    h = Halo{};
  }

  // The exchange of one padded full buffer: the halo when it is on, else the
  // in-place all-gather.
  void exchange(double* Context::*buf, size_t S, Halo& h) {
    if (!h.on) {
      allgather(buf, S);
      return;
    }
    if (comm == nullptr) {
      for (auto& dst : shards)
        for (auto& src : shards) {
          const int p = dst->shard_rank, q = src->shard_rank;
          if (p == q || h.cnt[p][q] == 0) continue;
          k_halo_copy<<<blocks_for(h.cnt[p][q]), kBlock, 0, stream>>>(
              src.get()->*buf + static_cast<size_t>(q) * S, dst.get()->*buf + static_cast<size_t>(q) * S,
              h.need[p][q], h.cnt[p][q]);
        }
      CKL("halo copy");
      return;
    }
    double* b = s0().*buf;
    long long so = 0, ro = 0;
    for (int p = 0; p < P; ++p) {  // pack what each peer needs from this rank
      if (p == rank || h.cnt[p][rank] == 0) continue;
      k_halo_pack<<<blocks_for(h.cnt[p][rank]), kBlock, 0, stream>>>(b + static_cast<size_t>(rank) * S,
                                                                      h.need[p][rank], h.cnt[p][rank],
                                                                      h.sendbuf + so);
      so += h.cnt[p][rank];
    }
    CKL("halo pack");
    nck(nccl().GroupStart(), "ncclGroupStart");
    so = 0;
    for (int p = 0; p < P; ++p) {
      if (p == rank) continue;
      if (h.cnt[p][rank] > 0) {
        nck(nccl().Send(h.sendbuf + so, h.cnt[p][rank], ncclDouble, p, comm, stream), "ncclSend");
        so += h.cnt[p][rank];
      }
      if (h.cnt[rank][p] > 0) {
        nck(nccl().Recv(h.recvbuf + ro, h.cnt[rank][p], ncclDouble, p, comm, stream), "ncclRecv");
        ro += h.cnt[rank][p];
      }
    }
    nck(nccl().GroupEnd(), "ncclGroupEnd");
    ro = 0;
    for (int p = 0; p < P; ++p) {
      if (p == rank || h.cnt[rank][p] == 0) continue;
      k_halo_unpack<<<blocks_for(h.cnt[rank][p]), kBlock, 0, stream>>>(h.recvbuf + ro, h.need[rank][p],
                                                                        h.cnt[rank][p],
                                                                        b + static_cast<size_t>(p) * S);
      ro += h.cnt[rank][p];
    }
    CKL("halo unpack");
  }

  ~Sharded() {
    if (graph) cudaGraphExecDestroy(graph);
    if (stream) cudaStreamSynchronize(stream);
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
    if (full)
      for (unsigned char* mk : masks) full->release(mk);
    shards.clear();
    if (full) {
      release_halo(halo_x);
      release_halo(halo_y);
      full->release(vx_full);
      full->release(vy_full);
      full->release(vz_full);
      full->release(vparts_full);
    }
    full.reset();
    if (comm) nccl().CommDestroy(comm);
  }

  Context& s0() { return *shards[0]; }

  // ---- push transport ------------------------------------------------------
  bool push = false;
  std::vector<void*> ipc_opened;  // peers' buffers opened over CUDA IPC
  std::vector<unsigned char*> masks;

  // Per-row / per-column bitmasks of the shards that gather each entry of
  // this shard's slice (from the halo need lists; all shards without a halo).
  unsigned char* build_mask(const Halo& h, int owner, int len) {
    if (!h.on) return nullptr;
    std::vector<unsigned char> mk(static_cast<size_t>(std::max(len, 1)), 0);
    for (int j = 0; j < len; ++j) mk[j] = static_cast<unsigned char>(1u << owner);
    for (int q = 0; q < P; ++q) {
      if (q == owner || h.cnt[q][owner] == 0) continue;
      std::vector<int> lst(h.cnt[q][owner]);
      CK(cudaMemcpy(lst.data(), h.need[q][owner], sizeof(int) * lst.size(), cudaMemcpyDeviceToHost));
      for (int j : lst) mk[j] |= static_cast<unsigned char>(1u << q);
    }
    unsigned char* d = full->alloc<unsigned char>(mk.size());
    CK(cudaMemcpy(d, mk.data(), mk.size(), cudaMemcpyHostToDevice));
    masks.push_back(d);
    return d;
  }

  void barrier() { agree(kStopNone); }  // every rank past this point (multi-process only)

  // Host-side stop requests (cancel, time limit) taken by any rank apply to
  // all ranks, so no rank is left waiting on peers that stopped launching.
  // Every rank all-gathers its request code and takes the same decision with
  // a fixed priority (cancel over time limit), so all shards also report the
  // same stop reason although their wall clocks differ.
  enum StopReq : char { kStopNone = 0, kStopTime = 1, kStopCancel = 2 };
  StopReq agree(StopReq local) {
    if (!multi()) return local;
    const char v = static_cast<char>(local);
    const std::vector<char> all = gather_bytes(&v, 1);
    char best = kStopNone;
    for (char a : all) best = a > best ? a : best;
    return static_cast<StopReq>(best);
  }

  // All-gather of `bytes` host bytes per rank, in rank order (NCCL through a
  // device buffer, or the caller's host callback).
  std::vector<char> gather_bytes(const void* mine, size_t bytes) {
    std::vector<char> all(bytes * P);
    if (have_hcomm) {
      if (hcomm.allgather(mine, bytes, all.data(), hcomm.user) != 0)
        throw Error(CCLP_CU_ENCCL, "host all-gather callback failed");
      return all;
    }
    char* d = full->alloc<char>(std::max<size_t>(1, bytes * P));
    CK(cudaMemcpyAsync(d + bytes * rank, mine, bytes, cudaMemcpyHostToDevice, stream));
    nck(nccl().AllGather(d + bytes * rank, d, bytes, ncclChar, comm, stream), "ncclAllGather");
    CK(cudaMemcpyAsync(all.data(), d, all.size(), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    full->release(d);
    return all;
  }

  void setup_push() {
    for (unsigned char* mk : masks) full->release(mk);
    masks.clear();
    for (void* q : ipc_opened) cudaIpcCloseMemHandle(q);
    ipc_opened.clear();
    std::vector<double*> Y(P), X(P), PT(P);
    std::vector<unsigned long long*> F(P);
    if (!multi()) {
      for (auto& s : shards) {
        Y[s->shard_rank] = s->y_full;
        X[s->shard_rank] = s->x_full;
        PT[s->shard_rank] = s->xpart;
        F[s->shard_rank] = s->push_flags;
      }
    } else {  // CUDA IPC: every rank exports its four buffers, all-gathers the handles
      Context& me = s0();
      cudaIpcMemHandle_t hs[4];
      void* bufs[4] = {me.y_full, me.x_full, me.xpart, me.push_flags};
      for (int k = 0; k < 4; ++k) CK(cudaIpcGetMemHandle(&hs[k], bufs[k]));
      const size_t hb = sizeof(hs);
      const std::vector<char> all = gather_bytes(hs, hb);
      for (int q = 0; q < P; ++q) {
        if (q == rank) {
          Y[q] = me.y_full;
          X[q] = me.x_full;
          PT[q] = me.xpart;
          F[q] = me.push_flags;
          continue;
        }
        void* ptr[4];
        for (int k = 0; k < 4; ++k) {
          cudaIpcMemHandle_t h;
          std::memcpy(&h, all.data() + hb * q + sizeof(cudaIpcMemHandle_t) * k, sizeof h);
          CK(cudaIpcOpenMemHandle(&ptr[k], h, cudaIpcMemLazyEnablePeerAccess));
          ipc_opened.push_back(ptr[k]);
        }
        Y[q] = static_cast<double*>(ptr[0]);
        X[q] = static_cast<double*>(ptr[1]);
        PT[q] = static_cast<double*>(ptr[2]);
        F[q] = static_cast<unsigned long long*>(ptr[3]);
      }
    }
    for (auto& s : shards) {
      PushArgs a{};
      a.on = 1;
      a.gpu_scope = multi() ? 0 : 1;  // one process, one device: GPU scope suffices
      a.P = P;
      a.rank = s->shard_rank;
      a.Sm = s->Sm;
      a.Sn = s->Sn;
      for (int q = 0; q < P; ++q) {
        a.y[q] = Y[q];
        a.x[q] = X[q];
        a.part[q] = PT[q];
        a.flags[q] = F[q];
      }
      a.my_flags = s->push_flags;
      a.mask_y = build_mask(halo_y, s->shard_rank, s->m);
      a.mask_x = build_mask(halo_x, s->shard_rank, s->n);
      a.counter = s->push_counter;
      s->params.push = a;
    }
    CK(cudaStreamSynchronize(stream));
    barrier();  // flags are zero everywhere before anyone pushes
  }

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

  void create(const cclp_cu_lp* lp, int dev, int local_shards, int rk, int nr, const ncclUniqueId* id,
              const cclp_cu_host_comm* hc = nullptr) {
    if (lp == nullptr || lp->m < 0 || lp->n < 0 || lp->colptr == nullptr)
      throw std::invalid_argument("sharded: bad LP");
    validate_csc(lp);
    device = dev;
    rank = rk;
    nranks = nr;
    if (hc != nullptr) {
      if (hc->allgather == nullptr) throw std::invalid_argument("sharded: host comm needs an all-gather");
      if (local_shards != 1) throw std::invalid_argument("sharded: one shard per process with a host comm");
      have_hcomm = true;
      hcomm = *hc;
    }
    P = (nr > 1 || id != nullptr || hc != nullptr) ? nr : local_shards;
    m = lp->m;
    n = lp->n;
    if (P < 1) throw std::invalid_argument("sharded: need at least one shard");
    if (nr > 1 && local_shards != 1)
      throw std::invalid_argument("sharded: one shard per process with NCCL");
    full = std::make_unique<Context>();
    full->init_aux(dev);
    stream = full->stream;
    // equality form, checked on the host view (lp.hpp:66-70)
    for (int i = 0; i < m && equality; ++i)
      equality = lp->row_lower[i] == lp->row_upper[i] && std::isfinite(lp->row_lower[i]);
    // nnz-balanced row blocks of A (row counts from the caller's CSC) and of
    // A^T (its column pointers): the same split on every rank
    std::vector<int> rowptr_h(static_cast<size_t>(m) + 1, 0);
    {
      const long long nz = lp->colptr[n];
      std::vector<std::atomic<int>> cnt(static_cast<size_t>(m));
      for (auto& c : cnt) c.store(0, std::memory_order_relaxed);
      host_parallel(nz, [&](int, long long a, long long b) {
        for (long long q = a; q < b; ++q) cnt[lp->rowind[q]].fetch_add(1, std::memory_order_relaxed);
      });
      for (int i = 0; i < m; ++i) rowptr_h[i + 1] = rowptr_h[i] + cnt[i].load(std::memory_order_relaxed);
    }
    rb.assign(P + 1, 0);
    cb.assign(P + 1, 0);
    host_partition(rowptr_h.data(), m, P, 4, rb.data());
    host_partition(lp->colptr, n, P, 4, cb.data());
    panel_G = host_panel_groups(lp);
    gnnz = lp->colptr[n];
    {  // transport: push (P2P stores fused into the producers) or NCCL / device-copy gathers
      const char* e = std::getenv("CCLP_CU_TRANSPORT");
      const bool want_push = e == nullptr || std::string(e) != "gather";  // push unless asked
      push = (want_push || have_hcomm) && P <= kMaxPushShards;
      if (have_hcomm && !push) throw std::invalid_argument("sharded: host comm needs P <= 8 (push)");
    }
    if (id != nullptr) {  // NCCL transport (also with one rank: exercises the collective path)
      if (local_shards != 1) throw std::invalid_argument("sharded: one shard per process with NCCL");
      if (!nccl().ok) throw Error(CCLP_CU_ENCCL, nccl().err);
      nck(nccl().CommInitRank(&comm, nr, *id, rk), "ncclCommInitRank");
    }
    // this process's shards, each holding only its slices of A / A^T and
    // of the vectors (device memory ~ 1/P of the LP per shard)
    const int first = multi() ? rank : 0;
    const int count = multi() ? 1 : P;
    for (int q = first; q < first + count; ++q) {
      auto sh = std::make_unique<Context>();
      sh->device = dev;
      sh->ipc_buffers = push && multi();
      sh->shard_from_host(lp, q, P, rb, cb, stream, panel_G);
      shards.push_back(std::move(sh));
    }
    const char* e = dev_knob("CCLP_CU_HALO");  // 0: always all-gather (A/B)
    if (e == nullptr || std::atoi(e) != 0) {
      build_halo(halo_x, true, lp);
      build_halo(halo_y, false, lp);
    }
    halo_built = true;
    // the start vector of the default seed (full length: a shard takes its slice)
    v0_seed = 0;
    h_v0.resize(static_cast<size_t>(n));
    if (n > 0) gaussian_start(0, n, h_v0.data());
  }

  // ---- distributed setup (scaling.cpp:46-90, pdhg.cpp:46-65, :253-267) -----
  // Every rank works on its own slices; the setup exchanges are in-place
  // all-gathers of the padded full r / s / v / w (x_full, y_full) and small
  // host gathers of per-shard scalars. The maxima are order-free and the
  // sums are the partition-free reproducible sums (k_repro_*), so every
  // scale factor, ||A||, tau and sigma equal the single device's bit for bit.
  void allgather_any(double* Context::*buf, size_t count) {
    if (have_hcomm) {
      Context& me = s0();
      std::vector<double> mine(count);
      CK(cudaMemcpyAsync(mine.data(), me.*buf + static_cast<size_t>(rank) * count, sizeof(double) * count,
                         cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      const std::vector<char> all = gather_bytes(mine.data(), sizeof(double) * count);
      CK(cudaMemcpyAsync(me.*buf, all.data(), all.size(), cudaMemcpyHostToDevice, stream));
      CK(cudaStreamSynchronize(stream));
      return;
    }
    allgather(buf, count);
  }
  // Combine per-shard host values over all shards of all ranks.
  std::vector<double> combine(const std::vector<double>& local, bool is_max) {
    std::vector<double> out = local;
    if (!multi()) return out;
    const std::vector<char> all = gather_bytes(local.data(), sizeof(double) * local.size());
    const size_t K = local.size();
    for (size_t k = 0; k < K; ++k) out[k] = is_max ? 0.0 : 0.0;
    for (int q = 0; q < P; ++q)
      for (size_t k = 0; k < K; ++k) {
        double v;
        std::memcpy(&v, all.data() + (q * K + k) * sizeof(double), sizeof v);
        if (is_max)
          out[k] = (v != v || out[k] != out[k]) ? NAN : std::max(out[k], v);
        else
          out[k] = out[k] + v;  // exact level sums: any order
      }
    return out;
  }
  // Reproducible global sum(s) of a per-shard term vector (mode as k_repro_*).
  template <class A, class B, class L>
  std::vector<double> global_sum(int mode, A a, B b, L len, long long N) {
    const int K = mode == 3 ? 2 : 1;
    std::vector<double> M(K, 0.0);
    for (auto& sp : shards) {
      double Ms[2];
      sp->repro_local_max(mode, a(*sp), b(*sp), len(*sp), Ms);
      for (int k = 0; k < K; ++k) M[k] = (Ms[k] != Ms[k] || M[k] != M[k]) ? NAN : std::max(M[k], Ms[k]);
    }
    M = combine(M, true);
    std::vector<double> S(3 * K, 0.0);
    for (auto& sp : shards) {
      double Ss[6];
      sp->repro_local_sums(mode, a(*sp), b(*sp), len(*sp), M.data(), N, Ss);
      for (int k = 0; k < 3 * K; ++k) S[k] += Ss[k];
    }
    S = combine(S, false);
    std::vector<double> out(K);
    for (int k = 0; k < K; ++k) out[k] = repro_final(S.data() + 3 * k);
    return out;
  }
  bool any_true(bool local) {
    std::vector<double> v{local ? 1.0 : 0.0};
    return combine(v, true)[0] > 0.0;
  }
  // r into every shard's y_full and s into its x_full (padded, in full)
  void publish(double* Context::*own_m, double* Context::*own_n) {
    for (auto& sp : shards) {
      if (own_m && sp->m > 0)
        CK(cudaMemcpyAsync(sp->y_full + static_cast<size_t>(sp->shard_rank) * sp->Sm, (*sp).*own_m,
                           sizeof(double) * sp->m, cudaMemcpyDeviceToDevice, stream));
      if (own_n && sp->n > 0)
        CK(cudaMemcpyAsync(sp->x_full + static_cast<size_t>(sp->shard_rank) * sp->Sn, (*sp).*own_n,
                           sizeof(double) * sp->n, cudaMemcpyDeviceToDevice, stream));
    }
    if (own_m) allgather_any(&Context::y_full, static_cast<size_t>(s0().Sm));
    if (own_n) allgather_any(&Context::x_full, static_cast<size_t>(s0().Sn));
  }

  void dist_setup(const cclp_cu_config& cfg) {
    for (auto& sp : shards) sp->exact = cfg.exact_spmv != 0;
    auto none = [](Context&) -> const double* { return nullptr; };
    auto lm = [](Context& c) { return static_cast<long long>(c.m); };
    auto ln = [](Context& c) { return static_cast<long long>(c.n); };
    // norms on the unscaled model (pdhg.cpp:253-254)
    const double bn = std::sqrt(global_sum(0, [](Context& c) -> const double* { return c.b; }, none, lm, m)[0]);
    const double cn = std::sqrt(global_sum(0, [](Context& c) -> const double* { return c.c; }, none, ln, n)[0]);
    // Ruiz (scaling.cpp:46-90): row maxima need the gathered s, column maxima the gathered r
    for (auto& sp : shards) sp->ruiz_init();
    for (int t = 0; t < cfg.scaling_iterations; ++t) {
      publish(&Context::r, &Context::s);
      bool notdone = false;
      for (auto& sp : shards) notdone = sp->ruiz_maxima(sp->x_full, sp->y_full) || notdone;
      if (!any_true(notdone)) break;
      for (auto& sp : shards) sp->ruiz_update();
    }
    publish(&Context::r, &Context::s);
    for (auto& sp : shards) {  // A' = R A S on both slices, the reference's exact products
      Context& c = *sp;
      if (!c.sval_csr) c.sval_csr = c.alloc<double>(c.nnz);
      if (!c.sval_csc) c.sval_csc = c.alloc<double>(c.nnz);
      k_scale_values<<<blocks_for(static_cast<long long>(c.m) * 32), kBlock, 0, stream>>>(
          c.rowptr, c.m, c.colind, c.val_csr, c.r, c.x_full, 1, c.sval_csr);
      k_scale_values<<<blocks_for(static_cast<long long>(c.n) * 32), kBlock, 0, stream>>>(
          c.colptr, c.n, c.rowind, c.val_csc, c.s, c.y_full, 0, c.sval_csc);
      for (auto& pn : c.panels)
        if (pn.nnz > 0)
          k_gather_vals<<<blocks_for(pn.nnz), kBlock, 0, stream>>>(pn.perm, pn.nnz, c.sval_csr, pn.val);
      CKL("shard scale");
    }
    // ||A||_2 by the power iteration (pdhg.cpp:46-65) over the shards
    double norm = 0.0;
    if (m > 0 && n > 0 && gnnz > 0) {
      if (v0_seed != cfg.seed) {
        h_v0.resize(static_cast<size_t>(n));
        gaussian_start(cfg.seed, n, h_v0.data());
        v0_seed = cfg.seed;
      }
      for (auto& sp : shards) {
        sp->ensure_tuned();
        if (sp->n > 0)
          CK(cudaMemcpyAsync(sp->wn, h_v0.data() + sp->c0, sizeof(double) * sp->n, cudaMemcpyHostToDevice,
                             stream));
      }
      auto vv = [](Context& c) -> const double* { return c.wn; };
      double nv = global_sum(0, vv, none, ln, n)[0];
      if (std::sqrt(nv) == 0.0) {
        for (auto& sp : shards) k_fill<<<blocks_for(sp->n), kBlock, 0, stream>>>(sp->wn, sp->n, 1.0);
        nv = global_sum(0, vv, none, ln, n)[0];
      }
      auto set_nu = [&](double nu) {
        for (auto& sp : shards) {
          PowerCtrl pc{nu, 0.0, 0, 0};
          CK(cudaMemcpyAsync(sp->pctrl, &pc, sizeof pc, cudaMemcpyHostToDevice, stream));
        }
      };
      set_nu(std::sqrt(nv));
      for (auto& sp : shards)
        k_div_scalar<<<blocks_for(sp->n), kBlock, 0, stream>>>(sp->wn, &sp->pctrl->nu, sp->wn, sp->n);
      double lambda = 0.0;
      bool zero = false;
      for (int t = 0; t < cfg.norm_iterations; ++t) {
        publish(nullptr, &Context::wn);  // v in full
        for (auto& sp : shards) sp->power_rows(sp->x_full, sp->wm, true);  // w = A v
        publish(&Context::wm, nullptr);  // w in full
        for (auto& sp : shards) sp->power_cols(sp->y_full, sp->wn2, true);  // u = A' w
        const std::vector<double> r2 = global_sum(
            3, [](Context& c) -> const double* { return c.wn2; }, vv, ln, n);
        const double nu = std::sqrt(r2[0]);
        if (nu == 0.0) {
          zero = true;
          break;
        }
        lambda = r2[1];
        set_nu(nu);
        for (auto& sp : shards)
          k_div_scalar<<<blocks_for(sp->n), kBlock, 0, stream>>>(sp->wn2, &sp->pctrl->nu, sp->wn, sp->n);
        CKL("shard power");
      }
      norm = zero ? 0.0 : std::sqrt(std::max(lambda, 0.0));
    } else {
      for (auto& sp : shards) sp->ensure_tuned();
    }
    const double a_norm = norm > 0.0 ? norm : 1.0;
    double omega = cfg.primal_weight;
    if (omega <= 0.0) {  // pdhg.cpp:260-265 on the scaled model
      const double cs = std::sqrt(global_sum(1, [](Context& c) -> const double* { return c.c; },
                                             [](Context& c) -> const double* { return c.s; }, ln, n)[0]);
      const double bs = std::sqrt(global_sum(1, [](Context& c) -> const double* { return c.b; },
                                             [](Context& c) -> const double* { return c.r; }, lm, m)[0]);
      omega = (cs > 0.0 && bs > 0.0) ? cs / bs : 1.0;
    }
    for (auto& sp : shards) {
      sp->b_norm = bn;
      sp->c_norm = cn;
      sp->norm_est = norm;
      sp->omega = omega;
      sp->tau = cfg.step_scale * omega / a_norm;
      sp->sigma = cfg.step_scale / (omega * a_norm);
    }
    CK(cudaStreamSynchronize(stream));
  }

  void build_shards(const cclp_cu_config& cfg) {
    if (graph) {
      cudaGraphExecDestroy(graph);
      graph = nullptr;
    }
    dist_setup(cfg);
    for (auto& sh : shards) {
      k_stamp<<<1, 1, 0, stream>>>(sh->t0);
      CKL("stamp");
    }
  }

  // One iteration on every local shard. With the push transport the
  // exchanges are inside the producers (k_dual, k_primal's last block,
  // k_select_x) and the consumers wait on peer flags: no collective call.
  void launch_round(bool init) {
    for (auto& s : shards) s->launch_rows_half(init);
    if (!push) exchange(&Context::y_full, static_cast<size_t>(s0().Sm), halo_y);
    for (auto& s : shards) s->launch_cols_half(init);
    if (!push) allgather(&Context::xpart, kRowParts + kColParts);
    for (auto& s : shards) {
      k_finalize_shard<<<1, kEpiBlock, 0, stream>>>(s->params, s->xpart, P, init ? 1 : 0);
      k_select_x<<<blocks_for(s->n), kBlock, 0, stream>>>(
          s->params, s->x_full + static_cast<size_t>(s->shard_rank) * s->Sn, 0);
    }
    CKL("shard finalize");
    if (!push) exchange(&Context::x_full, static_cast<size_t>(s0().Sn), halo_x);
    launches += static_cast<long long>(shards.size()) * (kKernelsPerIteration + 2);
  }

  void begin(const cclp_cu_config& cfg, const cclp_cu_tolerances& tol, const double* thr, int nthr) {
    build_shards(cfg);
    for (auto& s : shards) s->init_state(cfg, tol, thr, nthr, false);
    if (push) {
      setup_push();
      for (auto& s : shards)  // x_0 into every shard that gathers it (epoch 1)
        k_select_x<<<blocks_for(s->n), kBlock, 0, stream>>>(s->params, nullptr, 1);
      CKL("push x0");
    } else {
      allgather(&Context::x_full, static_cast<size_t>(s0().Sn));  // x_0: once, in full
    }
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
      s->extract_view(view, st);
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
    if (have_hcomm) {  // every rank ends with the full vectors, through the caller's all-gather
      auto gather_dev = [&](double* fullbuf, size_t S) {
        std::vector<double> mine(S);
        CK(cudaMemcpyAsync(mine.data(), fullbuf + static_cast<size_t>(rank) * S, sizeof(double) * S,
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        const std::vector<char> all = gather_bytes(mine.data(), sizeof(double) * S);
        CK(cudaMemcpyAsync(fullbuf, all.data(), all.size(), cudaMemcpyHostToDevice, stream));
      };
      gather_dev(vx_full, Sn);
      gather_dev(vz_full, Sn);
      gather_dev(vy_full, Sm);
      gather_dev(vparts_full, W);
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
