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
  release(d_rb);
  release(d_cb);
  panel_gn = F.n;  // column panels on the full matrix's column space
  panel_cb = cb;
  for (const auto& pn : F.panels) panel_G_hint.push_back(pn.G);
  partition();  // setup-kernel grids, the local SpMV plans and their tuned geometry
  for (auto& pn : panels)  // the shard never runs setup(): its panels take the scaled values here
    if (pn.nnz > 0)
      k_gather_vals<<<blocks_for(pn.nnz), kBlock, 0, stream>>>(pn.perm, pn.nnz, sval_csr, pn.val);
  CKL("shard panel values");
}

// ---- the sharded solve ---------------------------------------------------------
struct Sharded {
  int P = 1, rank = 0, nranks = 1, device = 0;
  int m = 0, n = 0;  // global
  std::unique_ptr<Context> full;                 // full matrix: setup (replicated per rank)
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

  void build_halo(Halo& h, bool x_side) {
    // x side: rows of A owned by p (full CSR), columns owned by q; y side:
    // rows of A' = columns of A owned by p (the CSC), rows of A owned by q
    const int* ptr = x_side ? full->rowptr : full->colptr;
    const int* idx = x_side ? full->colind : full->rowind;
    const std::vector<int>& own = x_side ? rb : cb;     // rows of this side's matrix per shard
    const std::vector<int>& tgt = x_side ? cb : rb;     // gathered vector's split
    const int len = x_side ? n : m;
    const long long S = x_side ? s0().Sn : s0().Sm;
    const long long allgather = static_cast<long long>(P) * (P - 1) * S;
    unsigned char* flags = full->alloc<unsigned char>(len);
    std::vector<unsigned char> hf(static_cast<size_t>(len));
    h.need.assign(P, std::vector<int*>(P, nullptr));
    h.cnt.assign(P, std::vector<int>(P, 0));
    std::vector<std::vector<std::vector<int>>> lists(P, std::vector<std::vector<int>>(P));
    h.volume = 0;
    for (int p = 0; p < P; ++p) {
      CK(cudaMemsetAsync(flags, 0, std::max(1, len), stream));
      if (own[p + 1] > own[p])
        k_mark_cols<<<blocks_for(1 << 20), kBlock, 0, stream>>>(ptr, idx, own[p], own[p + 1], flags);
      CKL("halo mark");
      CK(cudaMemcpyAsync(hf.data(), flags, len, cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      for (int q = 0; q < P; ++q) {
        if (q == p) continue;
        for (int j = tgt[q]; j < tgt[q + 1]; ++j)
          if (hf[j]) lists[p][q].push_back(j - tgt[q]);
        h.cnt[p][q] = static_cast<int>(lists[p][q].size());
        h.volume += h.cnt[p][q];
      }
    }
    full->release(flags);
    h.on = P > 1 && h.volume * 2 < allgather;
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
    const int first = multi() ? rank : 0;
    const int count = multi() ? 1 : P;
    for (int q = first; q < first + count; ++q) {
      auto sh = std::make_unique<Context>();
      sh->ipc_buffers = push && multi();
      sh->shard_from(*full, q, P, rb, cb, stream);
      k_stamp<<<1, 1, 0, stream>>>(sh->t0);
      CKL("stamp");
      shards.push_back(std::move(sh));
    }
    if (!halo_built) {
      const char* e = std::getenv("CCLP_CU_HALO");  // 0: always all-gather (A/B)
      if (e == nullptr || std::atoi(e) != 0) {
        build_halo(halo_x, true);
        build_halo(halo_y, false);
      }
      halo_built = true;
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
