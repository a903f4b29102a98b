// The four kernels of one PDHG iteration, plus the on-device decision tail.
// Step t (state t -> t+1, pdhg_step, pdhg.cpp:118-143) is:
//
//   k_spmv_rows(t): ax_{t+1} = A x_{t+1}       (x_{t+1} produced by k_primal(t-1))
//   k_dual(t):      y_{t+1} = y' + sigma (b - (2 ax_{t+1} - ax'))   (:125-126)
//                   y_sum, ax_sum += ; row-side report partials for check(t+1)
//   k_spmv_cols(t): aty_{t+1} = A' y_{t+1}
//   k_primal(t):    x_sum, aty_sum += ; column-side report partials; next-x
//                   candidates x_{t+2} = proj(x - tau (c - aty)) for both
//                   outcomes of the restart test at check(t+1) (continue /
//                   restart from the average), so no restart kernel is ever
//                   launched; last block: finalize = check(t+1) decisions
//                   (:311-368).
//
// The SpMV kernels are lean (few registers, high occupancy: the products are
// gather-bound); the epilogues are coalesced streams. (x', y', ax', aty') is
// state t after restart_if_improved (:145-165): when check(t) restarted, the
// kernels read sums * (1/window) instead of the current vectors — the same
// values the reference stores — and restart the sums at zero.
#pragma once

#include "kernels.cuh"

namespace cclp_cu {
namespace {  // internal linkage: compiled into engine.cu and sharded.cu

constexpr unsigned kRowMaxMask = (1u << 1) | (1u << 4);
constexpr unsigned kColMaxMask = (1u << 1) | (1u << 2) | (1u << 3) | (1u << 7) | (1u << 8) | (1u << 9);

struct StepInfo {
  long long t;   // state index before the step (-1 for the initial products)
  long long t1;  // t + 1
  int R;         // restart applied by this step
  int s0, s1;    // ping-pong slots of states t and t+1
  int a0, a1;    // ax slots of states t and t+1 (index mod 3)
  int xs;        // candidate slot holding x_{t+1}
  int xs2;       // candidate slot receiving x_{t+2}
  double inv;    // 1/window_t (restart average)
  double inv1;   // 1/window_{t+1} (average view at check(t+1))
  bool check;    // check(t+1) happens
  bool init;
  // the pending ladder snapshot of state t (inline extraction, decide())
  bool snap;
  int snap_slot, snap_avg, snap_rprev;
  double snap_inv;
};

__device__ __forceinline__ bool step_from(const Ctrl* C, const IterParams& p, bool init, StepInfo& si) {
  if (C->stop >= 0 || C->halt) return false;
  if (init) {
    si.t = -1;
    si.t1 = 0;
    si.R = 0;
    si.s0 = 0;
    si.s1 = 0;
    si.a0 = 0;
    si.a1 = 0;
    si.xs = 0;
    si.xs2 = 1;
    si.inv = 0.0;
    si.inv1 = 0.0;
    si.check = true;
    si.init = true;
    si.snap = false;
    return true;
  }
  si.t = C->iteration;
  si.t1 = si.t + 1;
  si.R = C->R;
  const long long win = C->window;
  const long long win1 = (si.R ? 0 : win) + 1;
  si.inv = si.R ? 1.0 / static_cast<double>(win) : 0.0;
  si.inv1 = 1.0 / static_cast<double>(win1);
  si.s0 = static_cast<int>(si.t & 1);
  si.s1 = si.s0 ^ 1;
  si.a0 = static_cast<int>(si.t % 3);
  si.a1 = static_cast<int>(si.t1 % 3);
  si.xs = static_cast<int>(si.t1 % 3);
  si.xs2 = static_cast<int>((si.t1 + 1) % 3);
  si.check = (si.t1 % p.check_interval) == 0;
  si.init = false;
  si.snap = p.snap_inline && C->snap_pending;
  if (si.snap) {
    si.snap_slot = C->snaps_done % kSnapSlots;
    si.snap_avg = C->snap_use_avg;
    si.snap_rprev = C->snap_rprev;
    si.snap_inv = C->snap_inv;
  }
  return true;
}

__device__ __forceinline__ unsigned ld_relaxed_sys(const volatile unsigned* a) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}

// In-graph phase stamps: block 0 of each of the step's four kernels records
// %globaltimer once the previous kernel has completed (after the PDL wait),
// into a ring of kStampRing steps; consecutive stamps split the iteration
// into rows / dual / cols / primal+decide as they run inside the CUDA graph
// (cclp_cu_phase_profile). A store by one thread per kernel: no load, no wait.
__device__ __forceinline__ void stamp_phase(const IterParams& p, const StepInfo& si, int phase) {
  if (phase >= 0 && p.stamps != nullptr && !si.init && blockIdx.x == 0 && threadIdx.x == 0)
    p.stamps[(si.t % kStampRing) * 4 + phase] = globaltimer();
}

__device__ __forceinline__ bool read_step(const IterParams& p, bool init, StepInfo& si, int phase = -1) {
  pdl_wait();  // the previous kernel of the step (or step) must be complete
  const bool go = step_from(p.ctrl, p, init, si);
  if (go) stamp_phase(p, si, phase);
  return go;
}

// ---- push transport (PushArgs, kernels.cuh) --------------------------------
// Memory scope of the pushes' fences and flags: system scope between
// processes / GPUs (CUDA IPC over NVLink), GPU scope when every shard lives on
// this device in this process (PushArgs::gpu_scope) — the system-scope fences
// cost ~40 us per shard and iteration there (C4, 8 shards on one GPU: 1,624 ->
// 1,300 us per iteration).
__device__ __forceinline__ void st_release(const PushArgs& ps, unsigned long long* a, unsigned long long v) {
  if (ps.gpu_scope)
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
  else
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const PushArgs& ps, const unsigned long long* a) {
  unsigned long long v;
  if (ps.gpu_scope)
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  else
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void push_fence(const PushArgs& ps) {
  if (ps.gpu_scope)
    __threadfence();
  else
    __threadfence_system();
}
// Consumer side: wait until every peer has released epoch `value` for
// `kind` (threads < P poll; bounded: a lost peer traps instead of hanging).
__device__ __forceinline__ void push_wait(const PushArgs& ps, int kind, unsigned long long value) {
  if (threadIdx.x < ps.P && static_cast<int>(threadIdx.x) != ps.rank) {
    const unsigned long long* f = ps.my_flags + kind * kMaxPushShards + threadIdx.x;
    long long spins = 0;
    while (ld_acquire(ps, f) < value) {
      __nanosleep(32);
      if (++spins > (1LL << 30)) __trap();
    }
  }
  __syncthreads();
}
// Producer side, after every thread's stores: the grid's last block
// releases `value` for `kind` in every peer's flag array.
__device__ __forceinline__ void push_signal_grid(const PushArgs& ps, int kind, unsigned long long value,
                                                 unsigned* counter) {
  __shared__ bool last_blk;
  push_fence(ps);
  __syncthreads();
  if (threadIdx.x == 0) last_blk = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last_blk || threadIdx.x != 0) return;
  push_fence(ps);
  for (int q = 0; q < ps.P; ++q) st_release(ps, ps.flags[q] + kind * kMaxPushShards + ps.rank, value);
  *counter = 0u;
}

// The global values decide() reads, loaded into shared memory by a thread the
// partial reduction leaves idle, so their latency overlaps it: the cancel
// request block 0 of the column kernel mirrored, the loop's start time and
// the next ladder threshold.
constexpr int kPrefetchThread = 480;  // reduce_partials uses threads 0..351
struct DecidePrefetch {
  unsigned cancel;
  unsigned long long t0;
  double thr;
};
__device__ __forceinline__ DecidePrefetch decide_prefetch(const IterParams& p) {
  DecidePrefetch f{0u, 0ull, 0.0};
  if (p.cancel_dev != nullptr) f.cancel = *reinterpret_cast<volatile unsigned*>(p.cancel_dev);
  f.t0 = *p.t0_ns;
  const int nt = __ldcg(&p.ctrl->next_threshold);
  if (nt < p.nthr) f.thr = __ldcg(p.thr + nt);
  return f;
}

// check(t+1) and everything after the step in the reference pass
// (pdhg.cpp:128-130 error, 301-368 next pass: time, check, limit), taken by
// thread 0 on a shared-memory copy of the control block. `rep` holds the two
// reports of check(t+1) (current, average), assembled beforehand by two
// other threads.
__device__ __forceinline__ void decide(const IterParams& p, const StepInfo& si, Ctrl* C,
                                       const double* rowv, const double* colv, const double (*rep)[kRepN],
                                       const DecidePrefetch& pf, bool write_log = true) {
  if (!si.init && p.snap_inline && C->snap_pending) {  // this step extracted the pending snapshot
    SnapMeta& mt = C->snap_meta[C->snaps_done % kSnapSlots];
    mt.iteration = C->snap_iteration;
    mt.maxresid = C->snap_maxresid;
    mt.thr_idx = C->snap_thr_idx;
    mt.use_avg = C->snap_use_avg;
    C->snaps_done++;
    C->snap_pending = 0;
  }
  if (!si.init) {
    if (rowv[6] + colv[12] > 0.0) {  // PdhgNumericalError before commit
      C->stop = 5;
      C->error_iteration = si.t;
      C->result_view = kViewCurEff;
      C->result_report_valid = C->checked;
      if (C->checked) {
        const double* src = C->R ? C->avg : C->cur;
        for (int k = 0; k < kRepN; ++k) C->result_report[k] = src[k];
      }
      return;
    }
    C->R_prev = C->R;
    C->window = (C->R ? 0 : C->window) + 1;
    C->iteration = si.t1;
    C->R = 0;
  }
  const long long t1 = si.t1;
  const long long win = C->window;
  C->checked = si.check ? 1 : 0;
  if (si.check) {
    for (int k = 0; k < kRepN; ++k) C->cur[k] = rep[0][k];
    if (win > 0)
      for (int k = 0; k < kRepN; ++k) C->avg[k] = rep[1][k];
  }
  // cancel poll at the top of the pass (pdhg.cpp:301-305): the request the
  // host mirrored into mapped memory, read by k_primal's block 0 this step
  if (pf.cancel != 0u) {
    C->stop = 3;
    C->result_view = kViewCur;
    C->result_report_valid = C->checked;
    if (C->checked)
      for (int k = 0; k < kRepN; ++k) C->result_report[k] = C->cur[k];
    return;
  }
  if (isfin(p.time_limit)) {  // pdhg.cpp:306-310
    const double el = 1e-9 * static_cast<double>(globaltimer() - pf.t0);
    if (el > p.time_limit) {
      C->stop = 2;
      C->result_view = kViewCur;
      C->result_report_valid = C->checked;
      if (C->checked)
        for (int k = 0; k < kRepN; ++k) C->result_report[k] = C->cur[k];
      return;
    }
  }
  if (si.check) {  // pdhg.cpp:311-363
    const bool use_avg = win > 0 && C->avg[kMaxResid] < C->cur[kMaxResid];
    C->use_avg = use_avg ? 1 : 0;
    const double* better = use_avg ? C->avg : C->cur;
    if (!C->have_best || better[kMaxResid] < C->best[kMaxResid]) {
      for (int k = 0; k < kRepN; ++k) C->best[k] = better[k];
      C->have_best = 1;
    }
    if (C->last_restart_resid == CCLP_INF) C->last_restart_resid = C->cur[kMaxResid];
    if (p.log_interval > 0 && t1 % p.log_interval == 0) {
      if (write_log) {
        LogEntry& e = p.log[C->log_count % p.log_cap];
        e.iteration = t1;
        e.rel_primal = better[kRelP];
        e.rel_dual = better[kRelD];
        e.rel_gap = better[kRelGap];
        e.elapsed = 1e-9 * static_cast<double>(globaltimer() - pf.t0);
      }
      C->log_count++;
    }
    if (better[kMaxResid] <= p.eps_rel) {
      C->stop = 0;
      C->result_view = use_avg ? kViewAvg : kViewCur;
      C->result_report_valid = 1;
      for (int k = 0; k < kRepN; ++k) C->result_report[k] = better[k];
      return;
    }
    if (C->next_threshold < p.nthr && better[kMaxResid] <= pf.thr) {
      // a free slot: the next step extracts the view and the loop runs on;
      // else halt and let the host extract it (pdhg.cpp:346-358)
      const int copied = p.host_flags != nullptr ? static_cast<int>(ld_relaxed_sys(p.host_flags + 1)) : 0;
      const bool inl = p.snap_inline && p.host_flags != nullptr && C->snaps_done - copied < kSnapSlots;
      if (!inl) C->halt = 1;
      C->snap_rprev = C->R_prev;
      C->snap_inv = win > 0 ? 1.0 / static_cast<double>(win) : 0.0;
      C->snap_pending = 1;
      C->snap_use_avg = use_avg ? 1 : 0;
      C->snap_thr_idx = C->next_threshold;
      C->snap_maxresid = better[kMaxResid];
      C->snap_iteration = t1;
      C->next_threshold++;
    }
    if (win > 0 && C->avg[kMaxResid] <= p.restart_factor * C->last_restart_resid) {
      C->R = 1;  // applied by the next step's kernels
      C->last_restart_resid = C->avg[kMaxResid];
      C->restarts++;
    }
  }
  if (t1 >= p.max_iter) {  // pdhg.cpp:364-368
    C->stop = 1;
    C->result_view = kViewCurEff;
    C->result_report_valid = C->checked;
    if (C->checked) {
      const double* src = C->R ? C->avg : C->cur;
      for (int k = 0; k < kRepN; ++k) C->result_report[k] = src[k];
    }
  }
}

static_assert(sizeof(Ctrl) % 8 == 0, "Ctrl is copied as 8-byte words");

// Reduces every epilogue block's partials (field-major: field f of block b at
// src[f * nblocks + b]) into rowv[kRowParts] and colv[kColParts] (shared
// memory), deterministically.
__device__ __forceinline__ void reduce_partials(const double* rowsrc, int nrow, const double* colsrc,
                                                int ncol, double* rowv, double* colv) {
  // half-warp h takes field h (all 22 fields in one round with >= 11 warps);
  // lane l of the half takes blocks l, l+16, ... with 16 loads in flight (one
  // round up to 256 blocks; consecutive lanes read consecutive blocks),
  // accumulates them in order, then a fixed butterfly within the half
  const int hl = threadIdx.x & 15;
  for (int fld = threadIdx.x >> 4; fld - static_cast<int>(threadIdx.x >> 4) < kRowParts + kColParts;
       fld += blockDim.x / 16) {
    const bool live = fld < kRowParts + kColParts;
    const bool is_row = fld < kRowParts;
    const int f = is_row ? fld : fld - kRowParts;
    const bool is_max = is_row ? ((kRowMaxMask >> f) & 1u) : ((kColMaxMask >> f) & 1u);
    const int nb = live ? (is_row ? nrow : ncol) : 0;
    const double* src = (is_row ? rowsrc : colsrc) + static_cast<long long>(f) * nb;
    double a = 0.0;
    for (int b0 = hl; b0 < nb; b0 += 16 * 16) {
      double v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int b = b0 + 16 * k;
        v[k] = b < nb ? __ldcg(src + b) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k)
        if (b0 + 16 * k < nb) a = is_max ? amax(a, v[k]) : a + v[k];
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, a, off);
      a = is_max ? amax(a, o) : a + o;
    }
    if (hl == 0 && live) (is_row ? rowv : colv)[f] = a;
  }
  __syncthreads();
}

// The control block's shared copy; loaded before the partial reduction so
// the two round trips overlap.
__device__ __forceinline__ Ctrl& ctrl_smem() {
  __shared__ Ctrl cs;
  return cs;
}
__device__ __forceinline__ void load_ctrl(const IterParams& p) {
  constexpr int kWords = sizeof(Ctrl) / 8;
  long long* csw = reinterpret_cast<long long*>(&ctrl_smem());
  const long long* gw = reinterpret_cast<const long long*>(p.ctrl);
  for (int w = threadIdx.x; w < kWords; w += blockDim.x) csw[w] = __ldcg(gw + w);
}

// Expects load_ctrl() and a block barrier before it, and `pf` in shared memory.
__device__ void decide_and_store(const IterParams& p, const StepInfo& si, const double* rowv,
                                 const double* colv, const DecidePrefetch& pf) {
  Ctrl& cs = ctrl_smem();
  constexpr int kWords = sizeof(Ctrl) / 8;
  long long* csw = reinterpret_cast<long long*>(&cs);
  __shared__ double rep[2][kRepN];
  // the two reports of check(t+1) in parallel (make_report: sqrt and divisions)
  if (si.check) {
    if (threadIdx.x == 32) make_report(rowv, colv, p.b_norm, p.c_norm, rep[0]);
    if (threadIdx.x == 64) make_report(rowv + 3, colv + 6, p.b_norm, p.c_norm, rep[1]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cs.t_cols_start = globaltimer();  // debug: reuse as "partials reduced" stamp
    decide(p, si, &cs, rowv, colv, rep, pf);
    cs.t_fin_end = globaltimer();
  }
  __syncthreads();
  long long* out = reinterpret_cast<long long*>(p.ctrl);
  for (int w = threadIdx.x; w < kWords; w += blockDim.x) out[w] = csw[w];
}

// Runs on the last block of k_primal: all partials, then the decisions. In
// sharded mode it only publishes this shard's sums (k_finalize_shard decides
// once every shard's sums have been exchanged).
__device__ void finalize(const IterParams& p, const StepInfo& si) {
  __shared__ double rowv[kRowParts];
  __shared__ double colv[kColParts];
  const bool deciding = p.xpart_loc == nullptr && !p.push.on;
  __shared__ DecidePrefetch pf;
  if (deciding && threadIdx.x == kPrefetchThread % blockDim.x) pf = decide_prefetch(p);
  if (deciding) load_ctrl(p);
  reduce_partials(p.rowp, p.row_grid, p.colp, p.col_grid, rowv, colv);  // ends with a barrier
  if (p.push.on) {  // this shard's sums into every shard's [P][22], then release
    constexpr int W = kRowParts + kColParts;
    for (int k = threadIdx.x; k < p.push.P * W; k += blockDim.x) {
      const int q = k / W, f = k % W;
      p.push.part[q][p.push.rank * W + f] = f < kRowParts ? rowv[f] : colv[f - kRowParts];
    }
    push_fence(p.push);
    __syncthreads();
    if (threadIdx.x == 0)
      for (int q = 0; q < p.push.P; ++q)
        st_release(p.push, p.push.flags[q] + kPushPart * kMaxPushShards + p.push.rank,
                   static_cast<unsigned long long>(si.t1 + 1));
    return;
  }
  if (p.xpart_loc != nullptr) {
    if (threadIdx.x < kRowParts) p.xpart_loc[threadIdx.x] = rowv[threadIdx.x];
    if (threadIdx.x < kColParts) p.xpart_loc[kRowParts + threadIdx.x] = colv[threadIdx.x];
    return;
  }
  decide_and_store(p, si, rowv, colv, pf);
}

// Sharded mode: every shard reduces the exchanged per-shard sums
// xpart[P][kRowParts + kColParts] in shard order (so all shards take
// identical decisions), then decides.
__global__ void __launch_bounds__(kEpiBlock) k_finalize_shard(const IterParams p, const double* xpart,
                                                              int nshards, int init) {
  StepInfo si;
  if (!read_step(p, init != 0, si)) return;
  __shared__ double rowv[kRowParts];
  __shared__ double colv[kColParts];
  if (p.push.on) push_wait(p.push, kPushPart, static_cast<unsigned long long>(si.t1 + 1));
  __shared__ DecidePrefetch pf;
  if (threadIdx.x == kPrefetchThread % blockDim.x) pf = decide_prefetch(p);
  load_ctrl(p);
  constexpr int W = kRowParts + kColParts;
  if (threadIdx.x < W) {
    const int f = threadIdx.x;
    const bool is_row = f < kRowParts;
    const int k = is_row ? f : f - kRowParts;
    const bool is_max = is_row ? ((kRowMaxMask >> k) & 1u) : ((kColMaxMask >> k) & 1u);
    double a = 0.0;
    for (int b = 0; b < nshards; ++b) {
      const double v = __ldcg(xpart + b * W + f);
      a = is_max ? amax(a, v) : a + v;
    }
    (is_row ? rowv : colv)[k] = a;
  }
  __syncthreads();
  decide_and_store(p, si, rowv, colv, pf);
}

// Sharded mode: this shard's slice of the next iterate, x_{t+2} =
// xc[(t+1) % 3][R] after check(t+1), into its region of the full x
// (idempotent, so it may run after a stop or halt).
// With the push transport it stores the slice into every shard that gathers
// it and releases epoch t+2 (the consuming step's t1 + 1); `initial` pushes
// x_0 for the initial products (epoch 1).
__global__ void k_select_x(const IterParams p, double* __restrict__ x_full_loc, int initial) {
  pdl_wait();
  const Ctrl* C = p.ctrl;
  const double* __restrict__ src = initial ? p.xc[0][0] : p.xc[(C->iteration + 1) % 3][C->R];
  if (!p.push.on) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.n; j += gridDim.x * blockDim.x)
      x_full_loc[j] = src[j];
    return;
  }
  const PushArgs& ps = p.push;
  const long long off = static_cast<long long>(ps.rank) * ps.Sn;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.n; j += gridDim.x * blockDim.x) {
    const double v = src[j];
    const unsigned mk = ps.mask_x != nullptr ? ps.mask_x[j] : 0xFFu;
    for (int q = 0; q < ps.P; ++q)
      if ((mk >> q) & 1u) ps.x[q][off + j] = v;
  }
  push_signal_grid(ps, kPushX, initial ? 1ull : static_cast<unsigned long long>(C->iteration + 2),
                   ps.counter + 1);
}

// Lean SpMV of one half-step: out[r] = sum_k M[r,k] vec[k] over CSR M.
// Block b owns the contiguous, nnz-balanced row range [start[b], start[b+1])
// and its warps walk it together (so on structured LPs their gathers share an
// L1-resident window of vec); G lanes per row. The per-row summation order
// depends only on G, never on the launch geometry, so the geometry can be
// autotuned without changing a bit of the result; G = 1 sums each row in the
// reference's own order.
template <class Gather>
__device__ __forceinline__ void spmv_long_segments(const SpmvPlan& P, const int* __restrict__ idx,
                                                   const double* __restrict__ val, const Gather& g,
                                                   double* __restrict__ out, int accumulate);

template <int G, bool LONG, class Gather>
__device__ __forceinline__ void spmv_block_range(const SpmvPlan& P, const int* __restrict__ ptr,
                                                 const int* __restrict__ idx,
                                                 const double* __restrict__ val, const Gather& g,
                                                 double* __restrict__ out, int rpg = 1,
                                                 int accumulate = 0) {
  const int gl = threadIdx.x % G;
  const int gpb = blockDim.x / G;
  const int rb = P.start[blockIdx.x], re = P.start[blockIdx.x + 1];
  const int thr = LONG ? P.thr : 0x7fffffff;
  if (rpg == 2) {  // two rows per group in flight: rows r and r + gpb of a 2*gpb round
    for (int row = rb + static_cast<int>(threadIdx.x / G); row - static_cast<int>(threadIdx.x / G) < re;
         row += 2 * gpb) {
      const int row1 = row + gpb;
      bool ok0 = row < re, ok1 = row1 < re;
      int b0 = ok0 ? __ldg(ptr + row) : 0, e0 = ok0 ? __ldg(ptr + row + 1) : 0;
      int b1 = ok1 ? __ldg(ptr + row1) : 0, e1 = ok1 ? __ldg(ptr + row1 + 1) : 0;
      if (LONG && e0 - b0 > thr) ok0 = false, e0 = b0;  // long row: summed by segments
      if (LONG && e1 - b1 > thr) ok1 = false, e1 = b1;
      double s0, s1;
      group_dot2<G, 2>(b0, e0, b1, e1, gl, idx, val, g, s0, s1);
      if (gl == 0 && ok0) out[row] = (accumulate ? out[row] : 0.0) + s0;
      if (gl == 0 && ok1) out[row1] = (accumulate ? out[row1] : 0.0) + s1;
    }
  } else {
    for (int row = rb + static_cast<int>(threadIdx.x / G); row - static_cast<int>(threadIdx.x / G) < re;
         row += gpb) {
      bool ok = row < re;
      int b = ok ? __ldg(ptr + row) : 0, e = ok ? __ldg(ptr + row + 1) : 0;
      if (LONG && e - b > thr) ok = false, e = b;
      const double s = group_dot<G, 4>(b, e, gl, idx, val, g);
      if (gl == 0 && ok) out[row] = (accumulate ? out[row] : 0.0) + s;
    }
  }
  if (LONG) spmv_long_segments(P, idx, val, g, out, accumulate);
}

// Long-row segments of block blockIdx.x: one warp per segment, 32 lanes
// strided, then the last segment of a row to finish combines them in order.
template <class Gather>
__device__ __forceinline__ void spmv_long_segments(const SpmvPlan& P, const int* __restrict__ idx,
                                                   const double* __restrict__ val, const Gather& g,
                                                   double* __restrict__ out, int accumulate) {
  const int lane = threadIdx.x & 31;
  const int sb = P.start[P.grid + 1 + blockIdx.x], se = P.start[P.grid + 2 + blockIdx.x];
  for (int k = sb + static_cast<int>(threadIdx.x >> 5); k < se; k += static_cast<int>(blockDim.x >> 5)) {
    const int4 sg = P.seg[k];  // row, begin, end, long-row index
    const double s = group_dot<32, 4>(sg.y, sg.z, lane, idx, val, g);
    if (lane == 0) {
      const int f0 = __ldg(P.lr_first + sg.w), f1 = __ldg(P.lr_first + sg.w + 1);
      if (f1 - f0 == 1) {  // a single-segment row: no combine
        out[sg.x] = (accumulate ? out[sg.x] : 0.0) + s;
      } else {
        P.part[k] = s;
        __threadfence();
        if (atomicAdd(P.cnt + sg.w, 1u) == static_cast<unsigned>(f1 - f0 - 1)) {
          __threadfence();
          double acc = 0.0;
          for (int q = f0; q < f1; ++q) acc = acc + __ldcg(P.part + q);
          out[sg.x] = (accumulate ? out[sg.x] : 0.0) + acc;
          P.cnt[sg.w] = 0u;
        }
      }
    }
  }
}

template <int G, bool LONG, class Gather>
__global__ void __launch_bounds__(kSpmvBlock) k_spmv_range(const SpmvPlan P, const int* __restrict__ ptr,
                                                           const int* __restrict__ idx,
                                                           const double* __restrict__ val, Gather g,
                                                           double* __restrict__ out, int rpg = 1,
                                                           int accumulate = 0) {
  pdl_wait();  // a no-op unless launched programmatically (the power iteration)
  spmv_block_range<G, LONG>(P, ptr, idx, val, g, out, rpg, accumulate);
}

// One column panel of ax_{t+1} = A x_{t+1} (panels run in panel order; the
// first writes, the others add).
template <int G, bool LONG>
__global__ void __launch_bounds__(kSpmvBlock) k_spmv_rows_panel(const IterParams p, int init,
                                                                const PanelArgs a) {
  StepInfo si;
  if (!read_step(p, init != 0, si, a.accumulate ? -1 : 0)) return;
  if (p.push.on) push_wait(p.push, kPushX, static_cast<unsigned long long>(si.t1 + 1));
  spmv_block_range<G, LONG>(a.plan, a.ptr, a.idx, a.val,
                            GatherPlain{p.xg != nullptr ? p.xg : p.xc[si.xs][si.R]}, p.ax[si.a1], 1,
                            a.accumulate);
}

// Row product ax_{t+1} = A x_{t+1} of step t, `rows(x, ax)`. On the
// single-device loop (p.spec) it does not wait for k_primal(t-1)'s decision
// tail: that kernel's last block publishes t and the candidates-ready epoch,
// then triggers this launch while it reduces the partials and runs decide().
// The product runs on the no-restart candidate xc[(t+1) % 3][0]; each block
// then waits for the decided epoch and, in the rare step that restarts,
// recomputes its rows from the restart candidate (stop / halt: the result is
// never read; ax has three slots, so states t and t-1 stay intact). Per-row
// order is unchanged, so ax is bit-identical to the waiting form. Without a
// pending decision (PDL off, init, k_primal exited early) it takes the
// waiting form.
template <class Rows>
__device__ __forceinline__ void row_step(const IterParams& p, int init, const Rows& rows) {
  if (p.spec != nullptr && !init) {
    __shared__ long long sp_t;
    __shared__ unsigned long long sp_d;
    __shared__ int sp_go, sp_r;
    if (threadIdx.x == 0) {
      const unsigned long long S = ld_acquire_gpu(p.spec);
      const unsigned long long D = ld_relaxed_gpu(p.spec + 1);
      sp_go = S != D ? 1 : 0;
      sp_d = D;
      sp_t = static_cast<long long>(ld_relaxed_gpu(p.spec + 2));
    }
    __syncthreads();
    if (sp_go) {
      const long long t = sp_t;
      if (p.stamps != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
        p.stamps[(t % kStampRing) * 4] = globaltimer();
      const int xs = static_cast<int>((t + 1) % 3);
      double* out = p.ax[xs];
      rows(p.xc[xs][0], out);
      if (threadIdx.x == 0) {
        long long spins = 0;  // bounded: a lost decision traps instead of hanging
        while (ld_relaxed_gpu(p.spec + 1) == sp_d) {
          __nanosleep(32);
          if (++spins > (1LL << 30)) __trap();
        }
        ld_acquire_gpu(p.spec + 1);  // one acquire orders the control-block reads
        const volatile Ctrl* C = p.ctrl;
        sp_r = (C->stop >= 0 || C->halt) ? 0 : C->R;
      }
      __syncthreads();
      if (sp_r) rows(p.xc[xs][1], out);
      pdl_wait();
      return;
    }
  }
  StepInfo si;
  if (!read_step(p, init != 0, si, 0)) return;
  if (p.push.on) push_wait(p.push, kPushX, static_cast<unsigned long long>(si.t1 + 1));
  rows(p.xg != nullptr ? p.xg : p.xc[si.xs][si.R], p.ax[si.a1]);
}

template <int G, bool LONG>
__global__ void __launch_bounds__(kSpmvBlock, 2048 / kSpmvBlock) k_spmv_rows(const IterParams p, int init) {
  row_step(p, init, [&](const double* x, double* out) {
    spmv_block_range<G, LONG>(p.plan_r, p.rowptr, p.colind, p.aval, GatherPlain{x}, out, p.rpg_rows);
  });
}

// SELL-32 column product of block blockIdx.x's slices: lane = column, its
// elements in ascending position with one accumulator (the reference's
// sequential order, as the G = 1 path), 4 gathers in flight. Columns longer
// than S.thr are written by the long-row segments instead.
template <class Gather>
__device__ __forceinline__ void sell_block(const SellPlan& S, const Gather& g, double* __restrict__ out) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  // block-contiguous slice ranges (S.start), or, with S.start == nullptr,
  // slices dealt round-robin over every warp of the grid
  int s0, se, step;
  if (S.start != nullptr) {
    s0 = S.start[blockIdx.x] + static_cast<int>(threadIdx.x >> 5);
    se = S.start[blockIdx.x + 1];
    step = static_cast<int>(blockDim.x >> 5);
  } else {
    s0 = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    se = (S.n + 31) / 32;
    step = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  }
  for (int s = s0; s < se; s += step) {
    const long long off = S.off[s];
    const int w = static_cast<int>((S.off[s + 1] - off) >> 5);
    const int j = s * 32 + lane;
    int len = j < S.n ? __ldg(S.ptr + j + 1) - __ldg(S.ptr + j) : 0;
    const bool seg = len > S.thr;
    if (seg) len = 0;
    const int* __restrict__ ib = S.idx + off + lane;
    const double* __restrict__ vb = S.val + off + lane;
    // U index/value loads, then U gathers, then U multiply-adds in order:
    // 32 registers, two 1024-thread blocks per SM (C3 columns 77.7 -> 69.6
    // us against the software-pipelined loop's 44 registers and one block;
    // profiles/r2/history/r2_sell_cols_occupancy.txt)
    double acc = 0.0;
    for (int k = 0; k < w; k += U) {
      int ii[U];
      double vv[U], xx[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = k + u < len;
        ii[u] = ok ? ld_stream(ib + 32 * (k + u)) : -1;
        vv[u] = ok ? ld_stream(vb + 32 * (k + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xx[u] = ii[u] >= 0 ? g(ii[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ii[u] >= 0) acc = acc + vv[u] * xx[u];
    }
    if (j < S.n && !seg) out[j] = acc;
  }
}

// SELL-G row product of block blockIdx.x's slices: 32/G rows per slice, lane
// gl of a row's group takes the row's elements gl, gl+G, ... in order (4 in
// flight) and the group ends with the xor butterfly — the CSR-G kernel's
// exact per-lane order and combine, so the sums are bit-identical to it
// while every index/value load is one 128-byte line. Rows longer than S.thr
// are written by the long-row segments.
template <int G, class Gather>
__device__ __forceinline__ void sellg_block(const SellPlan& S, const Gather& g, double* __restrict__ out) {
  constexpr int U = 4, R = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int r = lane / G, gl = lane % G;
  const int sb = S.start[blockIdx.x], se = S.start[blockIdx.x + 1];
  for (int s = sb + warp; s < se; s += nw) {
    const long long off = S.off[s];
    const int w = static_cast<int>((S.off[s + 1] - off) >> 5);
    const int row = s * R + r;
    int len = row < S.n ? __ldg(S.ptr + row + 1) - __ldg(S.ptr + row) : 0;
    const bool seg = len > S.thr;
    if (seg) len = 0;
    const int* __restrict__ ib = S.idx + off + lane;
    const double* __restrict__ vb = S.val + off + lane;
    double acc = 0.0;
    for (int k = 0; k < w; k += U) {
      int ii[U];
      double vv[U], xx[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = (k + u) * G + gl < len;
        ii[u] = ok ? ld_line(ib + 32 * (k + u)) : -1;
        vv[u] = ok ? ld_line(vb + 32 * (k + u)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) xx[u] = ii[u] >= 0 ? g(ii[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (ii[u] >= 0) acc = acc + vv[u] * xx[u];
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (gl == 0 && row < S.n && !seg) out[row] = 0.0 + acc;
  }
}

template <int G, bool LONG, int BS>
__global__ void __launch_bounds__(BS) k_sellg_range(const SellPlan S, const SpmvPlan P, const int* __restrict__ idx,
                                                    const double* __restrict__ val, GatherPlain g,
                                                    double* __restrict__ out) {
  sellg_block<G>(S, g, out);
  if (LONG) spmv_long_segments(P, idx, val, g, out, 0);
}

template <int G, bool LONG, int BS>
__global__ void __launch_bounds__(BS, 2048 / BS) k_spmv_rows_sellg(const IterParams p, int init) {
  row_step(p, init, [&](const double* x, double* out) {
    const GatherPlain g{x};
    sellg_block<G>(p.sell_r, g, out);
    if (LONG) spmv_long_segments(p.plan_r, p.colind, p.aval, g, out, 0);
  });
}

template <int G, bool LONG, int BS>
__global__ void __launch_bounds__(BS) k_spmv_cols_sellg(const IterParams p, int init) {
  StepInfo si;
  if (!read_step(p, init != 0, si, 2)) return;
  if (p.push.on) push_wait(p.push, kPushY, static_cast<unsigned long long>(si.t1 + 1));
  const GatherPlain g{p.yg != nullptr ? p.yg : p.y[si.s1]};
  sellg_block<G>(p.sell_cg, g, p.aty[si.s1]);
  if (LONG) spmv_long_segments(p.plan_c, p.rowind, p.atval, g, p.aty[si.s1], 0);
}

// Stand-alone SELL product (geometry tuning in Context::build_sell_cols).
template <int BS>
__global__ void __launch_bounds__(BS, 2048 / BS) k_sell_range(const SellPlan S, GatherPlain g, double* __restrict__ out) {
  sell_block(S, g, out);
}

template <bool LONG, int BS>
__global__ void __launch_bounds__(BS, 2048 / BS) k_spmv_cols_sell(const IterParams p, int init) {
  StepInfo si;
  if (!read_step(p, init != 0, si, 2)) return;
  if (p.push.on) push_wait(p.push, kPushY, static_cast<unsigned long long>(si.t1 + 1));
  const GatherPlain g{p.yg != nullptr ? p.yg : p.y[si.s1]};
  sell_block(p.sell_c, g, p.aty[si.s1]);
  if (LONG) spmv_long_segments(p.plan_c, p.rowind, p.atval, g, p.aty[si.s1], 0);
}

template <int G, bool LONG>
__global__ void __launch_bounds__(kSpmvBlock) k_spmv_cols(const IterParams p, int init) {
  StepInfo si;
  if (!read_step(p, init != 0, si, 2)) return;
  if (p.push.on) push_wait(p.push, kPushY, static_cast<unsigned long long>(si.t1 + 1));
  spmv_block_range<G, LONG>(p.plan_c, p.colptr, p.rowind, p.atval,
                            GatherPlain{p.yg != nullptr ? p.yg : p.y[si.s1]},
                      p.aty[si.s1], p.rpg_cols);
}

// ---- the epilogues' operand streams, moved by the TMA engine -------------
// 1-D bulk async copies (cp.async.bulk) of kTile-element tiles of every
// operand stream into a kStages-deep shared-memory ring: one thread issues, an
// mbarrier per stage counts the bytes in. An SM keeps up to kStages tiles of
// all streams in flight (112-128 KB) without holding registers. Block b takes
// tiles b, b + grid, ..., thread t element t of each: body(j, v) with
// v[q] = stream q's element j (streams outside `mask` are not copied and
// read as 0). The grid is fixed (one block per SM), so every thread's
// partial sums cover the same elements on every run.
constexpr int kTile = 512;
constexpr int kStages = 4;
template <int NS>
__host__ __device__ constexpr size_t bulk_smem() {
  return static_cast<size_t>(kStages) * NS * kTile * sizeof(double) + kStages * 8;
}
template <int NS, class Body>
__device__ __forceinline__ void bulk_stream(int n, const double* const (&src)[NS], unsigned mask, Body&& body) {
  extern __shared__ __align__(16) double sbuf[];  // [stage][stream][tile]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(sbuf + kStages * NS * kTile);
  const int ntiles = (n + kTile - 1) / kTile;
  const int b = static_cast<int>(blockIdx.x), g = static_cast<int>(gridDim.x);
  const int mine = b < ntiles ? (ntiles - 1 - b) / g + 1 : 0;
  auto issue = [&](int k) {  // my k-th tile into stage k % kStages
    const int j0 = (b + k * g) * kTile;
    // whole 16-byte units: an odd tail reads one element past the end
    // (every device vector is allocated with slack, Context::alloc)
    const unsigned bytes = static_cast<unsigned>((min(kTile, n - j0) + 1) & ~1) * 8u;
    const int st = k % kStages;
    mbar_expect_tx(&full[st], bytes * static_cast<unsigned>(__popc(mask)));
#pragma unroll
    for (int q = 0; q < NS; ++q)
      if ((mask >> q) & 1u) bulk_g2s(sbuf + (st * NS + q) * kTile, src[q] + j0, bytes, &full[st]);
  };
  if (threadIdx.x == 0) {
    for (int st = 0; st < kStages; ++st) mbar_init(&full[st], 1);
    mbar_init_fence();
    for (int k = 0; k < min(kStages, mine); ++k) issue(k);
  }
  __syncthreads();
  double v[NS];
  for (int k = 0; k < mine; ++k) {
    const int st = k % kStages;
    mbar_wait(&full[st], static_cast<unsigned>((k / kStages) & 1));
    const int j = (b + k * g) * kTile + static_cast<int>(threadIdx.x);
    if (j < n) {
#pragma unroll
      for (int q = 0; q < NS; ++q) v[q] = ((mask >> q) & 1u) ? sbuf[(st * NS + q) * kTile + threadIdx.x] : 0.0;
      body(j, v);
    }
    __syncthreads();  // every thread is done with this stage
    if (threadIdx.x == 0 && k + kStages < mine) {
      fence_proxy_async();
      issue(k + kStages);
    }
  }
}

// The same walk without the shared-memory ring, for short vectors (a block
// gets only a few tiles, so the ring's first-tile latency is not amortized):
// thread t of block b takes elements b * kTile + t + k * grid * kTile,
// k = 0, 1, ... in order — the elements and order of bulk_stream, so every
// thread's partial sums, the block partials and all results are identical —
// with two elements' loads in flight.
template <int NS, class Body>
__device__ __forceinline__ void reg_stream(int n, const double* const (&src)[NS], unsigned mask, Body&& body) {
  const int stride = static_cast<int>(gridDim.x) * kTile;
  for (int j0 = static_cast<int>(blockIdx.x) * kTile + static_cast<int>(threadIdx.x); j0 < n; j0 += 2 * stride) {
    const int j1 = j0 + stride;
    double v0[NS], v1[NS];
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      const bool on = (mask >> q) & 1u;
      v0[q] = on ? src[q][j0] : 0.0;
      v1[q] = on && j1 < n ? src[q][j1] : 0.0;
    }
    body(j0, v0);
    if (j1 < n) body(j1, v1);
  }
}

// k_dual's operand streams: r, b, ax_{t+1}, then state t: y, ax, y_sum, ax_sum.
enum DualStream : int { kDsR = 0, kDsB, kDsAxn, kDsY, kDsAx, kDsYs, kDsAxs, kDualStreams };

// One row of k_dual's work (pdhg.cpp:125-126, :139-140, :179-189): y_{t+1},
// the sums, the push of y_{t+1} (sharded) and the row-side report partials.
__device__ __forceinline__ void dual_row(const IterParams& p, const StepInfo& si, int i, const double* v,
                                         double* acc) {
  const double r = v[kDsR], b = v[kDsB], axn = v[kDsAxn];
  const double rinv = pow2_recip(r);
  if (si.init) {
    row_report(axn, v[kDsY], r, rinv, b, acc);
    return;
  }
  double y_old = v[kDsY], ax_old = v[kDsAx];
  if (si.R) {
    y_old = v[kDsYs] * si.inv;
    ax_old = v[kDsAxs] * si.inv;
  }
  const double bs = b * r;  // row_lower.cwiseProduct(r)
  double t = 2.0 * axn;
  t = t - ax_old;
  t = bs - t;
  t = p.sigma * t;
  const double yn = y_old + t;
  const double ysn = (si.R ? 0.0 : v[kDsYs]) + yn;
  const double axsn = (si.R ? 0.0 : v[kDsAxs]) + axn;
  p.y[si.s1][i] = yn;
  if (p.push.on) {  // fused push: into every shard that gathers this row
    const unsigned mk = p.push.mask_y != nullptr ? p.push.mask_y[i] : 0xFFu;
    const long long off = static_cast<long long>(p.push.rank) * p.push.Sm;
    for (int q = 0; q < p.push.P; ++q)
      if ((mk >> q) & 1u) p.push.y[q][off + i] = yn;
  } else if (p.y_full_loc != nullptr) {
    p.y_full_loc[i] = yn;
  }
  p.ysum[si.s1][i] = ysn;
  p.axsum[si.s1][i] = axsn;
  if (nonfinite(yn)) acc[6] += 1.0;
  if (si.check) {
    row_report(axn, yn, r, rinv, b, acc);
    row_report(axsn * si.inv1, ysn * si.inv1, r, rinv, b, acc + 3);
  }
}

// Unscaled y of the pending snapshot's state t (view_of, pdhg.cpp:271-283;
// the same operations as k_view_rows) into its slot.
__device__ __forceinline__ void snap_rows(const IterParams& p, const StepInfo& si) {
  const double* __restrict__ src = si.snap_avg ? p.ysum[si.s0] : p.y[si.s0];
  double* __restrict__ out = p.snap_y[si.snap_slot];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.m; i += gridDim.x * blockDim.x) {
    const double ys = si.snap_avg ? src[i] * si.snap_inv : src[i];
    out[i] = ys * p.r[i];
  }
}

// Unscaled x and clipped z of the pending snapshot's state t (k_view_cols).
__device__ __forceinline__ void snap_cols(const IterParams& p, const StepInfo& si) {
  const double* __restrict__ xsrc = si.snap_avg ? p.xsum[si.s0] : p.xc[si.t % 3][si.snap_rprev];
  const double* __restrict__ asrc = si.snap_avg ? p.atysum[si.s0] : p.aty[si.s0];
  double* __restrict__ xo = p.snap_x[si.snap_slot];
  double* __restrict__ zo = p.snap_z[si.snap_slot];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.n; j += gridDim.x * blockDim.x) {
    double xs = xsrc[j], as = asrc[j];
    if (si.snap_avg) {
      xs = xs * si.snap_inv;
      as = as * si.snap_inv;
    }
    const double sj = p.s[j];
    const double sinv = pow2_recip(sj);
    const double x = xs * sj;
    xo[j] = x;
    zo[j] = clip_z(p.c[j], as * sinv, x, p.l[j], p.u[j]);
  }
}

// Dual update + row-side report partials, the operand streams staged by the
// TMA engine (bulk_stream) or, on short vectors, loaded by the threads
// (reg_stream): the same results either way.
template <bool BULK>
__global__ void __launch_bounds__(kTile, 1) k_dual(const IterParams p, int init) {
  StepInfo si;
  if (!read_step(p, init != 0, si, 1)) return;
  __shared__ double red[(kTile / 32) * kRowParts];
  __shared__ double out[kRowParts];
  double acc[kRowParts];
#pragma unroll
  for (int k = 0; k < kRowParts; ++k) acc[k] = 0.0;
  const double* const src[kDualStreams] = {p.r, p.b, p.ax[si.a1], p.y[si.s0], p.ax[si.a0], p.ysum[si.s0],
                                           p.axsum[si.s0]};
  // state t's ax is read when no restart is applied, the sums except at init
  const unsigned mask = 0xFu | (si.init || si.R ? 0u : (1u << kDsAx)) |
                        (si.init ? 0u : ((1u << kDsYs) | (1u << kDsAxs)));
  auto body = [&](int i, const double* v) { dual_row(p, si, i, v, acc); };
  if constexpr (BULK)
    bulk_stream<kDualStreams>(p.m, src, mask, body);
  else
    reg_stream<kDualStreams>(p.m, src, mask, body);
  if (si.snap) snap_rows(p, si);
  block_reduce<kRowParts, kRowMaxMask, kTile>(acc, red, out);
  if (threadIdx.x < kRowParts) p.rowp[threadIdx.x * gridDim.x + blockIdx.x] = out[threadIdx.x];  // field-major
  if (p.push.on) push_signal_grid(p.push, kPushY, static_cast<unsigned long long>(si.t1 + 1), p.push.counter);
}

// One column of k_primal's work: the sums, both next-x candidates and the
// column-side report partials (pdhg.cpp:121-123, :138, :141, :190-210).
__device__ __forceinline__ void primal_column(const IterParams& p, const StepInfo& si, int j, double s, double c,
                                              double l, double u, double x1, double atyn, double xs0, double as0,
                                              double* acc) {
  const double sinv = pow2_recip(s);
  // apply_scaling: c*s, l/s, u/s (l/s == l*(1/s) exactly)
  const double cs = c * s, ls = l * sinv, us = u * sinv;
  p.xc[si.xs2][0][j] = primal_update(x1, atyn, cs, ls, us, p.tau);
  if (si.init) {
    col_report(x1, atyn, s, sinv, c, l, u, acc);
    return;
  }
  const double xsn = (si.R ? 0.0 : xs0) + x1;
  const double asn = (si.R ? 0.0 : as0) + atyn;
  p.xsum[si.s1][j] = xsn;
  p.atysum[si.s1][j] = asn;
  if (nonfinite(x1)) acc[12] += 1.0;
  if (si.check) {
    col_report(x1, atyn, s, sinv, c, l, u, acc);
    const double xa = xsn * si.inv1, aa = asn * si.inv1;
    col_report(xa, aa, s, sinv, c, l, u, acc + 6);
    p.xc[si.xs2][1][j] = primal_update(xa, aa, cs, ls, us, p.tau);
  }
}

// k_primal's operand streams: s, c, l, u, x_{t+1}, aty_{t+1}, x_sum, aty_sum.
enum PrimalStream : int { kPsS = 0, kPsC, kPsL, kPsU, kPsX, kPsAty, kPsXs, kPsAs, kPrimalStreams };

// Primal side: sums, column-side report partials, both next-x candidates,
// the operand streams staged by the TMA engine (bulk_stream) or, on short
// vectors, loaded by the threads (reg_stream); the last block to finish runs
// finalize().
template <bool BULK>
__global__ void __launch_bounds__(kTile, 1) k_primal(const IterParams p, int init) {
  StepInfo si;
  if (!read_step(p, init != 0, si, 3)) return;
  __shared__ double red[(kTile / 32) * kColParts];
  __shared__ double out[kColParts];
  __shared__ bool last;
  // block 0 samples the host's cancel request early (a PCIe read that
  // completes behind the column stream) for this step's decide()
  const bool sampler = blockIdx.x == 0 && threadIdx.x == 0 && p.host_flags != nullptr;
  const unsigned cancel_req = sampler ? ld_relaxed_sys(p.host_flags) : 0u;
  double acc[kColParts];
#pragma unroll
  for (int k = 0; k < kColParts; ++k) acc[k] = 0.0;
  const double* const src[kPrimalStreams] = {p.s, p.c, p.l, p.u, p.xc[si.xs][si.R], p.aty[si.s1],
                                             p.xsum[si.s0], p.atysum[si.s0]};
  // the sums are read only when they carry on (not at init, not after a restart)
  const unsigned mask = (si.init || si.R) ? 0x3Fu : 0xFFu;
  auto body = [&](int j, const double* v) {
    primal_column(p, si, j, v[kPsS], v[kPsC], v[kPsL], v[kPsU], v[kPsX], v[kPsAty], v[kPsXs], v[kPsAs], acc);
  };
  if constexpr (BULK)
    bulk_stream<kPrimalStreams>(p.n, src, mask, body);
  else
    reg_stream<kPrimalStreams>(p.n, src, mask, body);
  if (si.snap) snap_cols(p, si);
  block_reduce<kColParts, kColMaxMask, kTile>(acc, red, out);
  if (threadIdx.x < kColParts) p.colp[threadIdx.x * gridDim.x + blockIdx.x] = out[threadIdx.x];  // field-major
  if (sampler && p.cancel_dev != nullptr) *p.cancel_dev = cancel_req;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(p.counter, 1u) == gridDim.x - 1;
  __syncthreads();
  // Every block fenced its partials before its counter increment, and the
  // last block reads them with L2 (.cg) loads, so no second fence is needed
  // here (the classic last-block reduction; 0.45 us off the decision tail).
  if (!last) return;
  if (p.spec != nullptr) {  // every candidate of x_{t+1} is written: let row_step start
    if (threadIdx.x == 0) {
      p.spec[2] = static_cast<unsigned long long>(si.t1);
      __threadfence();
      st_release_gpu(p.spec, ld_acquire_gpu(p.spec) + 1);
    }
    __syncthreads();
    pdl_trigger();
  }
  if (threadIdx.x == 0) p.ctrl->t_fin_start = globaltimer();
  finalize(p, si);
  if (threadIdx.x == 0) *p.counter = 0u;
  if (p.spec != nullptr) {  // the decisions (the whole control block) are stored
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(p.spec + 1, ld_acquire_gpu(p.spec));
  }
}

// ---------------------------------------------------------------------------
// View extraction for results and ladder snapshots: unscaled x, y, z of the
// current or averaged iterate of state t (view_of, pdhg.cpp:271-283), plus
// report partials for an independent recomputation when no check ran.
// ---------------------------------------------------------------------------
struct ViewParams {
  IterParams it;
  int view;  // kViewCur / kViewAvg (kViewCurEff resolved on the host)
  long long t;
  int R_prev;
  double inv;  // 1/window_t for kViewAvg
  double* x_out;
  double* y_out;
  double* z_out;
  double* rowp;
  double* colp;
  unsigned* counter;
  double* report;     // [kRepN]
  double* parts_out;  // optional: the reduced sums [kRowParts + kColParts] (sharded mode)
};

__global__ void __launch_bounds__(kBlock) k_view_rows(const ViewParams v) {
  const IterParams& p = v.it;
  __shared__ double red[(kBlock / 32) * kRowParts];
  __shared__ double out[kRowParts];
  double acc[kRowParts];
#pragma unroll
  for (int k = 0; k < kRowParts; ++k) acc[k] = 0.0;
  const int sl = static_cast<int>(v.t & 1);
  for (int i = blockIdx.x * kBlock + threadIdx.x; i < p.m; i += gridDim.x * kBlock) {
    double ys, axs;
    if (v.view == kViewAvg) {
      ys = p.ysum[sl][i] * v.inv;
      axs = p.axsum[sl][i] * v.inv;
    } else {
      ys = p.y[sl][i];
      axs = p.ax[v.t % 3][i];
    }
    const double r = p.r[i];
    v.y_out[i] = ys * r;
    row_report(axs, ys, r, pow2_recip(r), p.b[i], acc);
  }
  block_reduce<kRowParts, kRowMaxMask>(acc, red, out);
  if (threadIdx.x < kRowParts) v.rowp[blockIdx.x * kRowParts + threadIdx.x] = out[threadIdx.x];
}

__global__ void __launch_bounds__(kBlock) k_view_cols(const ViewParams v, int row_blocks) {
  const IterParams& p = v.it;
  __shared__ double red[(kBlock / 32) * kColParts];
  __shared__ double out[kColParts];
  __shared__ double rowv[kRowParts];
  __shared__ double colv[kColParts];
  __shared__ bool last;
  double acc[kColParts];
#pragma unroll
  for (int k = 0; k < kColParts; ++k) acc[k] = 0.0;
  const int sl = static_cast<int>(v.t & 1);
  const double* xcur = p.xc[v.t % 3][v.R_prev];
  for (int j = blockIdx.x * kBlock + threadIdx.x; j < p.n; j += gridDim.x * kBlock) {
    double xs, as;
    if (v.view == kViewAvg) {
      xs = p.xsum[sl][j] * v.inv;
      as = p.atysum[sl][j] * v.inv;
    } else {
      xs = xcur[j];
      as = p.aty[sl][j];
    }
    const double s = p.s[j], c = p.c[j], l = p.l[j], u = p.u[j];
    const double sinv = pow2_recip(s);
    const double x = xs * s;
    v.x_out[j] = x;
    v.z_out[j] = clip_z(c, as * sinv, x, l, u);
    col_report(xs, as, s, sinv, c, l, u, acc);
  }
  block_reduce<kColParts, kColMaxMask>(acc, red, out);
  if (threadIdx.x < kColParts) v.colp[blockIdx.x * kColParts + threadIdx.x] = out[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(v.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double ra[kRowParts], ca[kColParts];
#pragma unroll
  for (int k = 0; k < kRowParts; ++k) ra[k] = 0.0;
#pragma unroll
  for (int k = 0; k < kColParts; ++k) ca[k] = 0.0;
  for (int b = threadIdx.x; b < row_blocks; b += kBlock)
    for (int k = 0; k < kRowParts; ++k) {
      const double x = __ldcg(v.rowp + b * kRowParts + k);
      ra[k] = ((kRowMaxMask >> k) & 1u) ? amax(ra[k], x) : ra[k] + x;
    }
  for (int b = threadIdx.x; b < gridDim.x; b += kBlock)
    for (int k = 0; k < kColParts; ++k) {
      const double x = __ldcg(v.colp + b * kColParts + k);
      ca[k] = ((kColMaxMask >> k) & 1u) ? amax(ca[k], x) : ca[k] + x;
    }
  block_reduce<kRowParts, kRowMaxMask>(ra, red, rowv);
  block_reduce<kColParts, kColMaxMask>(ca, red, colv);
  if (v.parts_out != nullptr) {
    if (threadIdx.x < kRowParts) v.parts_out[threadIdx.x] = rowv[threadIdx.x];
    if (threadIdx.x < kColParts) v.parts_out[kRowParts + threadIdx.x] = colv[threadIdx.x];
  }
  if (threadIdx.x == 0) {
    make_report(rowv, colv, p.b_norm, p.c_norm, v.report);
    *v.counter = 0u;
  }
}

}  // namespace
}  // namespace cclp_cu
