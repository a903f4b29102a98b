// Device kernels of the cclp_cu PDHG engine (sm_100a). Compiled with
// --fmad=false so every a*b+c rounds twice, as the reference's x86-64 build
// does (no FMA contraction); elementwise operations follow the reference's
// operation order exactly (cited per function).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "engine.cuh"

namespace cclp_cu {

// Loads of the matrix streams (index/value arrays read once per product):
// evict-first. ld_line is for the SELL-G row slices, where every load of a
// warp is one whole 128-byte line: no L1 allocation (the x lines gathered
// next stay in L1) and a 256-byte L2 prefetch of the slice's next line
// (C3 row product 85.8 -> 83.8 us; on CSR rows, whose lanes re-read a line
// over several loads, and on the SELL-32 columns it costs:
// profiles/r2/history/r2_stream_hints.txt).
__device__ __forceinline__ int ld_stream(const int* p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ int ld_line(const int* p) {
  int v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_line(const double* p) {
  double v;
  asm("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

#define CCLP_INF (__longlong_as_double(0x7ff0000000000000LL))

// std::max / std::min argument semantics (pdhg.cpp uses both).
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
// Accumulating max that ignores NaN exactly like `acc = std::max(acc, v)` with
// a finite accumulator (the comparison is false for NaN, keeping acc).
__device__ __forceinline__ double amax(double acc, double v) { return (acc < v) ? v : acc; }
__device__ __forceinline__ bool isfin(double v) { return v > -CCLP_INF && v < CCLP_INF; }
__device__ __forceinline__ bool nonfinite(double v) { return isnan(v - v); }

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization is set up while its
// predecessor drains; pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible. No early launch_dependents trigger:
// measured on C4, successor blocks launched early squat on SMs the draining
// grid still needs (+300 us/iteration); without it PDL is neutral-to-positive.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// The one early trigger: the last block of k_primal, once every candidate of
// x_{t+1} is written (the other blocks have exited), lets the next step's row
// product start on the no-restart candidate while it runs the decision tail
// (row_step, iter_kernels.cuh).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
// Polling without the acquire's L1 invalidation (an ld.acquire.gpu drops the
// SM's whole L1, which the other block on the SM may be gathering from).
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// 1-D bulk async copies (the TMA engine: cp.async.bulk) into shared memory,
// completing on an mbarrier (transaction bytes), for the streaming kernels.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      " @!P bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// the generic proxy's reads of a buffer before the async proxy rewrites it
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Work plan of one SpMV side (A or A^T) for a given launch geometry. Block b
// owns rows [start[b], start[b+1]) and long-row segments [start[grid+1+b],
// start[grid+2+b]). Rows longer than `thr` nonzeros are not summed by their
// lane group: they are cut into fixed kSegLen-element segments (a function of
// the matrix alone, so the result never depends on the geometry), each summed
// by a full warp; the last segment of a row to finish adds the segment sums in
// segment order (deterministic). The unified row+segment sequence is split by
// weight, so power-law row lengths stay balanced (merge-path in spirit).
// ---------------------------------------------------------------------------
constexpr int kSegLen = 4096;

struct SpmvPlan {
  const int* start;     // [2 * (grid + 1)]
  const int4* seg;      // [nseg]: row, begin, end, long-row index
  const int* lr_first;  // [nlong + 1]: first segment of each long row
  double* part;         // [nseg] segment sums
  unsigned* cnt;        // [nlong] finished segments per long row (self-resetting)
  int thr;              // rows with more nonzeros are segmented (INT_MAX: none)
  int grid;
};

// SELL-32 layout of one SpMV side (engine.cu, Context::build_sell_cols):
// 32 consecutive rows per slice, slice s holding 32 * width_s slots, slot k
// of lane l at off[s] + 32k + l (row s*32 + l's k-th element). Rows longer
// than `thr` are left to the long-row segments of the side's SpmvPlan.
struct SellPlan {
  const long long* off;  // [nsl + 1]
  const int* start;      // [grid + 1] slice range of each block
  const int* ptr;        // the side's row pointer (lengths)
  const int* idx;
  const double* val;
  int n;                 // rows of the side
  int thr;
};

// One column panel of the row SpMV (engine.cu, Context::build_panels).
struct PanelArgs {
  SpmvPlan plan;
  const int* ptr;
  const int* idx;
  const double* val;
  int accumulate;  // 0: out = sum; 1: out += sum (panel order)
};

// Sharded push transport (sharded.cuh): the producers store their slice of
// y, x and the report sums straight into every peer shard's full buffers
// (NVLink P2P stores across GPUs, plain stores between shards on one GPU),
// then release a per-(kind, source) epoch flag in every peer's flag array;
// the consumers acquire the flags before gathering. No collective call.
constexpr int kMaxPushShards = 8;
enum PushKind : int { kPushY = 0, kPushX = 1, kPushPart = 2 };
struct PushArgs {
  int on, P, rank;
  int gpu_scope;                 // every shard on this device in this process: GPU-scope fences/flags
  long long Sm, Sn;
  double* y[kMaxPushShards];     // every shard's padded full y
  double* x[kMaxPushShards];     // every shard's padded full x
  double* part[kMaxPushShards];  // every shard's [P][22] report sums
  unsigned long long* flags[kMaxPushShards];  // every shard's flags [3][kMaxPushShards]
  unsigned long long* my_flags;
  const unsigned char* mask_y;   // [m_loc]: bit q = shard q gathers this row's y (null: all)
  const unsigned char* mask_x;   // [n_loc]
  unsigned* counter;             // [2] last-block counters (k_dual, k_select_x)
};

// ---------------------------------------------------------------------------
// Parameters of the fused iteration kernels (passed by value, captured into
// CUDA graphs once per solve).
// ---------------------------------------------------------------------------
constexpr int kStampRing = 128;

struct IterParams {
  int m, n;
  // CSR(A), scaled values
  const int* rowptr;
  const int* colind;
  const double* aval;
  // CSR(A^T) == CSC(A), scaled values
  const int* colptr;
  const int* rowind;
  const double* atval;
  // balanced block partitions [grid+1]
  const int* row_start;
  const int* col_start;
  int row_grid, col_grid;
  // work plans of the iteration SpMV kernels (autotuned grids)
  SpmvPlan plan_r, plan_c;
  SellPlan sell_c;     // SELL-32 copy of A' for the column product
  int use_sell_c;      // k_spmv_cols_sell instead of k_spmv_cols
  SellPlan sell_r;     // SELL-G copy of A for the row product (same sums as CSR-G)
  int use_sell_r;      // k_spmv_rows_sellg instead of k_spmv_rows
  SellPlan sell_cg;    // SELL-G copy of A' (same sums as CSR-G), when SELL-32 is not used
  int use_sell_cg;     // k_spmv_cols_sellg
  // unscaled problem data and Ruiz factors
  const double *c, *l, *u, *b, *r, *s;
  // state
  double* xc[3][2];
  double* aty[2];
  double* xsum[2];
  double* atysum[2];
  double* y[2];
  double* ax[3];  // by state index mod 3: the speculative row product of step t
                  // writes state t+1's slot while states t and t-1 stay intact
  double* ysum[2];
  double* axsum[2];
  // partials and control
  double* rowp;
  double* colp;
  unsigned* counter;
  Ctrl* ctrl;
  LogEntry* log;
  int log_cap;
  long long log_interval;
  // scalars
  double tau, sigma, eps_rel, restart_factor, b_norm, c_norm, time_limit;
  long long max_iter;
  int check_interval;
  int nthr;
  const double* thr;
  const unsigned long long* t0_ns;
  int rpg_rows, rpg_cols;  // rows per lane group in flight in the SpMV (1 or 2)
  // sharded mode (row-block partition, sharded.cuh); all null on one device
  const double* xg;    // gather source of the row SpMV: the full (padded) x
  const double* yg;    // gather source of the column SpMV: the full (padded) y
  double* y_full_loc;  // this shard's region of the full y (k_dual also writes y there)
  double* xpart_loc;   // k_primal's last block writes the shard's 22 report sums here
  PushArgs push;       // sharded push transport (push.on == 0 otherwise)
  // ladder snapshots extracted by the step after the check (single device;
  // 0: halt the loop and let the host extract, as the sharded solve does)
  int snap_inline;
  double* snap_x[kSnapSlots];
  double* snap_y[kSnapSlots];
  double* snap_z[kSnapSlots];
  // host flags in mapped pinned memory ([0] cancel request, [1] snapshots the
  // host has copied out), read by block 0 of k_primal / by decide(); null:
  // none. cancel_dev: block 0's copy of the cancel request for decide().
  const volatile unsigned* host_flags;
  unsigned* cancel_dev;
  // in-graph phase stamps (stamp_phase): u64[kStampRing * 4] or null
  unsigned long long* stamps;
  // speculative row products (row_step): u64[3] = {candidates-ready epoch,
  // decided epoch, t of the next row product}; null: off (sharded, panels)
  unsigned long long* spec;
};

// Power-iteration scalars on the device (Context::power_norm, setup_kernels.cuh).
struct PowerCtrl {
  double nu;      // ||u_prev|| (v = u_prev / nu)
  double lambda;  // Rayleigh quotient v.u
  int zero;       // ||u|| == 0 -> result 0
  int pad;
};

// ---------------------------------------------------------------------------
// Block reductions (deterministic: fixed shuffle tree, fixed warp order).
// ---------------------------------------------------------------------------
template <int N, unsigned MAXMASK, int BS = kBlock>
__device__ __forceinline__ void block_reduce(double (&v)[N], double* smem, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double a = v[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_down_sync(0xffffffffu, a, off);
      a = ((MAXMASK >> k) & 1u) ? amax(a, o) : a + o;
    }
    if (lane == 0) smem[warp * N + k] = a;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    const int k = threadIdx.x;
    double a = smem[k];
    for (int w = 1; w < BS / 32; ++w) {
      const double o = smem[w * N + k];
      a = ((MAXMASK >> k) & 1u) ? amax(a, o) : a + o;
    }
    out[k] = a;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Gathers of the dense operand of an SpMV.
// ---------------------------------------------------------------------------
struct GatherPlain {
  const double* v;
  __device__ __forceinline__ double operator()(int j) const { return __ldg(v + j); }
};
struct GatherDiv {  // v_j = u_j / nu (power iteration: v = u / norm, pdhg.cpp:62)
  const double* v;
  const double* nu;
  __device__ __forceinline__ double operator()(int j) const { return __ldg(v + j) / *nu; }
};

// Group-of-G-lanes row dot product: lane l of the group accumulates the row's
// elements l, l+G, l+2G, ... in order (U independent idx/val loads and U
// gathers in flight), then a fixed xor butterfly. Deterministic run to run.
// With G = 1 a lane sums its row sequentially in ascending position — the
// reference's (Eigen's) own order, so the result is bit-identical to it.
template <int G, int U, class Gather>
__device__ __forceinline__ double group_dot(int beg, int end, int lane, const int* __restrict__ idx,
                                            const double* __restrict__ val, const Gather& g) {
  double acc = 0.0;
  for (int p = beg + lane; p < end; p += G * U) {
    int ii[U];
    double vv[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int q = p + k * G;
      const bool ok = q < end;
      ii[k] = ok ? ld_stream(idx + q) : -1;
      vv[k] = ok ? ld_stream(val + q) : 0.0;
    }
    double xx[U];
#pragma unroll
    for (int k = 0; k < U; ++k) xx[k] = ii[k] >= 0 ? g(ii[k]) : 0.0;
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (ii[k] >= 0) acc = acc + vv[k] * xx[k];
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  return acc;
}

// Two rows per G-lane group in flight: the same per-row, per-lane order as
// group_dot (so bit-identical results), with both rows' loads and gathers
// issued before either row's multiply-adds.
template <int G, int U, class Gather>
__device__ __forceinline__ void group_dot2(int b0, int e0, int b1, int e1, int lane,
                                           const int* __restrict__ idx,
                                           const double* __restrict__ val, const Gather& g,
                                           double& s0, double& s1) {
  double a0 = 0.0, a1 = 0.0;
  for (int p0 = b0 + lane, p1 = b1 + lane; p0 < e0 || p1 < e1; p0 += G * U, p1 += G * U) {
    int i0[U], i1[U];
    double v0[U], v1[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int q0 = p0 + k * G, q1 = p1 + k * G;
      const bool ok0 = q0 < e0, ok1 = q1 < e1;
      i0[k] = ok0 ? ld_stream(idx + q0) : -1;
      v0[k] = ok0 ? ld_stream(val + q0) : 0.0;
      i1[k] = ok1 ? ld_stream(idx + q1) : -1;
      v1[k] = ok1 ? ld_stream(val + q1) : 0.0;
    }
    double x0[U], x1[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      x0[k] = i0[k] >= 0 ? g(i0[k]) : 0.0;
      x1[k] = i1[k] >= 0 ? g(i1[k]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (i0[k] >= 0) a0 = a0 + v0[k] * x0[k];
#pragma unroll
    for (int k = 0; k < U; ++k)
      if (i1[k] >= 0) a1 = a1 + v1[k] * x1[k];
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, off);
    a1 += __shfl_xor_sync(0xffffffffu, a1, off);
  }
  s0 = a0;
  s1 = a1;
}

// Barrier-free warp tiles shared by every "row" kernel. The block owns rows
// [rb, re); its warps take 32-row tiles round-robin. Per tile: lane l first
// issues pre(row) — the epilogue's operand loads for row tile+l — so their
// latency overlaps the SpMV; then G passes in which each G-lane group
// reduces one row (32/G rows per pass); the 32 sums go to a warp-private
// shared slot and all 32 lanes run epi(row, sum, operands) on the tile's rows
// (coalesced). Only __syncwarp, no block barrier.
struct NoPre {
  __device__ __forceinline__ int operator()(int) const { return 0; }
};

template <int G, class Gather, class Pre, class Epi>
__device__ __forceinline__ void warp_tiles(int rb, int re, const int* __restrict__ ptr,
                                           const int* __restrict__ idx,
                                           const double* __restrict__ val, const Gather& g,
                                           double* wsum, const Pre& pre, Epi&& epi) {
  constexpr int GPW = 32 / G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gid = lane / G, gl = lane % G;
  for (int tile = rb + warp * 32; tile < re; tile += nw * 32) {
    const int nrows = min(32, re - tile);
    const int pl = lane <= nrows ? __ldg(ptr + tile + lane) : 0;
    const int pend = __ldg(ptr + tile + nrows);
    const auto ops = pre(lane < nrows ? tile + lane : tile);
#pragma unroll 1
    for (int k = 0; k < G; ++k) {
      const int local = k * GPW + gid;
      const int b = __shfl_sync(0xffffffffu, pl, local & 31);
      const int e1 = __shfl_sync(0xffffffffu, pl, (local + 1) & 31);
      const int e = local + 1 < 32 ? e1 : pend;
      const bool ok = local < nrows;
      const double s = group_dot<G, 4>(ok ? b : 0, ok ? e : 0, gl, idx, val, g);
      if (gl == 0 && ok) wsum[local] = s;
    }
    __syncwarp();
    if (lane < nrows) epi(tile + lane, wsum[lane], ops);
    __syncwarp();
  }
}

// Exact reciprocal of a Ruiz factor (a power of two, scaling.hpp:22-26):
// x / s == x * (1/s) bit for bit, without a double division. Falls back to
// the division if s is not a normal power of two.
__device__ __forceinline__ double pow2_recip(double s) {
  const long long bits = __double_as_longlong(s);
  const double r = __longlong_as_double(0x7FE0000000000000LL - bits);
  return (bits & 0x000FFFFFFFFFFFFFLL) == 0 && bits > 0x0010000000000000LL &&
                 bits < 0x7FE0000000000000LL
             ? r
             : 1.0 / s;
}

// ---------------------------------------------------------------------------
// Report contributions (report_from_products, pdhg.cpp:170-220) on the
// unscaled model, computed from scaled values exactly as view_of does
// (pdhg.cpp:271-283: x*s, y*r, ax/r, aty/s).
// ---------------------------------------------------------------------------
// acc: [0] rp2 (sum), [1] rp_inf (max), [2] b.y (sum)
__device__ __forceinline__ void row_report(double axs, double ys, double r, double rinv, double b,
                                           double* acc) {
  const double ax = axs * rinv;  // == axs / r exactly (r is a power of two)
  const double y = ys * r;
  double v = 0.0;
  if (ax < b) {
    v = b - ax;
  } else if (ax > b) {
    v = ax - b;
  }
  acc[0] += v * v;
  acc[1] = amax(acc[1], v);
  acc[2] += b * y;
}

// clipped_reduced_costs (pdhg.cpp:89-108) for one column.
__device__ __forceinline__ double clip_z(double c, double aty, double x, double l, double u) {
  double z = c - aty;
  const bool lo = isfin(l), up = isfin(u);
  if (!lo && !up) {
    z = 0.0;
  } else if (lo && up) {
    const double dl = x - l, du = u - x;
    z = dl <= du ? smax(z, 0.0) : smin(z, 0.0);
  } else if (lo) {
    z = smax(z, 0.0);
  } else {
    z = smin(z, 0.0);
  }
  return z;
}

// acc: [0] rd2 (sum), [1] rd_inf (max), [2] bound violation inf (max),
//      [3] complementarity (max), [4] dual bound terms (sum), [5] c.x (sum)
__device__ __forceinline__ void col_report(double xs, double atys, double s, double sinv, double c,
                                           double l, double u, double* acc) {
  const double x = xs * s;
  const double aty = atys * sinv;  // == atys / s exactly (s is a power of two)
  const double z = clip_z(c, aty, x, l, u);
  double rd = aty + z;
  rd = rd - c;
  acc[0] += rd * rd;
  acc[1] = amax(acc[1], fabs(rd));
  double bv = l - x;  // std::max({l - x, x - u, 0.0})
  if (bv < x - u) bv = x - u;
  if (bv < 0.0) bv = 0.0;
  acc[2] = amax(acc[2], bv);
  double dist = CCLP_INF;
  if (isfin(l)) dist = smin(dist, fabs(x - l));
  if (isfin(u)) dist = smin(dist, fabs(x - u));
  if (isfin(dist)) acc[3] = amax(acc[3], dist * fabs(z));
  if (z > 0.0 && isfin(l)) {
    acc[4] += l * z;
  } else if (z < 0.0 && isfin(u)) {
    acc[4] += u * z;
  }
  acc[5] += c * x;
}

// pdhg_step primal update (pdhg.cpp:121-123): (x - tau*(c - aty)) clamped.
__device__ __forceinline__ double primal_update(double x, double aty, double cs, double ls,
                                                double us, double tau) {
  double t = cs - aty;
  t = tau * t;
  t = x - t;
  t = smax(t, ls);  // cwiseMax(col_lower)
  return smin(t, us);  // cwiseMin(col_upper)
}

// Assembles a ResidualReport (pdhg.cpp:211-219).
__device__ __forceinline__ void make_report(const double* rowv, const double* colv, double bn,
                                            double cn, double* rep) {
  rep[kRpNorm2] = sqrt(rowv[0]);
  rep[kRdNorm2] = sqrt(colv[0]);
  rep[kRpInf] = amax(rowv[1], colv[2]);
  rep[kRdInf] = colv[1];
  rep[kCompl] = colv[3];
  rep[kPobj] = colv[5];
  rep[kDobj] = rowv[2] + colv[4];
  rep[kGap] = fabs(rep[kPobj] - rep[kDobj]);
  rep[kRelP] = rep[kRpNorm2] / (1.0 + bn);
  rep[kRelD] = rep[kRdNorm2] / (1.0 + cn);
  rep[kRelGap] = rep[kGap] / (1.0 + fabs(rep[kPobj]) + fabs(rep[kDobj]));
  double mx = rep[kRelP];  // std::max({p, d, g})
  if (mx < rep[kRelD]) mx = rep[kRelD];
  if (mx < rep[kRelGap]) mx = rep[kRelGap];
  rep[kMaxResid] = mx;
}

}  // namespace cclp_cu
