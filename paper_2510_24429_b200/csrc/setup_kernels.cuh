// One-time kernels: CSR(A) construction, balanced partitions, plain SpMV,
// Ruiz equilibration (scaling.cpp:46-90), power iteration for ||A||
// (pdhg.cpp:46-65) and deterministic vector reductions.
#pragma once

#include "kernels.cuh"

namespace cclp_cu {
namespace {  // internal linkage: compiled into engine.cu and sharded.cu

__global__ void k_expand_major(const int* __restrict__ ptr, int outer, int* __restrict__ major) {
  // major[p] = outer index owning nonzero p
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < outer; j += gridDim.x * blockDim.x)
    for (int p = ptr[j]; p < ptr[j + 1]; ++p) major[p] = j;
}

__global__ void k_iota(int* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = static_cast<int>(i);
}

// ptr[i] = first position with sorted_key >= i (sorted keys -> CSR offsets).
__global__ void k_offsets_from_sorted(const int* __restrict__ keys, long long nnz, int rows,
                                      int* __restrict__ ptr) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= rows; i += gridDim.x * blockDim.x) {
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) / 2;
      if (keys[mid] >= i) hi = mid; else lo = mid + 1;
    }
    ptr[i] = static_cast<int>(lo);
  }
}

__global__ void k_gather_csr(const int* __restrict__ perm, long long nnz,
                             const int* __restrict__ col_of, const double* __restrict__ val_in,
                             int* __restrict__ colind, double* __restrict__ val_out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nnz;
       q += (long long)gridDim.x * blockDim.x) {
    const int p = perm[q];
    colind[q] = col_of[p];
    val_out[q] = val_in[p];
  }
}

// Column panels (Context::build_panels): entries of row i with column in
// [lo, hi) - a contiguous run, since rows keep ascending column order.
__device__ __forceinline__ int lower_in_row(const int* __restrict__ idx, int b, int e, int key) {
  while (b < e) {
    const int mid = b + (e - b) / 2;
    if (idx[mid] < key) b = mid + 1; else e = mid;
  }
  return b;
}

__global__ void k_panel_count(const int* __restrict__ ptr, const int* __restrict__ idx, int rows, int lo,
                              int hi, int* __restrict__ cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= rows; i += gridDim.x * blockDim.x) {
    if (i == rows) {
      cnt[i] = 0;
      continue;
    }
    const int b = ptr[i], e = ptr[i + 1];
    cnt[i] = lower_in_row(idx, b, e, hi) - lower_in_row(idx, b, e, lo);
  }
}

__global__ void k_panel_fill(const int* __restrict__ ptr, const int* __restrict__ idx, int rows, int lo,
                             const int* __restrict__ pptr, int* __restrict__ pidx, int* __restrict__ perm) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
    const int b = lower_in_row(idx, ptr[i], ptr[i + 1], lo);
    const int base = pptr[i], len = pptr[i + 1] - base;
    for (int q = 0; q < len; ++q) {
      pidx[base + q] = idx[b + q];
      perm[base + q] = b + q;
    }
  }
}

__global__ void k_gather_vals(const int* __restrict__ perm, long long cnt, const double* __restrict__ src,
                              double* __restrict__ dst) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < cnt;
       q += (long long)gridDim.x * blockDim.x)
    dst[q] = src[perm[q]];
}

// Number of rows with more than `thr` nonzeros.
__global__ void k_count_long(const int* __restrict__ ptr, int rows, int thr, int* count) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x)
    if (ptr[i + 1] - ptr[i] > thr) atomicAdd(count, 1);
}

// Block b owns rows [start[b], start[b+1]) with ~equal weight
// w(i) = ptr[i] + alpha * i (nonzeros plus a per-row epilogue cost).
__global__ void k_partition(const int* __restrict__ ptr, int rows, int grid, long long alpha,
                            int* __restrict__ start) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > grid) return;
  if (b == grid) {
    start[b] = rows;
    return;
  }
  const long long total = static_cast<long long>(ptr[rows]) + alpha * rows;
  const long long target = total * b / grid;
  int lo = 0, hi = rows;
  while (lo < hi) {
    const int mid = (lo + hi) / 2;
    if (static_cast<long long>(ptr[mid]) + alpha * mid >= target) hi = mid; else lo = mid + 1;
  }
  start[b] = lo;
}

// Plain y = M v over a CSR (used for matvec / matvec_transpose and the power
// iteration's A v; G = 1 gives the reference's exact sequential order).
template <int G, class Gather>
__global__ void __launch_bounds__(kBlock) k_spmv(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                 const double* __restrict__ val, Gather g,
                                                 const int* __restrict__ start,
                                                 double* __restrict__ out, const int* stop_flag) {
  if (stop_flag != nullptr && *stop_flag) return;
  __shared__ double wsum[kBlock];
  warp_tiles<G>(start[blockIdx.x], start[blockIdx.x + 1], ptr, idx, val, g, wsum + (threadIdx.x & ~31),
                NoPre{}, [&](int i, double s, int) { out[i] = 0.0 + s; });
}

// ---- power iteration (estimate_matrix_norm, pdhg.cpp:46-65) ---------------


// u = A' w, partial sums of u.u and v.u with v = u_prev / nu; the last block
// finalizes nu and lambda.
template <int G>
__global__ void __launch_bounds__(kBlock) k_power_cols(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                       const double* __restrict__ val,
                                                       const double* __restrict__ w,
                                                       const int* __restrict__ start,
                                                       const double* __restrict__ u_prev,
                                                       double* __restrict__ u, double* part,
                                                       unsigned* counter, PowerCtrl* pc) {
  if (pc->zero) return;
  __shared__ double wsum[kBlock];
  __shared__ double red[(kBlock / 32) * 2];
  __shared__ double out[2];
  __shared__ bool last;
  double acc[2] = {0.0, 0.0};
  const double nu = pc->nu;
  warp_tiles<G>(start[blockIdx.x], start[blockIdx.x + 1], ptr, idx, val, GatherPlain{w},
                wsum + (threadIdx.x & ~31), [&](int j) { return u_prev[j]; }, [&](int j, double s, double up) {
    const double uj = 0.0 + s;
    u[j] = uj;
    const double vj = up / nu;
    acc[0] += uj * uj;
    acc[1] += vj * uj;
  });
  block_reduce<2, 0u>(acc, red, out);
  if (threadIdx.x < 2) part[blockIdx.x * 2 + threadIdx.x] = out[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a2[2] = {0.0, 0.0};
  for (int b = threadIdx.x; b < gridDim.x; b += kBlock) {
    a2[0] += __ldcg(part + 2 * b);
    a2[1] += __ldcg(part + 2 * b + 1);
  }
  block_reduce<2, 0u>(a2, red, out);
  if (threadIdx.x == 0) {
    const double norm = sqrt(out[0]);
    if (norm == 0.0) {
      pc->zero = 1;
    } else {
      pc->lambda = out[1];
      pc->nu = norm;
    }
    *counter = 0u;
  }
}

// nu = ||u||, lambda = v.u (pdhg.cpp:59-61) over the materialized u and v;
// the last block finalizes (a zero norm sets `zero`: the reference returns 0).
__global__ void __launch_bounds__(kBlock) k_power_reduce(const double* __restrict__ u,
                                                         const double* __restrict__ v, long long n,
                                                         double* part, unsigned* counter,
                                                         PowerCtrl* pc) {
  if (pc->zero) return;
  __shared__ double red[(kBlock / 32) * 2];
  __shared__ double out[2];
  __shared__ bool last;
  double acc[2] = {0.0, 0.0};
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n;
       i += (long long)gridDim.x * kBlock) {
    const double ui = u[i];
    acc[0] += ui * ui;
    acc[1] += v[i] * ui;
  }
  block_reduce<2, 0u>(acc, red, out);
  if (threadIdx.x < 2) part[blockIdx.x * 2 + threadIdx.x] = out[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a2[2] = {0.0, 0.0};
  for (int b = threadIdx.x; b < gridDim.x; b += kBlock) {
    a2[0] += __ldcg(part + 2 * b);
    a2[1] += __ldcg(part + 2 * b + 1);
  }
  block_reduce<2, 0u>(a2, red, out);
  if (threadIdx.x == 0) {
    const double norm = sqrt(out[0]);
    if (norm == 0.0) {
      pc->zero = 1;
    } else {
      pc->lambda = out[1];
      pc->nu = norm;
    }
    *counter = 0u;
  }
}

// ---- deterministic reductions over a vector --------------------------------
// mode 0: sum a[i]^2      mode 1: sum (a[i]*b[i])^2      mode 2: sum a[i]*b[i]
__global__ void __launch_bounds__(kBlock) k_reduce(const double* __restrict__ a, const double* __restrict__ b,
                                                   long long n, int mode, double* part,
                                                   unsigned* counter, double* result) {
  __shared__ double red[kBlock / 32];
  __shared__ double out[1];
  __shared__ bool last;
  double acc[1] = {0.0};
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n;
       i += (long long)gridDim.x * kBlock) {
    double v;
    if (mode == 0) {
      v = a[i] * a[i];
    } else if (mode == 1) {
      const double t = a[i] * b[i];
      v = t * t;
    } else {
      v = a[i] * b[i];
    }
    acc[0] += v;
  }
  block_reduce<1, 0u>(acc, red, out);
  if (threadIdx.x == 0) part[blockIdx.x] = out[0];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s[1] = {0.0};
  for (int q = threadIdx.x; q < gridDim.x; q += kBlock) s[0] += __ldcg(part + q);
  block_reduce<1, 0u>(s, red, out);
  if (threadIdx.x == 0) {
    *result = out[0];
    *counter = 0u;
  }
}

// ---- partition-independent (reproducible) sums ------------------------------
// The setup's scalars (||b||, ||c||, omega's norms, the power iteration's
// ||u|| and v.u; pdhg.cpp:53-61, :253-265) are sums whose rounding depends on
// the order of the terms. To make the sharded solve bit-identical to one
// device, every such sum is computed by error-free pre-rounding: with
// M = max |term| and N the global term count (both partition-free), level k
// rounds each term's remainder to a multiple of a quantum u_k (the extraction
// (T_k + v) - T_k with T_k = 1.5 * 2^E_k), chosen so that any partial sum of N
// such multiples is exactly representable. Each level's sum is then EXACT in
// any order and over any split into blocks, shards or ranks, and the result
// (S_1 + S_2) + S_3 carries ~3(53 - log2 N) bits below 2^E_1: the same
// double on one device and on P shards. (Terms with M = 0, inf or nan fall
// back to a plain sum, still order-dependent only in the degenerate case.)
struct ReproConsts {
  double T[3];
  int ok;
};
__host__ __device__ inline ReproConsts repro_consts(double M, long long N) {
  ReproConsts c{{0.0, 0.0, 0.0}, 0};
  if (!(M > 0.0) || !(M <= 1.7e308) || N <= 0) return c;
  int k = 1;
  while ((1LL << k) <= N) ++k;  // N < 2^k
  int e;
  (void)frexp(M, &e);  // M < 2^e
  const int E1 = e + k;
  const int E2 = E1 - 53 + k;
  const int E3 = E2 - 53 + k;
  if (E1 > 1020 || E3 < -1000) return c;
  c.T[0] = ldexp(1.5, E1);
  c.T[1] = ldexp(1.5, E2);
  c.T[2] = ldexp(1.5, E3);
  c.ok = 1;
  return c;
}
__host__ __device__ inline double repro_final(const double* S) { return (S[0] + S[1]) + S[2]; }

// Terms of the reductions: mode 0 a_i^2, 1 (a_i b_i)^2, 2 a_i b_i,
// 3 (two sums, the power iteration) a_i^2 and b_i a_i (= u^2, v.u).
template <int MODE>
struct ReproTerms {
  static constexpr int K = MODE == 3 ? 2 : 1;
  __device__ __forceinline__ static void at(const double* __restrict__ a, const double* __restrict__ b,
                                            long long i, double* t) {
    if (MODE == 0) {
      t[0] = a[i] * a[i];
    } else if (MODE == 1) {
      const double q = a[i] * b[i];
      t[0] = q * q;
    } else if (MODE == 2) {
      t[0] = a[i] * b[i];
    } else {
      const double ui = a[i];
      t[0] = ui * ui;
      t[1] = b[i] * ui;
    }
  }
};

// NaN-absorbing max (the reduction of k_repro_max: a nan term wins) and a
// block-wide reduction of K such maxima or K exact sums. Both operations are
// order-free (max; sums of the level quanta are exact), so the tree shape
// never changes a bit of the result.
__device__ __forceinline__ double nanmax(double a, double b) { return (b != b) ? b : amax(a, b); }
template <int K, bool MAX>
__device__ __forceinline__ void block_reduce_free(double (&v)[K], double* smem, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double a = v[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_down_sync(0xffffffffu, a, off);
      a = MAX ? nanmax(a, o) : a + o;
    }
    if (lane == 0) smem[warp * K + k] = a;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double a = smem[threadIdx.x];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
      const double o = smem[w * K + threadIdx.x];
      a = MAX ? nanmax(a, o) : a + o;
    }
    out[threadIdx.x] = a;
  }
  __syncthreads();
}

// Pass 1: out[k] = max |term_k| (exact, order-free); the last block to finish
// reduces the per-block maxima with all its threads.
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_repro_max(const double* __restrict__ a, const double* __restrict__ b,
                                                      long long n, double* part, unsigned* counter,
                                                      double* out) {
  using F = ReproTerms<MODE>;
  constexpr int K = F::K;
  __shared__ double red[(kBlock / 32) * K];
  __shared__ double o[K];
  __shared__ bool last;
  pdl_wait();  // no-op unless launched programmatically (the power iteration)
  double acc[K];
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock) {
    double t[K];
    F::at(a, b, i, t);
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = nanmax(acc[q], fabs(t[q]));
  }
  block_reduce_free<K, true>(acc, red, o);
  if (threadIdx.x < K) part[blockIdx.x * K + threadIdx.x] = o[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int q = 0; q < K; ++q) acc[q] = 0.0;
  for (int bl = threadIdx.x; bl < static_cast<int>(gridDim.x); bl += kBlock)
#pragma unroll
    for (int q = 0; q < K; ++q) acc[q] = nanmax(acc[q], __ldcg(part + bl * K + q));
  block_reduce_free<K, true>(acc, red, o);
  if (threadIdx.x < K) out[threadIdx.x] = o[threadIdx.x];
  if (threadIdx.x == 0) *counter = 0u;
}

// The power iteration's scalars from the level sums of mode 3 (pdhg.cpp:59-61):
// nu = ||u||, lambda = v.u; a zero norm sets `zero` (the reference returns 0).
__device__ __forceinline__ void power_finish(const double* S, PowerCtrl* pc) {
  if (pc->zero) return;
  const double norm = sqrt(repro_final(S));
  if (norm == 0.0) {
    pc->zero = 1;
  } else {
    pc->lambda = repro_final(S + 3);
    pc->nu = norm;
  }
}
__global__ void k_power_finish(const double* __restrict__ S, PowerCtrl* pc) { power_finish(S, pc); }

// Pass 2: out[3k + l] = the exact level-l sum of term k, given its global
// max Mx[k] and global count N (repro_consts); plain sums when !ok.
template <int MODE>
__global__ void __launch_bounds__(kBlock) k_repro_sum(const double* __restrict__ a, const double* __restrict__ b,
                                                      long long n, const double* __restrict__ Mx, long long N,
                                                      double* part, unsigned* counter, double* out,
                                                      PowerCtrl* pc = nullptr) {
  using F = ReproTerms<MODE>;
  constexpr int K = F::K;
  constexpr int K3 = 3 * K;
  __shared__ double red[(kBlock / 32) * K3];
  __shared__ double o[K3];
  __shared__ bool last;
  pdl_wait();
  ReproConsts c[K];
#pragma unroll
  for (int q = 0; q < K; ++q) c[q] = repro_consts(Mx[q], N);
  double acc[K3];
#pragma unroll
  for (int q = 0; q < K3; ++q) acc[q] = 0.0;
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < n; i += (long long)gridDim.x * kBlock) {
    double t[K];
    F::at(a, b, i, t);
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (!c[q].ok) {
        acc[3 * q] += t[q];
        continue;
      }
      double v = t[q];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const double T = c[q].T[l];
        const double x = (T + v) - T;  // v rounded to the level's quantum (exact)
        acc[3 * q + l] += x;           // exact
        v = v - x;                     // exact remainder
      }
    }
  }
  block_reduce_free<K3, false>(acc, red, o);
  if (threadIdx.x < K3) part[blockIdx.x * K3 + threadIdx.x] = o[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int q = 0; q < K3; ++q) acc[q] = 0.0;
  for (int bl = threadIdx.x; bl < static_cast<int>(gridDim.x); bl += kBlock)
#pragma unroll
    for (int q = 0; q < K3; ++q) acc[q] += __ldcg(part + bl * K3 + q);
  block_reduce_free<K3, false>(acc, red, o);  // exact level sums: any order
  if (threadIdx.x < K3) out[threadIdx.x] = o[threadIdx.x];
  if (threadIdx.x == 0) {
    *counter = 0u;
    if (pc != nullptr) power_finish(o, pc);
  }
}

__global__ void k_div_scalar(const double* __restrict__ a, const double* den, double* __restrict__ out,
                             long long n) {
  pdl_wait();
  const double d = *den;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = a[i] / d;
}

__global__ void k_fill(double* a, long long n, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = v;
}

// ---- Ruiz equilibration (scaling.cpp:46-90) --------------------------------
// max over the row of (|a| * r_row) * s_col: exact (order-free).
template <int G>
__global__ void __launch_bounds__(kBlock) k_scaled_absmax(const int* __restrict__ ptr, const int* __restrict__ idx,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ self_scale,
                                                          const double* __restrict__ other_scale,
                                                          int self_is_row, const int* __restrict__ start,
                                                          double* __restrict__ out) {
  constexpr int GPB = kBlock / G;
  const int gid = threadIdx.x / G, lane = threadIdx.x % G;
  const int rb = start[blockIdx.x], re = start[blockIdx.x + 1];
  for (int tile = rb; tile < re; tile += GPB) {
    const int row = tile + gid;
    double mx = 0.0;
    if (row < re) {
      const double sr = self_scale[row];
      for (int p = ptr[row] + lane; p < ptr[row + 1]; p += G) {
        const double so = other_scale[idx[p]];
        // v = |a_ij| * r_i * s_j evaluated left to right (scaling.cpp:60-61)
        const double v = self_is_row ? (fabs(val[p]) * sr) * so : (fabs(val[p]) * so) * sr;
        if (v > mx) mx = v;
      }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, mx, off);
      if (o > mx) mx = o;
    }
    if (lane == 0 && row < re) out[row] = mx;
  }
}

// flag |= some max outside [1/2, 2) (scaling.cpp:64-80)
__global__ void k_ruiz_notdone(const double* __restrict__ mx, int n, int* flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double v = mx[i];
    if (v > 0.0 && (v < 0.5 || v >= 2.0)) *flag = 1;
  }
}

// pow2_sqrt(v) = exp2(round(0.5 * log2(v))) (scaling.cpp:23-25), bit-exact
// with glibc: exact powers of two are decided in integer arithmetic; values
// whose half-log lies within 1e-9 of a rounding boundary are listed for the
// host to evaluate with glibc (never observed on generated LPs).
__device__ __forceinline__ bool pow2_sqrt_dev(double v, double* out) {
  int e;
  const double f = frexp(v, &e);  // v = f 2^e, f in [0.5, 1)
  if (f == 0.5) {
    const int L = e - 1;  // log2(v), exact
    int k;                // round(L / 2), halves away from zero
    if (L >= 0) k = (L + 1) / 2; else k = -((-L + 1) / 2);
    *out = ldexp(1.0, k);
    return true;
  }
  const double h = 0.5 * log2(v);
  const double fl = floor(h);
  const double frac = h - fl;
  if (fabs(frac - 0.5) < 1e-9) return false;
  *out = ldexp(1.0, static_cast<int>(frac < 0.5 ? fl : fl + 1.0));
  return true;
}

__global__ void k_ruiz_update(const double* __restrict__ mx, int n, double* __restrict__ scale,
                              int* amb_count, int* amb_idx, int amb_cap) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double v = mx[i];
    if (!(v > 0.0)) continue;
    double p2;
    if (pow2_sqrt_dev(v, &p2)) {
      scale[i] /= p2;
    } else {
      const int k = atomicAdd(amb_count, 1);
      if (k < amb_cap) amb_idx[k] = i;
    }
  }
}

// scaled values: val * (r_row * s_col)  (apply_scaling, scaling.cpp:33-37)
__global__ void k_scale_values(const int* __restrict__ ptr, int outer, const int* __restrict__ idx,
                               const double* __restrict__ val, const double* __restrict__ outer_scale,
                               const double* __restrict__ inner_scale, int outer_is_row,
                               double* __restrict__ out) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int o = warp; o < outer; o += nwarps) {
    const double so = outer_scale[o];
    for (int p = ptr[o] + lane; p < ptr[o + 1]; p += 32) {
      const double si = inner_scale[idx[p]];
      const double f = outer_is_row ? so * si : si * so;  // r_i * s_j
      out[p] = val[p] * f;
    }
  }
}

// x_0 = Zero.cwiseMax(l').cwiseMin(u') on the scaled bounds (pdhg.cpp:71-73)
__global__ void k_init_x(const double* __restrict__ l, const double* __restrict__ u,
                         const double* __restrict__ s, int n, double* __restrict__ x) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double ls = l[j] / s[j], us = u[j] / s[j];
    x[j] = smin(smax(0.0, ls), us);
  }
}

__global__ void k_stamp(unsigned long long* t) { *t = globaltimer(); }

}  // namespace
}  // namespace cclp_cu

// ---------------------------------------------------------------------------
// Verification side (kkt.cpp:37-149): relative_report / absolute_violation
// of a given iterate (x, y, z) on the unscaled equality-form LP, from
// ax = A x and aty = A' y of the reference-order (G = 1) SpMV. Per-row and
// per-column terms go to block partials (field-major); one block then sums
// each field over the blocks in block order (deterministic).
// ---------------------------------------------------------------------------
namespace cclp_cu {
namespace {  // internal linkage: compiled into engine.cu and sharded.cu

constexpr int kKktRowF = 4;   // 0 sum r^2, 1 max |r|, 2 b.y, 3 sum b^2   (r = b - ax, kkt.cpp:37-52)
constexpr int kKktColF = 7;   // 0 sum rd^2, 1 max |rd|, 2 max bound violation, 3 complementarity,
                              // 4 c.x, 5 dual bound terms, 6 sum c^2
constexpr unsigned kKktRowMax = (1u << 1);
constexpr unsigned kKktColMax = (1u << 1) | (1u << 2) | (1u << 3);

__global__ void __launch_bounds__(kBlock) k_kkt_rows(int m, const double* __restrict__ ax,
                                                     const double* __restrict__ y,
                                                     const double* __restrict__ b, double* part) {
  __shared__ double red[(kBlock / 32) * kKktRowF];
  __shared__ double out[kKktRowF];
  double acc[kKktRowF] = {0.0, 0.0, 0.0, 0.0};
  for (int i = blockIdx.x * kBlock + threadIdx.x; i < m; i += gridDim.x * kBlock) {
    const double r = b[i] - ax[i];  // equality row: rl - ax (kkt.cpp:42-43)
    acc[0] += r * r;
    acc[1] = amax(acc[1], fabs(r));
    acc[2] += b[i] * y[i];
    acc[3] += b[i] * b[i];
  }
  block_reduce<kKktRowF, kKktRowMax>(acc, red, out);
  if (threadIdx.x < kKktRowF) part[threadIdx.x * gridDim.x + blockIdx.x] = out[threadIdx.x];
}

__global__ void __launch_bounds__(kBlock) k_kkt_cols(int n, const double* __restrict__ x,
                                                     const double* __restrict__ z,
                                                     const double* __restrict__ aty,
                                                     const double* __restrict__ c,
                                                     const double* __restrict__ l,
                                                     const double* __restrict__ u, double* part) {
  __shared__ double red[(kBlock / 32) * kKktColF];
  __shared__ double out[kKktColF];
  double acc[kKktColF] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int j = blockIdx.x * kBlock + threadIdx.x; j < n; j += gridDim.x * kBlock) {
    const double xj = x[j], zj = z[j], cj = c[j], lj = l[j], uj = u[j];
    const double rd = (aty[j] + zj) - cj;  // dual_residual (kkt.cpp:66-69)
    acc[0] += rd * rd;
    acc[1] = amax(acc[1], fabs(rd));
    double bv = lj - xj;  // bound_violations: max({l - x, x - u, 0}) (:55-63)
    if (bv < xj - uj) bv = xj - uj;
    if (bv < 0.0) bv = 0.0;
    acc[2] = amax(acc[2], bv);
    const bool lf = isfin(lj), uf = isfin(uj);  // complementarity_inf (:90-104)
    double dist = CCLP_INF;
    if (lf) dist = fmin(dist, fabs(xj - lj));
    if (uf) dist = fmin(dist, fabs(xj - uj));
    if (isfin(dist)) acc[3] = amax(acc[3], dist * fabs(zj));  // free column: skipped
    acc[4] += cj * xj;  // objective_gap (:71-86)
    if (zj > 0.0 && lf) {
      acc[5] += lj * zj;
    } else if (zj < 0.0 && uf) {
      acc[5] += uj * zj;
    }
    acc[6] += cj * cj;
  }
  block_reduce<kKktColF, kKktColMax>(acc, red, out);
  if (threadIdx.x < kKktColF) part[threadIdx.x * gridDim.x + blockIdx.x] = out[threadIdx.x];
}

// One block: field f (thread f) sums / maxes its blocks in block order.
__global__ void k_kkt_finish(const double* __restrict__ rpart, int rblocks, const double* __restrict__ cpart,
                             int cblocks, double* out) {
  const int f = threadIdx.x;
  if (f < kKktRowF) {
    const bool mx = (kKktRowMax >> f) & 1u;
    double a = 0.0;
    for (int k = 0; k < rblocks; ++k) a = mx ? amax(a, rpart[f * rblocks + k]) : a + rpart[f * rblocks + k];
    out[f] = a;
  } else if (f < kKktRowF + kKktColF) {
    const int g = f - kKktRowF;
    const bool mx = (kKktColMax >> g) & 1u;
    double a = 0.0;
    for (int k = 0; k < cblocks; ++k) a = mx ? amax(a, cpart[g * cblocks + k]) : a + cpart[g * cblocks + k];
    out[f] = a;
  }
}

}  // namespace
}  // namespace cclp_cu

// SELL-32 build (Context::build_sell_cols): slice widths, then the slots.
namespace cclp_cu {
namespace {  // internal linkage: compiled into engine.cu and sharded.cu

__global__ void k_sell_width(const int* __restrict__ ptr, int n, int thr, int nsl, int* __restrict__ width) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x) {
    int w = 0;
    for (int l = 0; l < 32; ++l) {
      const int j = s * 32 + l;
      if (j >= n) break;
      const int len = ptr[j + 1] - ptr[j];
      if (len <= thr && len > w) w = len;
    }
    width[s] = w;
  }
}

// warp per slice: lane l writes row s*32+l's elements (zero padding) into
// slots off + 32k + l — coalesced stores, strided loads (setup only)
__global__ void k_sell_fill(const int* __restrict__ ptr, const int* __restrict__ idx,
                            const double* __restrict__ val, int n, int thr, int nsl,
                            const long long* __restrict__ off, int* __restrict__ sidx,
                            double* __restrict__ sval) {
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nsl; s += nwarps) {
    const long long o = off[s];
    const int w = static_cast<int>((off[s + 1] - o) >> 5);
    const int j = s * 32 + lane;
    int b = 0, len = 0;
    if (j < n) {
      b = ptr[j];
      len = ptr[j + 1] - b;
      if (len > thr) len = 0;
    }
    for (int k = 0; k < w; ++k) {
      const bool ok = k < len;
      sidx[o + 32LL * k + lane] = ok ? idx[b + k] : 0;
      sval[o + 32LL * k + lane] = ok ? val[b + k] : 0.0;
    }
  }
}

}  // namespace
}  // namespace cclp_cu

// SELL-G build (Context::build_sell_rows): 32/G rows per slice, G lanes per
// row; slot k of lane (r, gl) holds row s*R + r's element k*G + gl.
namespace cclp_cu {
namespace {  // internal linkage: compiled into engine.cu and sharded.cu

__global__ void k_sellg_width(const int* __restrict__ ptr, int n, int thr, int nsl, int G,
                              int* __restrict__ width) {
  const int R = 32 / G;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < nsl; s += gridDim.x * blockDim.x) {
    int w = 0;
    for (int r = 0; r < R; ++r) {
      const int j = s * R + r;
      if (j >= n) break;
      const int len = ptr[j + 1] - ptr[j];
      if (len <= thr) w = max(w, (len + G - 1) / G);
    }
    width[s] = w;
  }
}

__global__ void k_sellg_fill(const int* __restrict__ ptr, const int* __restrict__ idx,
                             const double* __restrict__ val, int n, int thr, int nsl, int G,
                             const long long* __restrict__ off, int* __restrict__ sidx,
                             double* __restrict__ sval) {
  const int lane = threadIdx.x & 31, R = 32 / G, r = lane / G, gl = lane % G;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nsl; s += nwarps) {
    const long long o = off[s];
    const int w = static_cast<int>((off[s + 1] - o) >> 5);
    const int j = s * R + r;
    int b = 0, len = 0;
    if (j < n) {
      b = ptr[j];
      len = ptr[j + 1] - b;
      if (len > thr) len = 0;
    }
    for (int k = 0; k < w; ++k) {
      const int e = k * G + gl;
      const bool ok = e < len;
      sidx[o + 32LL * k + lane] = ok ? idx[b + e] : 0;
      sval[o + 32LL * k + lane] = ok ? val[b + e] : 0.0;
    }
  }
}

}  // namespace
}  // namespace cclp_cu

// ---------------------------------------------------------------------------
// Crossover pricing on the device: the reference's price()
// (simplex.cpp:266-296) over the EngineModel's n structural + m logical
// columns. d_j = cost_j - column_dot(j, y) with column_dot's own sequential
// order (basis.cpp:35-42; a logical column j >= n has column_dot = y[j-n]),
// then the same status tests; the pick is the largest violation, first
// index on ties (the reference's strict '>'), or with Bland's rule the first
// violating index. Block candidates are combined by the same total order, so
// the pick is the reference's.
// ---------------------------------------------------------------------------
namespace cclp_cu {
namespace {  // internal linkage: compiled into engine.cu and sharded.cu

struct PriceCand {
  double viol;
  long long j;  // -1: none
  int dir;
};

__device__ __forceinline__ bool price_better(const PriceCand& a, const PriceCand& b, int bland) {
  if (a.j < 0) return false;
  if (b.j < 0) return true;
  if (bland) return a.j < b.j;
  return a.viol > b.viol || (a.viol == b.viol && a.j < b.j);
}

__global__ void __launch_bounds__(kBlock) k_price(int n, int m, const int* __restrict__ colptr,
                                                  const int* __restrict__ rowind, const double* __restrict__ val,
                                                  const double* __restrict__ c, const double* __restrict__ y,
                                                  const char* __restrict__ status, const unsigned char* __restrict__ skip,
                                                  int phase1, double dtol, int bland, PriceCand* part) {
  PriceCand best{0.0, -1, 0};
  const long long total = static_cast<long long>(n) + m;
  for (long long j = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; j < total;
       j += static_cast<long long>(gridDim.x) * kBlock) {
    const char st = status[j];
    if (st == 'B' || st == 'X') continue;
    if (skip != nullptr && skip[j]) continue;
    double dot;
    if (j >= n) {
      dot = y[j - n];
    } else {
      dot = 0.0;  // column_dot: acc += value * v[row], ascending position
      for (int p = colptr[j]; p < colptr[j + 1]; ++p) dot = dot + val[p] * y[rowind[p]];
    }
    const double cost = phase1 ? 0.0 : (j < n ? c[j] : 0.0);
    const double d = cost - dot;
    double viol = 0.0;
    int dir = 0;
    if (st == 'L' && d < -dtol) {
      viol = -d;
      dir = 1;
    } else if (st == 'U' && d > dtol) {
      viol = d;
      dir = -1;
    } else if (st == 'Z' && fabs(d) > dtol) {
      viol = fabs(d);
      dir = d < 0.0 ? 1 : -1;
    } else {
      continue;
    }
    const PriceCand cand{viol, j, dir};
    if (price_better(cand, best, bland)) best = cand;
  }
  // block: warp shuffles, then warp 0 over the warps (the order is total)
  for (int off = 16; off > 0; off >>= 1) {
    PriceCand o;
    o.viol = __shfl_down_sync(0xffffffffu, best.viol, off);
    o.j = __shfl_down_sync(0xffffffffu, best.j, off);
    o.dir = __shfl_down_sync(0xffffffffu, best.dir, off);
    if (price_better(o, best, bland)) best = o;
  }
  __shared__ PriceCand wb[kBlock / 32];
  if ((threadIdx.x & 31) == 0) wb[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    PriceCand b = wb[0];
    for (int w = 1; w < kBlock / 32; ++w)
      if (price_better(wb[w], b, bland)) b = wb[w];
    part[blockIdx.x] = b;
  }
}

__global__ void k_price_finish(const PriceCand* __restrict__ part, int nblocks, int bland, PriceCand* out) {
  PriceCand b{0.0, -1, 0};
  for (int k = 0; k < nblocks; ++k)
    if (price_better(part[k], b, bland)) b = part[k];
  *out = b;
}

}  // namespace
}  // namespace cclp_cu
