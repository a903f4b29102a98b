// Dev microbenchmark: SELL-32-sigma (32-row slices, column-major within a
// slice, rows sorted by length inside sigma-row windows, one lane per row,
// sequential per-row sums = the reference's order) against the engine's
// G-lanes-per-row CSR kernel (two rows per group in flight), on dumps made by
// tools/dump_csr.py. Steady state (x resident, no flush) and flushed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sell_bench sell_bench.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
template <class T> std::vector<T> readf(const char* path, size_t n) {
  std::vector<T> v(n); FILE* f = fopen(path, "rb");
  if (!f || fread(v.data(), sizeof(T), n, f) != n) { printf("read %s failed\n", path); exit(1); }
  fclose(f); return v;
}

template <int G, int U>
__global__ void __launch_bounds__(1024) v_csr2(const int* __restrict__ st, const int* __restrict__ ptr,
    const int* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const int gl = threadIdx.x % G, gpb = blockDim.x / G;
  const int rb = st[blockIdx.x], re = st[blockIdx.x + 1];
  for (int row = rb + (int)(threadIdx.x / G); row - (int)(threadIdx.x / G) < re; row += 2 * gpb) {
    const int row1 = row + gpb;
    const bool ok0 = row < re, ok1 = row1 < re;
    const int b0 = ok0 ? __ldg(ptr + row) : 0, e0 = ok0 ? __ldg(ptr + row + 1) : 0;
    const int b1 = ok1 ? __ldg(ptr + row1) : 0, e1 = ok1 ? __ldg(ptr + row1 + 1) : 0;
    double a0 = 0, a1 = 0;
    for (int p0 = b0 + gl, p1 = b1 + gl; p0 < e0 || p1 < e1; p0 += G * U, p1 += G * U) {
      int i0[U], i1[U]; double v0[U], v1[U], x0[U], x1[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int q0 = p0 + k * G, q1 = p1 + k * G;
        i0[k] = q0 < e0 ? __ldcs(idx + q0) : -1; v0[k] = q0 < e0 ? __ldcs(val + q0) : 0.0;
        i1[k] = q1 < e1 ? __ldcs(idx + q1) : -1; v1[k] = q1 < e1 ? __ldcs(val + q1) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < U; ++k) { x0[k] = i0[k] >= 0 ? __ldg(x + i0[k]) : 0.0; x1[k] = i1[k] >= 0 ? __ldg(x + i1[k]) : 0.0; }
#pragma unroll
      for (int k = 0; k < U; ++k) if (i0[k] >= 0) a0 = a0 + v0[k] * x0[k];
#pragma unroll
      for (int k = 0; k < U; ++k) if (i1[k] >= 0) a1 = a1 + v1[k] * x1[k];
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) { a0 += __shfl_xor_sync(~0u, a0, off); a1 += __shfl_xor_sync(~0u, a1, off); }
    if (gl == 0 && ok0) y[row] = a0;
    if (gl == 0 && ok1) y[row1] = a1;
  }
}

// rpg = 1 CSR-G kernel with U loads in flight per lane (engine's group_dot<G, U>)
template <int G, int U>
__global__ void __launch_bounds__(1024) v_csr1(const int* __restrict__ st, const int* __restrict__ ptr,
    const int* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
  const int gl = threadIdx.x % G, gpb = blockDim.x / G;
  const int rb = st[blockIdx.x], re = st[blockIdx.x + 1];
  for (int row = rb + (int)(threadIdx.x / G); row - (int)(threadIdx.x / G) < re; row += gpb) {
    const bool ok = row < re;
    const int b = ok ? __ldg(ptr + row) : 0, e = ok ? __ldg(ptr + row + 1) : 0;
    double acc = 0.0;
    for (int p = b + gl; p < e; p += G * U) {
      int ii[U]; double vv[U], xx[U];
#pragma unroll
      for (int k = 0; k < U; ++k) { const int q = p + k * G; ii[k] = q < e ? __ldcs(idx + q) : -1; vv[k] = q < e ? __ldcs(val + q) : 0.0; }
#pragma unroll
      for (int k = 0; k < U; ++k) xx[k] = ii[k] >= 0 ? __ldg(x + ii[k]) : 0.0;
#pragma unroll
      for (int k = 0; k < U; ++k) if (ii[k] >= 0) acc = acc + vv[k] * xx[k];
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(~0u, acc, off);
    if (gl == 0 && ok) y[row] = acc;
  }
}

// SELL: warp per slice (grid-stride over slices); lane = row; U elements per round.
template <int U, bool PIPE>
__global__ void __launch_bounds__(1024) v_sell(int nsl, const long long* __restrict__ soff, const int* __restrict__ swid,
    const int* __restrict__ prow, const int* __restrict__ plen, const int* __restrict__ sidx,
    const double* __restrict__ sval, const double* __restrict__ x, double* __restrict__ y, int m) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nsl; s += nw) {
    const long long off = soff[s];
    const int w = swid[s];
    const int p = s * 32 + lane;
    const int len = p < m ? __ldg(plen + p) : 0;
    const int row = p < m ? __ldg(prow + p) : -1;
    const int* ib = sidx + off + lane;
    const double* vb = sval + off + lane;
    double acc = 0.0;
    if (!PIPE) {
      for (int k = 0; k < w; k += U) {
        int ii[U]; double vv[U], xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const bool ok = k + u < len; ii[u] = ok ? __ldcs(ib + (k + u) * 32) : 0; vv[u] = ok ? __ldcs(vb + (k + u) * 32) : 0.0; }
#pragma unroll
        for (int u = 0; u < U; ++u) xx[u] = k + u < len ? __ldg(x + ii[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) if (k + u < len) acc = acc + vv[u] * xx[u];
      }
    } else {
      int ii[U]; double vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { const bool ok = u < len; ii[u] = ok ? __ldcs(ib + u * 32) : 0; vv[u] = ok ? __ldcs(vb + u * 32) : 0.0; }
      for (int k = 0; k < w; k += U) {
        double xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) xx[u] = k + u < len ? __ldg(x + ii[u]) : 0.0;
        int in[U]; double vn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const bool ok = k + U + u < len; in[u] = ok ? __ldcs(ib + (k + U + u) * 32) : 0; vn[u] = ok ? __ldcs(vb + (k + U + u) * 32) : 0.0; }
#pragma unroll
        for (int u = 0; u < U; ++u) if (k + u < len) acc = acc + vv[u] * xx[u];
#pragma unroll
        for (int u = 0; u < U; ++u) { ii[u] = in[u]; vv[u] = vn[u]; }
      }
    }
    if (row >= 0) y[row] = acc;
  }
}

// SELL-G: 32/G rows per slice, G lanes per row; lane gl of row r takes the
// row's elements gl, gl+G, ... (stored at off + k*32 + r*G + gl), then the
// same xor butterfly as the CSR-G kernel: bit-identical to it.
template <int G, int U, bool PIPE>
__global__ void __launch_bounds__(1024) v_sellg(int nsl, const long long* __restrict__ soff, const int* __restrict__ swid,
    const int* __restrict__ plen, const int* __restrict__ sidx, const double* __restrict__ sval,
    const double* __restrict__ x, double* __restrict__ y, int m) {
  constexpr int R = 32 / G;
  const int lane = threadIdx.x & 31, r = lane / G, gl = lane % G;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = gw; s < nsl; s += nw) {
    const long long off = soff[s];
    const int w = swid[s];
    const int row = s * R + r;
    const int len = row < m ? __ldg(plen + row) : 0;
    const int* ib = sidx + off + lane;
    const double* vb = sval + off + lane;
    double acc = 0.0;
    if (!PIPE) {
      for (int k = 0; k < w; k += U) {
        int ii[U]; double vv[U], xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const bool ok = (k + u) * G + gl < len; ii[u] = ok ? __ldcs(ib + (k + u) * 32) : -1; vv[u] = ok ? __ldcs(vb + (k + u) * 32) : 0.0; }
#pragma unroll
        for (int u = 0; u < U; ++u) xx[u] = ii[u] >= 0 ? __ldg(x + ii[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) if (ii[u] >= 0) acc = acc + vv[u] * xx[u];
      }
    } else {
      int ii[U]; double vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) { const bool ok = u * G + gl < len; ii[u] = ok ? __ldcs(ib + u * 32) : -1; vv[u] = ok ? __ldcs(vb + u * 32) : 0.0; }
      for (int k = 0; k < w; k += U) {
        double xx[U];
#pragma unroll
        for (int u = 0; u < U; ++u) xx[u] = ii[u] >= 0 ? __ldg(x + ii[u]) : 0.0;
        int in[U]; double vn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { const bool ok = (k + U + u) * G + gl < len; in[u] = ok ? __ldcs(ib + (k + U + u) * 32) : -1; vn[u] = ok ? __ldcs(vb + (k + U + u) * 32) : 0.0; }
#pragma unroll
        for (int u = 0; u < U; ++u) if (ii[u] >= 0) acc = acc + vv[u] * xx[u];
#pragma unroll
        for (int u = 0; u < U; ++u) { ii[u] = in[u]; vv[u] = vn[u]; }
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(~0u, acc, o);
    if (gl == 0 && row < m) y[row] = acc;
  }
}

int main(int argc, char** argv) {
  char path[512];
  snprintf(path, sizeof path, "%s.meta", argv[1]);
  auto meta = readf<long long>(path, 3);
  const int m = (int)meta[0], ncols = (int)meta[1];
  const long long nnz = meta[2];
  snprintf(path, sizeof path, "%s.ptr", argv[1]); auto hp = readf<int>(path, m + 1);
  snprintf(path, sizeof path, "%s.idx", argv[1]); auto hi = readf<int>(path, nnz);
  snprintf(path, sizeof path, "%s.val", argv[1]); auto hv = readf<double>(path, nnz);
  snprintf(path, sizeof path, "%s.x", argv[1]); auto hx = readf<double>(path, ncols);
  const int G = argc > 2 ? atoi(argv[2]) : 8;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  std::vector<double> ref(m);
  for (int i = 0; i < m; ++i) { double a = 0; for (int p = hp[i]; p < hp[i + 1]; ++p) a = a + hv[p] * hx[hi[p]]; ref[i] = a; }
  int *dp, *di; double *dv, *dx, *dy;
  CK(cudaMalloc(&dp, 4 * (m + 1))); CK(cudaMalloc(&di, 4 * nnz)); CK(cudaMalloc(&dv, 8 * nnz));
  CK(cudaMalloc(&dx, 8 * ncols)); CK(cudaMalloc(&dy, 8 * m));
  CK(cudaMemcpy(dp, hp.data(), 4 * (m + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(di, hi.data(), 4 * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), 8 * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, hx.data(), 8 * ncols, cudaMemcpyHostToDevice));
  double* flush; const size_t fl = 256ull << 20; CK(cudaMalloc(&flush, fl));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, bool fl_on, auto launch) {
    std::vector<double> hy(m); float sum = 0; const int reps = 30;
    CK(cudaMemset(dy, 0, 8 * m));
    for (int r = 0; r < reps + 3; ++r) {
      if (fl_on) CK(cudaMemset(flush, r, fl));
      CK(cudaEventRecord(e0)); launch(); CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (r >= 3) sum += ms;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpy(hy.data(), dy, 8 * m, cudaMemcpyDeviceToHost));
    int exact = 0; double maxrel = 0;
    for (int i = 0; i < m; ++i) { exact += hy[i] == ref[i]; double d = fabs(hy[i] - ref[i]) / (fabs(ref[i]) + 1e-300); maxrel = std::max(maxrel, d); }
    printf("%-40s %s %8.2f us  exact %d/%d maxrel %.1e\n", name, fl_on ? "flush" : "warm ", sum / reps * 1e3, exact, m, maxrel);
  };
  printf("m=%d ncols=%d nnz=%lld avg %.1f\n", m, ncols, nnz, (double)nnz / m);
  // CSR contiguous ranges balanced by nnz + 4 per row
  for (int per : {1, 2}) {
    const int grid = sms * per;
    std::vector<int> st(grid + 1);
    for (int b = 0; b <= grid; ++b) {
      const long long target = ((long long)hp[m] + 4LL * m) * b / grid; int lo = 0, h2 = m;
      while (lo < h2) { int mid = (lo + h2) / 2; if ((long long)hp[mid] + 4LL * mid >= target) h2 = mid; else lo = mid + 1; }
      st[b] = b == grid ? m : lo;
    }
    int* dst; CK(cudaMalloc(&dst, 4 * (grid + 1))); CK(cudaMemcpy(dst, st.data(), 4 * (grid + 1), cudaMemcpyHostToDevice));
    char nm[64];
#define C1(GG, UU) if (G == GG) { snprintf(nm, sizeof nm, "csr1 G%d U%d x%d", GG, UU, per); \
      run(nm, false, [&] { v_csr1<GG, UU><<<grid, 1024>>>(dst, dp, di, dv, dx, dy); }); }
    C1(2, 4) C1(2, 8) C1(4, 2) C1(4, 3) C1(4, 4) C1(4, 6) C1(4, 8) C1(8, 2) C1(8, 4) C1(8, 6) C1(8, 7) C1(8, 8) C1(16, 2) C1(16, 3) C1(16, 4)
    for (bool f : {false, true}) {
      snprintf(nm, sizeof nm, "csr G%d U2 rpg2 x%d", G, per);
      if (G == 4) run(nm, f, [&] { v_csr2<4, 2><<<grid, 1024>>>(dst, dp, di, dv, dx, dy); });
      if (G == 8) run(nm, f, [&] { v_csr2<8, 2><<<grid, 1024>>>(dst, dp, di, dv, dx, dy); });
      if (G == 16) run(nm, f, [&] { v_csr2<16, 2><<<grid, 1024>>>(dst, dp, di, dv, dx, dy); });
    }
  }
  {
    // SELL-G in natural row order (no sorting), same G as the CSR kernel
    const int R = 32 / G;
    const int nsl = (m + R - 1) / R;
    std::vector<long long> soff(nsl + 1); std::vector<int> swid(nsl), plen(m);
    for (int i = 0; i < m; ++i) plen[i] = hp[i + 1] - hp[i];
    soff[0] = 0;
    for (int s = 0; s < nsl; ++s) {
      int w = 0; for (int r = 0; r < R && s * R + r < m; ++r) w = std::max(w, (plen[s * R + r] + G - 1) / G);
      swid[s] = w; soff[s + 1] = soff[s] + 32LL * w;
    }
    const long long tot = soff[nsl];
    std::vector<int> si(tot, -1); std::vector<double> sv(tot, 0.0);
    for (int i = 0; i < m; ++i) {
      const int s = i / R, r = i % R;
      for (int e = 0; e < plen[i]; ++e) { const long long q = soff[s] + 32LL * (e / G) + r * G + e % G; si[q] = hi[hp[i] + e]; sv[q] = hv[hp[i] + e]; }
    }
    long long *d_off; int *d_w, *d_plen, *d_si; double* d_sv;
    CK(cudaMalloc(&d_off, 8 * (nsl + 1))); CK(cudaMalloc(&d_w, 4 * nsl)); CK(cudaMalloc(&d_plen, 4 * m));
    CK(cudaMalloc(&d_si, 4 * tot)); CK(cudaMalloc(&d_sv, 8 * tot));
    CK(cudaMemcpy(d_off, soff.data(), 8 * (nsl + 1), cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_w, swid.data(), 4 * nsl, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_plen, plen.data(), 4 * m, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_si, si.data(), 4 * tot, cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_sv, sv.data(), 8 * tot, cudaMemcpyHostToDevice));
    printf("SELL-G%d: padding %.2f%%\n", G, 100.0 * (tot - nnz) / nnz);
    std::vector<double> csr_y(m), sg_y(m);
    for (int bs : {256, 1024}) for (int per : {1, 2}) {
      const int grid = bs == 256 ? sms * per * 4 : sms * per;
      char nm[80];
#define SG(GG, UU, PP) \
      if (G == GG) { snprintf(nm, sizeof nm, "sellG%d U%d%s bs%d g%d", GG, UU, PP ? " pipe" : "", bs, grid); \
        run(nm, false, [&] { v_sellg<GG, UU, PP><<<grid, bs>>>(nsl, d_off, d_w, d_plen, d_si, d_sv, dx, dy, m); }); }
      SG(2, 2, false) SG(2, 4, false) SG(2, 8, false)
      SG(4, 2, false) SG(4, 4, false) SG(4, 2, true) SG(4, 4, true)
      SG(8, 2, false) SG(8, 4, false) SG(8, 2, true)
      SG(16, 2, false) SG(16, 2, true)
    }
    CK(cudaMemcpy(sg_y.data(), dy, 8 * m, cudaMemcpyDeviceToHost));
    cudaFree(d_off); cudaFree(d_w); cudaFree(d_plen); cudaFree(d_si); cudaFree(d_sv);
    // bit-identity against the CSR-G kernel
    int* dst; const int grid = sms; std::vector<int> st(grid + 1);
    for (int b = 0; b <= grid; ++b) st[b] = (int)((long long)m * b / grid);
    CK(cudaMalloc(&dst, 4 * (grid + 1))); CK(cudaMemcpy(dst, st.data(), 4 * (grid + 1), cudaMemcpyHostToDevice));
    if (G == 2) v_csr2<2, 2><<<grid, 1024>>>(dst, dp, di, dv, dx, dy);
    if (G == 4) v_csr2<4, 2><<<grid, 1024>>>(dst, dp, di, dv, dx, dy);
    if (G == 8) v_csr2<8, 2><<<grid, 1024>>>(dst, dp, di, dv, dx, dy);
    if (G == 16) v_csr2<16, 2><<<grid, 1024>>>(dst, dp, di, dv, dx, dy);
    CK(cudaMemcpy(csr_y.data(), dy, 8 * m, cudaMemcpyDeviceToHost));
    int same = 0; for (int i = 0; i < m; ++i) same += memcmp(&csr_y[i], &sg_y[i], 8) == 0;
    printf("SELL-G%d vs CSR-G%d bit-identical rows: %d/%d\n", G, G, same, m);
    cudaFree(dst);
  }
  if (argc > 3) return 0;
  for (int sigma : {32, 256, 4096}) {
    std::vector<int> perm(m); std::iota(perm.begin(), perm.end(), 0);
    for (int w0 = 0; w0 < m; w0 += sigma) {
      const int w1 = std::min(m, w0 + sigma);
      std::stable_sort(perm.begin() + w0, perm.begin() + w1, [&](int a, int b) { return hp[a + 1] - hp[a] > hp[b + 1] - hp[b]; });
    }
    const int nsl = (m + 31) / 32;
    std::vector<long long> soff(nsl + 1); std::vector<int> swid(nsl), plen(m);
    for (int p = 0; p < m; ++p) plen[p] = hp[perm[p] + 1] - hp[perm[p]];
    soff[0] = 0;
    for (int s = 0; s < nsl; ++s) {
      int w = 0; for (int l = 0; l < 32 && s * 32 + l < m; ++l) w = std::max(w, plen[s * 32 + l]);
      swid[s] = w; soff[s + 1] = soff[s] + 32LL * w;
    }
    const long long tot = soff[nsl];
    std::vector<int> si(tot, 0); std::vector<double> sv(tot, 0.0);
    for (int p = 0; p < m; ++p) {
      const int s = p / 32, l = p % 32, r = perm[p];
      for (int k = 0; k < plen[p]; ++k) { si[soff[s] + 32LL * k + l] = hi[hp[r] + k]; sv[soff[s] + 32LL * k + l] = hv[hp[r] + k]; }
    }
    long long *d_off; int *d_w, *d_prow, *d_plen, *d_si; double* d_sv;
    CK(cudaMalloc(&d_off, 8 * (nsl + 1))); CK(cudaMalloc(&d_w, 4 * nsl)); CK(cudaMalloc(&d_prow, 4 * m)); CK(cudaMalloc(&d_plen, 4 * m));
    CK(cudaMalloc(&d_si, 4 * tot)); CK(cudaMalloc(&d_sv, 8 * tot));
    CK(cudaMemcpy(d_off, soff.data(), 8 * (nsl + 1), cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_w, swid.data(), 4 * nsl, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_prow, perm.data(), 4 * m, cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_plen, plen.data(), 4 * m, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_si, si.data(), 4 * tot, cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_sv, sv.data(), 8 * tot, cudaMemcpyHostToDevice));
    printf("sigma %d: padding %.2f%%\n", sigma, 100.0 * (tot - nnz) / nnz);
    for (int bs : {256, 1024}) for (int per : {1, 2, 4}) {
      if (bs * per > 2048) continue;
      const int grid = sms * per * (1024 / bs) / (1024 / bs) * (bs == 256 ? 4 : 1);
      char nm[80];
      for (bool f : {false, true}) {
        snprintf(nm, sizeof nm, "sell s%d U4 bs%d g%d", sigma, bs, grid);
        run(nm, f, [&] { v_sell<4, false><<<grid, bs>>>(nsl, d_off, d_w, d_prow, d_plen, d_si, d_sv, dx, dy, m); });
        snprintf(nm, sizeof nm, "sell s%d U8 bs%d g%d", sigma, bs, grid);
        run(nm, f, [&] { v_sell<8, false><<<grid, bs>>>(nsl, d_off, d_w, d_prow, d_plen, d_si, d_sv, dx, dy, m); });
        snprintf(nm, sizeof nm, "sell s%d U4 pipe bs%d g%d", sigma, bs, grid);
        run(nm, f, [&] { v_sell<4, true><<<grid, bs>>>(nsl, d_off, d_w, d_prow, d_plen, d_si, d_sv, dx, dy, m); });
      }
    }
    cudaFree(d_off); cudaFree(d_w); cudaFree(d_prow); cudaFree(d_plen); cudaFree(d_si); cudaFree(d_sv);
  }
  return 0;
}
