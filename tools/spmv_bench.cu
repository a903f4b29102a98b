// Standalone SpMV variant microbenchmark (development tool, not product).
// Reads a CSR (rowptr i32[m+1], colind i32[nnz], val f64[nnz]) and a dense
// vector of length ncols from raw files and times y = A x for several kernel
// designs, checking each against the sequential-order result.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o spmv_bench spmv_bench.cu
//   ./spmv_bench prefix   (prefix.ptr, prefix.idx, prefix.val, prefix.x, prefix.meta)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

template <class T>
std::vector<T> readf(const char* path, size_t n) {
  std::vector<T> v(n);
  FILE* f = fopen(path, "rb");
  if (!f || fread(v.data(), sizeof(T), n, f) != n) {
    printf("read %s failed\n", path);
    exit(1);
  }
  fclose(f);
  return v;
}

// V0: thread per row, sequential (reference order), unroll loads by U
template <int U>
__global__ void v_scalar(int m, const int* __restrict__ ptr, const int* __restrict__ idx,
                         const double* __restrict__ val, const double* __restrict__ x,
                         double* __restrict__ y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
    const int b = ptr[i], e = ptr[i + 1];
    double acc = 0.0;
    int p = b;
    for (; p + U <= e; p += U) {
      int ii[U];
      double vv[U], xx[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        ii[k] = __ldcs(idx + p + k);
        vv[k] = __ldcs(val + p + k);
      }
#pragma unroll
      for (int k = 0; k < U; ++k) xx[k] = __ldg(x + ii[k]);
#pragma unroll
      for (int k = 0; k < U; ++k) acc = acc + vv[k] * xx[k];
    }
    for (; p < e; ++p) acc = acc + __ldcs(val + p) * __ldg(x + __ldcs(idx + p));
    y[i] = acc;
  }
}

// V1: G lanes per row, strided partial sums + butterfly (deterministic, not
// reference order), warp-independent (no block barriers).
template <int G, int U>
__global__ void v_vector(int m, const int* __restrict__ ptr, const int* __restrict__ idx,
                         const double* __restrict__ val, const double* __restrict__ x,
                         double* __restrict__ y) {
  const int lane = threadIdx.x % G;
  const int gpb = blockDim.x / G;
  for (int row = blockIdx.x * gpb + threadIdx.x / G; row - (threadIdx.x / G) < m;
       row += gridDim.x * gpb) {
    double acc = 0.0;
    if (row < m) {
      const int b = ptr[row], e = ptr[row + 1];
      for (int p = b + lane; p < e; p += G * U) {
        int ii[U];
        double vv[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
          const int q = p + k * G;
          ii[k] = q < e ? __ldcs(idx + q) : -1;
          vv[k] = q < e ? __ldcs(val + q) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < U; ++k)
          if (ii[k] >= 0) acc = acc + vv[k] * __ldg(x + ii[k]);
      }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0 && row < m) y[row] = acc;
  }
}

// V2: warp-private 32-row tiles staged through smem, sequential per-row sum
// by the owner lane from a products buffer filled coalesced by the warp.
// No block barriers (only __syncwarp). Window = the tile's nnz, processed in
// pieces of 32*K.
template <int K>
__global__ void v_warpstream(int m, const int* __restrict__ ptr, const int* __restrict__ idx,
                             const double* __restrict__ val, const double* __restrict__ x,
                             double* __restrict__ y) {
  extern __shared__ double sh[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* prod = sh + warp * 32 * K;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int tile = (blockIdx.x * (blockDim.x >> 5) + warp) * 32; tile < m; tile += nwarps * 32) {
    const int nrows = min(32, m - tile);
    const int my_b = lane < nrows ? ptr[tile + lane] : 0;
    const int my_e = lane < nrows ? ptr[tile + lane + 1] : 0;
    const int pb = __shfl_sync(0xffffffffu, my_b, 0);
    const int pe = __shfl_sync(0xffffffffu, my_e, nrows - 1);
    double acc = 0.0;
    for (int c0 = pb; c0 < pe; c0 += 32 * K) {
      const int len = min(32 * K, pe - c0);
      int ii[K];
      double vv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int q = lane + 32 * k;
        ii[k] = q < len ? __ldcs(idx + c0 + q) : 0;
        vv[k] = q < len ? __ldcs(val + c0 + q) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int q = lane + 32 * k;
        if (q < len) prod[q] = vv[k] * __ldg(x + ii[k]);
      }
      __syncwarp();
      const int a = max(my_b, c0), e = min(my_e, c0 + len);
      for (int q = a; q < e; ++q) acc = acc + prod[q - c0];
      __syncwarp();
    }
    if (lane < nrows) y[tile + lane] = acc;
  }
}

int main(int argc, char** argv) {
  char path[512];
  snprintf(path, sizeof path, "%s.meta", argv[1]);
  auto meta = readf<long long>(path, 3);
  const int m = (int)meta[0], ncols = (int)meta[1];
  const long long nnz = meta[2];
  snprintf(path, sizeof path, "%s.ptr", argv[1]);
  auto hp = readf<int>(path, m + 1);
  snprintf(path, sizeof path, "%s.idx", argv[1]);
  auto hi = readf<int>(path, nnz);
  snprintf(path, sizeof path, "%s.val", argv[1]);
  auto hv = readf<double>(path, nnz);
  snprintf(path, sizeof path, "%s.x", argv[1]);
  auto hx = readf<double>(path, ncols);
  int *dp, *di;
  double *dv, *dx, *dy;
  CK(cudaMalloc(&dp, sizeof(int) * (m + 1)));
  CK(cudaMalloc(&di, sizeof(int) * nnz));
  CK(cudaMalloc(&dv, sizeof(double) * nnz));
  CK(cudaMalloc(&dx, sizeof(double) * ncols));
  CK(cudaMalloc(&dy, sizeof(double) * m));
  CK(cudaMemcpy(dp, hp.data(), sizeof(int) * (m + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(di, hi.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv, hv.data(), sizeof(double) * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, hx.data(), sizeof(double) * ncols, cudaMemcpyHostToDevice));
  // flush buffer > L2
  double* flush;
  const size_t fl = 256ull << 20;
  CK(cudaMalloc(&flush, fl));
  std::vector<double> ref(m);
  for (int i = 0; i < m; ++i) {
    double a = 0.0;
    for (int p = hp[i]; p < hp[i + 1]; ++p) a = a + hv[p] * hx[hi[p]];
    ref[i] = a;
  }
  const double bytes = 12.0 * nnz + 4.0 * (m + 1) + 8.0 * ncols + 8.0 * m;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    std::vector<double> hy(m);
    float best = 1e9, sum = 0;
    const int reps = 20;
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaMemset(flush, r, fl));
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) {
        best = ms < best ? ms : best;
        sum += ms;
      }
    }
    CK(cudaGetLastError());
    CK(cudaMemcpy(hy.data(), dy, sizeof(double) * m, cudaMemcpyDeviceToHost));
    int exact = 0;
    double maxrel = 0;
    for (int i = 0; i < m; ++i) {
      exact += hy[i] == ref[i];
      double d = fabs(hy[i] - ref[i]) / (fabs(ref[i]) + 1e-300);
      if (d > maxrel) maxrel = d;
    }
    printf("%-28s avg %7.2f us  best %7.2f us  %6.0f GB/s  exact %d/%d  maxrel %.1e\n", name,
           sum / reps * 1e3, best * 1e3, bytes / (sum / reps * 1e-3) / 1e9, exact, m, maxrel);
  };
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("m=%d ncols=%d nnz=%lld avg=%.1f bytes=%.1f MB\n", m, ncols, nnz, (double)nnz / m, bytes / 1e6);
  for (int bs : {128, 256}) {
    for (int mult : {4, 8, 16}) {
      const int grid = sms * mult * (256 / bs);
      char nm[64];
      snprintf(nm, sizeof nm, "scalar U4 bs%d g%d", bs, grid);
      run(nm, [&] { v_scalar<4><<<grid, bs>>>(m, dp, di, dv, dx, dy); });
      snprintf(nm, sizeof nm, "scalar U8 bs%d g%d", bs, grid);
      run(nm, [&] { v_scalar<8><<<grid, bs>>>(m, dp, di, dv, dx, dy); });
    }
  }
#define VEC(G, U)                                                                          \
  for (int mult : {8, 16, 32}) {                                                           \
    const int grid = sms * mult;                                                           \
    char nm[64];                                                                           \
    snprintf(nm, sizeof nm, "vector G%d U%d g%d", G, U, grid);                             \
    run(nm, [&] { v_vector<G, U><<<grid, 256>>>(m, dp, di, dv, dx, dy); });                \
  }
  VEC(2, 4) VEC(4, 4) VEC(8, 2) VEC(8, 4) VEC(16, 2) VEC(16, 4) VEC(32, 2) VEC(32, 4)
#define WS(K)                                                                              \
  for (int mult : {4, 8, 16}) {                                                            \
    const int grid = sms * mult;                                                           \
    char nm[64];                                                                           \
    snprintf(nm, sizeof nm, "warpstream K%d g%d", K, grid);                                \
    run(nm, [&] { v_warpstream<K><<<grid, 256, 8 * 32 * K * 8>>>(m, dp, di, dv, dx, dy); }); \
  }
  WS(4) WS(8) WS(16)
  return 0;
}
