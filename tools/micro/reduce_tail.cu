// Dev micro: cost of the finalize-block partial reduction (reduce_partials in
// iter_kernels.cuh) in isolation: 22 fields x 148 block partials, 512 threads,
// half-warp per field, 16 loads in flight, butterfly, shared store, barrier.
#include <cstdio>
#include <vector>
constexpr int kRowParts = 8, kColParts = 14;
constexpr unsigned kRowMax = (1u << 1) | (1u << 4), kColMax = (1u << 1) | (1u << 2) | (1u << 3) | (1u << 7) | (1u << 8) | (1u << 9);
__device__ __forceinline__ double amax(double a, double v) { return a < v ? v : a; }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

template <bool LOADS>
__global__ void k(const double* rowsrc, int nrow, const double* colsrc, int ncol, double* out, unsigned long long* times) {
  __shared__ double rowv[kRowParts], colv[kColParts];
  const long long c0 = clock64();
  const unsigned long long g0 = gt();
  const int hl = threadIdx.x & 15;
  for (int fld = threadIdx.x >> 4; fld - (int)(threadIdx.x >> 4) < kRowParts + kColParts; fld += blockDim.x / 16) {
    const bool live = fld < kRowParts + kColParts;
    const bool is_row = fld < kRowParts;
    const int f = is_row ? fld : fld - kRowParts;
    const bool is_max = is_row ? ((kRowMax >> f) & 1u) : ((kColMax >> f) & 1u);
    const int nb = live ? (is_row ? nrow : ncol) : 0;
    const double* src = (is_row ? rowsrc : colsrc) + (long long)f * nb;
    double a = 0.0;
    for (int b0 = hl; b0 < nb; b0 += 256) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) { const int b = b0 + 16 * q; v[q] = b < nb ? (LOADS ? __ldcg(src + b) : (double)b) : 0.0; }
#pragma unroll
      for (int q = 0; q < 16; ++q) if (b0 + 16 * q < nb) a = is_max ? amax(a, v[q]) : a + v[q];
    }
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) { const double o = __shfl_xor_sync(0xffffffffu, a, off); a = is_max ? amax(a, o) : a + o; }
    if (hl == 0 && live) (is_row ? rowv : colv)[f] = a;
  }
  __syncthreads();
  const long long c1 = clock64();
  const unsigned long long g1 = gt();
  if (threadIdx.x == 0) { times[0] = c1 - c0; times[1] = g1 - g0; out[0] = rowv[0] + colv[0]; }
}

int main() {
  double *r, *c, *o; unsigned long long* t;
  cudaMalloc(&r, 148 * kRowParts * 8); cudaMalloc(&c, 148 * kColParts * 8); cudaMalloc(&o, 8); cudaMalloc(&t, 16);
  cudaMemset(r, 0, 148 * kRowParts * 8); cudaMemset(c, 0, 148 * kColParts * 8);
  for (int rep = 0; rep < 4; ++rep) {
    for (int loads = 0; loads < 2; ++loads) {
      if (loads) k<true><<<1, 512>>>(r, 148, c, 148, o, t); else k<false><<<1, 512>>>(r, 148, c, 148, o, t);
      unsigned long long h[2]; cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
      printf("loads=%d: %llu cycles, %llu ns\n", loads, h[0], h[1]);
    }
  }
}
