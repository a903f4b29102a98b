// Microbenchmark: random fp64 gathers from L2 (global, __ldg) vs from
// distributed shared memory (the gathered vector split across a cluster's
// CTAs). Question: can the column SpMV of a small-m LP (C2: m = 100k, 800 KB)
// gather y from DSMEM faster than the L1TEX/L2 sector path?
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
namespace cg = cooperative_groups;

__global__ void k_global(const int* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ y,
                         long long N, double* out) {
  double acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N; e += stride)
    acc += __ldcs(val + e) * __ldg(y + __ldcs(idx + e));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int SHIFT>
__global__ void k_dsmem(const int* __restrict__ idx, const double* __restrict__ val, const double* __restrict__ y,
                        int m, long long N, double* out) {
  extern __shared__ double sy[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  const int S = 1 << SHIFT;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    const int g = rank * S + i;
    sy[i] = g < m ? y[g] : 0.0;
  }
  cl.sync();
  double* parts[16];
  const int cs = cl.num_blocks();
  for (int q = 0; q < cs; ++q) parts[q] = cl.map_shared_rank(sy, q);
  double acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < N; e += stride) {
    const int j = __ldcs(idx + e);
    acc += __ldcs(val + e) * parts[j >> SHIFT][j & (S - 1)];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  cl.sync();
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 100000;
  const long long N = 5000000;
  std::vector<int> hi(N);
  std::vector<double> hv(N), hy(m);
  std::mt19937 rng(1);
  for (long long e = 0; e < N; ++e) { hi[e] = rng() % m; hv[e] = 1.0 + (e % 7); }
  for (int i = 0; i < m; ++i) hy[i] = i * 0.5;
  int* idx; double *val, *y, *out;
  cudaMalloc(&idx, N * 4); cudaMalloc(&val, N * 8); cudaMalloc(&y, m * 8); cudaMalloc(&out, 1 << 24);
  cudaMemcpy(idx, hi.data(), N * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(val, hv.data(), N * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(y, hy.data(), m * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int bs : {512, 1024}) {
    for (int per : {1, 2, 4}) {
      if (bs * per > 2048) continue;
      k_global<<<148 * per, bs>>>(idx, val, y, N, out);
      cudaEventRecord(a);
      for (int r = 0; r < 20; ++r) k_global<<<148 * per, bs>>>(idx, val, y, N, out);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
      printf("global  block %4d x %d/SM: %.2f us per 5M gathers\n", bs, per, ms / 20 * 1e3);
    }
  }
  // DSMEM: S = 2^SHIFT doubles per CTA, cluster size cs with cs * S >= m
  auto run = [&](auto kern, int shift, int cs, int bs) {
    const size_t smem = sizeof(double) << shift;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(bs); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
    int ncl = 0;
    cfg.gridDim = dim3(cs);
    cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
    cfg.gridDim = dim3(ncl * cs);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, (const int*)idx, (const double*)val, (const double*)y, m, N, out);
    if (e != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(e)); return; }
    cudaEventRecord(a);
    for (int r = 0; r < 20; ++r) cudaLaunchKernelEx(&cfg, kern, (const int*)idx, (const double*)val, (const double*)y, m, N, out);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("dsmem   cluster %2d, %3d KB/CTA, block %4d, %d clusters (%d CTAs): %.2f us  [%s]\n", cs,
           (int)(smem >> 10), bs, ncl, ncl * cs, ms / 20 * 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bs : {512, 1024}) {
    if (m <= 8 * 16384) run(k_dsmem<14>, 14, 8, bs);
    if (m <= 16 * 8192) run(k_dsmem<13>, 13, 16, bs);
    if (m <= 4 * 16384 * 2) run(k_dsmem<15>, 15, 4, bs);
  }
  return 0;
}
