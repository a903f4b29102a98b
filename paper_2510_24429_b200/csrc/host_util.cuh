// Host-side utilities shared by the engine's translation units (engine.cu,
// sharded.cu, capi.cu): errors, the pinned-memory cache, the stream-ordered
// pool, launch helpers and the LP's CSC validation.
#pragma once
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <condition_variable>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <type_traits>
#include <random>
#include <stdexcept>
#include <memory>
#include <thread>
#include <string>
#include <vector>

#include "../../include/cclp_cu.h"

#include "engine.cuh"
#include "kernels.cuh"

namespace cclp_cu {

inline thread_local std::string g_err;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? CCLP_CU_ENOMEM : CCLP_CU_ECUDA;
    cudaGetLastError();
    throw Error(code, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(x) ::cclp_cu::ck((x), #x)
#define CKL(what) ::cclp_cu::ck(cudaGetLastError(), what)

// one pinned-buffer cache per process, shared by every translation unit
inline std::mutex g_pinned_mu;
inline std::multimap<size_t, void*> g_pinned_free;

namespace {

// Device memory comes from the device's default stream-ordered pool with an
// unbounded release threshold: a solve's buffers return to the pool on
// destroy and the next context reuses them, so create/destroy never touch
// the driver's allocator (cudaMalloc/cudaFree synchronize the device and cost
// milliseconds each at these sizes).
void ensure_pool(int device) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> g(mu);
  if (std::find(done.begin(), done.end(), device) != done.end()) return;
  cudaMemPool_t pool;
  CK(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done.push_back(device);
}

// Pinned host buffers (control block, log, snapshot staging) are recycled
// process-wide for the same reason: cudaHostAlloc/cudaFreeHost pin and unpin
// pages synchronously.

void* pinned_alloc(size_t bytes) {
  {
    std::lock_guard<std::mutex> g(g_pinned_mu);
    auto it = g_pinned_free.lower_bound(bytes);
    if (it != g_pinned_free.end() && it->first <= 2 * bytes + 4096) {
      void* p = it->second;
      g_pinned_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  CK(cudaHostAlloc(&p, std::max<size_t>(bytes, 1), cudaHostAllocDefault));
  return p;
}

void pinned_release(void* p, size_t bytes) {
  if (p == nullptr) return;
  std::lock_guard<std::mutex> g(g_pinned_mu);
  g_pinned_free.emplace(std::max<size_t>(bytes, 1), p);
}

// Lanes per row from the mean row length L. A fixed rule (never timing
// based): G sets the per-row summation order, so it must not vary between
// runs. Thresholds measured on B200 (profiles/r1/history/): L <= 8 -> 2
// (C1 columns, C5 column panels at L ~ 5.5: G 1/2/4 = 4.40/4.22/4.69 ms),
// L 9-24 -> 4 (C2/C4 columns, C4 rows), L ~ 50 -> 8, L ~ 100 -> 16,
// L >= 160 -> 32.
int pick_group(long long nnz, long long rows) {
  const double L = rows > 0 ? static_cast<double>(nnz) / static_cast<double>(rows) : 0.0;
  if (L <= 8.0) return 2;
  if (L <= 24.0) return 4;
  if (L <= 64.0) return 8;
  if (L <= 160.0) return 16;
  return 32;
}

int blocks_for(long long n, int per = kBlock, int cap = 148 * 8) {
  long long b = (n + per - 1) / per;
  return static_cast<int>(std::max<long long>(1, std::min<long long>(b, cap)));
}

// Development knobs (A/B experiments and tests: lanes per row, panel width,
// SELL layouts, launch geometry, PDL, halo): read only when
// CCLP_CU_DEV_KNOBS=1, so a user's environment cannot change the engine's
// summation order or layouts. (CCLP_CU_TRANSPORT, a bit-identical transport
// choice of the sharded solve, is a documented user option.)
const char* dev_knob(const char* name) {
  static const bool on = [] {
    const char* e = std::getenv("CCLP_CU_DEV_KNOBS");
    return e != nullptr && std::atoi(e) == 1;
  }();
  return on ? std::getenv(name) : nullptr;
}

// Launch with programmatic stream serialization (PDL): the kernel may begin
// launching while its predecessor drains; it synchronizes with griddepcontrol.
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = dev_knob("CCLP_CU_PDL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

template <class... KArgs, class... Args>
void launch_pdl_smem(void (*kernel)(KArgs...), int grid, int block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  ck(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t st, Args&&... args) {
  launch_pdl_smem(kernel, grid, block, 0, st, std::forward<Args>(args)...);
}
// More than 48 KB of dynamic shared memory needs the kernel's opt-in
// attribute, per device (set once each).
void allow_smem(const void* kernel, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> set;
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = set[{kernel, dev}];
  if (smem > have) {
    ck(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
       "cudaFuncSetAttribute");
    have = smem;
  }
}

// Calls f(std::integral_constant<int, G>) for the runtime group size G.
// Host <-> device copies of the caller's arrays (the LP in, the result out).
// Pinned memory goes straight to the DMA engine; large pageable arrays are
// staged through two pinned chunks filled (or drained) by several host
// threads while the other chunk is in flight - the driver's own pageable path
// is a single-threaded bounce (~8 GB/s).
constexpr size_t kStageChunk = size_t(32) << 20;

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  if (bytes < (size_t(4) << 20) || hw == 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = (bytes + hw - 1) / hw;
  std::vector<std::thread> th;
  for (unsigned t = 1; t < hw && size_t(t) * per < bytes; ++t) {
    const size_t a = size_t(t) * per;
    th.emplace_back([=] {
      std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, std::min(per, bytes - a));
    });
  }
  std::memcpy(dst, src, std::min(per, bytes));
  for (auto& t : th) t.join();
}

// The CSC checks of LinearProgram::validate (lp.cpp:71-83) that guard memory
// safety: colptr[0] == 0, non-decreasing offsets, 0 <= row < m, rows strictly
// ascending within a column. Same messages; host threads over column ranges.
void validate_csc(const cclp_cu_lp* lp) {
  const int m = lp->m, n = lp->n;
  const int32_t* cp = lp->colptr;
  const int32_t* ri = lp->rowind;
  if (cp[0] != 0) throw std::invalid_argument("colptr[0] != 0");
  for (int j = 0; j < n; ++j)
    if (cp[j] > cp[j + 1]) throw std::invalid_argument("decreasing column offsets");
  const long long nnz = cp[n];
  if (nnz > 0 && ri == nullptr) throw std::invalid_argument("null row indices");
  const unsigned hw = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  const unsigned T = nnz < (1LL << 20) ? 1u : hw;
  std::vector<int> bad(T, 0);
  auto work = [&](unsigned t) {
    const int j0 = static_cast<int>(static_cast<long long>(n) * t / T);
    const int j1 = static_cast<int>(static_cast<long long>(n) * (t + 1) / T);
    for (int j = j0; j < j1 && !bad[t]; ++j)
      for (int q = cp[j]; q < cp[j + 1]; ++q) {
        const int i = ri[q];
        if (i < 0 || i >= m) { bad[t] = 1; break; }
        if (q > cp[j] && i <= ri[q - 1]) { bad[t] = 2; break; }
      }
  };
  std::vector<std::thread> th;
  for (unsigned t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (int b : bad) {
    if (b == 1) throw std::invalid_argument("row index out of range");
    if (b == 2) throw std::invalid_argument("unsorted or duplicate row indices");
  }
}

template <class F>
void with_group(int G, F&& f) {
  switch (G) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    case 8: f(std::integral_constant<int, 8>{}); break;
    case 16: f(std::integral_constant<int, 16>{}); break;
    default: f(std::integral_constant<int, 32>{}); break;
  }
}

// Calls f(G constant, LONG constant): long-row segments compiled in only when
// the matrix has rows past the threshold.
template <class F>
void with_group_long(int G, bool lng, F&& f) {
  if (lng) {
    with_group(G, [&](auto g) { f(g, std::true_type{}); });
  } else {
    with_group(G, [&](auto g) { f(g, std::false_type{}); });
  }
}

}  // namespace

}  // namespace cclp_cu
