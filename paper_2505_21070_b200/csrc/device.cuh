// Device-side shared declarations: error checking, buffers, launch helpers.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "common.hpp"

namespace bp {

constexpr int kNumSms = 148;  // B200
constexpr uint64_t kGoldenDev = 0x9E3779B97F4A7C15ULL;

#define BP_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      ::bp::fail(BP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// NVTX range for the host scope (pass / stage / sublayer structure of the
// reference's run_pipeline and forward_chunk in nsys and `ncu --nvtx`
// timelines); header-only NVTX3, a no-op unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Counts our own kernel launches (reported as gpu_launches by bench.py).
extern std::atomic<int64_t> g_launches;
inline void count_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
#ifdef BP_DEBUG_SYNC
  BP_CUDA(cudaDeviceSynchronize());
#endif
  BP_CUDA(cudaPeekAtLastError());
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device);
// the attribute is per device context, and the bookkeeping is thread-safe.
void set_smem_attr_impl(const void* fn, int bytes);
template <typename F>
inline void set_smem_attr(F* fn, int bytes) { set_smem_attr_impl(reinterpret_cast<const void*>(fn), bytes); }

// Device allocation tracking for the peak-HBM report.
extern std::atomic<int64_t> g_dev_bytes, g_dev_peak;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t n) {
    release();
    if (n == 0) return;
    BP_CUDA(cudaMalloc(&p, n));
    bytes = n;
    const int64_t now = g_dev_bytes.fetch_add(static_cast<int64_t>(n)) + static_cast<int64_t>(n);
    int64_t peak = g_dev_peak.load();
    while (now > peak && !g_dev_peak.compare_exchange_weak(peak, now)) {}
  }
  // Grows (never shrinks) to at least n bytes; contents are not preserved.
  void reserve(size_t n) { if (n > bytes) alloc(n); }
  void release() {
    if (p) {
      cudaFree(p);
      g_dev_bytes.fetch_sub(static_cast<int64_t>(bytes));
    }
    p = nullptr;
    bytes = 0;
  }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

// Up to 4 source row ranges concatenated into one destination.
struct GatherSegs {
  int n = 0;
  const double* src[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t start[5] = {0, 0, 0, 0, 0};
  void add(const double* s, int64_t rows) {
    src[n] = s;
    start[n + 1] = start[n] + rows;
    ++n;
  }
};

void launch_normal_fill(uint64_t state, int64_t n, double sigma, double* out, cudaStream_t st);
void launch_pool_differs(const double* pool, int m, int64_t per, int* differs, cudaStream_t st);
void launch_gather_rows(const GatherSegs& segs, int64_t cols, double* dst, cudaStream_t st);
void launch_gather_ids(const double* pool, int64_t per, const int32_t* ids, int n, double* out, cudaStream_t st);
void launch_elementwise(int op, const double* a, const double* b, int64_t n, double s, double* out, cudaStream_t st);
template <typename TE>
void launch_scheduler_step(const double* x, const TE* eps, int64_t n, int steps, double* out,
                           cudaStream_t st);

}  // namespace bp
