// Microbenchmark: cycles per tcgen05.mma (bf16, M=128, K=16) for SS and TS
// operand modes and N in {128, 256}, one CTA per SM, back-to-back issue.
// Also exercises fma.rn.f32x2 / add.f32x2 / 3-input max so their SASS can be
// inspected (cuobjdump -sass). Build: nvcc -gencode arch=compute_100a,code=sm_100a
//   -O3 -std=c++17 -I../../paper_2505_21070_b200/csrc mma_floor.cu -lcuda -o mma_floor
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "tc_common.cuh"

using namespace bp;

template <int mode>
__global__ void __launch_bounds__(128, 1) k_floor(int reps, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc<512>(&slot);
  tc::fence_proxy_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint32_t a = tc::smem_u32(smem), b = tc::smem_u32(smem + 32768);
    const uint32_t id128 = tc::idesc_bf16(128, 128, 0, 0), id256 = tc::idesc_bf16(128, 256, 0, 0);
    const uint32_t idv = tc::idesc_bf16(128, 128, 0, 1);
    const uint32_t id64 = tc::idesc_bf16(128, 64, 0, 0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t ad = tc::desc_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32, 1024, 16);
        const uint64_t bd = tc::desc_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32, 1024, 16);
        const uint64_t vd = tc::desc_sw128(b + kk * 2048, 1024, 16384);
        if constexpr (mode == 0) tc::mma_bf16_ss_elect(tmem, ad, bd, id128, 1u);                   // SS N=128
        if constexpr (mode == 1) tc::mma_bf16_ts_elect(tmem, tmem + 384 + kk * 8, bd, id128, 1u);  // TS N=128
        if constexpr (mode == 2) tc::mma_bf16_ss_elect(tmem, ad, bd, id256, 1u);                   // SS N=256
        if constexpr (mode == 3) {                                                                  // SS QK + TS PV
          tc::mma_bf16_ss_elect(tmem, ad, bd, id128, 1u);
          tc::mma_bf16_ts_elect(tmem + 128, tmem + 384 + kk * 8, vd, idv, 1u);
        }
        if constexpr (mode == 4) tc::mma_bf16_ts_elect(tmem + 128, tmem + 384 + kk * 8, vd, idv, 1u);  // TS MN-major
        if constexpr (mode == 5) tc::mma_bf16_ss_elect(tmem, ad, bd, id64, 1u);                   // SS N=64
        if constexpr (mode == 6) tc::mma_bf16_ts_elect(tmem, tmem + 384 + kk * 8, bd, id64, 1u);  // TS N=64
      }
    }
    tc::mma_commit_elect(&bar);
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = static_cast<unsigned long long>(t1 - t0);
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

// Packed f32x2 math and 3-input max (SASS check only).
__global__ void k_packed(const float2* x, float2* y, float s, float m) {
  float2 v = x[threadIdx.x];
  unsigned long long xv = *reinterpret_cast<unsigned long long*>(&v), r, acc;
  const float2 sc = make_float2(s, s), mm = make_float2(-m, -m);
  const unsigned long long scv = *reinterpret_cast<const unsigned long long*>(&sc);
  const unsigned long long mv = *reinterpret_cast<const unsigned long long*>(&mm);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(xv), "l"(scv), "l"(mv));
  asm("add.f32x2 %0, %1, %2;" : "=l"(acc) : "l"(r), "l"(xv));
  float m3;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(m3) : "f"(v.x), "f"(v.y), "f"(s));
  float2 o = *reinterpret_cast<float2*>(&acc);
  o.x += m3;
  y[threadIdx.x] = o;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  void (*kern[7])(int, unsigned long long*) = {k_floor<0>, k_floor<1>, k_floor<2>, k_floor<3>,
                                                k_floor<4>, k_floor<5>, k_floor<6>};
  const char* names[] = {"SS 128x128x16", "TS 128x128x16", "SS 128x256x16", "SS+TS pairs", "TS MN-major B",
                         "SS 128x64x16", "TS 128x64x16"};
  for (int mode = 0; mode < 7; ++mode) {
    cudaFuncSetAttribute(kern[mode], cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int reps = mode == 3 ? 1000 : 2000;
    for (int it = 0; it < 2; ++it) kern[mode]<<<148, 128, 100 * 1024>>>(reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const int n = mode == 2 ? 256 : mode >= 5 ? 64 : 128;
    const double per = static_cast<double>(cyc) / (reps * 8.0 * (mode == 3 ? 2 : 1));
    printf("%-20s %8.2f cyc/mma  floor %d  -> %.1f%% of floor (%s)\n", names[mode], per, 128 * n / 256,
           100.0 * (128.0 * n / 256) / per, cudaGetErrorString(e));
  }
  return 0;
}
