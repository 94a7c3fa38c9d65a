// MUFU exp2 throughput: ex2.approx.f32 vs ex2.approx.f16x2 vs ex2.approx.ftz.bf16x2
// (exps per SM per clock, all SMs busy).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_probe.cu -o mufu_probe && ./mufu_probe
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void k(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * 2654435761u + i);
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = -0.001f * (threadIdx.x + i);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
    }
  }
  const long long t1 = clock64();
  float acc = 0;
  for (int i = 0; i < 8; ++i) acc += f[i] + __uint_as_float(a[i]);
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = static_cast<float>(t1 - t0);
  if (acc == 12345.f) out[1] = acc;
}

int main() {
  float* d;
  cudaMalloc(&d, 8);
  const int iters = 4096, threads = 1024;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<148, threads>>>(d, iters);
      if (mode == 1) k<1><<<148, threads>>>(d, iters);
      if (mode == 2) k<2><<<148, threads>>>(d, iters);
    }
    cudaDeviceSynchronize();
    float cyc;
    cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
    const double insts = static_cast<double>(iters) * 8 * threads;  // per SM (one CTA per SM)
    const double values = insts * (mode == 0 ? 1 : 2);
    std::printf("%-18s %.2f instr/clk/SM  %.2f exp/clk/SM\n",
                mode == 0 ? "ex2.f32" : (mode == 1 ? "ex2.f16x2" : "ex2.bf16x2"), insts / cyc, values / cyc);
  }
  return 0;
}
