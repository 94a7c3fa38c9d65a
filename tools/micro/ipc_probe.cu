// Two processes on one GPU: cross-process counter signalling through CUDA
// IPC memory with one-warp polling / release-store kernels (the IPC
// transport's primitives). Prints the round-trip latency of a ping-pong.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 ipc_probe.cu -o ipc_probe && ./ipc_probe [iters]
#include <cuda_runtime.h>
#include <sys/wait.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); std::exit(1); } } while (0)

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void k_wait(const unsigned* a, unsigned v, int* timeout) {
  if (threadIdx.x) return;
  const unsigned long long t0 = gt();
  for (;;) {
    unsigned c;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(c) : "l"(a) : "memory");
    if (static_cast<int>(c - v) >= 0) return;
    __nanosleep(256);
    if (gt() - t0 > 5000000000ULL) { *timeout = 1; return; }
  }
}
__global__ void k_write(unsigned* a, unsigned v) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
  }
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? std::atoi(argv[1]) : 200;
  int p2c[2], c2p[2];
  if (pipe(p2c) || pipe(c2p)) return 1;
  const pid_t pid = fork();
  const bool parent = pid != 0;
  CK(cudaSetDevice(0));
  unsigned* mine;  // [0] = ping counter written by the other process
  CK(cudaMalloc(&mine, 256));
  CK(cudaMemset(mine, 0, 256));
  int* to;
  CK(cudaMallocManaged(&to, 4));
  *to = 0;
  cudaIpcMemHandle_t h, ph;
  CK(cudaIpcGetMemHandle(&h, mine));
  if (parent) {
    if (write(p2c[1], &h, sizeof h) != sizeof h || read(c2p[0], &ph, sizeof ph) != sizeof ph) return 1;
  } else {
    if (read(p2c[0], &ph, sizeof ph) != sizeof ph || write(c2p[1], &h, sizeof h) != sizeof h) return 1;
  }
  void* peer;
  CK(cudaIpcOpenMemHandle(&peer, ph, cudaIpcMemLazyEnablePeerAccess));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaDeviceSynchronize());
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 1; i <= iters; ++i) {
    if (parent) {
      k_write<<<1, 32, 0, s>>>(static_cast<unsigned*>(peer), i);
      k_wait<<<1, 32, 0, s>>>(mine, i, to);
    } else {
      k_wait<<<1, 32, 0, s>>>(mine, i, to);
      k_write<<<1, 32, 0, s>>>(static_cast<unsigned*>(peer), i);
    }
  }
  CK(cudaStreamSynchronize(s));
  const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
  std::printf("%s: %d round trips, %.1f us each, timeout=%d\n", parent ? "parent" : "child", iters, us / iters, *to);
  if (parent) waitpid(pid, nullptr, 0);
  return 0;
}
