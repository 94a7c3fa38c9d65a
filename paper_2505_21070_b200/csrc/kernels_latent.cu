// K1 rng_normal_fill, K2 gather_block_noise, payload assembly and K9
// scheduler_step: the fp64 latent-side kernels. All are HBM/latency-bound
// integer or elementwise work (coalesced, grid-stride, 148-SM multiples).
#include <cuda_runtime.h>

#include "device.cuh"
#include "glibc_port.h"

namespace bp {

// RandomSource(state).normal_tensor({n}, sigma) (rng.cpp:24-39): normal k
// consumes raw draws 2k+1 and 2k+2 of the splitmix64 stream, so every thread
// derives its own counter: state + (2k+1)*phi. Bit-exact with glibc (see
// glibc_port.h). Writes fp64 and optionally a converted copy.
__global__ void k_normal_fill(uint64_t state, int64_t n, double sigma, double* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n; k += stride) {
    const uint64_t s1 = state + static_cast<uint64_t>(2 * k + 1) * kGoldenDev;
    const uint64_t a = bp_splitmix_mix(s1);
    const uint64_t b = bp_splitmix_mix(s1 + kGoldenDev);
    out[k] = bp_box_muller(a, b, sigma);
  }
}

void launch_normal_fill(uint64_t state, int64_t n, double sigma, double* out, cudaStream_t st) {
  if (n <= 0) return;
  const int threads = 256;
  const int64_t want = (n + threads - 1) / threads;
  const int blocks = static_cast<int>(want < kNumSms * 16 ? want : kNumSms * 16);
  k_normal_fill<<<blocks, threads, 0, st>>>(state, n, sigma, out);
  count_launch();
}

// build_pool's collision check (noise.cpp:41-47): flags[i*M+j] = 1 if entry
// i and entry j differ anywhere.
__global__ void k_pool_differs(const double* __restrict__ pool, int m, int64_t per,
                               int* __restrict__ differs) {
  const int i = blockIdx.y, j = blockIdx.z;
  if (j <= i) return;
  const unsigned long long* a = reinterpret_cast<const unsigned long long*>(pool + i * per);
  const unsigned long long* b = reinterpret_cast<const unsigned long long*>(pool + j * per);
  int local = 0;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < per;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    local |= a[k] != b[k];
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(&differs[i * m + j], 1);
}

void launch_pool_differs(const double* pool, int m, int64_t per, int* differs, cudaStream_t st) {
  dim3 grid(8, m, m);
  k_pool_differs<<<grid, 256, 0, st>>>(pool, m, per, differs);
  count_launch();
}

// Gathers rows of fp64 latents: dst[r] = src_rows[r] where row r of the
// destination comes from segment s (r in [seg_start[s], seg_start[s+1])),
// source pointer seg_src[s] + (r - seg_start[s]) * cols. Covers stack_entries
// (noise.cpp:12-22), vcat of explicit context + center (engine.cpp:373-383),
// take_rows and slice_rows. Vectorised 16-byte copies.
__global__ void k_gather_rows(GatherSegs segs, int64_t cols, double* __restrict__ dst) {
  const int64_t total = segs.start[segs.n] * cols;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t r = e / cols, c = e - r * cols;
    int s = 0;
    while (r >= segs.start[s + 1]) ++s;
    dst[e] = segs.src[s][(r - segs.start[s]) * cols + c];
  }
}

void launch_gather_rows(const GatherSegs& segs, int64_t cols, double* dst, cudaStream_t st) {
  const int64_t total = segs.start[segs.n] * cols;
  if (total <= 0) return;
  const int threads = 256;
  const int64_t want = (total + threads - 1) / threads;
  const int blocks = static_cast<int>(want < kNumSms * 8 ? want : kNumSms * 8);
  k_gather_rows<<<blocks, threads, 0, st>>>(segs, cols, dst);
  count_launch();
}

// stack_entries (noise.cpp:12-22) for an arbitrary id list: out[i] = pool[ids[i]].
__global__ void k_gather_ids(const double* __restrict__ pool, int64_t per, const int32_t* __restrict__ ids, int n,
                             double* __restrict__ out) {
  const int64_t total = static_cast<int64_t>(n) * per;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t i = e / per;
    out[e] = pool[static_cast<int64_t>(ids[i]) * per + (e - i * per)];
  }
}

void launch_gather_ids(const double* pool, int64_t per, const int32_t* ids, int n, double* out, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(n) * per;
  if (total <= 0) return;
  const int64_t want = (total + 255) / 256;
  k_gather_ids<<<static_cast<int>(want < kNumSms * 8 ? want : kNumSms * 8), 256, 0, st>>>(pool, per, ids, n, out);
  count_launch();
}

// add / sub / scale (tensor.cpp:148-172): one IEEE operation per element, as
// the reference (out = a; out op= b), so results are bitwise the reference's.
__global__ void k_elementwise(int op, const double* __restrict__ a, const double* __restrict__ b, int64_t n, double s,
                              double* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = op == 0 ? __dadd_rn(a[i], b[i]) : op == 1 ? __dsub_rn(a[i], b[i]) : op == 3 ? __dadd_rn(a[i], s)
                                                                        : __dmul_rn(a[i], s);
}

void launch_elementwise(int op, const double* a, const double* b, int64_t n, double s, double* out, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t want = (n + 255) / 256;
  k_elementwise<<<static_cast<int>(want < kNumSms * 8 ? want : kNumSms * 8), 256, 0, st>>>(op, a, b, n, s, out);
  count_launch();
}

// scheduler_step (model.cpp:338-345): x - eps * (1/steps), exactly the
// reference's two roundings (scale, then sub). eps is the center rows of the
// last stage's output, converted to fp64.
template <typename TE>
__global__ void k_scheduler_step(const double* __restrict__ x, const TE* __restrict__ eps,
                                 int64_t n, double inv_steps, double* __restrict__ out) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __dsub_rn(x[i], __dmul_rn(static_cast<double>(eps[i]), inv_steps));
}

template <typename TE>
void launch_scheduler_step(const double* x, const TE* eps, int64_t n, int steps, double* out,
                           cudaStream_t st) {
  if (n <= 0) return;
  const int threads = 256;
  const int64_t want = (n + threads - 1) / threads;
  const int blocks = static_cast<int>(want < kNumSms * 8 ? want : kNumSms * 8);
  k_scheduler_step<TE><<<blocks, threads, 0, st>>>(x, eps, n, 1.0 / static_cast<double>(steps), out);
  count_launch();
}
template void launch_scheduler_step<double>(const double*, const double*, int64_t, int, double*, cudaStream_t);
template void launch_scheduler_step<float>(const double*, const float*, int64_t, int, double*, cudaStream_t);

}  // namespace bp
