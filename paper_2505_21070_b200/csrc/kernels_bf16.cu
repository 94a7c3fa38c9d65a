// bf16 path: LayerNorm into the GEMM operand, and the SIMT "check" versions
// of the GEMM / attention (set_*_impl(0)) used to cross-validate the tcgen05
// kernels on the device. The production GEMM/attention live in
// gemm_sm100.cu / attn_sm100.cu.
#include <cuda_bf16.h>

#include <cstdlib>
#include <cuda_runtime.h>

#include "device.cuh"
#include "kernels_bf16.cuh"

namespace bp {

// ---- LayerNorm: one warp per row, fp32 two-pass statistics ------------------------
__global__ void __launch_bounds__(256) k_ln_bf16(const float* __restrict__ x, int64_t ldx,
                                                 const float* __restrict__ g,
                                                 const float* __restrict__ b, int64_t rows, int n,
                                                 bf16* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float* xr = x + r * ldx;
  const int n4 = n >> 2;  // n % 4 == 0 on this path
  const float4* x4 = reinterpret_cast<const float4*>(xr);
  float s = 0.f;
  for (int j = lane; j < n4; j += 32) {
    const float4 v = x4[j];
    s += (v.x + v.y) + (v.z + v.w);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / static_cast<float>(n);
  float q = 0.f;
  for (int j = lane; j < n4; j += 32) {
    const float4 v = x4[j];
    const float a = v.x - mean, bb = v.y - mean, c = v.z - mean, d = v.w - mean;
    q += (a * a + bb * bb) + (c * c + d * d);
  }
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float inv = 1.0f / sqrtf(q / static_cast<float>(n) + 1e-5f);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  __nv_bfloat162* y2 = reinterpret_cast<__nv_bfloat162*>(y + r * n);
  for (int j = lane; j < n4; j += 32) {
    const float4 v = x4[j], gg = g4[j], bbv = b4[j];
    const float o0 = (v.x - mean) * inv * gg.x + bbv.x;
    const float o1 = (v.y - mean) * inv * gg.y + bbv.y;
    const float o2 = (v.z - mean) * inv * gg.z + bbv.z;
    const float o3 = (v.w - mean) * inv * gg.w + bbv.w;
    y2[2 * j] = __floats2bfloat162_rn(o0, o1);
    y2[2 * j + 1] = __floats2bfloat162_rn(o2, o3);
  }
}

void launch_ln_bf16(const float* x, int64_t ldx, const float* g, const float* b, int64_t rows,
                    int n, bf16* y, cudaStream_t st) {
  if (rows <= 0) return;
  if (n % 4 != 0 || ldx % 4 != 0) fail(BP_ERR_CONFIG, "bf16 path needs hidden % 4 == 0");
  const int64_t blocks = (rows + 7) / 8;
  k_ln_bf16<<<static_cast<unsigned>(blocks), 256, 0, st>>>(x, ldx, g, b, rows, n, y);
  count_launch();
}

__device__ __forceinline__ float gelu_erf(float v) {
  return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f));
}

// ---- SIMT check GEMM: C = A . W^T, fp32 accumulate, k ascending --------------------
__global__ void __launch_bounds__(256) k_gemm_simt(const bf16* __restrict__ A, int64_t lda,
                                                   const bf16* __restrict__ W, int M, int N, int K,
                                                   void* __restrict__ Cv, int64_t ldc, int epi) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 1];
  __shared__ float Ws[BK][BN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      const int mm = e / BK, kk = e % BK, gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? __bfloat162float(A[static_cast<int64_t>(gm) * lda + gk]) : 0.f;
      const int gn = n0 + mm;
      Ws[kk][mm] = (gn < N && gk < K) ? __bfloat162float(W[static_cast<int64_t>(gn) * K + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[kk][ty * 4 + i], Ws[kk][tx * 4 + j], acc[i][j]);
    __syncthreads();
  }
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      const int64_t o = static_cast<int64_t>(gm) * ldc + gn;
      const float v = acc[i][j];
      if (epi == kGemmStoreBf16) static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(v);
      else if (epi == kGemmGeluBf16) static_cast<bf16*>(Cv)[o] = __float2bfloat16_rn(gelu_erf(v));
      else if (epi == kGemmResidualF32) static_cast<float*>(Cv)[o] += v;
      else static_cast<float*>(Cv)[o] = v;
    }
  }
}

void launch_gemm_simt(const bf16* A, int64_t lda, const bf16* W, int M, int N, int K, void* C,
                      int64_t ldc, int epi, cudaStream_t st) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  k_gemm_simt<<<grid, 256, 0, st>>>(A, lda, W, M, N, K, C, ldc, epi);
  count_launch();
}

// ---- SIMT check attention: one block per (row, head), online softmax in fp32 ------------
__global__ void __launch_bounds__(128) k_attn_simt(AttnBf16Args a) {
  __shared__ float qs[256];
  __shared__ float ps[128];
  __shared__ float red[4];
  const int64_t i = blockIdx.x;
  const int c0 = blockIdx.y * a.dh;
  for (int t = threadIdx.x; t < a.dh; t += 128) qs[t] = __bfloat162float(a.q[i * a.ldq + c0 + t]);
  __syncthreads();
  const int64_t nkv = a.n0 + a.n1;
  float m_run = -INFINITY, l_run = 0.f, acc0 = 0.f, acc1 = 0.f;
  for (int64_t j0 = 0; j0 < nkv; j0 += 128) {
    const int64_t j = j0 + threadIdx.x;
    float s = -INFINITY;
    if (j < nkv) {
      const bf16* kr = j < a.n0 ? a.k0 + j * a.ldk0 + c0 : a.k1 + (j - a.n0) * a.ldk1 + c0;
      float acc = 0.f;
      for (int t = 0; t < a.dh; ++t) acc = fmaf(qs[t], __bfloat162float(kr[t]), acc);
      s = acc * a.scale;
    }
    float mx = s;
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
    const float m_new = fmaxf(m_run, mx);
    const float p = (j < nkv) ? __expf(s - m_new) : 0.f;
    ps[threadIdx.x] = p;
    float ls = p;
    for (int o = 16; o > 0; o >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ls;
    __syncthreads();
    ls = (red[0] + red[1]) + (red[2] + red[3]);
    const float corr = __expf(m_run - m_new);
    l_run = l_run * corr + ls;
    acc0 *= corr;
    acc1 *= corr;
    m_run = m_new;
    const int jn = static_cast<int>((nkv - j0) < 128 ? (nkv - j0) : 128);
    for (int jj = 0; jj < jn; ++jj) {
      const int64_t jg = j0 + jj;
      const bf16* vr = jg < a.n0 ? a.v0 + jg * a.ldv0 + c0 : a.v1 + (jg - a.n0) * a.ldv1 + c0;
      const float pj = ps[jj];
      if (threadIdx.x < a.dh) acc0 = fmaf(pj, __bfloat162float(vr[threadIdx.x]), acc0);
      if (threadIdx.x + 128 < a.dh) acc1 = fmaf(pj, __bfloat162float(vr[threadIdx.x + 128]), acc1);
    }
    __syncthreads();
  }
  bf16* orow = a.out + i * a.ldo + c0;
  if (threadIdx.x < a.dh) orow[threadIdx.x] = __float2bfloat16_rn(acc0 / l_run);
  if (threadIdx.x + 128 < a.dh) orow[threadIdx.x + 128] = __float2bfloat16_rn(acc1 / l_run);
}

void launch_attn_simt(const AttnBf16Args& a, int64_t rows, cudaStream_t st) {
  if (a.dh > 256) fail(BP_ERR_CONFIG, "head dim > 256 unsupported");
  dim3 grid(static_cast<unsigned>(rows), a.heads);
  k_attn_simt<<<grid, 128, 0, st>>>(a);
  count_launch();
}

}  // namespace bp

namespace bp {

void launch_gemm_tc(const bf16* A, int64_t lda, const bf16* W, int M, int N, int K, void* C, int64_t ldc,
                    int epi, cudaStream_t st, int variant);
void launch_attn_tc(const AttnBf16Args& a, int64_t rows, cudaStream_t st, int variant);

namespace {
// GEMM: 0 = SIMT check path, 1 = tcgen05 one CTA per tile, 2 = tcgen05 cluster
// pair sharing the weight tile. BP_GEMM_IMPL overrides the default.
int default_gemm_impl() {
  const char* e = std::getenv("BP_GEMM_IMPL");
  return e ? std::atoi(e) : 2;
}
int g_gemm_impl = default_gemm_impl();
// 0 = SIMT check path, 1 = tcgen05 one Q tile/CTA, 2 = tcgen05 ping-pong.
// BP_ATTN_IMPL overrides the default (A/B runs of the whole suite).
int default_attn_impl() {
  const char* e = std::getenv("BP_ATTN_IMPL");
  return e ? std::atoi(e) : 2;
}
int g_attn_impl = default_attn_impl();
}  // namespace

void set_gemm_impl(int impl) { g_gemm_impl = impl; }
int gemm_impl() { return g_gemm_impl; }
void set_attn_impl(int impl) { g_attn_impl = impl; }
int attn_impl() { return g_attn_impl; }

void launch_gemm_bf16(const bf16* A, int64_t lda, const bf16* W, int M, int N, int K, void* C, int64_t ldc,
                      int epi, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  if (g_gemm_impl >= 1) launch_gemm_tc(A, lda, W, M, N, K, C, ldc, epi, st, g_gemm_impl);
  else launch_gemm_simt(A, lda, W, M, N, K, C, ldc, epi, st);
}

void launch_attn_bf16(const AttnBf16Args& a, int64_t rows, cudaStream_t st) {
  if (rows <= 0) return;
  if (g_attn_impl >= 1) launch_attn_tc(a, rows, st, g_attn_impl);
  else launch_attn_simt(a, rows, st);
}

}  // namespace bp
