// SIMT kernels for the fp64 parity mode and the fp32 verification mode.
// fp64 follows the reference's arithmetic order: matmul accumulates k
// ascending with separate multiply/add roundings (tensor.cpp:84-109), the
// LayerNorm is two-pass (tensor.cpp:128-146) followed by *g + b
// (model.cpp:32-41), softmax divides by the sum (tensor.cpp:111-126) and the
// attention output accumulates keys ascending (model.cpp:63-69). nvcc's FMA
// contraction is suppressed with explicit _rn intrinsics. fp32 uses FMA.
#include <cuda_runtime.h>

#include "device.cuh"
#include "kernels_simt.cuh"

namespace bp {

template <typename T> struct Ar;
template <> struct Ar<double> {
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
  static __device__ __forceinline__ double madd(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));
  }
  static __device__ __forceinline__ double ex(double x) { return exp(x); }
  static __device__ __forceinline__ double erf_(double x) { return erf(x); }
  static __device__ __forceinline__ double sqrt_(double x) { return __dsqrt_rn(x); }
};
template <> struct Ar<float> {
  static __device__ __forceinline__ float add(float a, float b) { return a + b; }
  static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
  static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
  static __device__ __forceinline__ float div(float a, float b) { return a / b; }
  static __device__ __forceinline__ float madd(float acc, float a, float b) { return fmaf(a, b, acc); }
  static __device__ __forceinline__ float ex(float x) { return expf(x); }
  static __device__ __forceinline__ float erf_(float x) { return erff(x); }
  static __device__ __forceinline__ float sqrt_(float x) { return sqrtf(x); }
};

template <typename T>
__device__ __forceinline__ T block_reduce(T v, T* red, bool is_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const T other = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? (other > v ? other : v) : Ar<T>::add(v, other);
  }
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  T r = red[0];
  for (int w = 1; w < nw; ++w) r = is_max ? (red[w] > r ? red[w] : r) : Ar<T>::add(r, red[w]);
  return r;
}

// ---- patchify + embeddings (model.cpp:245-260, 155-169) ----------------------
// x[r,j] = (sum_c lat[r,c] w_in[c,j]) + (pe[j] + te[j]) in fp64 for every
// precision (arguments reach ~4e5 rad), then stored as TO.
template <typename TO>
__global__ void k_embed(const double* __restrict__ lat, const double* __restrict__ w_in,
                        const double* __restrict__ freq, const int32_t* __restrict__ levels,
                        const int64_t* __restrict__ frame_ids, int64_t tokens, int C, int h,
                        int tpf, TO* __restrict__ x) {
  const int64_t total = tokens * h;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / h;
    const int j = static_cast<int>(e - r * h);
    double acc = 0.0;
    for (int c = 0; c < C; ++c) acc = __dadd_rn(acc, __dmul_rn(lat[r * C + c], w_in[static_cast<int64_t>(c) * h + j]));
    const int64_t f = r / tpf, t = r - f * tpf;
    const int64_t pos = frame_ids[f] * tpf + t;
    const int64_t tpos = static_cast<int64_t>(levels[f]) + 1000000;
    const double fr = freq[j >> 1];
    const double ap = __dmul_rn(static_cast<double>(pos), fr);
    const double at = __dmul_rn(static_cast<double>(tpos), fr);
    const double pe = (j & 1) ? cos(ap) : sin(ap);
    const double te = (j & 1) ? cos(at) : sin(at);
    x[e] = static_cast<TO>(__dadd_rn(acc, __dadd_rn(pe, te)));
  }
}

template <typename TO>
void launch_embed(const double* lat, const double* w_in, const double* freq, const int32_t* levels,
                  const int64_t* frame_ids, int64_t tokens, int C, int h, int tpf, TO* x,
                  cudaStream_t st) {
  const int64_t total = tokens * h;
  if (total <= 0) return;
  const int64_t want = (total + 255) / 256;
  k_embed<TO><<<static_cast<int>(want < kNumSms * 16 ? want : kNumSms * 16), 256, 0, st>>>(
      lat, w_in, freq, levels, frame_ids, tokens, C, h, tpf, x);
  count_launch();
}
template void launch_embed<double>(const double*, const double*, const double*, const int32_t*,
                                   const int64_t*, int64_t, int, int, int, double*, cudaStream_t);
template void launch_embed<float>(const double*, const double*, const double*, const int32_t*,
                                  const int64_t*, int64_t, int, int, int, float*, cudaStream_t);

// ---- ln_affine (model.cpp:32-41 over tensor.cpp:128-146) ---------------------
template <typename T>
__global__ void k_ln(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b,
                     int64_t rows, int n, T eps, T* __restrict__ y) {
  __shared__ T red[32];
  const int64_t r = blockIdx.x;
  const T* xr = x + r * n;
  T s = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) s = Ar<T>::add(s, xr[j]);
  const T mean = Ar<T>::div(block_reduce<T>(s, red, false), static_cast<T>(n));
  T v = 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const T d = Ar<T>::sub(xr[j], mean);
    v = Ar<T>::madd(v, d, d);
  }
  const T var = Ar<T>::div(block_reduce<T>(v, red, false), static_cast<T>(n));
  const T inv = Ar<T>::div(static_cast<T>(1), Ar<T>::sqrt_(Ar<T>::add(var, eps)));
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const T yn = Ar<T>::mul(Ar<T>::sub(xr[j], mean), inv);
    y[r * n + j] = g ? Ar<T>::add(Ar<T>::mul(yn, g[j]), b[j]) : yn;  // g == nullptr: plain layer_norm
  }
}

template <typename T>
void launch_ln(const T* x, const T* g, const T* b, int64_t rows, int n, T* y, cudaStream_t st) {
  if (rows <= 0) return;
  k_ln<T><<<static_cast<unsigned>(rows), 128, 0, st>>>(x, g, b, rows, n, static_cast<T>(1e-5), y);
  count_launch();
}
template void launch_ln<double>(const double*, const double*, const double*, int64_t, int, double*, cudaStream_t);

// Plain layer_norm(x, eps) (tensor.cpp:128-146): no affine.
void launch_layer_norm(const double* x, int64_t rows, int n, double eps, double* y, cudaStream_t st) {
  if (rows <= 0) return;
  k_ln<double><<<static_cast<unsigned>(rows), 128, 0, st>>>(x, nullptr, nullptr, rows, n, eps, y);
  count_launch();
}

// ---- softmax_rows (tensor.cpp:111-126) -------------------------------------------
// One block per row: row max, then e = exp(x - max) and their sum, then e / sum.
__global__ void k_softmax_rows(const double* __restrict__ x, int64_t n, double* __restrict__ y) {
  __shared__ double red[32];
  const double* xr = x + blockIdx.x * n;
  double* yr = y + blockIdx.x * n;
  double mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) mx = fmax(mx, xr[j]);
  mx = block_reduce<double>(mx, red, true);
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const double e = exp(xr[j] - mx);
    yr[j] = e;
    s += e;
  }
  s = block_reduce<double>(s, red, false);
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) yr[j] = yr[j] / s;
}

void launch_softmax_rows(const double* x, int64_t rows, int64_t n, double* y, cudaStream_t st) {
  if (rows <= 0 || n <= 0) return;
  k_softmax_rows<<<static_cast<unsigned>(rows), 128, 0, st>>>(x, n, y);
  count_launch();
}
template void launch_ln<float>(const float*, const float*, const float*, int64_t, int, float*, cudaStream_t);

// ---- matmul (tensor.cpp:84-109) with fused epilogues ---------------------------
// C[M,N] = A[M,K] (row stride lda) @ B[K,N] (row-major). Each thread owns a
// 4x4 micro-tile and accumulates k in ascending order.
template <typename T, int EPI>
__global__ void __launch_bounds__(256) k_matmul(const T* __restrict__ A, int64_t lda,
                                                const T* __restrict__ B, int64_t ldb, int M, int N, int K,
                                                T* __restrict__ Cm, int64_t ldc,
                                                const T* __restrict__ R, int64_t ldr) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int k0 = 0; k0 < K; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      const int mm = e / BK, kk = e % BK;
      const int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[static_cast<int64_t>(gm) * lda + gk] : T(0);
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      Bs[kk][nn] = (gk < K && gn < N) ? B[static_cast<int64_t>(gk) * ldb + gn] : T(0);
    }
    __syncthreads();
    const int kmax = (K - k0) < BK ? (K - k0) : BK;
    for (int kk = 0; kk < kmax; ++kk) {
      T a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = Ar<T>::madd(acc[i][j], a[i], bb[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      T v = acc[i][j];
      if (EPI == kEpiGelu) {
        // gelu (model.cpp:43): 0.5*x*(1 + erf(x/sqrt(2)))
        const T t = Ar<T>::div(v, static_cast<T>(1.4142135623730951));
        v = Ar<T>::mul(Ar<T>::mul(static_cast<T>(0.5), v), Ar<T>::add(static_cast<T>(1), Ar<T>::erf_(t)));
      } else if (EPI == kEpiResidual) {
        // add(x, y) (tensor.cpp:148-156): x + y
        v = Ar<T>::add(R[static_cast<int64_t>(gm) * ldr + gn], v);
      }
      Cm[static_cast<int64_t>(gm) * ldc + gn] = v;
    }
  }
}

// fp32 tile GEMM (the fp32 verification path at Wan shapes, and the bf16
// path's fp32 side GEMMs): 128 x 64 tile per CTA, 8 x 4 outputs per thread as
// packed FFMA2 pairs, k ascending from zero with one FMA per k -- the same
// per-element sequence as k_matmul<float>, so results do not depend on which
// of the two kernels ran (nor on an output row's position: cached == recompute).
// Needs K % 32 == 0, N % 64 == 0 and 16-byte aligned rows.
template <int EPI>
__global__ void __launch_bounds__(256) k_matmul_f32_tile(const float* __restrict__ A, int64_t lda,
                                                         const float* __restrict__ B, int64_t ldb, int M, int N,
                                                         int K, float* Cm, int64_t ldc, const float* R, int64_t ldr) {
  constexpr int BM = 128, BN = 64, BK = 32;
  __shared__ __align__(16) float As[BK][BM + 4];  // transposed A tile
  __shared__ __align__(16) float Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // cols tx*4.., rows ty*8..
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float2 acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = make_float2(0.f, 0.f);
  for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {  // A: 128 rows x 8 float4
      const int e = tid + v * 256, r = e >> 3, c4 = e & 7;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if (m0 + r < M) a = *reinterpret_cast<const float4*>(A + static_cast<int64_t>(m0 + r) * lda + k0 + c4 * 4);
      As[c4 * 4 + 0][r] = a.x;
      As[c4 * 4 + 1][r] = a.y;
      As[c4 * 4 + 2][r] = a.z;
      As[c4 * 4 + 3][r] = a.w;
    }
#pragma unroll
    for (int v = 0; v < 2; ++v) {  // B: 32 rows x 16 float4
      const int e = tid + v * 256, r = e >> 4, c4 = e & 15;
      *reinterpret_cast<float4*>(&Bs[r][c4 * 4]) =
          *reinterpret_cast<const float4*>(B + static_cast<int64_t>(k0 + r) * ldb + n0 + c4 * 4);
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][ty * 8 + 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float2 b01 = make_float2(b.x, b.y), b23 = make_float2(b.z, b.w);
      const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 aa = make_float2(av[i], av[i]);
        acc[i][0] = __ffma2_rn(aa, b01, acc[i][0]);
        acc[i][1] = __ffma2_rn(aa, b23, acc[i][1]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = m0 + ty * 8 + i;
    if (r >= M) continue;
    float o[4] = {acc[i][0].x, acc[i][0].y, acc[i][1].x, acc[i][1].y};
    if (EPI == kEpiGelu) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        o[j] = Ar<float>::mul(Ar<float>::mul(0.5f, o[j]),
                              Ar<float>::add(1.f, erff(Ar<float>::div(o[j], 1.4142135623730951f))));
    } else if (EPI == kEpiResidual) {
      const float4 c = *reinterpret_cast<const float4*>(R + static_cast<int64_t>(r) * ldr + n0 + tx * 4);
      o[0] = c.x + o[0]; o[1] = c.y + o[1]; o[2] = c.z + o[2]; o[3] = c.w + o[3];
    }
    *reinterpret_cast<float4*>(Cm + static_cast<int64_t>(r) * ldc + n0 + tx * 4) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

template <typename T>
void launch_matmul(const T* A, int64_t lda, const T* B, int64_t ldb, int M, int N, int K, T* C,
                   int64_t ldc, int epi, const T* R, int64_t ldr, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  if constexpr (sizeof(T) == 4) {
    const bool fits = K % 32 == 0 && N % 64 == 0 && K > 0 && lda % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 &&
                      (epi != kEpiResidual || ldr % 4 == 0) &&
                      ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) |
                        reinterpret_cast<uintptr_t>(C) | reinterpret_cast<uintptr_t>(R)) & 15) == 0;
    if (fits) {
      dim3 grid(static_cast<unsigned>(N / 64), static_cast<unsigned>((M + 127) / 128));
      switch (epi) {
        case kEpiNone: k_matmul_f32_tile<kEpiNone><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, C, ldc, R, ldr); break;
        case kEpiGelu: k_matmul_f32_tile<kEpiGelu><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, C, ldc, R, ldr); break;
        default: k_matmul_f32_tile<kEpiResidual><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, C, ldc, R, ldr); break;
      }
      count_launch();
      return;
    }
  }
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  switch (epi) {
    case kEpiNone: k_matmul<T, kEpiNone><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, C, ldc, R, ldr); break;
    case kEpiGelu: k_matmul<T, kEpiGelu><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, C, ldc, R, ldr); break;
    default: k_matmul<T, kEpiResidual><<<grid, 256, 0, st>>>(A, lda, B, ldb, M, N, K, C, ldc, R, ldr); break;
  }
  count_launch();
}
template void launch_matmul<double>(const double*, int64_t, const double*, int64_t, int, int, int, double*, int64_t, int, const double*, int64_t, cudaStream_t);
template void launch_matmul<float>(const float*, int64_t, const float*, int64_t, int, int, int, float*, int64_t, int, const float*, int64_t, cudaStream_t);

// ---- attention (model.cpp:47-72) over two KV segments ---------------------------
// One block per (query row, head). Pass 1: row max of the scaled scores;
// pass 2: sum of exp(s - max); pass 3: p = e / sum, out = sum_j p_j v_j in
// ascending key order (prefix segment first, like vcat_rows(prefix, k)).
template <typename T>
__global__ void __launch_bounds__(128) k_attention(AttnArgs<T> a) {
  extern __shared__ unsigned char smem_raw[];
  T* qs = reinterpret_cast<T*>(smem_raw);  // dh
  T* ps = qs + a.dh;                        // 128
  __shared__ T red[32];
  const int64_t i = blockIdx.x;
  const int hd = blockIdx.y;
  const int c0 = hd * a.dh;
  const T* qrow = a.q + i * a.ldq + c0;
  for (int t = threadIdx.x; t < a.dh; t += blockDim.x) qs[t] = qrow[t];
  __syncthreads();
  const int64_t nkv = a.n0 + a.n1;
  auto krow = [&](int64_t j) -> const T* {
    return j < a.n0 ? a.k0 + j * a.ldk0 + c0 : a.k1 + (j - a.n0) * a.ldk1 + c0;
  };
  auto vrow = [&](int64_t j) -> const T* {
    return j < a.n0 ? a.v0 + j * a.ldv0 + c0 : a.v1 + (j - a.n0) * a.ldv1 + c0;
  };
  auto score = [&](int64_t j) -> T {
    const T* kr = krow(j);
    T acc = 0;
    for (int t = 0; t < a.dh; ++t) acc = Ar<T>::madd(acc, qs[t], kr[t]);
    return Ar<T>::mul(acc, a.scale);
  };
  T mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < nkv; j += blockDim.x) {
    const T s = score(j);
    mx = s > mx ? s : mx;
  }
  mx = block_reduce<T>(mx, red, true);
  T sum = 0;
  for (int64_t j = threadIdx.x; j < nkv; j += blockDim.x) sum = Ar<T>::add(sum, Ar<T>::ex(Ar<T>::sub(score(j), mx)));
  sum = block_reduce<T>(sum, red, false);
  T acc0 = 0, acc1 = 0;  // dims threadIdx.x and threadIdx.x + 128 (dh <= 256)
  for (int64_t j0 = 0; j0 < nkv; j0 += blockDim.x) {
    __syncthreads();
    const int64_t j = j0 + threadIdx.x;
    if (j < nkv) ps[threadIdx.x] = Ar<T>::div(Ar<T>::ex(Ar<T>::sub(score(j), mx)), sum);
    __syncthreads();
    const int jn = static_cast<int>((nkv - j0) < blockDim.x ? (nkv - j0) : blockDim.x);
    for (int jj = 0; jj < jn; ++jj) {
      const T* vr = vrow(j0 + jj);
      const T p = ps[jj];
      if (threadIdx.x < a.dh) acc0 = Ar<T>::madd(acc0, p, vr[threadIdx.x]);
      if (threadIdx.x + 128 < a.dh) acc1 = Ar<T>::madd(acc1, p, vr[threadIdx.x + 128]);
    }
  }
  T* orow = a.out + i * a.ldo + c0;
  if (threadIdx.x < a.dh) orow[threadIdx.x] = acc0;
  if (threadIdx.x + 128 < a.dh) orow[threadIdx.x + 128] = acc1;
}

// fp32 verification attention at Wan shapes: flash-style tiles of 64 query
// rows x 64 keys for one head per CTA, online softmax (running max / sum,
// expf), the two KV segments walked in order. Scores are (q.k) * scale as in
// model.cpp:55-58; the normalisation divides once at the end. S = Q K^T and
// O += P V run from shared memory as 4x4 / 4x(DH/16) register tiles.
template <int DH>
__global__ void __launch_bounds__(256, 2) k_attn_f32_flash(AttnArgs<float> a, int64_t rows) {
  constexpr int BQ = 64, BK = 64, CPT = DH / 16, D4 = DH / 4;
  extern __shared__ __align__(16) float fsm[];
  float* Qt = fsm;             // [DH][BQ]
  float* Kt = Qt + DH * BQ;    // [DH][BK]
  float* Vs = Kt + DH * BK;    // [BK][DH]
  float* Pt = Vs + BK * DH;    // [BK][BQ]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * BQ;
  const int c0 = blockIdx.y * DH;
  for (int e = tid; e < BQ * D4; e += 256) {
    const int r = e % BQ, d4 = e / BQ;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q0 + r < rows) v = *reinterpret_cast<const float4*>(a.q + (q0 + r) * a.ldq + c0 + d4 * 4);
    Qt[(d4 * 4 + 0) * BQ + r] = v.x;
    Qt[(d4 * 4 + 1) * BQ + r] = v.y;
    Qt[(d4 * 4 + 2) * BQ + r] = v.z;
    Qt[(d4 * 4 + 3) * BQ + r] = v.w;
  }
  float m[4], l[4], o[4][CPT];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    m[i] = -INFINITY;
    l[i] = 0.f;
#pragma unroll
    for (int c = 0; c < CPT; ++c) o[i][c] = 0.f;
  }
  const int64_t nkv = a.n0 + a.n1;
  for (int64_t k0 = 0; k0 < nkv; k0 += BK) {
    __syncthreads();  // the previous tile's P.V is done with Vs / Pt
    for (int e = tid; e < BK * D4; e += 256) {  // K transposed: key index fastest (conflict-free stores)
      const int r = e % BK, d4 = e / BK;
      const int64_t j = k0 + r;
      float4 kv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < nkv) {
        const float* kp = j < a.n0 ? a.k0 + j * a.ldk0 : a.k1 + (j - a.n0) * a.ldk1;
        kv = *reinterpret_cast<const float4*>(kp + c0 + d4 * 4);
      }
      Kt[(d4 * 4 + 0) * BK + r] = kv.x;
      Kt[(d4 * 4 + 1) * BK + r] = kv.y;
      Kt[(d4 * 4 + 2) * BK + r] = kv.z;
      Kt[(d4 * 4 + 3) * BK + r] = kv.w;
    }
    for (int e = tid; e < BK * D4; e += 256) {  // V row-major: column fastest (coalesced)
      const int r = e / D4, d4 = e % D4;
      const int64_t j = k0 + r;
      float4 vv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < nkv) {
        const float* vp = j < a.n0 ? a.v0 + j * a.ldv0 : a.v1 + (j - a.n0) * a.ldv1;
        vv = *reinterpret_cast<const float4*>(vp + c0 + d4 * 4);
      }
      *reinterpret_cast<float4*>(Vs + r * DH + d4 * 4) = vv;
    }
    __syncthreads();
    float s[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 4
    for (int d = 0; d < DH; ++d) {
      const float4 qa = *reinterpret_cast<const float4*>(Qt + d * BQ + ty * 4);
      const float4 kb = *reinterpret_cast<const float4*>(Kt + d * BK + tx * 4);
      const float qv[4] = {qa.x, qa.y, qa.z, qa.w}, kw[4] = {kb.x, kb.y, kb.z, kb.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = fmaf(qv[i], kw[j], s[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s[i][j] = (k0 + tx * 4 + j < nkv) ? s[i][j] * a.scale : -INFINITY;
        mx = fmaxf(mx, s[i][j]);
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mn = fmaxf(m[i], mx);
      const float alpha = expf(m[i] - mn);
      float rs = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s[i][j] = expf(s[i][j] - mn);
        rs += s[i][j];
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
      l[i] = l[i] * alpha + rs;
      m[i] = mn;
#pragma unroll
      for (int c = 0; c < CPT; ++c) o[i][c] *= alpha;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      *reinterpret_cast<float4*>(Pt + (tx * 4 + j) * BQ + ty * 4) = make_float4(s[0][j], s[1][j], s[2][j], s[3][j]);
    __syncthreads();
#pragma unroll 2
    for (int k = 0; k < BK; ++k) {
      const float4 pa = *reinterpret_cast<const float4*>(Pt + k * BQ + ty * 4);
      const float pv[4] = {pa.x, pa.y, pa.z, pa.w};
#pragma unroll
      for (int c4 = 0; c4 < CPT / 4; ++c4) {
        const float4 vb = *reinterpret_cast<const float4*>(Vs + k * DH + tx * CPT + c4 * 4);
        const float vv[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < 4; ++c) o[i][c4 * 4 + c] = fmaf(pv[i], vv[c], o[i][c4 * 4 + c]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = q0 + ty * 4 + i;
    if (r >= rows) continue;
    const float inv = 1.f / l[i];
    float* orow = a.out + r * a.ldo + c0 + tx * CPT;
#pragma unroll
    for (int c4 = 0; c4 < CPT / 4; ++c4)
      *reinterpret_cast<float4*>(orow + c4 * 4) =
          make_float4(o[i][c4 * 4] * inv, o[i][c4 * 4 + 1] * inv, o[i][c4 * 4 + 2] * inv, o[i][c4 * 4 + 3] * inv);
  }
}

template <int DH>
void launch_attn_f32_flash(const AttnArgs<float>& a, int64_t rows, int heads, cudaStream_t st) {
  const size_t smem = sizeof(float) * (2 * DH * 64 + 64 * DH + 64 * 64);
  set_smem_attr(k_attn_f32_flash<DH>, static_cast<int>(smem));
  dim3 grid(static_cast<unsigned>((rows + 63) / 64), heads);
  k_attn_f32_flash<DH><<<grid, 256, smem, st>>>(a, rows);
  count_launch();
}

template <typename T>
void launch_attention(const AttnArgs<T>& a, int64_t rows, int heads, cudaStream_t st) {
  if (rows <= 0) return;
  if (a.dh > 256) fail(BP_ERR_CONFIG, "SIMT attention supports head dim <= 256");
  if constexpr (sizeof(T) == 4) {
    const bool aligned = ((a.ldq | a.ldk1 | a.ldv1 | a.ldo | (a.n0 ? (a.ldk0 | a.ldv0) : 0)) & 3) == 0 &&
                         ((reinterpret_cast<uintptr_t>(a.q) | reinterpret_cast<uintptr_t>(a.k1) |
                           reinterpret_cast<uintptr_t>(a.v1) | reinterpret_cast<uintptr_t>(a.out) |
                           (a.n0 ? (reinterpret_cast<uintptr_t>(a.k0) | reinterpret_cast<uintptr_t>(a.v0)) : 0)) & 15) == 0;
    if (aligned && a.n0 + a.n1 > 0 && (a.dh == 128 || a.dh == 64)) {
      if (a.dh == 128) launch_attn_f32_flash<128>(a, rows, heads, st);
      else launch_attn_f32_flash<64>(a, rows, heads, st);
      return;
    }
  }
  dim3 grid(static_cast<unsigned>(rows), heads);
  const size_t smem = sizeof(T) * (a.dh + 128);
  k_attention<T><<<grid, 128, smem, st>>>(a);
  count_launch();
}

template void launch_attention<double>(const AttnArgs<double>&, int64_t, int, cudaStream_t);
template void launch_attention<float>(const AttnArgs<float>&, int64_t, int, cudaStream_t);

// ---- strided row copy / bitwise compare / conversion --------------------------
__global__ void k_copy_rows(const uint32_t* __restrict__ src, int64_t src_ld, uint32_t* __restrict__ dst,
                            int64_t dst_ld, int64_t rows, int64_t words) {
  const int64_t total = rows * words;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / words, c = e - r * words;
    dst[r * dst_ld + c] = src[r * src_ld + c];
  }
}

// 16-byte rows: a warp-strided row walk, one uint4 per thread per step
// (the KV-cache capture moves [P, 2h] bf16 out of the [S, 3h] QKV buffer).
__global__ void k_copy_rows16(const uint4* __restrict__ src, int64_t src_ld, uint4* __restrict__ dst, int64_t dst_ld,
                              int rows, int vecs) {
  for (int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < rows; r += gridDim.x * (blockDim.x / 32)) {
    const uint4* s = src + static_cast<int64_t>(r) * src_ld;
    uint4* d = dst + static_cast<int64_t>(r) * dst_ld;
    for (int c = threadIdx.x & 31; c < vecs; c += 32) d[c] = __ldg(s + c);
  }
}

void launch_copy_rows(const void* src, int64_t src_ld_bytes, void* dst, int64_t dst_ld_bytes,
                      int64_t rows, int64_t row_bytes, cudaStream_t st) {
  if (rows <= 0 || row_bytes <= 0) return;
  if (((row_bytes | src_ld_bytes | dst_ld_bytes | reinterpret_cast<uintptr_t>(src) |
        reinterpret_cast<uintptr_t>(dst)) & 15) == 0 && rows < (1LL << 31)) {
    const int64_t want = (rows + 7) / 8;
    k_copy_rows16<<<static_cast<int>(want < kNumSms * 16 ? want : kNumSms * 16), 256, 0, st>>>(
        static_cast<const uint4*>(src), src_ld_bytes / 16, static_cast<uint4*>(dst), dst_ld_bytes / 16,
        static_cast<int>(rows), static_cast<int>(row_bytes / 16));
    count_launch();
    return;
  }
  if ((row_bytes | src_ld_bytes | dst_ld_bytes) & 3) fail(BP_ERR_INTERNAL, "copy_rows needs 4-byte rows");
  const int64_t words = row_bytes / 4, total = rows * words;
  const int64_t want = (total + 255) / 256;
  k_copy_rows<<<static_cast<int>(want < kNumSms * 8 ? want : kNumSms * 8), 256, 0, st>>>(
      static_cast<const uint32_t*>(src), src_ld_bytes / 4, static_cast<uint32_t*>(dst),
      dst_ld_bytes / 4, rows, words);
  count_launch();
}

// First flat index where a[r*lda + c] and b[r*ldb + c] differ bitwise (words);
// *first is initialised to INT64_MAX by the caller.
__global__ void k_first_diff(const uint32_t* __restrict__ a, int64_t lda, const uint32_t* __restrict__ b,
                             int64_t ldb, int64_t rows, int64_t words, unsigned long long* first) {
  const int64_t total = rows * words;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / words, c = e - r * words;
    if (a[r * lda + c] != b[r * ldb + c]) atomicMin(first, static_cast<unsigned long long>(e));
  }
}

void launch_first_diff(const void* a, int64_t lda_bytes, const void* b, int64_t ldb_bytes,
                       int64_t rows, int64_t row_bytes, unsigned long long* first, cudaStream_t st) {
  if (rows <= 0) return;
  const int64_t words = row_bytes / 4, total = rows * words;
  const int64_t want = (total + 255) / 256;
  k_first_diff<<<static_cast<int>(want < kNumSms * 8 ? want : kNumSms * 8), 256, 0, st>>>(
      static_cast<const uint32_t*>(a), lda_bytes / 4, static_cast<const uint32_t*>(b), ldb_bytes / 4,
      rows, words, first);
  count_launch();
}

template <typename TI, typename TO>
__global__ void k_convert(const TI* __restrict__ in, TO* __restrict__ out, int64_t n) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[e] = static_cast<TO>(in[e]);
}
template <typename TI, typename TO>
void launch_convert(const TI* in, TO* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  const int64_t want = (n + 255) / 256;
  k_convert<TI, TO><<<static_cast<int>(want < kNumSms * 8 ? want : kNumSms * 8), 256, 0, st>>>(in, out, n);
  count_launch();
}
template void launch_convert<double, float>(const double*, float*, int64_t, cudaStream_t);
template void launch_convert<float, double>(const float*, double*, int64_t, cudaStream_t);
template void launch_convert<double, double>(const double*, double*, int64_t, cudaStream_t);

// bumps one double / float / bf16 value by one ulp towards +inf
__global__ void k_bump_ulp(void* p, int kind) {
  if (kind == 0) {
    double* d = static_cast<double*>(p);
    *d = nextafter(*d, INFINITY);
  } else if (kind == 1) {
    float* f = static_cast<float*>(p);
    *f = nextafterf(*f, INFINITY);
  } else {
    uint16_t* u = static_cast<uint16_t*>(p);
    const uint16_t v = *u;
    // bf16 nextafter towards +inf (finite values)
    if ((v & 0x7fff) == 0) *u = 0x0001;
    else if (v & 0x8000) *u = static_cast<uint16_t>(v - 1);
    else *u = static_cast<uint16_t>(v + 1);
  }
}
void launch_bump_ulp(void* p, int kind, cudaStream_t st) {
  k_bump_ulp<<<1, 1, 0, st>>>(p, kind);
  count_launch();
}

}  // namespace bp

namespace bp {
// Places an fp64 [rows, cols] tensor into a destination of type TO with row
// stride ld (optionally transposed: dst[c*ld + r]).
template <typename TO>
__global__ void k_place(const double* __restrict__ src, int64_t rows, int64_t cols, TO* __restrict__ dst,
                        int64_t ld, int transpose) {
  const int64_t total = rows * cols;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / cols, c = e - r * cols;
    const TO v = static_cast<TO>(src[e]);
    if (transpose) dst[c * ld + r] = v; else dst[r * ld + c] = v;
  }
}
template <typename TO>
void launch_place(const double* src, int64_t rows, int64_t cols, TO* dst, int64_t ld, int transpose,
                  cudaStream_t st) {
  const int64_t total = rows * cols;
  if (total <= 0) return;
  const int64_t want = (total + 255) / 256;
  k_place<TO><<<static_cast<int>(want < kNumSms * 16 ? want : kNumSms * 16), 256, 0, st>>>(src, rows, cols, dst, ld, transpose);
  count_launch();
}
template void launch_place<double>(const double*, int64_t, int64_t, double*, int64_t, int, cudaStream_t);
template void launch_place<float>(const double*, int64_t, int64_t, float*, int64_t, int, cudaStream_t);
template void launch_place<__nv_bfloat16>(const double*, int64_t, int64_t, __nv_bfloat16*, int64_t, int, cudaStream_t);
}  // namespace bp
