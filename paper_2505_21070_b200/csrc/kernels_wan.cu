// Wan-block bandwidth kernels (see kernels_wan.cuh). Everything here is
// row-parallel and memory-bound except the tiny per-frame timestep MLP, which
// runs as three small SIMT GEMMs (launch_matmul) plus bias / SiLU passes.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "device.cuh"
#include "kernels_wan.cuh"
#include "tc_common.cuh"

namespace bp {

namespace {

template <typename T> __device__ __forceinline__ double to_d(T v) { return static_cast<double>(v); }

template <typename T>
__global__ void k_wan_sinus(const int32_t* __restrict__ levels, int nframes, T* __restrict__ out) {
  const int f = blockIdx.x, k = threadIdx.x;  // 128 threads
  if (f >= nframes) return;
  const double t = static_cast<double>(levels[f]);
  const double w = pow(10000.0, -static_cast<double>(k) / (kWanFreqDim / 2));
  double s, c;
  sincos(t * w, &s, &c);
  out[static_cast<int64_t>(f) * kWanFreqDim + k] = static_cast<T>(c);
  out[static_cast<int64_t>(f) * kWanFreqDim + kWanFreqDim / 2 + k] = static_cast<T>(s);
}

template <typename T>
__device__ __forceinline__ T silu_t(T v) {
  return v / (T(1) + exp(-v));
}

template <typename T>
__global__ void k_bias_act(T* __restrict__ y, int64_t rows, int n, const T* __restrict__ bias, int act,
                           T* __restrict__ y_silu) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * n) return;
  T v = y[i] + bias[i % n];
  if (act == 1) v = silu_t(v);
  y[i] = v;
  if (y_silu) y_silu[i] = silu_t(v);
}

template <typename T>
__global__ void k_wan_modt(const T* __restrict__ mod, int64_t mod_stride, int nl, const T* __restrict__ e,
                           int64_t e_stride, int nframes, int h, int chunks, bool bcast, T* __restrict__ out) {
  const int64_t per = static_cast<int64_t>(chunks) * h;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<int64_t>(nl) * nframes * per) return;
  const int64_t kc = i % per;
  const int64_t f = (i / per) % nframes;
  const int64_t l = i / (per * nframes);
  const int k = static_cast<int>(kc / h);
  const int64_t c = kc % h;
  const bool scale = chunks == 6 ? (k == 1 || k == 4) : k == 1;
  T v = mod[l * mod_stride + kc] + e[f * e_stride + (bcast ? c : kc)];
  if (scale) v += T(1);
  out[i] = v;
}

// One block (128 threads) per row: two-pass mean / variance in fp64, like the
// reference's layer_norm (tensor.cpp:128-146) but with a per-group affine.
template <typename T>
__global__ void __launch_bounds__(128) k_ln_mod(const T* __restrict__ x, int64_t ldx, const T* __restrict__ g,
                                               const T* __restrict__ b, int grp_rows, int64_t grp_stride,
                                               int n, double eps, T* __restrict__ y, int64_t ldy) {
  __shared__ double red[4];
  const int64_t r = blockIdx.x;
  const T* xr = x + r * ldx;
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += 128) s += to_d(xr[j]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  const double mean = (red[0] + red[1] + red[2] + red[3]) / n;
  __syncthreads();
  double q = 0.0;
  for (int j = threadIdx.x; j < n; j += 128) {
    const double d = to_d(xr[j]) - mean;
    q += d * d;
  }
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = q;
  __syncthreads();
  const double inv = 1.0 / sqrt((red[0] + red[1] + red[2] + red[3]) / n + eps);
  const int64_t go = grp_stride ? (r / grp_rows) * grp_stride : 0;
  for (int j = threadIdx.x; j < n; j += 128)
    y[r * ldy + j] = static_cast<T>((to_d(xr[j]) - mean) * inv * to_d(g[go + j]) + to_d(b[go + j]));
}

__device__ __forceinline__ void wan_pair_angle_pos(int j, int nt, int nh, int64_t fid, int yy, int xx, double* pos,
                                                   double* w) {
  if (j < nt) {
    *pos = static_cast<double>(fid);
    *w = pow(10000.0, -static_cast<double>(j) / nt);
  } else if (j < nt + nh) {
    *pos = yy;
    *w = pow(10000.0, -static_cast<double>(j - nt) / nh);
  } else {
    *pos = xx;
    *w = pow(10000.0, -static_cast<double>(j - nt - nh) / nh);
  }
}

template <typename T>
__global__ void __launch_bounds__(128) k_wan_qk(T* __restrict__ base, int64_t ld, int h, int dh,
                                               const T* __restrict__ g, int nparts, int64_t part_stride,
                                               const int64_t* __restrict__ frame_ids, int tpf, int width, int rope) {
  __shared__ double red[4];
  const int64_t r = blockIdx.x;
  int nt, nh;
  wan_rope_split(dh, &nt, &nh);
  const int tok = static_cast<int>(r % tpf);
  const int yy = tok / width, xx = tok % width;
  const int64_t fid = rope ? frame_ids[r / tpf] : 0;
  for (int p = 0; p < nparts; ++p) {
    T* v = base + r * ld + p * part_stride;
    const T* gp = g + static_cast<int64_t>(p) * h;
    double s = 0.0;
    for (int j = threadIdx.x; j < h; j += 128) {
      const double a = to_d(v[j]);
      s += a * a;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    const double inv = 1.0 / sqrt((red[0] + red[1] + red[2] + red[3]) / h + kWanEps);
    __syncthreads();
    for (int i = threadIdx.x; i < h / 2; i += 128) {
      double a = to_d(v[2 * i]) * inv * to_d(gp[2 * i]);
      double b = to_d(v[2 * i + 1]) * inv * to_d(gp[2 * i + 1]);
      if (rope) {
        double pos, w, sn, cs;
        wan_pair_angle_pos(i % (dh / 2), nt, nh, fid, yy, xx, &pos, &w);
        sincos(pos * w, &sn, &cs);
        const double a2 = a * cs - b * sn;
        b = a * sn + b * cs;
        a = a2;
      }
      v[2 * i] = static_cast<T>(a);
      v[2 * i + 1] = static_cast<T>(b);
    }
  }
}

// bf16: one warp per (row, part), 8 bf16 (16 bytes) per lane access; the row
// is read twice (sum of squares, then normalise + rotate), the second time
// from L1.
__global__ void __launch_bounds__(256) k_wan_qk_bf16(bf16* __restrict__ base, int64_t ld, int64_t rows, int h,
                                                    int dh, const float* __restrict__ g, int nparts,
                                                    int64_t part_stride, const float2* __restrict__ ttab,
                                                    const float2* __restrict__ ytab, const float2* __restrict__ xtab,
                                                    int tpf, int width, int rope) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (wid >= rows * nparts) return;
  const int64_t r = wid / nparts;
  const int p = static_cast<int>(wid % nparts);
  uint4* v = reinterpret_cast<uint4*>(base + r * ld + p * part_stride);
  const float* gp = g + static_cast<int64_t>(p) * h;
  const int nv = h / 8;
  float s = 0.f;
  for (int c = lane; c < nv; c += 32) {
    const uint4 u = v[c];
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(b2[q]);
      s = fmaf(f.x, f.x, fmaf(f.y, f.y, s));
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = rsqrtf(s / static_cast<float>(h) + static_cast<float>(kWanEps));
  int nt, nh;
  wan_rope_split(dh, &nt, &nh);
  const int tok = static_cast<int>(r % tpf);
  const int yy = tok / width, xx = tok % width;
  const float2* tt = ttab + (r / tpf) * nt;
  const float2* yt = ytab + static_cast<int64_t>(yy) * nh;
  const float2* xt = xtab + static_cast<int64_t>(xx) * nh;
  for (int c = lane; c < nv; c += 32) {
    uint4 u = v[c];
    __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&u);
    const float4 g0 = *reinterpret_cast<const float4*>(gp + 8 * c);
    const float4 g1 = *reinterpret_cast<const float4*>(gp + 8 * c + 4);
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(b2[q]);
      float a = f.x * inv * gg[2 * q], b = f.y * inv * gg[2 * q + 1];
      if (rope) {
        const int j = ((8 * c + 2 * q) % dh) >> 1;
        const float2 cs = j < nt ? tt[j] : (j < nt + nh ? yt[j - nt] : xt[j - nt - nh]);
        const float a2 = a * cs.x - b * cs.y;
        b = a * cs.y + b * cs.x;
        a = a2;
      }
      b2[q] = __floats2bfloat162_rn(a, b);
    }
    v[c] = u;
  }
}

// Register-resident version for h % 256 == 0 and 32 % (dh / 8) == 0 (NV =
// h / 256 16-byte chunks per lane): one global read of the row; lane l's
// chunks l + 32 i all sit at the same offset inside their heads (32 is a
// multiple of the dh / 8 chunks per head), so its four rotary pairs' (cos,
// sin) are looked up once per row. Launched as a programmatic dependent of
// the QKV / cross-Q GEMM.
template <int NV>
__global__ void __launch_bounds__(256, (NV > 8 ? 1 : 3)) k_wan_qk_bf16_reg(bf16* __restrict__ base, int64_t ld, int64_t rows, int h,
                                                        int dh, const float* __restrict__ g, int nparts,
                                                        int64_t part_stride, const float2* __restrict__ ttab,
                                                        const float2* __restrict__ ytab,
                                                        const float2* __restrict__ xtab, int tpf, int width,
                                                        int rope) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t wid = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (wid >= rows * nparts) return;
  const int64_t r = wid / nparts;
  const int p = static_cast<int>(wid % nparts);
  uint4* v = reinterpret_cast<uint4*>(base + r * ld + p * part_stride);
  const float* gp = g + static_cast<int64_t>(p) * h;
  uint4 u[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) u[i] = v[lane + 32 * i];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u[i]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(b2[q]);
      s = fmaf(f.x, f.x, fmaf(f.y, f.y, s));
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv = rsqrtf(s / static_cast<float>(h) + static_cast<float>(kWanEps));
  float2 cs[4] = {make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f)};
  if (rope) {
    int nt, nh;
    wan_rope_split(dh, &nt, &nh);
    const int tok = static_cast<int>(r % tpf);
    const int yy = tok / width, xx = tok % width;
    const int j0 = (lane % (dh >> 3)) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      cs[q] = j < nt ? ttab[(r / tpf) * nt + j]
                     : (j < nt + nh ? ytab[static_cast<int64_t>(yy) * nh + j - nt]
                                    : xtab[static_cast<int64_t>(xx) * nh + j - nt - nh]);
    }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&u[i]);
    const float4 g0 = *reinterpret_cast<const float4*>(gp + 8 * c);
    const float4 g1 = *reinterpret_cast<const float4*>(gp + 8 * c + 4);
    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 f = __bfloat1622float2(b2[q]);
      const float a = f.x * inv * gg[2 * q], b = f.y * inv * gg[2 * q + 1];
      b2[q] = __floats2bfloat162_rn(a * cs[q].x - b * cs[q].y, a * cs[q].y + b * cs[q].x);
    }
    v[c] = u[i];
  }
}

// Both parts of a row (q and k, adjacent in the QKV buffer: part_stride ==
// h) in one warp: twice the bytes in flight per warp, two independent
// sum-of-squares chains, and the rotary (cos, sin) looked up once for both,
// since q and k of a row share the token's position.
template <int NV>
__global__ void __launch_bounds__(256, 2) k_wan_qk2_bf16_reg(bf16* __restrict__ base, int64_t ld, int64_t rows, int h,
                                                           int dh, const float* __restrict__ g,
                                                           const float2* __restrict__ ttab,
                                                           const float2* __restrict__ ytab,
                                                           const float2* __restrict__ xtab, int tpf, int width,
                                                           int rope) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  uint4* v = reinterpret_cast<uint4*>(base + r * ld);  // q chunks [0, h / 8), k chunks [h / 8, h / 4)
  const int hc = h >> 3;
  uint4 u[2][NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    u[0][i] = v[lane + 32 * i];
    u[1][i] = v[hc + lane + 32 * i];
  }
  float s[2] = {0.f, 0.f};
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&u[p][i]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(b2[q]);
        s[p] = fmaf(f.x, f.x, fmaf(f.y, f.y, s[p]));
      }
    }
  for (int o = 16; o > 0; o >>= 1) {
    s[0] += __shfl_xor_sync(0xffffffffu, s[0], o);
    s[1] += __shfl_xor_sync(0xffffffffu, s[1], o);
  }
  float2 cs[4] = {make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f)};
  if (rope) {
    int nt, nh;
    wan_rope_split(dh, &nt, &nh);
    const int tok = static_cast<int>(r % tpf);
    const int yy = tok / width, xx = tok % width;
    const int j0 = (lane % (dh >> 3)) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      cs[q] = j < nt ? ttab[(r / tpf) * nt + j]
                     : (j < nt + nh ? ytab[static_cast<int64_t>(yy) * nh + j - nt]
                                    : xtab[static_cast<int64_t>(xx) * nh + j - nt - nh]);
    }
  }
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const float inv = rsqrtf(s[p] / static_cast<float>(h) + static_cast<float>(kWanEps));
    const float* gp = g + static_cast<int64_t>(p) * h;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + 32 * i;
      __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&u[p][i]);
      const float4 g0 = *reinterpret_cast<const float4*>(gp + 8 * c);
      const float4 g1 = *reinterpret_cast<const float4*>(gp + 8 * c + 4);
      const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(b2[q]);
        const float a = f.x * inv * gg[2 * q], b = f.y * inv * gg[2 * q + 1];
        b2[q] = __floats2bfloat162_rn(a * cs[q].x - b * cs[q].y, a * cs[q].y + b * cs[q].x);
      }
      v[p * hc + c] = u[p][i];
    }
  }
}

__global__ void k_wan_rope_frames(const int64_t* __restrict__ frame_ids, int nframes, int nt, float2* __restrict__ ttab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nframes * nt) return;
  const int f = i / nt, j = i % nt;
  double s, c;
  sincos(static_cast<double>(frame_ids[f]) * pow(10000.0, -static_cast<double>(j) / nt), &s, &c);
  ttab[i] = make_float2(static_cast<float>(c), static_cast<float>(s));
}

template <typename T>
__global__ void k_gate_residual(T* __restrict__ x, const T* __restrict__ y, const T* __restrict__ gate, int grp_rows,
                                int64_t grp_stride, int64_t rows, int n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * n) return;
  const int64_t r = i / n, c = i % n;
  x[i] += gate[(r / grp_rows) * grp_stride + c] * y[i];
}

template <typename T>
__global__ void k_gelu_tanh(T* __restrict__ y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T v = y[i];
  const T k0 = T(0.7978845608028654);  // sqrt(2 / pi)
  y[i] = T(0.5) * v * (T(1) + tanh(k0 * (v + T(0.044715) * v * v * v)));
}

unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

template <typename T>
void launch_wan_sinus(const int32_t* levels, int nframes, T* out, cudaStream_t st) {
  if (nframes <= 0) return;
  k_wan_sinus<T><<<nframes, kWanFreqDim / 2, 0, st>>>(levels, nframes, out);
  count_launch();
}

template <typename T>
void launch_bias_act(T* y, int64_t rows, int n, const T* bias, int act, T* y_silu, cudaStream_t st) {
  if (rows * n <= 0) return;
  k_bias_act<T><<<blocks_for(rows * n, 256), 256, 0, st>>>(y, rows, n, bias, act, y_silu);
  count_launch();
}

template <typename T>
void launch_wan_modt(const T* mod, int64_t mod_stride, int nl, const T* e, int64_t e_stride, int nframes, int h,
                     int chunks, bool bcast, T* out, cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(nl) * nframes * chunks * h;
  if (n <= 0) return;
  k_wan_modt<T><<<blocks_for(n, 256), 256, 0, st>>>(mod, mod_stride, nl, e, e_stride, nframes, h, chunks, bcast, out);
  count_launch();
}

template <typename T>
void launch_ln_mod(const T* x, int64_t ldx, const T* g, const T* b, int grp_rows, int64_t grp_stride, int64_t rows,
                   int n, double eps, T* y, int64_t ldy, cudaStream_t st) {
  if (rows <= 0) return;
  k_ln_mod<T><<<static_cast<unsigned>(rows), 128, 0, st>>>(x, ldx, g, b, grp_rows, grp_stride, n, eps, y, ldy);
  count_launch();
}

template <typename T>
void launch_wan_qk(T* base, int64_t ld, int64_t rows, int h, int heads, const T* g, int nparts, int64_t part_stride,
                   const int64_t* frame_ids, int tpf, int width, int rope, cudaStream_t st) {
  if (rows <= 0) return;
  k_wan_qk<T><<<static_cast<unsigned>(rows), 128, 0, st>>>(base, ld, h, h / heads, g, nparts, part_stride, frame_ids,
                                                           tpf, width, rope);
  count_launch();
}

void launch_wan_qk_bf16(bf16* base, int64_t ld, int64_t rows, int h, int heads, const float* g, int nparts,
                        int64_t part_stride, const float2* ttab, const float2* ytab, const float2* xtab, int tpf,
                        int width, int rope, cudaStream_t st) {
  if (rows <= 0) return;
  if (h % 8 != 0 || ld % 8 != 0 || part_stride % 8 != 0) fail(BP_ERR_CONFIG, "wan qk kernel needs 16-byte rows");
  const int dh = h / heads;
  const unsigned blocks = blocks_for(rows * nparts, 8);
  auto reg = [&](auto kern) {
    launch_pdl(kern, dim3(blocks), dim3(256), 0, st, base, ld, rows, h, dh, g, nparts, part_stride, ttab, ytab, xtab,
               tpf, width, rope);
  };
  const bool lanes_fit = dh % 8 == 0 && 32 % (dh / 8) == 0;
  if (lanes_fit && nparts == 2 && part_stride == h && (h == 1536 || h == 256 || h == 512)) {
    auto reg2 = [&](auto kern) {
      launch_pdl(kern, dim3(blocks_for(rows, 8)), dim3(256), 0, st, base, ld, rows, h, dh, g, ttab, ytab, xtab, tpf,
                 width, rope);
    };
    if (h == 1536) reg2(k_wan_qk2_bf16_reg<6>);
    else if (h == 512) reg2(k_wan_qk2_bf16_reg<2>);
    else reg2(k_wan_qk2_bf16_reg<1>);
    count_launch();
    return;
  }
  switch (lanes_fit ? h : 0) {  // register-resident rows for the widths in use (Wan 1.3B / 14B, test models)
    case 256: reg(k_wan_qk_bf16_reg<1>); break;
    case 512: reg(k_wan_qk_bf16_reg<2>); break;
    case 1536: reg(k_wan_qk_bf16_reg<6>); break;
    case 5120: reg(k_wan_qk_bf16_reg<20>); break;
    default:
      k_wan_qk_bf16<<<blocks, 256, 0, st>>>(base, ld, rows, h, dh, g, nparts, part_stride, ttab, ytab, xtab, tpf,
                                            width, rope);
  }
  count_launch();
}

void launch_wan_rope_frames(const int64_t* frame_ids, int nframes, int nt, float2* ttab, cudaStream_t st) {
  if (nframes * nt <= 0) return;
  k_wan_rope_frames<<<blocks_for(static_cast<int64_t>(nframes) * nt, 128), 128, 0, st>>>(frame_ids, nframes, nt, ttab);
  count_launch();
}

template <typename T>
void launch_gate_residual(T* x, const T* y, const T* gate, int grp_rows, int64_t grp_stride, int64_t rows, int n,
                          cudaStream_t st) {
  if (rows * n <= 0) return;
  k_gate_residual<T><<<blocks_for(rows * n, 256), 256, 0, st>>>(x, y, gate, grp_rows, grp_stride, rows, n);
  count_launch();
}

template <typename T>
void launch_gelu_tanh(T* y, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_gelu_tanh<T><<<blocks_for(n, 256), 256, 0, st>>>(y, n);
  count_launch();
}

#define BP_WAN_INST(T)                                                                                              \
  template void launch_wan_sinus<T>(const int32_t*, int, T*, cudaStream_t);                                        \
  template void launch_bias_act<T>(T*, int64_t, int, const T*, int, T*, cudaStream_t);                             \
  template void launch_wan_modt<T>(const T*, int64_t, int, const T*, int64_t, int, int, int, bool, T*, cudaStream_t); \
  template void launch_ln_mod<T>(const T*, int64_t, const T*, const T*, int, int64_t, int64_t, int, double, T*,     \
                                 int64_t, cudaStream_t);                                                           \
  template void launch_wan_qk<T>(T*, int64_t, int64_t, int, int, const T*, int, int64_t, const int64_t*, int, int, \
                                 int, cudaStream_t);                                                               \
  template void launch_gate_residual<T>(T*, const T*, const T*, int, int64_t, int64_t, int, cudaStream_t);         \
  template void launch_gelu_tanh<T>(T*, int64_t, cudaStream_t);
BP_WAN_INST(double)
BP_WAN_INST(float)
#undef BP_WAN_INST

}  // namespace bp
