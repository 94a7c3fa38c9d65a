// Bandwidth kernels of the optional Wan2.1-style block (bp_block WAN; not a
// reference path, see DESIGN.md section 10 and oracle/wan_oracle.py): the
// per-frame timestep MLP, adaLN modulation tables, modulated LayerNorm,
// RMS-normalised Q/K with 3D RoPE, gated residual adds and tanh-GELU.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "kernels_bf16.cuh"

namespace bp {

constexpr int kWanFreqDim = 256;   // sinusoid width of the timestep embedding
constexpr double kWanEps = 1e-6;   // LayerNorm / RMSNorm epsilon of the Wan block

// RoPE split of a head dim dh into temporal / height / width pairs.
__host__ __device__ inline void wan_rope_split(int dh, int* nt, int* nh) {
  *nh = dh / 6;
  *nt = dh / 2 - 2 * *nh;
}

// [cos(t w_k), sin(t w_k)], w_k = 10000^(-k/128), t = levels[f]: out [nframes][256].
template <typename T>
void launch_wan_sinus(const int32_t* levels, int nframes, T* out, cudaStream_t st);
// y[r, c] = act(y[r, c] + bias[c]); act 0 = identity, 1 = SiLU. y_act (optional)
// receives SiLU(result) when act == 0 (the time MLP needs e and SiLU(e)).
template <typename T>
void launch_bias_act(T* y, int64_t rows, int n, const T* bias, int act, T* y_silu, cudaStream_t st);
// out[l][f][k h + c] = mod[l * mod_stride + k h + c] + e[f * e_stride + (bcast ? 0 : k) h + c],
// plus 1 on the scale chunks (k = 1, 4 of a 6-chunk table; k = 1 of a 2-chunk
// one), so the LayerNorm kernels apply (1 + scale) as their gain.
template <typename T>
void launch_wan_modt(const T* mod, int64_t mod_stride, int nl, const T* e, int64_t e_stride, int nframes, int h,
                     int chunks, bool bcast, T* out, cudaStream_t st);
// y = LN(x) * g[grp] + b[grp], grp = row / grp_rows, g/b advancing by
// grp_stride elements per group (0: one vector for all rows).
template <typename T>
void launch_ln_mod(const T* x, int64_t ldx, const T* g, const T* b, int grp_rows, int64_t grp_stride, int64_t rows,
                   int n, double eps, T* y, int64_t ldy, cudaStream_t st);
// In place, for parts p < nparts at column offset p * part_stride of each row:
// v = RMS(v) * g[p h ..], then (rope) 3D RoPE per head with the positions
// (frame_ids[row / tpf], (row % tpf) / width, row % width). fp64 angles.
template <typename T>
void launch_wan_qk(T* base, int64_t ld, int64_t rows, int h, int heads, const T* g, int nparts, int64_t part_stride,
                   const int64_t* frame_ids, int tpf, int width, int rope, cudaStream_t st);
// bf16 version: warp per (row, part), fp32 statistics, (cos, sin) tables:
// ttab [frames][nt] (per pass), ytab [height][nh], xtab [width][nh] (per stage).
void launch_wan_qk_bf16(bf16* base, int64_t ld, int64_t rows, int h, int heads, const float* g, int nparts,
                        int64_t part_stride, const float2* ttab, const float2* ytab, const float2* xtab, int tpf,
                        int width, int rope, cudaStream_t st);
// ttab[f][j] = (cos, sin)(frame_ids[f] * 10000^(-j / nt)) computed in fp64.
void launch_wan_rope_frames(const int64_t* frame_ids, int nframes, int nt, float2* ttab, cudaStream_t st);
// x[r, c] += gate[grp][c] * y[r, c]
template <typename T>
void launch_gate_residual(T* x, const T* y, const T* gate, int grp_rows, int64_t grp_stride, int64_t rows, int n,
                          cudaStream_t st);
template <typename T>
void launch_gelu_tanh(T* y, int64_t n, cudaStream_t st);

}  // namespace bp
