// bf16 tensor-core path: LayerNorm (fp32 residual -> bf16 operand), GEMMs
// with fused epilogues (tcgen05), attention over two KV segments.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace bp {

using bf16 = __nv_bfloat16;

// ln_affine (model.cpp:32-41): fp32 x [rows, n] -> bf16 y, fp32 stats.
// Embedding into the fp32 residual stream (bf16 path): per-stage table of
// (sin, cos)(t * f_k), t < tpf (ttab: tpf * h/2 double2), then per pass the
// per-frame terms (ftab: frames * h/2 double4) and x = pe + te + lat @ w_in.
void launch_embed_table(const double* freq, int h, int tpf, double* ttab, cudaStream_t st);
void launch_embed_fast(const double* lat, const float* w_in32, const double* freq, const double* ttab,
                       double* ftab, const int32_t* levels, const int64_t* frame_ids, int64_t tokens, int C, int h,
                       int tpf, float* lat32, float* x, cudaStream_t st);
// fp32 C[M,N] (+)= A[M,K] B[K,N] for the path's fp32 side GEMMs (embedding,
// head); falls back to the generic SIMT GEMM for shapes the tile kernel skips.
void launch_gemm_f32_tile(const float* A, int64_t lda, const float* B, int64_t ldb, int M, int N, int K, float* C,
                          int64_t ldc, bool residual, cudaStream_t st);
void launch_ln_bf16(const float* x, int64_t ldx, const float* g, const float* b, int64_t rows,
                    int n, bf16* y, cudaStream_t st);
// Same with a per-group affine (row r uses g/b + (r / grp_rows) * grp_stride;
// grp_stride 0: one vector) and a given epsilon: the Wan block's modulated
// LayerNorm (gain 1 + scale, bias shift per frame).
void launch_ln_bf16_grp(const float* x, int64_t ldx, const float* g, const float* b, int grp_rows,
                        int64_t grp_stride, float eps, int64_t rows, int n, bf16* y, cudaStream_t st);

enum GemmEpi {
  kGemmStoreBf16 = 0,    // C bf16 = acc
  kGemmGeluBf16 = 1,     // C bf16 = gelu_erf(acc)           (ffn_sublayer, model.cpp:221-225)
  kGemmResidualF32 = 2,  // C fp32 = C + acc (x += sublayer)  (forward_chunk, model.cpp:325-331)
  kGemmStoreF32 = 3,     // C fp32 = acc
  kGemmResidualGatedF32 = 4,  // C fp32 = C + gate[row group] * acc (Wan gated residual)
  kGemmGeluTanhBf16 = 5,      // C bf16 = gelu_tanh(acc)           (Wan FFN)
  kGemmResidualOutF32 = 6     // C fp32 = R + acc, R = gate.resid: the residual add written to
                              // another buffer (the next rank's receive slot, fused send)
};
// Per-row-group gate of kGemmResidualGatedF32: row r scales by
// gate + (r / grp_rows) * grp_stride (one fp32 vector of N per group).
// kGemmResidualOutF32 reads the residual from resid (row stride ldr).
struct GemmGate {
  const float* gate = nullptr;
  int grp_rows = 1;
  int64_t grp_stride = 0;
  const float* resid = nullptr;
  int64_t ldr = 0;
};
// C[M,N] = A[M,K] (bf16, row stride lda) x W[N,K]^T (bf16, K-major weights).
void launch_gemm_bf16(const bf16* A, int64_t lda, const bf16* W, int M, int N, int K, void* C,
                      int64_t ldc, int epi, cudaStream_t st, const GemmGate& gate = GemmGate{});
// Which GEMM implementation launch_gemm_bf16 uses: 1 = tcgen05 (default), 0 = SIMT check path.
void set_gemm_impl(int impl);
// SMs the persistent GEMM grids leave free (0 by default): the NCCL executor
// reserves a few for NCCL's send/recv kernels, which cannot co-reside with a
// ~200 KB-smem GEMM CTA -- a receive kernel parked on an SM would otherwise
// hold back one cluster's whole tile stream until its data arrives.
void set_sm_reserve(int sms);
int sm_reserve();
int gemm_impl();

struct AttnBf16Args {
  const bf16* q; int64_t ldq;
  const bf16* k0; int64_t ldk0; const bf16* v0; int64_t ldv0; int64_t n0;  // cached prefix
  const bf16* k1; int64_t ldk1; const bf16* v1; int64_t ldv1; int64_t n1;  // current block
  bf16* out; int64_t ldo;
  int heads, dh;
  float scale;
};
// Non-causal multi-head attention (model.cpp:47-72) of q rows against
// [prefix ++ current] keys; softmax in fp32.
void launch_attn_bf16(const AttnBf16Args& a, int64_t rows, cudaStream_t st);
// The cross-attention call (short key range; see kernels_bf16.cu).
void launch_attn_bf16_cross(const AttnBf16Args& a, int64_t rows, cudaStream_t st);
void set_attn_impl(int impl);
int attn_impl();

}  // namespace bp
