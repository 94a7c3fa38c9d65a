/* bp_cuda_test.h — kernel-level self-test hooks of libbp_cuda.so, used by the
 * parity tests to exercise one device kernel in isolation (not part of the
 * reference-facing API). */
#ifndef BP_CUDA_TEST_H_
#define BP_CUDA_TEST_H_

#include <stdint.h>

#include "bp_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Selects the bf16 GEMM / attention implementation: 1 = tcgen05 (default),
 * 0 = SIMT check kernels. Applies to subsequent launches in this process. */
BP_API bp_status bp_set_kernel_impl(int32_t gemm_impl, int32_t attn_impl);

/* C[M,N] (+)= A[M,K] . W[N,K]^T on the device, host buffers. A, W are bf16
 * bit patterns; C is bf16 (epi 0/1/5) or fp32 (epi 2/3), row stride ldc. */
BP_API bp_status bp_selftest_gemm(int32_t device, int32_t M, int32_t N, int32_t K, int32_t epi,
                           const uint16_t* A, int64_t lda, const uint16_t* W, void* C, int64_t ldc);

/* C[M,N] += gate[r / grp_rows][:] * (A . W^T) (fp32 C, the Wan gated residual
 * epilogue); gate holds ngroups fp32 rows of N. */
BP_API bp_status bp_selftest_gemm_gated(int32_t device, int32_t M, int32_t N, int32_t K, const uint16_t* A, int64_t lda,
                                 const uint16_t* W, float* C, int64_t ldc, const float* gate, int32_t grp_rows,
                                 int32_t ngroups);

/* Attention of q rows against [k0/v0 (n0 rows) ++ k1/v1 (n1 rows)], bf16 bit
 * patterns, all with row stride heads*dh; out bf16 [rows, heads*dh]. */
BP_API bp_status bp_selftest_attn(int32_t device, int64_t rows, int32_t heads, int32_t dh, const uint16_t* q,
                           const uint16_t* k0, const uint16_t* v0, int64_t n0, const uint16_t* k1,
                           const uint16_t* v1, int64_t n1, float scale, uint16_t* out);

/* The same through the stage's cross-attention launcher (one key segment). */
BP_API bp_status bp_selftest_attn_cross(int32_t device, int64_t rows, int32_t heads, int32_t dh, const uint16_t* q,
                                 const uint16_t* k1, const uint16_t* v1, int64_t n1, float scale, uint16_t* out);

/* Device time (ms, CUDA events on the launching stream) of `iters` back-to-back
 * launches of the current GEMM implementation on device-resident random data. */
BP_API bp_status bp_bench_gemm(int32_t device, int32_t M, int32_t N, int32_t K, int32_t epi, int32_t iters,
                        double* ms);
BP_API bp_status bp_bench_attn(int32_t device, int64_t rows, int32_t heads, int32_t dh, int64_t n0, int64_t n1,
                        int32_t iters, double* ms);

/* Device time (ms per launch) of `iters` back-to-back LayerNorm launches
 * (fp32 [rows, n] -> bf16, the bf16 path's k_ln_bf16_reg). */
BP_API bp_status bp_bench_ln(int32_t device, int64_t rows, int32_t n, int32_t iters, double* ms);

/* Device time (ms per launch) of the Wan block's bf16 Q/K RMSNorm + 3D RoPE
 * kernel over a [rows, 3h] QKV buffer (q and k parts, in place). */
BP_API bp_status bp_bench_wan_qk(int32_t device, int64_t rows, int32_t h, int32_t heads, int32_t height,
                                 int32_t width, int32_t iters, double* ms);

#ifdef __cplusplus
}
#endif
#endif
