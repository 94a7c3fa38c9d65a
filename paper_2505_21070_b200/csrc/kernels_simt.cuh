// Launchers of the SIMT (fp64 parity / fp32 verification) kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bp {

enum { kEpiNone = 0, kEpiGelu = 1, kEpiResidual = 2 };

template <typename T>
struct AttnArgs {
  const T* q; int64_t ldq;
  const T* k0; int64_t ldk0; const T* v0; int64_t ldv0; int64_t n0;  // prefix segment
  const T* k1; int64_t ldk1; const T* v1; int64_t ldv1; int64_t n1;  // current segment
  T* out; int64_t ldo;
  int dh;
  T scale;
};

template <typename TO>
void launch_embed(const double* lat, const double* w_in, const double* freq, const int32_t* levels,
                  const int64_t* frame_ids, int64_t tokens, int C, int h, int tpf, TO* x,
                  cudaStream_t st);
template <typename T>
void launch_ln(const T* x, const T* g, const T* b, int64_t rows, int n, T* y, cudaStream_t st);
void launch_layer_norm(const double* x, int64_t rows, int n, double eps, double* y, cudaStream_t st);
void launch_softmax_rows(const double* x, int64_t rows, int64_t n, double* y, cudaStream_t st);
template <typename T>
void launch_matmul(const T* A, int64_t lda, const T* B, int64_t ldb, int M, int N, int K, T* C,
                   int64_t ldc, int epi, const T* R, int64_t ldr, cudaStream_t st);
template <typename TO>
void launch_place(const double* src, int64_t rows, int64_t cols, TO* dst, int64_t ld, int transpose,
                  cudaStream_t st);
template <typename T>
void launch_attention(const AttnArgs<T>& a, int64_t rows, int heads, cudaStream_t st);

void launch_copy_rows(const void* src, int64_t src_ld_bytes, void* dst, int64_t dst_ld_bytes,
                      int64_t rows, int64_t row_bytes, cudaStream_t st);
void launch_first_diff(const void* a, int64_t lda_bytes, const void* b, int64_t ldb_bytes,
                       int64_t rows, int64_t row_bytes, unsigned long long* first, cudaStream_t st);
template <typename TI, typename TO>
void launch_convert(const TI* in, TO* out, int64_t n, cudaStream_t st);
void launch_bump_ulp(void* p, int kind, cudaStream_t st);

}  // namespace bp
