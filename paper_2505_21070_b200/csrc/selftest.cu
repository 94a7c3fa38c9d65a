// Kernel-level self-test and micro-benchmark hooks (include/bp_cuda_test.h).
#include <cuda_runtime.h>

#include <vector>

#include "bp_cuda_test.h"
#include "device.cuh"
#include "kernels_bf16.cuh"
#include "kernels_wan.cuh"

namespace bp {
__global__ void k_fill_rand_bf16(bf16* p, int64_t n, uint64_t seed, float scale) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t z = seed + static_cast<uint64_t>(i) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    const float u = static_cast<float>(z >> 40) * (1.0f / 16777216.0f) - 0.5f;
    p[i] = __float2bfloat16_rn(u * scale);
  }
}
}  // namespace bp

extern "C" {

bp_status bp_set_kernel_impl(int32_t gemm_impl, int32_t attn_impl) {
  return bp::guarded([&] {
    bp::set_gemm_impl(gemm_impl);
    bp::set_attn_impl(attn_impl);
  });
}

bp_status bp_selftest_gemm(int32_t device, int32_t M, int32_t N, int32_t K, int32_t epi, const uint16_t* A,
                           int64_t lda, const uint16_t* W, void* C, int64_t ldc) {
  return bp::guarded([&] {
    BP_CUDA(cudaSetDevice(device));
    if (epi == bp::kGemmResidualGatedF32) bp::fail(BP_ERR_CONFIG, "gated epilogue: use bp_selftest_gemm_gated");
    const size_t cb = (epi == bp::kGemmStoreBf16 || epi == bp::kGemmGeluBf16 || epi == bp::kGemmGeluTanhBf16) ? 2 : 4;
    bp::DevBuf da, dw, dc;
    da.alloc(static_cast<size_t>(M) * lda * 2);
    dw.alloc(static_cast<size_t>(N) * K * 2);
    dc.alloc(static_cast<size_t>(M) * ldc * cb);
    BP_CUDA(cudaMemcpy(da.p, A, static_cast<size_t>(M) * lda * 2, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(dw.p, W, static_cast<size_t>(N) * K * 2, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(dc.p, C, static_cast<size_t>(M) * ldc * cb, cudaMemcpyHostToDevice));
    if (epi == bp::kGemmResidualOutF32) {  // C (in) is the residual, C (out) = C + acc from another buffer
      bp::DevBuf dout;
      dout.alloc(static_cast<size_t>(M) * ldc * 4);
      BP_CUDA(cudaMemset(dout.p, 0xff, static_cast<size_t>(M) * ldc * 4));
      bp::GemmGate g{};
      g.resid = dc.as<float>();
      g.ldr = ldc;
      bp::launch_gemm_bf16(da.as<bp::bf16>(), lda, dw.as<bp::bf16>(), M, N, K, dout.p, ldc, epi, nullptr, g);
      BP_CUDA(cudaDeviceSynchronize());
      BP_CUDA(cudaMemcpy(C, dout.p, static_cast<size_t>(M) * ldc * 4, cudaMemcpyDeviceToHost));
      return;
    }
    bp::launch_gemm_bf16(da.as<bp::bf16>(), lda, dw.as<bp::bf16>(), M, N, K, dc.p, ldc, epi, nullptr);
    BP_CUDA(cudaDeviceSynchronize());
    BP_CUDA(cudaMemcpy(C, dc.p, static_cast<size_t>(M) * ldc * cb, cudaMemcpyDeviceToHost));
  });
}

bp_status bp_selftest_gemm_gated(int32_t device, int32_t M, int32_t N, int32_t K, const uint16_t* A, int64_t lda,
                                 const uint16_t* W, float* C, int64_t ldc, const float* gate, int32_t grp_rows,
                                 int32_t ngroups) {
  return bp::guarded([&] {
    BP_CUDA(cudaSetDevice(device));
    bp::DevBuf da, dw, dc, dg;
    da.alloc(static_cast<size_t>(M) * lda * 2);
    dw.alloc(static_cast<size_t>(N) * K * 2);
    dc.alloc(static_cast<size_t>(M) * ldc * 4);
    dg.alloc(static_cast<size_t>(ngroups) * N * 4);
    BP_CUDA(cudaMemcpy(da.p, A, static_cast<size_t>(M) * lda * 2, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(dw.p, W, static_cast<size_t>(N) * K * 2, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(dc.p, C, static_cast<size_t>(M) * ldc * 4, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(dg.p, gate, static_cast<size_t>(ngroups) * N * 4, cudaMemcpyHostToDevice));
    bp::launch_gemm_bf16(da.as<bp::bf16>(), lda, dw.as<bp::bf16>(), M, N, K, dc.p, ldc, bp::kGemmResidualGatedF32,
                         nullptr, bp::GemmGate{dg.as<float>(), grp_rows, N});
    BP_CUDA(cudaDeviceSynchronize());
    BP_CUDA(cudaMemcpy(C, dc.p, static_cast<size_t>(M) * ldc * 4, cudaMemcpyDeviceToHost));
  });
}

namespace {
bp_status selftest_attn(bool cross, int32_t device, int64_t rows, int32_t heads, int32_t dh, const uint16_t* q,
                        const uint16_t* k0, const uint16_t* v0, int64_t n0, const uint16_t* k1,
                        const uint16_t* v1, int64_t n1, float scale, uint16_t* out) {
  return bp::guarded([&] {
    BP_CUDA(cudaSetDevice(device));
    const int64_t H = static_cast<int64_t>(heads) * dh;
    bp::DevBuf dq, dk0, dv0, dk1, dv1, dout;
    auto up = [&](bp::DevBuf& b, const uint16_t* h, int64_t n) {
      b.alloc(static_cast<size_t>(n) * H * 2 + 16);
      if (n > 0) BP_CUDA(cudaMemcpy(b.p, h, static_cast<size_t>(n) * H * 2, cudaMemcpyHostToDevice));
    };
    up(dq, q, rows);
    up(dk0, k0, n0);
    up(dv0, v0, n0);
    up(dk1, k1, n1);
    up(dv1, v1, n1);
    dout.alloc(static_cast<size_t>(rows) * H * 2);
    bp::AttnBf16Args a{};
    a.q = dq.as<bp::bf16>(); a.ldq = H;
    a.k0 = dk0.as<bp::bf16>(); a.ldk0 = H; a.v0 = dv0.as<bp::bf16>(); a.ldv0 = H; a.n0 = n0;
    a.k1 = dk1.as<bp::bf16>(); a.ldk1 = H; a.v1 = dv1.as<bp::bf16>(); a.ldv1 = H; a.n1 = n1;
    a.out = dout.as<bp::bf16>(); a.ldo = H;
    a.heads = heads; a.dh = dh; a.scale = scale;
    if (cross) bp::launch_attn_bf16_cross(a, rows, nullptr);
    else bp::launch_attn_bf16(a, rows, nullptr);
    BP_CUDA(cudaDeviceSynchronize());
    BP_CUDA(cudaMemcpy(out, dout.p, static_cast<size_t>(rows) * H * 2, cudaMemcpyDeviceToHost));
  });
}
}  // namespace

bp_status bp_selftest_attn(int32_t device, int64_t rows, int32_t heads, int32_t dh, const uint16_t* q,
                           const uint16_t* k0, const uint16_t* v0, int64_t n0, const uint16_t* k1,
                           const uint16_t* v1, int64_t n1, float scale, uint16_t* out) {
  return selftest_attn(false, device, rows, heads, dh, q, k0, v0, n0, k1, v1, n1, scale, out);
}

bp_status bp_selftest_attn_cross(int32_t device, int64_t rows, int32_t heads, int32_t dh, const uint16_t* q,
                                 const uint16_t* k1, const uint16_t* v1, int64_t n1, float scale, uint16_t* out) {
  return selftest_attn(true, device, rows, heads, dh, q, nullptr, nullptr, 0, k1, v1, n1, scale, out);
}

bp_status bp_bench_gemm(int32_t device, int32_t M, int32_t N, int32_t K, int32_t epi, int32_t iters, double* ms) {
  return bp::guarded([&] {
    BP_CUDA(cudaSetDevice(device));
    if (epi == bp::kGemmResidualGatedF32) bp::fail(BP_ERR_CONFIG, "gated epilogue: use bp_selftest_gemm_gated");
    const size_t cb = (epi == bp::kGemmStoreBf16 || epi == bp::kGemmGeluBf16 || epi == bp::kGemmGeluTanhBf16) ? 2 : 4;
    bp::DevBuf da, dw, dc;
    da.alloc(static_cast<size_t>(M) * K * 2);
    dw.alloc(static_cast<size_t>(N) * K * 2);
    dc.alloc(static_cast<size_t>(M) * N * cb);
    bp::k_fill_rand_bf16<<<1024, 256>>>(da.as<bp::bf16>(), static_cast<int64_t>(M) * K, 1, 1.0f);
    bp::k_fill_rand_bf16<<<1024, 256>>>(dw.as<bp::bf16>(), static_cast<int64_t>(N) * K, 2, 0.05f);
    BP_CUDA(cudaMemset(dc.p, 0, static_cast<size_t>(M) * N * cb));
    bp::DevBuf dr;  // kGemmResidualOutF32: the residual input (the output goes to dc)
    bp::GemmGate g{};
    if (epi == bp::kGemmResidualOutF32) {
      dr.alloc(static_cast<size_t>(M) * N * 4);
      BP_CUDA(cudaMemset(dr.p, 0, static_cast<size_t>(M) * N * 4));
      g.resid = dr.as<float>();
      g.ldr = N;
    }
    cudaStream_t st;
    BP_CUDA(cudaStreamCreate(&st));
    for (int i = 0; i < 3; ++i) bp::launch_gemm_bf16(da.as<bp::bf16>(), K, dw.as<bp::bf16>(), M, N, K, dc.p, N, epi, st, g);
    cudaEvent_t e0, e1;
    BP_CUDA(cudaEventCreate(&e0));
    BP_CUDA(cudaEventCreate(&e1));
    BP_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) bp::launch_gemm_bf16(da.as<bp::bf16>(), K, dw.as<bp::bf16>(), M, N, K, dc.p, N, epi, st, g);
    BP_CUDA(cudaEventRecord(e1, st));
    BP_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    BP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

bp_status bp_bench_attn(int32_t device, int64_t rows, int32_t heads, int32_t dh, int64_t n0, int64_t n1,
                        int32_t iters, double* ms) {
  return bp::guarded([&] {
    BP_CUDA(cudaSetDevice(device));
    const int64_t H = static_cast<int64_t>(heads) * dh;
    // q/k/v interleaved like the QKV GEMM output [rows, 3H]; prefix [n0, 2H]
    bp::DevBuf qkv, pre, out;
    qkv.alloc(static_cast<size_t>(std::max(rows, n1)) * 3 * H * 2);
    pre.alloc(static_cast<size_t>(n0 + 1) * 2 * H * 2);
    out.alloc(static_cast<size_t>(rows) * H * 2);
    bp::k_fill_rand_bf16<<<1024, 256>>>(qkv.as<bp::bf16>(), std::max(rows, n1) * 3 * H, 3, 2.0f);
    bp::k_fill_rand_bf16<<<1024, 256>>>(pre.as<bp::bf16>(), (n0 + 1) * 2 * H, 4, 2.0f);
    bp::AttnBf16Args a{};
    a.q = qkv.as<bp::bf16>(); a.ldq = 3 * H;
    a.k0 = pre.as<bp::bf16>(); a.ldk0 = 2 * H; a.v0 = pre.as<bp::bf16>() + H; a.ldv0 = 2 * H; a.n0 = n0;
    a.k1 = qkv.as<bp::bf16>() + H; a.ldk1 = 3 * H; a.v1 = qkv.as<bp::bf16>() + 2 * H; a.ldv1 = 3 * H; a.n1 = n1;
    a.out = out.as<bp::bf16>(); a.ldo = H;
    a.heads = heads; a.dh = dh; a.scale = 1.0f / sqrtf(static_cast<float>(dh));
    cudaStream_t st;
    BP_CUDA(cudaStreamCreate(&st));
    for (int i = 0; i < 2; ++i) bp::launch_attn_bf16(a, rows, st);
    cudaEvent_t e0, e1;
    BP_CUDA(cudaEventCreate(&e0));
    BP_CUDA(cudaEventCreate(&e1));
    BP_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) bp::launch_attn_bf16(a, rows, st);
    BP_CUDA(cudaEventRecord(e1, st));
    BP_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    BP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

}  // extern "C"

bp_status bp_bench_ln(int32_t device, int64_t rows, int32_t n, int32_t iters, double* ms) {
  return bp::guarded([&] {
    BP_CUDA(cudaSetDevice(device));
    bp::DevBuf x, g, y;
    x.alloc(static_cast<size_t>(rows) * n * 4);
    g.alloc(static_cast<size_t>(2 * n) * 4);
    y.alloc(static_cast<size_t>(rows) * n * 2);
    BP_CUDA(cudaMemset(x.p, 0x3f, static_cast<size_t>(rows) * n * 4));
    BP_CUDA(cudaMemset(g.p, 0x3f, static_cast<size_t>(2 * n) * 4));
    cudaStream_t st;
    BP_CUDA(cudaStreamCreate(&st));
    const float* gp = g.as<float>();
    for (int i = 0; i < 3; ++i) bp::launch_ln_bf16(x.as<float>(), n, gp, gp + n, rows, n, y.as<bp::bf16>(), st);
    cudaEvent_t e0, e1;
    BP_CUDA(cudaEventCreate(&e0));
    BP_CUDA(cudaEventCreate(&e1));
    BP_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) bp::launch_ln_bf16(x.as<float>(), n, gp, gp + n, rows, n, y.as<bp::bf16>(), st);
    BP_CUDA(cudaEventRecord(e1, st));
    BP_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    BP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}

bp_status bp_bench_wan_qk(int32_t device, int64_t rows, int32_t h, int32_t heads, int32_t height, int32_t width,
                          int32_t iters, double* ms) {
  return bp::guarded([&] {
    BP_CUDA(cudaSetDevice(device));
    int nt, nh;
    bp::wan_rope_split(h / heads, &nt, &nh);
    const int tpf = height * width;
    const int nf = static_cast<int>((rows + tpf - 1) / tpf);
    bp::DevBuf qkv, g, tt, yt, xt;
    qkv.alloc(static_cast<size_t>(rows) * 3 * h * 2);
    g.alloc(static_cast<size_t>(2 * h) * 4);
    tt.alloc(static_cast<size_t>(nf) * nt * 8 + 8);
    yt.alloc(static_cast<size_t>(height) * nh * 8 + 8);
    xt.alloc(static_cast<size_t>(width) * nh * 8 + 8);
    bp::k_fill_rand_bf16<<<1024, 256>>>(qkv.as<bp::bf16>(), rows * 3 * h, 5, 2.0f);
    BP_CUDA(cudaMemset(g.p, 0x3f, static_cast<size_t>(2 * h) * 4));
    BP_CUDA(cudaMemset(tt.p, 0, tt.bytes));
    BP_CUDA(cudaMemset(yt.p, 0, yt.bytes));
    BP_CUDA(cudaMemset(xt.p, 0, xt.bytes));
    cudaStream_t st;
    BP_CUDA(cudaStreamCreate(&st));
    auto go = [&] {
      bp::launch_wan_qk_bf16(qkv.as<bp::bf16>(), 3 * h, rows, h, heads, g.as<float>(), 2, h, tt.as<float2>(),
                             yt.as<float2>(), xt.as<float2>(), tpf, width, 1, st);
    };
    for (int i = 0; i < 3; ++i) go();
    cudaEvent_t e0, e1;
    BP_CUDA(cudaEventCreate(&e0));
    BP_CUDA(cudaEventCreate(&e1));
    BP_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; ++i) go();
    BP_CUDA(cudaEventRecord(e1, st));
    BP_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    BP_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = t / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(st);
  });
}
