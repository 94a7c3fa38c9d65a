// tcgen05 GEMM for the DiT projections (K5a-K5f): C[M,N] = A[M,K] . W[N,K]^T
// with bf16 operands, fp32 accumulation in TMEM and fused epilogues (bf16
// store, erf-GELU, fp32 residual add by TMA reduce-add). One kernel,
// k_gemm_pair: persistent 2-CTA clusters issuing one cta_group::2 MMA
// (M = 256 x N = 256) per k-step (see its comment):
//   warp 0      TMA producer (one elected lane) into a 6-stage smem ring
//   warp 1      MMA issuer (leader CTA, one elected lane), TMEM alloc
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> smem -> global
// Two 256-column TMEM accumulators let the epilogue of tile i overlap the
// MMAs of tile i+1. K is consumed in a fixed ascending order and there is no
// split-K, so every output row is computed identically wherever it sits in
// M (the cached == recompute invariant). Losing variants of round
// 1 (one CTA per tile; a multicast pair with two M = 128 MMAs per step) are
// recorded in DESIGN.md and no longer built.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "device.cuh"
#include "kernels_bf16.cuh"
#include "tc_common.cuh"

namespace bp {

namespace {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr uint32_t A_BYTES = BM * BK * 2;
constexpr uint32_t B_BYTES = BN * BK * 2;
constexpr int kThreads = 192;

__device__ __forceinline__ float gelu_erf_f(float v) { return 0.5f * v * (1.0f + erff(v * 0.70710678118654752f)); }

// erf-GELU (ffn_sublayer, model.cpp:221-225) on a pair, for the bf16 epilogue:
// erf by Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7), t = 1/(1 + p|x|/sqrt2)
// and exp(-x^2/2) on MUFU, the rest as packed FFMA2 -- ~9 instructions per
// element instead of erff's ~25, which made the FFN-up epilogue the critical
// path. GELU error <= 2.2e-7 absolute, 20x below the bf16 output's rounding.
__device__ __forceinline__ float2 gelu_erf_f2(float2 v) {
  const float2 half = make_float2(0.5f, 0.5f);
  const float ax = fabsf(v.x), ay = fabsf(v.y);
  const float2 den = __ffma2_rn(make_float2(ax, ay), make_float2(0.23164085f, 0.23164085f), make_float2(1.f, 1.f));
  float2 t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.x) : "f"(den.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.y) : "f"(den.y));
  float2 poly = __ffma2_rn(t, make_float2(1.061405429f, 1.061405429f), make_float2(-1.453152027f, -1.453152027f));
  poly = __ffma2_rn(poly, t, make_float2(1.421413741f, 1.421413741f));
  poly = __ffma2_rn(poly, t, make_float2(-0.284496736f, -0.284496736f));
  poly = __ffma2_rn(poly, t, make_float2(0.254829592f, 0.254829592f));
  poly = __fmul2_rn(poly, t);
  // exp(-x^2/2) = 2^(-x^2 * log2(e)/2)
  const float2 arg = __fmul2_rn(__fmul2_rn(v, v), make_float2(-0.72134752f, -0.72134752f));
  float2 e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(arg.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(arg.y));
  const float2 q = __fmul2_rn(__fmul2_rn(half, v), __fmul2_rn(poly, e));  // 0.5 x (1 - erf(|x|/sqrt2))
  return make_float2(v.x >= 0.f ? v.x - q.x : q.x, v.y >= 0.f ? v.y - q.y : q.y);
}

// tanh-GELU (Wan FFN) on a pair: 0.5 x (1 + tanh(u)) = x / (1 + 2^(-2 u log2 e)),
// u = sqrt(2/pi) (x + 0.044715 x^3); the exponential and the reciprocal on MUFU.
__device__ __forceinline__ float2 gelu_tanh_f2(float2 v) {
  const float2 v2 = __fmul2_rn(v, v);
  const float2 inner = __ffma2_rn(v2, make_float2(0.044715f, 0.044715f), make_float2(1.f, 1.f));
  // -2 sqrt(2/pi) log2(e) = -2.3022082
  const float2 arg = __fmul2_rn(__fmul2_rn(v, inner), make_float2(-2.3022082f, -2.3022082f));
  float2 e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(arg.x));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(arg.y));
  const float2 den = __fadd2_rn(e, make_float2(1.f, 1.f));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.x) : "f"(den.x));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r.y) : "f"(den.y));
  return __fmul2_rn(v, r);
}

// ---- the cta_group::2 cluster pair ----------------------------------------------------
// The two CTAs of a (2,1,1) cluster compute vertically adjacent 128x256 tiles
// (m-blocks 2p, 2p+1) that share one weight tile, as ONE cta_group::2 MMA per
// k-step, M = 256 (each CTA's 128 A rows) x N = 256 (each CTA stages its
// 128-row half of the weight tile): 32 KB per stage and CTA, a 6-stage ring.
// The leader CTA issues every MMA, both CTAs' TMA loads complete on the
// leader's full barriers, every commit is multicast to both CTAs, and each
// CTA's epilogue drains its own 128 accumulator rows and reports to the
// leader's tempty barrier. Row results do not depend on which CTA computes
// them (same K order, no split-K), so cached == recompute holds bitwise.
//
// Epilogue: each 32-row x 32-column chunk goes TMEM -> registers (thread =
// row) -> a 4 KB per-warp smem slab (16-byte units XOR-swizzled by row) ->
// back with threads along columns, so every global load/store covers whole
// 128-byte rows (4 rows fp32, 8 rows bf16) instead of 32 scattered 16-byte
// pieces: the L1 work per tile drops 8x, which is what bounded the K = 1536
// residual GEMMs.
constexpr uint32_t B_HALF = B_BYTES / 2;
struct PairLayout {
  static constexpr int kStages = 6;
  static constexpr uint32_t kStageB = B_HALF;
  static constexpr uint32_t kStaging = (kStages * (A_BYTES + kStageB) + 256 + 1023) & ~1023u;  // after ring + mbarriers
  static constexpr uint32_t kSmem = kStaging + 2 * 4 * 4096 + 1024;  // two 4 KB slabs per epilogue warp
  static_assert(kSmem <= 232448, "pair GEMM exceeds the 227 KB smem limit");
};

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_pair(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_bh, int M, int N,
                int K, void* __restrict__ Cv, int64_t ldc, const __grid_constant__ CUtensorMap map_c,
                const GemmGate gate) {
  using L = PairLayout;
  constexpr int kSt = L::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;
  uint8_t* sb = smem + kSt * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sb + kSt * L::kStageB);
  uint64_t* empty = full + kSt;
  uint64_t* tfull = empty + kSt;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint8_t* staging = smem + L::kStaging;  // 4 epilogue warps x 2 x 4 KB (1024-aligned: TMA swizzle atoms)

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int rank = static_cast<int>(tc::cluster_ctarank());
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int n_tiles = (N + BN - 1) / BN;
  const int m_pairs = ((M + BM - 1) / BM + 1) / 2;
  const int total = n_tiles * m_pairs;
  const int num_k = (K + BK - 1) / BK;
  constexpr uint16_t kBoth = 0x3;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&map_a);
    tc::tma_prefetch(&map_bh);
    for (int s = 0; s < kSt; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast)
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 8);  // one lane per epilogue warp of both CTAs
    }
    tc::fence_mbarrier_init_cluster();
  }
  if (warp == 1) tc::tmem_alloc_cg2<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();  // barrier inits visible to the peer before any remote arrive / multicast
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot;
  tc::pdl_wait();  // A and the residual were produced by the previous kernel

  if (warp == 0) {
    // ---- TMA producer: own A tile + own half of the shared weight tile ----
    int stage = 0;
    uint32_t phase = 0;
    for (int pair = cluster; pair < total; pair += nclusters) {
      const int m_blk = (pair / n_tiles) * 2 + rank, n_blk = pair % n_tiles;
      for (int kb = 0; kb < num_k; ++kb) {
        tc::mbar_wait(&empty[stage], phase ^ 1);
        // own A rows + own weight half, both completing on the leader's barrier
        const uint32_t lf = tc::mapa_shared(tc::smem_u32(&full[stage]), 0);
        if (rank == 0) tc::mbar_arrive_expect_tx_elect(&full[stage], 2 * (A_BYTES + B_HALF));
        tc::tma_load_2d_cg2_elect(sa + stage * A_BYTES, &map_a, lf, kb * BK, m_blk * BM);
        tc::tma_load_2d_cg2_elect(sb + stage * L::kStageB, &map_bh, lf, kb * BK, n_blk * BN + rank * (BN / 2));
        if (++stage == kSt) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer (the leader only) -------------------------------------------------------
    if (rank == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(2 * BM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int pair = cluster; pair < total; pair += nclusters) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::fence_after_sync();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < num_k; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::fence_after_sync();
          const uint32_t a0 = tc::smem_u32(sa + stage * A_BYTES);
          const uint32_t b0 = tc::smem_u32(sb + stage * L::kStageB);
          tc::mma_ss_k64_cg2_elect(d, tc::desc_sw128(a0, 1024, 16), tc::desc_sw128(b0, 1024, 16), idesc,
                                   kb ? 1u : 0u);
          tc::mma_commit_cg2_multicast_elect(&empty[stage], kBoth);  // frees the stage in both CTAs
          if (++stage == kSt) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit_cg2_multicast_elect(&tfull[acc], kBoth);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---- epilogue (warps 2..5 -> TMEM lane quarters 2,3,0,1), transposed through smem ----
    const int q = warp & 3;
    const uint32_t slab = tc::smem_u32(staging + (warp - 2) * 8192);
    auto slab_addr = [&](int row, int unit) {
      return slab + static_cast<uint32_t>(row * 128 + ((unit ^ (row & 7)) << 4));
    };
    int red_buf = 0;  // residual epilogue: which of the warp's two slabs the next chunk uses
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int pair = cluster; pair < total; pair += nclusters) {
      const int m_blk = (pair / n_tiles) * 2 + rank, n_blk = pair % n_tiles;
      const int row0 = m_blk * BM + q * 32;  // this warp's 32 rows
      auto chunk = [&](int c) {
        uint32_t r[32];
        tc::tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN + c), r);
        tc::tmem_ld_wait();
        const int col0 = n_blk * BN + c;
        if (EPI == kGemmResidualF32 || EPI == kGemmResidualGatedF32) {
          // x += acc through a TMA reduce-add: the 32x32 fp32 chunk goes to a
          // 128B-swizzled slab (the tensor map's layout) and L2 performs the
          // read-modify-write, so the epilogue never waits on residual loads.
          if (EPI == kGemmResidualGatedF32) {  // Wan: x += gate[frame] * acc
            const int grow = row0 + lane < M ? row0 + lane : M - 1;
            const float4* g4 = reinterpret_cast<const float4*>(
                gate.gate + static_cast<int64_t>(grow / gate.grp_rows) * gate.grp_stride + col0);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float4 gv = col0 + 4 * u < N ? g4[u] : make_float4(0.f, 0.f, 0.f, 0.f);
              r[4 * u] = __float_as_uint(__uint_as_float(r[4 * u]) * gv.x);
              r[4 * u + 1] = __float_as_uint(__uint_as_float(r[4 * u + 1]) * gv.y);
              r[4 * u + 2] = __float_as_uint(__uint_as_float(r[4 * u + 2]) * gv.z);
              r[4 * u + 3] = __float_as_uint(__uint_as_float(r[4 * u + 3]) * gv.w);
            }
          }
          const uint32_t sl = slab + static_cast<uint32_t>(red_buf * 4096);
          tc::bulk_wait_group_read<1>();  // the slab's previous reduce has read it
          __syncwarp();
#pragma unroll
          for (int u = 0; u < 8; ++u)
            tc::st_shared_v4(sl + static_cast<uint32_t>(lane * 128 + ((u ^ (lane & 7)) << 4)), r[4 * u],
                             r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]);
          tc::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_reduce_add_2d(&map_c, staging + (warp - 2) * 8192 + red_buf * 4096, col0, row0);
            tc::bulk_commit_group();
          }
          red_buf ^= 1;
          return;
        }
        if (EPI == kGemmStoreBf16 || EPI == kGemmGeluBf16 || EPI == kGemmGeluTanhBf16) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x0 = __uint_as_float(r[2 * i]), x1 = __uint_as_float(r[2 * i + 1]);
            if (EPI == kGemmGeluBf16) {
              const float2 g = gelu_erf_f2(make_float2(x0, x1));
              x0 = g.x;
              x1 = g.y;
            } else if (EPI == kGemmGeluTanhBf16) {
              const float2 g = gelu_tanh_f2(make_float2(x0, x1));
              x0 = g.x;
              x1 = g.y;
            }
            __nv_bfloat162 h2 = __floats2bfloat162_rn(x0, x1);
            pk[i] = *reinterpret_cast<uint32_t*>(&h2);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            tc::st_shared_v4(slab_addr(lane, u), pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {  // 8 rows x 64 bytes per instruction
            const int rr = 8 * i + (lane >> 2), u = lane & 3;
            const uint4 v = tc::ld_shared_v4(slab_addr(rr, u));
            const int grow = row0 + rr, gcol = col0 + u * 8;
            if (grow < M && gcol < N)
              *reinterpret_cast<uint4*>(static_cast<bf16*>(Cv) + static_cast<int64_t>(grow) * ldc + gcol) = v;
          }
        } else {
          // fp32 store; kGemmResidualOutF32 adds the residual R (read here,
          // coalesced along rows) and writes R + acc to C, which may live on
          // another GPU (the next stage's receive slot): the residual add and
          // the stage-boundary send in one pass over the tile.
          float4 res[8];
          if (EPI == kGemmResidualOutF32) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int grow = row0 + 4 * i + (lane >> 3), gcol = col0 + (lane & 7) * 4;
              res[i] = grow < M && gcol < N
                           ? __ldg(reinterpret_cast<const float4*>(gate.resid + static_cast<int64_t>(grow) * gate.ldr + gcol))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
            tc::st_shared_v4(slab_addr(lane, u), r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + (lane >> 3), u = lane & 7;
            const uint4 v = tc::ld_shared_v4(slab_addr(rr, u));
            float4 o = make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w));
            const int grow = row0 + rr, gcol = col0 + u * 4;
            if (grow < M && gcol < N) {
              if (EPI == kGemmResidualOutF32) {
                o.x = res[i].x + o.x; o.y = res[i].y + o.y; o.z = res[i].z + o.z; o.w = res[i].w + o.w;
              }
              *reinterpret_cast<float4*>(static_cast<float*>(Cv) + static_cast<int64_t>(grow) * ldc + gcol) = o;
            }
          }
        }
        __syncwarp();  // the slab is rewritten by the next chunk
      };

      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::fence_after_sync();
#pragma unroll 1
      for (int c = 0; c < BN; c += 64) {
        chunk(c);
        chunk(c + 32);
      }
      tc::fence_before_sync();
      __syncwarp();  // the leader's MMA reuses the accumulator once both CTAs drained it
      if (lane == 0) tc::mbar_arrive_cluster(tc::mapa_shared(tc::smem_u32(&tempty[acc]), 0));
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (EPI == kGemmResidualF32 || EPI == kGemmResidualGatedF32)
      tc::bulk_wait_group<0>();  // this lane's reduce-adds are complete
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();  // the peer may still multicast into / arrive on this CTA's shared memory until here
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc_cg2<512>(tmem_base);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_map_mu;

struct MapKey {
  const void* p; uint64_t rows, cols, ld; uint32_t br, bc;
  bool operator==(const MapKey& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && br == o.br && bc == o.bc;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.p);
    h = h * 1000003u ^ k.rows;
    h = h * 1000003u ^ k.cols;
    h = h * 1000003u ^ k.ld;
    h = h * 1000003u ^ (static_cast<size_t>(k.br) << 16 | k.bc);
    return h;
  }
};
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

std::atomic<int> g_sm_reserve{0};

template <int EPI>
void launch_pair(const CUtensorMap& ma, const CUtensorMap& mbh, int M, int N, int K, void* C, int64_t ldc,
                 const CUtensorMap& mc, cudaStream_t st, const GemmGate& gate) {
  set_smem_attr(k_gemm_pair<EPI>, PairLayout::kSmem);
  const int pairs = (((M + BM - 1) / BM + 1) / 2) * ((N + BN - 1) / BN);
  const int avail = (kNumSms - g_sm_reserve.load(std::memory_order_relaxed)) / 2;
  const int clusters = pairs < avail ? pairs : avail;
  launch_pdl(k_gemm_pair<EPI>, dim3(2 * clusters), dim3(kThreads), PairLayout::kSmem, st, ma, mbh, M, N, K,
             C, ldc, mc, gate);
}

}  // namespace

static void load_encode() {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q{};
    void* fn = nullptr;
    BP_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) fail(BP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
}

void make_tmap_2d_f32(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                      uint32_t box_rows, uint32_t box_cols) {
  load_encode();
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(BP_ERR_CUDA, "cuTensorMapEncodeTiled (f32) failed (" + std::to_string(static_cast<int>(r)) + ")");
}

void make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                       uint32_t box_rows, uint32_t box_cols) {
  load_encode();
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(BP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
}

static const CUtensorMap& cached_map(const void* p, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t br,
                                     uint32_t bc) {
  std::lock_guard<std::mutex> lock(g_map_mu);
  const MapKey k{p, rows, cols, ld, br, bc};
  auto it = g_maps.find(k);
  if (it != g_maps.end()) return it->second;
  if (g_maps.size() > 4096) g_maps.clear();
  CUtensorMap m;
  make_tmap_2d_bf16(&m, p, rows, cols, ld, br, bc);
  return g_maps.emplace(k, m).first->second;
}

static const CUtensorMap& cached_map_f32(const void* p, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t br,
                                         uint32_t bc) {
  std::lock_guard<std::mutex> lock(g_map_mu);
  const MapKey k{p, rows, cols, ld | (1ull << 62), br, bc};  // tagged: fp32 maps never alias bf16 ones
  auto it = g_maps.find(k);
  if (it != g_maps.end()) return it->second;
  if (g_maps.size() > 4096) g_maps.clear();
  CUtensorMap m;
  make_tmap_2d_f32(&m, p, rows, cols, ld, br, bc);
  return g_maps.emplace(k, m).first->second;
}

void set_sm_reserve(int sms) {
  if (sms < 0 || sms > kNumSms - 2) fail(BP_ERR_CONFIG, "SM reservation out of range");
  g_sm_reserve.store(sms);
}
int sm_reserve() { return g_sm_reserve.load(); }

void launch_gemm_tc(const bf16* A, int64_t lda, const bf16* W, int M, int N, int K, void* C, int64_t ldc, int epi,
                    cudaStream_t st, const GemmGate& gate) {
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(W)) & 15)
    fail(BP_ERR_INTERNAL, "GEMM operands must be 16-byte aligned");
  if ((lda * 2) % 16 || (K * 2) % 16 || N % 32 || ldc % 8)
    fail(BP_ERR_INTERNAL, "GEMM strides must be 16-byte multiples and N % 32 == 0");
  const bool resid = epi == kGemmResidualF32 || epi == kGemmResidualGatedF32;
  if (epi == kGemmResidualGatedF32 &&
      ((reinterpret_cast<uintptr_t>(gate.gate) & 15) || gate.grp_stride % 4 || gate.grp_rows < 1))
    fail(BP_ERR_INTERNAL, "gate table must be 16-byte aligned");
  if (epi == kGemmResidualOutF32 &&
      ((reinterpret_cast<uintptr_t>(gate.resid) | reinterpret_cast<uintptr_t>(C)) & 15 || gate.ldr % 4 || ldc % 4))
    fail(BP_ERR_INTERNAL, "residual-out GEMM buffers must be 16-byte aligned");
  const CUtensorMap ma = cached_map(A, static_cast<uint64_t>(M), static_cast<uint64_t>(K), static_cast<uint64_t>(lda), BM, BK);
  // each CTA of the pair stages one 128-row half of the 256-row weight tile
  const CUtensorMap mbh =
      cached_map(W, static_cast<uint64_t>(N), static_cast<uint64_t>(K), static_cast<uint64_t>(K), BN / 2, BK);
  CUtensorMap mc = mbh;  // unused except by the residual epilogues
  if (resid) {
    if ((reinterpret_cast<uintptr_t>(C) & 15) || (ldc * 4) % 16) fail(BP_ERR_INTERNAL, "residual C must be 16-byte aligned");
    mc = cached_map_f32(C, static_cast<uint64_t>(M), static_cast<uint64_t>(N), static_cast<uint64_t>(ldc), 32, 32);
  }
  switch (epi) {
    case kGemmStoreBf16: launch_pair<kGemmStoreBf16>(ma, mbh, M, N, K, C, ldc, mc, st, gate); break;
    case kGemmGeluBf16: launch_pair<kGemmGeluBf16>(ma, mbh, M, N, K, C, ldc, mc, st, gate); break;
    case kGemmResidualF32: launch_pair<kGemmResidualF32>(ma, mbh, M, N, K, C, ldc, mc, st, gate); break;
    case kGemmResidualGatedF32: launch_pair<kGemmResidualGatedF32>(ma, mbh, M, N, K, C, ldc, mc, st, gate); break;
    case kGemmGeluTanhBf16: launch_pair<kGemmGeluTanhBf16>(ma, mbh, M, N, K, C, ldc, mc, st, gate); break;
    case kGemmResidualOutF32: launch_pair<kGemmResidualOutF32>(ma, mbh, M, N, K, C, ldc, mc, st, gate); break;
    default: launch_pair<kGemmStoreF32>(ma, mbh, M, N, K, C, ldc, mc, st, gate); break;
  }
  count_launch();
}

}  // namespace bp
