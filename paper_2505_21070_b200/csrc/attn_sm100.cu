// tcgen05 flash attention over two KV segments (K6/K7): every query row of
// one head attends to [cached prefix (previous pass on this GPU, resident in
// HBM) ++ current block] without concatenating them in memory
// (model.cpp:201-211, 302-318: vcat_rows(prefix, k) then attention()).
//
// Two kernels, both the ping-pong schedule of two 128-row query tiles over
// 64-key K/V tiles with S double-buffered in TMEM (described below):
//   k_attn_pp2  on a cta_group::2 CTA pair (M = 256 MMAs, each CTA staging
//               half of every K / V tile): the self-attention (launch_attn_tc
//               variant 4, the default);
//   k_attn_ps   one CTA per SM, persistent over (query pair, head) items, O
//               staged in the item's Q buffer and written by TMA bulk stores:
//               the cross-attention over the 512-token context (variant 2),
//               where a one-item CTA would be mostly fill and drain.
// Keys past a segment's end (a tile that straddles it) are masked; TMA
// zero-fills the rows. Losing variants measured in round 1 (one query tile
// per CTA with Q in TMEM; 128-key tiles with rows split over two softmax
// warps) are recorded in DESIGN.md and no longer built.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "device.cuh"
#include "kernels_bf16.cuh"
#include "tc_common.cuh"

namespace bp {

void launch_attn_simt(const AttnBf16Args& a, int64_t rows, cudaStream_t st);

namespace {

constexpr int kDh = 128, BQ = 128;
constexpr uint32_t HALF = 128 * 64 * 2;      // [128 rows][64 bf16] swizzled TMA box
constexpr uint32_t TILE = 2 * HALF;          // 32 KB: one 128-row query tile
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P values up to 2^8 before O is rescaled

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ============================================================================
// The ping-pong schedule: two query tiles, 64-key tiles, S double-buffered
// ============================================================================
// A work item is query rows [256 p, 256 p + 256) of one head as tiles A and B.
// K_j / V_j (64 keys each) stream through smem once for both tiles. Each tile
// has two S buffers, so QK_x(j+1) runs on the tensor core while the softmax of
// tile x works on S_x(j), and the softmax warpgroups of A and B run
// concurrently (two latency-bound softmax warps per SM sub-partition instead
// of one). TMEM: S_A0 [0,64) S_A1 [64,128) S_B0 [128,192) S_B1 [192,256)
// O_A [256,384) O_B [384,512); P_x(j) overwrites the first 32 columns of its S
// buffer as packed bf16 pairs. Q is an smem (SS) operand: an SS MMA sustains
// the tcgen05 issue floor (tools/micro/mma_floor.cu).
//   warp 0        TMA producer (Q_A, Q_B per item; K / V rings of 64-key tiles)
//   warp 1        MMA issuer: QK (M128 N64 K128, 8 MMAs), PV (M128 N128 K64, 4)
//   warps 2..5    softmax + epilogue of tile A  (thread <-> row <-> TMEM lane
//   warps 6..9    softmax + epilogue of tile B   quarter warp & 3)
// Softmax arithmetic is packed (FFMA2 / FADD2, three-input FMNMX); one exp2
// pair in eight runs on the FMA pipe.
constexpr int PBK = 64;                              // keys per K/V tile
constexpr uint32_t PHALF = PBK * 64 * 2;            // [64 keys][64 d] swizzled box, 8 KB
constexpr uint32_t PTILE = 2 * PHALF;               // 16 KB
constexpr int PP_THREADS = 320;

struct AttnMapsPP {
  CUtensorMap q, k0, v0, k1, v1;  // q: 128-row boxes; k/v: 64-row boxes
  CUtensorMap o;                  // output, 128-row boxes (epilogue TMA stores)
};

__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  // ex2_poly on a packed pair: round via 1.5*2^23, cubic on the fraction.
  const float2 big = make_float2(12582912.f, 12582912.f);
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 j = __fadd2_rn(x, big);
  const float2 jr = __fadd2_rn(j, make_float2(-12582912.f, -12582912.f));  // round(x)
  const float2 f = __fadd2_rn(x, make_float2(-jr.x, -jr.y));
  float2 p = __ffma2_rn(make_float2(0.0555041086f, 0.0555041086f), f, make_float2(0.2402264923f, 0.2402264923f));
  p = __ffma2_rn(p, f, make_float2(0.6931471806f, 0.6931471806f));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// ============================================================================
// k_attn_ps: the ping-pong schedule on one CTA, persistent (cross-attention)
// ============================================================================
// With 512 context keys a one-item CTA runs only 8 key steps between its
// prologue (barrier init, TMEM allocation, the Q load's DRAM latency, the
// first QK^T) and its epilogue, so most of its time is fill and drain (round
// 1's k_attn_pp: 821 TF/s at q 18720 x kv 512; this kernel 959). Here
// one CTA per SM walks work items (query pair, head) and keeps the pipeline
// running across items: Q is double-buffered (the next item's Q loads behind
// the current item's first K/V tiles, into the buffer the previous item's
// last QK^T released), the K/V rings continue across items, and the next
// item's first two QK^T are issued right behind the current item's last PV,
// so they overlap its epilogue. Every barrier phase derives from the global
// step counter g (all items' key steps in order) or the item counter n, never
// from an item's local step, so items whose key count is odd, even or an exact
// multiple of the tile chain their phases alike. O is staged in the item's
// own Q buffer (free once its last PV completed) and written by TMA stores;
// the epilogue, not the MMA warp, releases that buffer to the producer. The
// epilogue's TMEM reads complete before the same warps arrive P of the next
// item, which the MMA warp waits on before its first PV overwrites O.
constexpr int PS_KST = 3, PS_VST = 3;
constexpr uint32_t PS_Q = 0;                        // two Q buffers x (Q_A, Q_B): 128 KB
constexpr uint32_t PS_K = PS_Q + 4 * TILE;
constexpr uint32_t PS_V = PS_K + PS_KST * PTILE;
constexpr uint32_t PS_BAR = PS_V + PS_VST * PTILE;
constexpr uint32_t PS_SMEM_BYTES = PS_BAR + 256 + 1024;
static_assert(PS_SMEM_BYTES <= 232448, "persistent attention exceeds the 227 KB smem limit");

template <int kPoly8>
__global__ void __launch_bounds__(PP_THREADS, 1)
    k_attn_ps(const __grid_constant__ AttnMapsPP maps, int64_t rows, int64_t n0, int64_t n1, int heads,
              float scale_log2, bf16* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PS_BAR);
  uint64_t* q_full = bars + 0;              // [Q buffer]
  uint64_t* q_empty = q_full + 2;           // [Q buffer]
  uint64_t* k_full = q_empty + 2;           // [PS_KST]
  uint64_t* k_empty = k_full + PS_KST;      // [PS_KST]
  uint64_t* v_full = k_empty + PS_KST;      // [PS_VST]
  uint64_t* v_empty = v_full + PS_VST;      // [PS_VST]
  uint64_t* s_full = v_empty + PS_VST;      // [tile][buffer]
  uint64_t* p_full = s_full + 4;            // [tile][buffer] (128 arrivals)
  uint64_t* pv_done = p_full + 4;           // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int t0 = static_cast<int>((n0 + PBK - 1) / PBK);
  const int t1 = static_cast<int>((n1 + PBK - 1) / PBK);
  const int T = t0 + t1;
  const int npairs = static_cast<int>((rows + 2 * BQ - 1) / (2 * BQ));
  const int items = npairs * heads;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&maps.q);
    tc::tma_prefetch(&maps.k1);
    tc::tma_prefetch(&maps.v1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&q_full[b], 1);
      tc::mbar_init(&q_empty[b], 2);  // both tiles' epilogues have stored O out of the buffer
    }
    for (int s = 0; s < PS_KST; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < PS_VST; ++s) {
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], 128);
    }
    tc::mbar_init(&pv_done[0], 1);
    tc::mbar_init(&pv_done[1], 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  tc::pdl_wait();  // Q/K/V were produced by the previous kernel

  if (warp == 0) {
    // ---- TMA producer: Q of item n + 1 right behind item n's first K/V tiles --------------
    auto load_q = [&](int n, int item) {
      const int b = n & 1;
      tc::mbar_wait(&q_empty[b], ((n >> 1) & 1) ^ 1);
      const int qpair = item % npairs, head = item / npairs;
      uint8_t* qd = smem + PS_Q + b * 2 * TILE;
      tc::mbar_arrive_expect_tx_elect(&q_full[b], 2 * TILE);
      for (int x = 0; x < 2; ++x) {
        const int qrow = qpair * 2 * BQ + x * BQ;
        tc::tma_load_2d_elect(qd + x * TILE, &maps.q, &q_full[b], head * kDh, qrow);
        tc::tma_load_2d_elect(qd + x * TILE + HALF, &maps.q, &q_full[b], head * kDh + 64, qrow);
      }
    };
    int g = 0, n = 0;
    if (static_cast<int>(blockIdx.x) < items) load_q(0, blockIdx.x);
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
      const int head = item / npairs;
      for (int j = 0; j < T; ++j, ++g) {
        const bool seg0 = j < t0;
        const int row0 = (seg0 ? j : j - t0) * PBK;
        const int ks = g % PS_KST, vs = g % PS_VST;
        tc::mbar_wait(&k_empty[ks], ((g / PS_KST) & 1) ^ 1);
        uint8_t* kd = smem + PS_K + ks * PTILE;
        const CUtensorMap* mk = seg0 ? &maps.k0 : &maps.k1;
        tc::mbar_arrive_expect_tx_elect(&k_full[ks], PTILE);
        tc::tma_load_2d_elect(kd, mk, &k_full[ks], head * kDh, row0);
        tc::tma_load_2d_elect(kd + PHALF, mk, &k_full[ks], head * kDh + 64, row0);
        tc::mbar_wait(&v_empty[vs], ((g / PS_VST) & 1) ^ 1);
        uint8_t* vd = smem + PS_V + vs * PTILE;
        const CUtensorMap* mv = seg0 ? &maps.v0 : &maps.v1;
        tc::mbar_arrive_expect_tx_elect(&v_full[vs], PTILE);
        tc::tma_load_2d_elect(vd, mv, &v_full[vs], head * kDh, row0);
        tc::tma_load_2d_elect(vd + PHALF, mv, &v_full[vs], head * kDh + 64, row0);
        if (j == (T > 1 ? 1 : 0) && item + static_cast<int>(gridDim.x) < items)
          load_q(n + 1, item + gridDim.x);
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer -----------------------------------------------------------------------
    constexpr uint32_t idesc_s = tc::idesc_bf16(BQ, PBK, 0, 0);
    constexpr uint32_t idesc_o = tc::idesc_bf16(BQ, kDh, 0, 1);
    int g = 0, n = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
      const uint32_t q_base = tc::smem_u32(smem + PS_Q + (n & 1) * 2 * TILE);
      auto qk_pair = [&](int gg) {  // S_x(gg) into buffer gg & 1 of both tiles
        tc::mbar_wait(&k_full[gg % PS_KST], (gg / PS_KST) & 1);
        tc::fence_after_sync();
        const uint32_t k_addr = tc::smem_u32(smem + PS_K + (gg % PS_KST) * PTILE);
        for (int x = 0; x < 2; ++x) {
          const uint32_t d = tmem + static_cast<uint32_t>(x * 2 * PBK + (gg & 1) * PBK);
          tc::mma_ss_k128_elect<HALF / 16, PHALF / 16>(d, tc::desc_sw128(q_base + x * TILE, 1024, 16),
                                                       tc::desc_sw128(k_addr, 1024, 16), idesc_s, 0u);
          tc::mma_commit_elect(&s_full[x * 2 + (gg & 1)]);
        }
        tc::mma_commit_elect(&k_empty[gg % PS_KST]);
      };
      tc::mbar_wait(&q_full[n & 1], (n >> 1) & 1);
      tc::fence_after_sync();
      if (T > 0) qk_pair(g);
      if (T > 1) qk_pair(g + 1);
      for (int j = 0; j < T; ++j) {
        const int gg = g + j;
        tc::mbar_wait(&v_full[gg % PS_VST], (gg / PS_VST) & 1);
        const uint32_t v_addr = tc::smem_u32(smem + PS_V + (gg % PS_VST) * PTILE);
        for (int x = 0; x < 2; ++x) {
          tc::mbar_wait(&p_full[x * 2 + (gg & 1)], (gg >> 1) & 1);
          tc::fence_after_sync();
          const uint32_t p_tm = tmem + static_cast<uint32_t>(x * 2 * PBK + (gg & 1) * PBK);
          tc::mma_ts_k64_elect<2048 / 16>(tmem + 256 + x * kDh, p_tm, tc::desc_sw128(v_addr, 1024, PHALF), idesc_o,
                                          j > 0 ? 1u : 0u);
          tc::mma_commit_elect(&pv_done[x]);
        }
        tc::mma_commit_elect(&v_empty[gg % PS_VST]);
        if (j + 2 < T) qk_pair(gg + 2);  // S buffer gg & 1 is free once PV(gg) is issued (in-order)
      }
      g += T;
    }
  } else {
    // ---- softmax + epilogue of tile x -----------------------------------------------------
    const int x = (warp - 2) >> 2;
    const int qq = warp & 3;
    const int r = qq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(qq * 32) << 16;
    const uint32_t tm_o = tmem + lane_off + 256u + static_cast<uint32_t>(x * kDh);
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    const int n0i = static_cast<int>(n0), n1i = static_cast<int>(n1);
    int g = 0, n = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++n) {
      const int qpair = item % npairs, head = item / npairs;
      float m_used = -INFINITY;
      float2 l2 = make_float2(0.f, 0.f);
      for (int j = 0; j < T; ++j) {
        const int gg = g + j;
        const int b = gg & 1;
        const bool seg0 = j < t0;
        const int row0 = (seg0 ? j : j - t0) * PBK;
        const int rem = (seg0 ? n0i : n1i) - row0;
        const uint32_t tm_s = tmem + lane_off + static_cast<uint32_t>(x * 2 * PBK + b * PBK);
        tc::mbar_wait(&s_full[x * 2 + b], (gg >> 1) & 1);
        tc::fence_after_sync();
        uint32_t sr[64];
        tc::tmem_ld32(tm_s, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
        tc::tmem_ld32(tm_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
        tc::tmem_ld_wait();
        if (rem < PBK) {
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (c >= rem) sr[c] = __float_as_uint(-INFINITY);
        }
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 64; c += 8) {
          m4[0] = max3f(m4[0], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
          m4[1] = max3f(m4[1], __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
          m4[2] = max3f(m4[2], __uint_as_float(sr[c + 4]), __uint_as_float(sr[c + 5]));
          m4[3] = max3f(m4[3], __uint_as_float(sr[c + 6]), __uint_as_float(sr[c + 7]));
        }
        const float mx = max3f(m4[0], m4[1], fmaxf(m4[2], m4[3])) * scale_log2;
        const bool need = mx > m_used + kRescaleThreshold;
        const float m_new = need ? mx : m_used;
        const float corr = need ? ex2(m_used - m_new) : 1.f;
        const float2 neg_m2 = make_float2(-m_new, -m_new);
        uint32_t pk[32];
        float2 ls_a = make_float2(0.f, 0.f), ls_b = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float2 xv = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sc2,
                                       neg_m2);
          const float2 p = (c & 7) >= 8 - kPoly8 ? ex2_poly2(xv) : make_float2(ex2(xv.x), ex2(xv.y));
          if (c & 1) ls_b = __fadd2_rn(ls_b, p);
          else ls_a = __fadd2_rn(ls_a, p);
          pk[c] = pack_bf16(p.x, p.y);
        }
        l2 = __ffma2_rn(l2, make_float2(corr, corr), __fadd2_rn(ls_a, ls_b));
        m_used = m_new;
        // every PV completion is observed (one phase per step; compute-sanitizer
        // synccheck flags phases nobody waits on). PV(gg - 1) has normally
        // finished by now; O must hold it before it is rescaled.
        if (j >= 1) tc::mbar_wait(&pv_done[x], (gg - 1) & 1);
        if (j >= 1 && __any_sync(0xffffffffu, need)) {
          tc::fence_after_sync();
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            const uint32_t ta = tm_o + static_cast<uint32_t>(c * 32);
            tc::tmem_ld32(ta, o);
            tc::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
            tc::tmem_st32(ta, o);
          }
        }
        tc::tmem_st32(tm_s, pk);
        tc::tmem_st_wait();
        tc::fence_before_sync();
        tc::mbar_arrive(&p_full[x * 2 + b]);
      }
      g += T;
      if (T >= 1) {
        tc::mbar_wait(&pv_done[x], (g - 1) & 1);
        tc::fence_after_sync();
      }
      // O / l as bf16 into this item's Q buffer (every MMA that read it has
      // completed: PV(g - 1) is the item's last), in the output map's
      // 128B-swizzled layout, then two TMA stores per tile; the buffer is
      // released to the producer (q_empty) once the stores have read it
      const float inv_l = 1.f / (l2.x + l2.y);
      uint8_t* stage_o = smem + PS_Q + (n & 1) * 2 * TILE + x * TILE;
      const uint32_t so = tc::smem_u32(stage_o);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t o[32];
        tc::tmem_ld32(tm_o + static_cast<uint32_t>(c * 32), o);
        tc::tmem_ld_wait();
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const uint32_t unit = static_cast<uint32_t>((c & 1) * 4 + v);
          tc::st_shared_v4(so + static_cast<uint32_t>((c >> 1) * HALF + r * 128) + ((unit ^ static_cast<uint32_t>(r & 7)) << 4),
                           pack_bf16(__uint_as_float(o[8 * v]) * inv_l, __uint_as_float(o[8 * v + 1]) * inv_l),
                           pack_bf16(__uint_as_float(o[8 * v + 2]) * inv_l, __uint_as_float(o[8 * v + 3]) * inv_l),
                           pack_bf16(__uint_as_float(o[8 * v + 4]) * inv_l, __uint_as_float(o[8 * v + 5]) * inv_l),
                           pack_bf16(__uint_as_float(o[8 * v + 6]) * inv_l, __uint_as_float(o[8 * v + 7]) * inv_l));
        }
      }
      tc::fence_proxy_async_smem();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + x) : "memory");  // this tile's 128 softmax threads
      if (qq == 0 && lane == 0) {
        const int qrow = qpair * 2 * BQ + x * BQ;
        tc::tma_store_2d(&maps.o, stage_o, head * kDh, qrow);
        tc::tma_store_2d(&maps.o, stage_o + HALF, head * kDh + 64, qrow);
        tc::bulk_commit_group();
        tc::bulk_wait_group_read<0>();  // smem read out; the global writes drain on their own
        tc::mbar_arrive(&q_empty[n & 1]);
      }
      // the next item's P arrive (after these TMEM reads completed) gates the
      // MMA warp's first PV of that item, which overwrites O
      tc::fence_before_sync();
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<512>(tmem);
  }
}

// ============================================================================
// Variant 4: k_attn_pp on a CTA pair (cta_group::2)
// ============================================================================
// Two CTAs of a (2,1,1) cluster on one TPC run the ping-pong schedule of
// k_attn_pp on two adjacent query pairs of the same head as ONE M = 256 MMA
// per step: QK^T (M256 N64) takes its A rows from each CTA's own Q tile and
// splits the 64-key B tile by N, so each CTA stages only 32 keys of K (8 KB)
// and reads 5 KB of shared memory per K=16 step instead of 6 KB (the SS step
// that bounds k_attn_pp is smem-bound); PV (M256 N128) splits V by head-dim
// columns, so each CTA stages a [64 keys][64 d] half. K/V bytes per CTA halve.
// The leader CTA issues every MMA; both CTAs' TMA loads complete on the
// leader's full barriers, every commit is multicast to both CTAs, and each
// softmax warp reports P-ready to the leader with one remote arrive.
// TMEM layout and softmax are k_attn_pp's.
constexpr uint32_t P2_KH = 32 * 64 * 2;             // [32 keys][64 d] box, 4 KB
constexpr uint32_t P2_KT = 2 * P2_KH;               // this CTA's K half-tile, 8 KB
constexpr uint32_t P2_VT = PBK * 64 * 2;            // [64 keys][64 d] V half, 8 KB
constexpr int P2_KST = 6, P2_VST = 6;
constexpr uint32_t P2_Q = 0;
constexpr uint32_t P2_K = P2_Q + 2 * TILE;
constexpr uint32_t P2_V = P2_K + P2_KST * P2_KT;
constexpr uint32_t P2_BAR = P2_V + P2_VST * P2_VT;
constexpr uint32_t P2_SMEM_BYTES = P2_BAR + 512 + 1024;  // 37 mbarriers + the TMEM slot, then alignment slack
static_assert(P2_SMEM_BYTES <= 232448, "pair attention exceeds the 227 KB smem limit");

struct AttnMapsP2 {
  CUtensorMap q, k0, v0, k1, v1;  // q: 128-row boxes; k: 32-row boxes; v: 64-row boxes
  CUtensorMap o;                  // output, 128-row boxes (epilogue TMA stores)
};

// kPoly8: exp2 pairs in 8 evaluated on the FMA pipe
// kObserveAll: wait on every pv_done phase (the build compute-sanitizer's
// synccheck runs; see the rescale branch), otherwise only when rescaling.
template <int kPoly8, bool kObserveAll = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PP_THREADS, 1)
    k_attn_pp2(const __grid_constant__ AttnMapsP2 maps, int64_t rows, int64_t n0, int64_t n1, float scale_log2,
               bf16* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + P2_BAR);
  uint64_t* q_full = bars + 0;              // leader: both CTAs' Q
  uint64_t* k_full = bars + 1;              // [P2_KST] leader: both K halves
  uint64_t* k_empty = k_full + P2_KST;      // [P2_KST] each CTA (multicast commit)
  uint64_t* v_full = k_empty + P2_KST;      // [P2_VST] leader
  uint64_t* v_empty = v_full + P2_VST;      // [P2_VST] each CTA
  uint64_t* s_full = v_empty + P2_VST;      // [tile][buffer] each CTA
  uint64_t* p_full = s_full + 4;            // [tile][buffer] leader, 8 warp arrivals
  uint64_t* pv_done = p_full + 4;           // [tile] each CTA, one phase per PV
  uint64_t* o_done = pv_done + 2;           // [tile] each CTA, one phase: the last PV
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const int qpair = blockIdx.x, head = blockIdx.y;
  const int t0 = static_cast<int>((n0 + PBK - 1) / PBK);
  const int t1 = static_cast<int>((n1 + PBK - 1) / PBK);
  const int T = t0 + t1;
  constexpr uint16_t kBoth = 0x3;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&maps.q);
    tc::tma_prefetch(&maps.k1);
    tc::tma_prefetch(&maps.v1);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < P2_KST; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < P2_VST; ++s) {
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], 8);
    }
    tc::mbar_init(&pv_done[0], 1);
    tc::mbar_init(&pv_done[1], 1);
    tc::mbar_init(&o_done[0], 1);
    tc::mbar_init(&o_done[1], 1);
    tc::fence_mbarrier_init_cluster();
  }
  if (warp == 1) tc::tmem_alloc_cg2<512>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();  // barrier inits of both CTAs visible before any remote arrive / TMA
  tc::fence_after_sync();
  const uint32_t tmem = *tmem_slot;
  tc::pdl_wait();  // Q/K/V were produced by the previous kernel

  if (warp == 0) {
    // ---- TMA producer (both CTAs): own Q tiles, own K / V halves -> leader's barriers ----
    const uint32_t lq = tc::mapa_shared(tc::smem_u32(q_full), 0);
    if (rank == 0) tc::mbar_arrive_expect_tx_elect(q_full, 4 * TILE);
    for (int x = 0; x < 2; ++x) {
      const int qrow = qpair * 2 * BQ + x * BQ;
      tc::tma_load_2d_cg2_elect(smem + P2_Q + x * TILE, &maps.q, lq, head * kDh, qrow);
      tc::tma_load_2d_cg2_elect(smem + P2_Q + x * TILE + HALF, &maps.q, lq, head * kDh + 64, qrow);
    }
    for (int j = 0; j < T; ++j) {
      const bool seg0 = j < t0;
      const int row0 = (seg0 ? j : j - t0) * PBK;
      const int ks = j % P2_KST, vs = j % P2_VST;
      tc::mbar_wait_cluster(&k_empty[ks], ((j / P2_KST) & 1) ^ 1);
      uint8_t* kd = smem + P2_K + ks * P2_KT;
      const CUtensorMap* mk = seg0 ? &maps.k0 : &maps.k1;
      const uint32_t lk = tc::mapa_shared(tc::smem_u32(&k_full[ks]), 0);
      if (rank == 0) tc::mbar_arrive_expect_tx_elect(&k_full[ks], 2 * P2_KT);
      tc::tma_load_2d_cg2_elect(kd, mk, lk, head * kDh, row0 + static_cast<int>(rank) * 32);
      tc::tma_load_2d_cg2_elect(kd + P2_KH, mk, lk, head * kDh + 64, row0 + static_cast<int>(rank) * 32);
      tc::mbar_wait_cluster(&v_empty[vs], ((j / P2_VST) & 1) ^ 1);
      uint8_t* vd = smem + P2_V + vs * P2_VT;
      const CUtensorMap* mv = seg0 ? &maps.v0 : &maps.v1;
      const uint32_t lv = tc::mapa_shared(tc::smem_u32(&v_full[vs]), 0);
      if (rank == 0) tc::mbar_arrive_expect_tx_elect(&v_full[vs], 2 * P2_VT);
      tc::tma_load_2d_cg2_elect(vd, mv, lv, head * kDh + static_cast<int>(rank) * 64, row0);
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---- MMA issuer (leader) ---------------------------------------------------------------
      constexpr uint32_t idesc_s = tc::idesc_bf16(2 * BQ, PBK, 0, 0);  // Q x K^T, M256 N64
      constexpr uint32_t idesc_o = tc::idesc_bf16(2 * BQ, kDh, 0, 1);  // P (TMEM) x V, M256 N128
      const uint32_t q_base = tc::smem_u32(smem + P2_Q);
      auto qk = [&](int x, int j) {
        const uint32_t k_addr = tc::smem_u32(smem + P2_K + (j % P2_KST) * P2_KT);
        const uint32_t d = tmem + static_cast<uint32_t>(x * 2 * PBK + (j & 1) * PBK);
        tc::mma_ss_k128_cg2_elect<HALF / 16, P2_KH / 16>(d, tc::desc_sw128(q_base + x * TILE, 1024, 16),
                                                         tc::desc_sw128(k_addr, 1024, 16), idesc_s, 0u);
        tc::mma_commit_cg2_multicast_elect(&s_full[x * 2 + (j & 1)], kBoth);
      };
      auto pv = [&](int x, int j) {
        const uint32_t v_addr = tc::smem_u32(smem + P2_V + (j % P2_VST) * P2_VT);
        const uint32_t p_tm = tmem + static_cast<uint32_t>(x * 2 * PBK + (j & 1) * PBK);
        tc::mma_ts_k64_cg2_elect<2048 / 16>(tmem + 256 + x * kDh, p_tm, tc::desc_sw128(v_addr, 1024, P2_VT),
                                            idesc_o, j > 0 ? 1u : 0u);
        tc::mma_commit_cg2_multicast_elect(&pv_done[x], kBoth);
      };
      auto qk_pair = [&](int j) {
        tc::mbar_wait_cluster(&k_full[j % P2_KST], (j / P2_KST) & 1);
        tc::fence_after_sync();
        qk(0, j);
        qk(1, j);
        tc::mma_commit_cg2_multicast_elect(&k_empty[j % P2_KST], kBoth);
      };
      tc::mbar_wait_cluster(q_full, 0);
      if (T > 0) qk_pair(0);
      if (T > 1) qk_pair(1);
      for (int j = 0; j < T; ++j) {
        tc::mbar_wait_cluster(&v_full[j % P2_VST], (j / P2_VST) & 1);
        for (int x = 0; x < 2; ++x) {
          tc::mbar_wait_cluster(&p_full[x * 2 + (j & 1)], (j >> 1) & 1);
          tc::fence_after_sync();
          pv(x, j);
          // tile x's epilogue barrier: completes with its last PV (and every
          // MMA issued before it), not behind the other tile's last PV
          if (j == T - 1) tc::mma_commit_cg2_multicast_elect(&o_done[x], kBoth);
        }
        tc::mma_commit_cg2_multicast_elect(&v_empty[j % P2_VST], kBoth);
        if (j + 2 < T) qk_pair(j + 2);  // S buffer j & 1 is free once PV(j) is issued (in-order)
      }
    }
  } else {
    // ---- softmax + epilogue of tile x (each CTA, its own rows) ------------------------------
    const int x = (warp - 2) >> 2;
    const int qq = warp & 3;
    const int r = qq * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(qq * 32) << 16;
    const uint32_t tm_o = tmem + lane_off + 256u + static_cast<uint32_t>(x * kDh);
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    float m_used = -INFINITY;
    float2 l2 = make_float2(0.f, 0.f);
    const int n0i = static_cast<int>(n0), n1i = static_cast<int>(n1);
    const uint32_t p_full_leader = tc::mapa_shared(tc::smem_u32(&p_full[x * 2]), 0);
    for (int j = 0; j < T; ++j) {
      const int b = j & 1;
      const bool seg0 = j < t0;
      const int row0 = (seg0 ? j : j - t0) * PBK;
      const int rem = (seg0 ? n0i : n1i) - row0;
      const uint32_t tm_s = tmem + lane_off + static_cast<uint32_t>(x * 2 * PBK + b * PBK);
      tc::mbar_wait_cluster(&s_full[x * 2 + b], (j >> 1) & 1);
      tc::fence_after_sync();
      uint32_t sr[64];
      tc::tmem_ld32(tm_s, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tc::tmem_ld32(tm_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      tc::tmem_ld_wait();
      if (rem < PBK) {  // keys past the segment end (a segment's last tile)
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c >= rem) sr[c] = __float_as_uint(-INFINITY);
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 64; c += 8) {
        m4[0] = max3f(m4[0], __uint_as_float(sr[c]), __uint_as_float(sr[c + 1]));
        m4[1] = max3f(m4[1], __uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3]));
        m4[2] = max3f(m4[2], __uint_as_float(sr[c + 4]), __uint_as_float(sr[c + 5]));
        m4[3] = max3f(m4[3], __uint_as_float(sr[c + 6]), __uint_as_float(sr[c + 7]));
      }
      const float mx = max3f(m4[0], m4[1], fmaxf(m4[2], m4[3])) * scale_log2;  // scale > 0
      const bool need = mx > m_used + kRescaleThreshold;
      const float m_new = need ? mx : m_used;
      const float corr = need ? ex2(m_used - m_new) : 1.f;  // 0 on the first tile
      const float2 neg_m2 = make_float2(-m_new, -m_new);
      uint32_t pk[32];
      float2 ls_a = make_float2(0.f, 0.f), ls_b = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float2 xv = __ffma2_rn(make_float2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1])), sc2,
                                     neg_m2);
        const float2 p = (c & 7) >= 8 - kPoly8 ? ex2_poly2(xv) : make_float2(ex2(xv.x), ex2(xv.y));
        if (c & 1) ls_b = __fadd2_rn(ls_b, p);
        else ls_a = __fadd2_rn(ls_a, p);
        pk[c] = pack_bf16(p.x, p.y);
      }
      l2 = __ffma2_rn(l2, make_float2(corr, corr), __fadd2_rn(ls_a, ls_b));
      m_used = m_new;
      // O must hold PV(j-1) before it is rescaled. pv_done completes one phase
      // per step and is observed only here (rarely). A parity wait is exact
      // only when at most one phase can be outstanding, and here it is: S(j)
      // completing means PV(j-2) completed (QK(j) is issued after PV(j-2),
      // and a commit tracks every earlier MMA), and PV(j) cannot complete
      // before this warp arrives P(j). The epilogue has no S(T) to bound it
      // (a parity wait on pv_done there could pass on PV(T-3)'s phase while
      // PV(T-2) and PV(T-1) are still running; seen when another process
      // time-slices the GPU), so it waits on o_done, which completes once.
      // Observing every phase (which compute-sanitizer's synccheck asks for;
      // kObserveAll, BP_ATTN_OBSERVE_ALL=1) stalls the softmax behind the
      // tensor pipe: 1450 vs 1497 TF/s, round 2.
      if (j >= 1 && __any_sync(0xffffffffu, need)) {
        tc::mbar_wait_cluster(&pv_done[x], (j - 1) & 1);
        tc::fence_after_sync();
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          const uint32_t ta = tm_o + static_cast<uint32_t>(c * 32);
          tc::tmem_ld32(ta, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * corr);
          tc::tmem_st32(ta, o);
        }
      }
      tc::tmem_st32(tm_s, pk);
      tc::tmem_st_wait();
      if (kObserveAll && j >= 1) tc::mbar_wait_cluster(&pv_done[x], (j - 1) & 1);
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(p_full_leader + static_cast<uint32_t>(b * 8));
    }
    if (T >= 1) {
      if (kObserveAll) tc::mbar_wait_cluster(&pv_done[x], (T - 1) & 1);
      tc::mbar_wait_cluster(&o_done[x], 0);
      tc::fence_after_sync();
    }
    const int64_t row = static_cast<int64_t>(qpair) * 2 * BQ + x * BQ + r;
    const float inv_l = 1.f / (l2.x + l2.y);
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      tc::tmem_ld32(tm_o + static_cast<uint32_t>(c * 32), o);
      tc::tmem_ld_wait();
      if (row < rows) {
        uint4* dst = reinterpret_cast<uint4*>(out + row * ldo + head * kDh + c * 32);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          dst[v] = make_uint4(pack_bf16(__uint_as_float(o[8 * v]) * inv_l, __uint_as_float(o[8 * v + 1]) * inv_l),
                              pack_bf16(__uint_as_float(o[8 * v + 2]) * inv_l, __uint_as_float(o[8 * v + 3]) * inv_l),
                              pack_bf16(__uint_as_float(o[8 * v + 4]) * inv_l, __uint_as_float(o[8 * v + 5]) * inv_l),
                              pack_bf16(__uint_as_float(o[8 * v + 6]) * inv_l, __uint_as_float(o[8 * v + 7]) * inv_l));
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();  // the peer's MMAs / arrivals / TMA into this CTA are done
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc_cg2<512>(tmem);
  }
}

std::mutex g_mu;
struct Key {
  const void* p; int64_t rows, cols, ld, box_rows;
  bool operator==(const Key& o) const {
    return p == o.p && rows == o.rows && cols == o.cols && ld == o.ld && box_rows == o.box_rows;
  }
};
struct KeyHash {
  size_t operator()(const Key& k) const {
    return (reinterpret_cast<size_t>(k.p) * 1000003u) ^ (static_cast<size_t>(k.rows) * 7919u) ^
           (static_cast<size_t>(k.cols) << 20) ^ static_cast<size_t>(k.ld) ^ (static_cast<size_t>(k.box_rows) << 40);
  }
};
std::unordered_map<Key, CUtensorMap, KeyHash> g_maps;

CUtensorMap map_for(const bf16* p, int64_t rows, int64_t cols, int64_t ld, uint32_t box_rows = 128) {
  std::lock_guard<std::mutex> lock(g_mu);
  const Key k{p, rows, cols, ld, box_rows};
  auto it = g_maps.find(k);
  if (it != g_maps.end()) return it->second;
  if (g_maps.size() > 4096) g_maps.clear();
  CUtensorMap m;
  make_tmap_2d_bf16(&m, p, static_cast<uint64_t>(rows < 1 ? 1 : rows), static_cast<uint64_t>(cols),
                    static_cast<uint64_t>(ld), box_rows, 64);
  g_maps.emplace(k, m);
  return m;
}

}  // namespace

void launch_attn_tc(const AttnBf16Args& a, int64_t rows, cudaStream_t st, int variant) {
  const int64_t H = static_cast<int64_t>(a.heads) * a.dh;
  const bool aligned = ((a.ldq | a.ldk1 | a.ldv1 | a.ldo) * 2) % 16 == 0 &&
                       (a.n0 == 0 || ((a.ldk0 | a.ldv0) * 2) % 16 == 0);
  if (a.dh != kDh || !aligned || a.n0 + a.n1 == 0) {  // other head dims: SIMT kernel
    launch_attn_simt(a, rows, st);
    return;
  }
  if ((reinterpret_cast<uintptr_t>(a.out) | static_cast<uintptr_t>(a.ldo * 2)) % 16)
    fail(BP_ERR_INTERNAL, "attention output must be 16-byte aligned");
  const float scale_log2 = a.scale * 1.4426950408889634f;
  // K / V tensor maps of one segment; without a prefix the unused segment
  // maps alias the current block's
  auto seg_maps = [&](uint32_t k_box, uint32_t v_box, CUtensorMap* k0, CUtensorMap* v0, CUtensorMap* k1,
                      CUtensorMap* v1) {
    *k1 = map_for(a.k1, a.n1, H, a.ldk1, k_box);
    *v1 = map_for(a.v1, a.n1, H, a.ldv1, v_box);
    *k0 = a.n0 > 0 ? map_for(a.k0, a.n0, H, a.ldk0, k_box) : *k1;
    *v0 = a.n0 > 0 ? map_for(a.v0, a.n0, H, a.ldv0, v_box) : *v1;
  };
  if (variant == 4) {  // k_attn_pp on a CTA pair (cta_group::2): each CTA stages 32 keys of K, half of V
    set_smem_attr(k_attn_pp2<1>, P2_SMEM_BYTES);
    AttnMapsP2 pm;
    pm.q = map_for(a.q, rows, H, a.ldq);
    seg_maps(32, PBK, &pm.k0, &pm.v0, &pm.k1, &pm.v1);
    pm.o = map_for(a.out, rows, H, a.ldo);
    const unsigned pairs = static_cast<unsigned>((rows + 2 * BQ - 1) / (2 * BQ));
    dim3 grid(pairs + (pairs & 1u), static_cast<unsigned>(a.heads));
    // one exp2 pair in 8 on the FMA pipe: the pair's softmax is latency-bound,
    // so the polynomial pays only in small doses (1 in 8 beat all-MUFU and 1 in
    // 4 in the power-capped step, round 1: 15.47 vs 15.68 vs 16.22 s / video)
    static const bool observe_all = std::getenv("BP_ATTN_OBSERVE_ALL") != nullptr;  // the synccheck build
    if (observe_all) {
      set_smem_attr(k_attn_pp2<1, true>, P2_SMEM_BYTES);
      launch_pdl(k_attn_pp2<1, true>, grid, dim3(PP_THREADS), P2_SMEM_BYTES, st, pm, rows, a.n0, a.n1, scale_log2,
                 a.out, a.ldo);
    } else {
      launch_pdl(k_attn_pp2<1>, grid, dim3(PP_THREADS), P2_SMEM_BYTES, st, pm, rows, a.n0, a.n1, scale_log2, a.out,
                 a.ldo);
    }
  } else {  // cross-attention (variant 2): the persistent single-CTA ping-pong over (query pair, head) items
    set_smem_attr(k_attn_ps<1>, PS_SMEM_BYTES);
    AttnMapsPP pm;
    pm.q = map_for(a.q, rows, H, a.ldq);
    seg_maps(PBK, PBK, &pm.k0, &pm.v0, &pm.k1, &pm.v1);
    pm.o = map_for(a.out, rows, H, a.ldo);
    const int64_t items = ((rows + 2 * BQ - 1) / (2 * BQ)) * a.heads;
    const int64_t avail = kNumSms - sm_reserve();  // SMs left to NCCL's kernels (multi-process NCCL runs)
    const unsigned grid = static_cast<unsigned>(items < avail ? items : avail);
    // 1 exp2 pair in 8 on the FMA pipe (0, 1, 2, 3 in 8 measured within 1%)
    launch_pdl(k_attn_ps<1>, dim3(grid), dim3(PP_THREADS), PS_SMEM_BYTES, st, pm, rows, a.n0, a.n1, a.heads,
               scale_log2, a.out, a.ldo);
  }
  count_launch();
}

}  // namespace bp
