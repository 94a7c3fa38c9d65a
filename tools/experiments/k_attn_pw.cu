// EXPERIMENT (not built): the 128-key-tile pair attention of round 2, kept as
// the record behind profiles/r02e_attention_128key.md. It was a drop-in for
// attn_sm100.cu's anonymous namespace (launch_attn_tc variants 5-8 selected
// the kPoly8 = 1, 2, 0, 3 instantiations with seg_maps(32, PWK, ...)); it
// lost to k_attn_pp2 and was removed from the product.
// ============================================================================
// Variant 5: k_attn_pw -- 128-key tiles on a CTA pair, one S buffer per tile
// ============================================================================
// k_attn_pp2's QK^T (M256 N64 K16 per instruction) reads 4 KB of Q and 1 KB
// of K from each CTA's shared memory per 32-cycle step, 40 cycles at 128 B /
// clk: its tensor floor per 64 keys is 1152 cycles instead of 1024. Here a K
// tile holds 128 keys and a tile's S is written by two M256 N64 halves:
//   TMEM: S_A [0,128) S_B [128,256) O_A [256,384) O_B [384,512)
//   S_x columns [0,64) = keys 0..63 (QK "lo"), [64,128) = keys 64..127 ("hi");
//   P_x(j) (bf16 pairs) is written over the hi half: keys 0..63 at [64,96),
//   keys 64..127 at [96,128).
// Because P never touches the lo half, QK_lo_x(j + 1) is issued as soon as the
// softmax warps have loaded S_x(j) into registers (s_free), overlapping their
// exponentials; only QK_hi_x(j + 1) waits behind PV_x(j) (WAR on P, in issue
// order on the tensor pipe). P is released in two 64-key halves (p_full[x][h]),
// so PV_x(j)'s first half overlaps the second half's exponentials. A tile's
// serial chain is then softmax -> PV_hi -> QK_hi (512 tensor cycles), while
// the two tiles keep 2048 tensor cycles per 128 keys queued.
// Each CTA stages 64 keys of a tile as two 32-key runs, rows [32 r, 32 r + 32)
// and [64 + 32 r, ...) of the tile for CTA r, so that the lo MMA (first 32
// rows of both CTAs) covers keys 0..63 in order and the hi MMA keys 64..127.
// The commit of S_x(j + 1) follows PV_x(j) in issue order, so when a softmax
// warp sees S_x(j + 1) its O holds PV_x(j) and can be rescaled without a PV
// barrier; pv_done[x] fires once, after the tile's last PV, for the epilogue.
constexpr int PWK = 128;                             // keys per K/V tile
constexpr uint32_t PW_KR = 32 * 64 * 2;             // [32 keys][64 d] box, 4 KB
constexpr uint32_t PW_KH = 2 * PW_KR;               // one d-half of this CTA's 64 keys, 8 KB
constexpr uint32_t PW_KT = 2 * PW_KH;               // 16 KB
constexpr uint32_t PW_VT = PWK * 64 * 2;            // [128 keys][64 d] V half (this CTA's d columns), 16 KB
constexpr int PW_ST = 4;                            // K / V ring depth (tiles of 128 keys)
constexpr uint32_t PW_Q = 0;
constexpr uint32_t PW_K = PW_Q + 2 * TILE;
constexpr uint32_t PW_V = PW_K + PW_ST * PW_KT;
constexpr uint32_t PW_BAR = PW_V + PW_ST * PW_VT;
constexpr uint32_t PW_SMEM_BYTES = PW_BAR + 256 + 1024;
static_assert(PW_SMEM_BYTES <= 232448, "128-key pair attention exceeds the 227 KB smem limit");

template <int kPoly8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PP_THREADS, 1)
    k_attn_pw(const __grid_constant__ AttnMapsP2 maps, int64_t rows, int64_t n0, int64_t n1, float scale_log2,
              bf16* __restrict__ out, int64_t ldo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PW_BAR);
  uint64_t* q_full = bars + 0;              // leader: both CTAs' Q
  uint64_t* k_full = bars + 1;              // [PW_ST] leader: both CTAs' keys
  uint64_t* k_empty = k_full + PW_ST;       // [PW_ST] each CTA (multicast commit)
  uint64_t* v_full = k_empty + PW_ST;       // [PW_ST] leader
  uint64_t* v_empty = v_full + PW_ST;       // [PW_ST] each CTA
  uint64_t* s_full = v_empty + PW_ST;       // [tile] each CTA
  uint64_t* s_free = s_full + 2;            // [tile] leader, 8 warp arrivals: S_x loaded to registers
  uint64_t* p_full = s_free + 2;            // [tile][half] leader, 8 warp arrivals
  uint64_t* pv_done = p_full + 4;           // [tile] each CTA, once per launch
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const int qpair = blockIdx.x, head = blockIdx.y;
  const int t0 = static_cast<int>((n0 + PWK - 1) / PWK);
  const int t1 = static_cast<int>((n1 + PWK - 1) / PWK);
  const int T = t0 + t1;
  constexpr uint16_t kBoth = 0x3;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&maps.q);
    tc::tma_prefetch(&maps.k1);
    tc::tma_prefetch(&maps.v1);
    tc::mbar_init(q_full, 1);
    for (int s = 0; s < PW_ST; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], 1);
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_free[i], 8);
      tc::mbar_init(&pv_done[i], 1);
    }
    for (int i = 0; i < 4; ++i) tc::mbar_init(&p_full[i], 8);
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
    // ---- TMA producer (both CTAs): own Q tiles, own key runs / V columns -> leader's barriers ----
    const uint32_t lq = tc::mapa_shared(tc::smem_u32(q_full), 0);
    if (rank == 0) tc::mbar_arrive_expect_tx_elect(q_full, 4 * TILE);
    for (int x = 0; x < 2; ++x) {
      const int qrow = qpair * 2 * BQ + x * BQ;
      tc::tma_load_2d_cg2_elect(smem + PW_Q + x * TILE, &maps.q, lq, head * kDh, qrow);
      tc::tma_load_2d_cg2_elect(smem + PW_Q + x * TILE + HALF, &maps.q, lq, head * kDh + 64, qrow);
    }
    for (int j = 0; j < T; ++j) {
      const bool seg0 = j < t0;
      const int row0 = (seg0 ? j : j - t0) * PWK + static_cast<int>(rank) * 32;
      const int s = j % PW_ST;
      const uint32_t ph = ((j / PW_ST) & 1) ^ 1;
      tc::mbar_wait_cluster(&k_empty[s], ph);
      uint8_t* kd = smem + PW_K + s * PW_KT;
      const CUtensorMap* mk = seg0 ? &maps.k0 : &maps.k1;
      const uint32_t lk = tc::mapa_shared(tc::smem_u32(&k_full[s]), 0);
      if (rank == 0) tc::mbar_arrive_expect_tx_elect(&k_full[s], 2 * PW_KT);
      for (int dh = 0; dh < 2; ++dh)
        for (int run = 0; run < 2; ++run)
          tc::tma_load_2d_cg2_elect(kd + dh * PW_KH + run * PW_KR, mk, lk, head * kDh + dh * 64, row0 + run * 64);
      tc::mbar_wait_cluster(&v_empty[s], ph);
      uint8_t* vd = smem + PW_V + s * PW_VT;
      const CUtensorMap* mv = seg0 ? &maps.v0 : &maps.v1;
      const uint32_t lv = tc::mapa_shared(tc::smem_u32(&v_full[s]), 0);
      if (rank == 0) tc::mbar_arrive_expect_tx_elect(&v_full[s], 2 * PW_VT);
      tc::tma_load_2d_cg2_elect(vd, mv, lv, head * kDh + static_cast<int>(rank) * 64, row0 - static_cast<int>(rank) * 32);
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---- MMA issuer (leader) ---------------------------------------------------------------
      constexpr uint32_t idesc_s = tc::idesc_bf16(2 * BQ, 64, 0, 0);   // Q x K^T half, M256 N64
      constexpr uint32_t idesc_o = tc::idesc_bf16(2 * BQ, kDh, 0, 1);  // P (TMEM) x V, M256 N128
      const uint32_t q_base = tc::smem_u32(smem + PW_Q);
      auto qk = [&](int x, int j, int hi) {  // keys 64 hi .. 64 hi + 63 of tile j into S_x
        const uint32_t k_addr = tc::smem_u32(smem + PW_K + (j % PW_ST) * PW_KT) + static_cast<uint32_t>(hi) * PW_KR;
        tc::mma_ss_k128_cg2_elect<HALF / 16, PW_KH / 16>(tmem + static_cast<uint32_t>(x * PWK + hi * 64),
                                                         tc::desc_sw128(q_base + x * TILE, 1024, 16),
                                                         tc::desc_sw128(k_addr, 1024, 16), idesc_s, 0u);
        if (hi) tc::mma_commit_cg2_multicast_elect(&s_full[x], kBoth);
      };
      tc::mbar_wait_cluster(q_full, 0);
      if (T > 0) {
        tc::mbar_wait_cluster(&k_full[0], 0);
        tc::fence_after_sync();
        for (int x = 0; x < 2; ++x) {
          qk(x, 0, 0);
          qk(x, 0, 1);
        }
        tc::mma_commit_cg2_multicast_elect(&k_empty[0], kBoth);
      }
      for (int j = 0; j < T; ++j) {
        const int s = j % PW_ST;
        const bool more = j + 1 < T;
        const uint32_t v_addr = tc::smem_u32(smem + PW_V + s * PW_VT);
        for (int x = 0; x < 2; ++x) {
          const uint32_t o_tm = tmem + 256u + static_cast<uint32_t>(x * kDh);
          const uint32_t p_tm = tmem + static_cast<uint32_t>(x * PWK + 64);
          if (more) {  // S_x lo of tile j + 1 once the softmax holds S_x(j) in registers
            if (x == 0) tc::mbar_wait_cluster(&k_full[(j + 1) % PW_ST], ((j + 1) / PW_ST) & 1);
            tc::mbar_wait_cluster(&s_free[x], j & 1);
            tc::fence_after_sync();
            qk(x, j + 1, 0);
          }
          if (x == 0) tc::mbar_wait_cluster(&v_full[s], (j / PW_ST) & 1);
          for (int h = 0; h < 2; ++h) {
            tc::mbar_wait_cluster(&p_full[x * 2 + h], j & 1);
            tc::fence_after_sync();
            tc::mma_ts_k64_cg2_elect<2048 / 16>(o_tm, p_tm + static_cast<uint32_t>(h * 32),
                                                tc::desc_sw128(v_addr + static_cast<uint32_t>(h * 8192), 1024, PW_VT),
                                                idesc_o, (j > 0 || h > 0) ? 1u : 0u);
          }
          if (x == 1) tc::mma_commit_cg2_multicast_elect(&v_empty[s], kBoth);
          if (more) {
            qk(x, j + 1, 1);  // over P_x(j): behind PV_x(j) on the in-order tensor pipe
            if (x == 1) tc::mma_commit_cg2_multicast_elect(&k_empty[(j + 1) % PW_ST], kBoth);
          } else {
            tc::mma_commit_cg2_multicast_elect(&pv_done[x], kBoth);
          }
        }
      }
    }
  } else {
    // ---- softmax + epilogue of tile x (each CTA, its own rows) ------------------------------
    const int x = (warp - 2) >> 2;
    const int qq = warp & 3;
    const uint32_t lane_off = static_cast<uint32_t>(qq * 32) << 16;
    const uint32_t tm_s = tmem + lane_off + static_cast<uint32_t>(x * PWK);
    const uint32_t tm_o = tmem + lane_off + 256u + static_cast<uint32_t>(x * kDh);
    const float2 sc2 = make_float2(scale_log2, scale_log2);
    float m_used = -INFINITY;
    float2 l2 = make_float2(0.f, 0.f);
    const int n0i = static_cast<int>(n0), n1i = static_cast<int>(n1);
    const uint32_t p_full_leader = tc::mapa_shared(tc::smem_u32(&p_full[x * 2]), 0);
    const uint32_t s_free_leader = tc::mapa_shared(tc::smem_u32(&s_free[x]), 0);
    for (int j = 0; j < T; ++j) {
      const bool seg0 = j < t0;
      const int row0 = (seg0 ? j : j - t0) * PWK;
      const int rem = (seg0 ? n0i : n1i) - row0;
      tc::mbar_wait_cluster(&s_full[x], j & 1);
      tc::fence_after_sync();
      uint32_t sr[128];
      tc::tmem_ld32(tm_s, *reinterpret_cast<uint32_t(*)[32]>(&sr[0]));
      tc::tmem_ld32(tm_s + 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[32]));
      tc::tmem_ld32(tm_s + 64, *reinterpret_cast<uint32_t(*)[32]>(&sr[64]));
      tc::tmem_ld32(tm_s + 96, *reinterpret_cast<uint32_t(*)[32]>(&sr[96]));
      tc::tmem_ld_wait();
      // S_x(j) is in registers: the lo half may be overwritten by QK_lo_x(j + 1)
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(s_free_leader);
      if (rem < PWK) {  // keys past the segment end (a segment's last tile)
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c >= rem) sr[c] = __float_as_uint(-INFINITY);
      }
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < 128; c += 8) {
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
      float2 ls_a = make_float2(0.f, 0.f), ls_b = make_float2(0.f, 0.f);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int e = h * 64 + 2 * c;
          const float2 xv = __ffma2_rn(make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), sc2, neg_m2);
          const float2 p = (c & 7) >= 8 - kPoly8 ? ex2_poly2(xv) : make_float2(ex2(xv.x), ex2(xv.y));
          if (c & 1) ls_b = __fadd2_rn(ls_b, p);
          else ls_a = __fadd2_rn(ls_a, p);
          pk[c] = pack_bf16(p.x, p.y);
        }
        // O holds PV_x(j - 1) (its commit preceded S_x(j)'s): rescale it
        // before the first half of P releases PV_x(j)
        if (h == 0 && j >= 1 && __any_sync(0xffffffffu, need)) {
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
        tc::tmem_st32(tm_s + static_cast<uint32_t>(64 + h * 32), pk);
        tc::tmem_st_wait();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(p_full_leader + static_cast<uint32_t>(h * 8));
      }
      l2 = __ffma2_rn(l2, make_float2(corr, corr), __fadd2_rn(ls_a, ls_b));
      m_used = m_new;
    }
    if (T >= 1) {
      tc::mbar_wait_cluster(&pv_done[x], 0);
      tc::fence_after_sync();
    }
    const int64_t row = static_cast<int64_t>(qpair) * 2 * BQ + x * BQ + qq * 32 + lane;
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

