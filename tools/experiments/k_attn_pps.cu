// EXPERIMENT (not built): k_attn_ps's persistent schedule on a cta_group::2
// pair (round 2), kept as the record behind
// profiles/r02f_cross_attention_pair.md. Correct on every kernel-test shape
// (45/45 with impl 3) but 932 vs 951 TF/s for k_attn_ps at q 18720 x kv 512,
// so it was removed. Drop-in for attn_sm100.cu's anonymous namespace; launch:
//
//   } else if (variant == 3) {  // persistent ping-pong on a CTA pair over (query quad, head) items
//     set_smem_attr(k_attn_pps<1>, PQ_SMEM_BYTES);
//     AttnMapsP2 pm;
//     pm.q = map_for(a.q, rows, H, a.ldq);
//     seg_maps(32, PBK, &pm.k0, &pm.v0, &pm.k1, &pm.v1);
//     pm.o = map_for(a.out, rows, H, a.ldo);
//     const int64_t items = ((rows + 4 * BQ - 1) / (4 * BQ)) * a.heads;
//     const int64_t avail = (kNumSms - sm_reserve()) / 2;
//     const unsigned clusters = static_cast<unsigned>(items < avail ? items : avail);
//     launch_pdl(k_attn_pps<1>, dim3(2 * clusters), dim3(PP_THREADS), PQ_SMEM_BYTES, st, pm, rows, a.n0, a.n1, a.heads,
//                scale_log2);

// ============================================================================
// k_attn_pps: k_attn_ps's persistent schedule on a cta_group::2 pair
// ============================================================================
// The single-CTA cross-attention kernel's QK^T (M128 N64 K16 per instruction)
// reads 4 KB of Q and 2 KB of K from shared memory per 32-cycle step: 48
// cycles at 128 B / clk, so its QK^T runs at 2/3 of the MMA rate. On a CTA
// pair the same step is M256 N64 with 4 KB + 1 KB per CTA (40 cycles), and
// each CTA stages and reads from L2 only half of every K / V tile (k_attn_pp2's
// split: 32 keys of K, 64 head-dim columns of V). A work item is (query quad,
// head): 512 query rows, CTA r owning rows [256 r, 256 r + 256) of the quad as
// its tiles A and B. The cluster walks items persistently exactly like
// k_attn_ps: Q double-buffered per CTA, K / V rings continuing across items,
// the next item's first two QK^T issued behind the current item's last PV,
// every phase derived from the global step counter g or the item counter n,
// O staged in the item's Q buffer and written by TMA stores. The leader CTA
// issues every MMA; both CTAs' TMA loads complete on the leader's full
// barriers; every commit is multicast to both CTAs; P-ready is one remote
// arrive per softmax warp on the leader (8 per tile and buffer).
constexpr int PQ_KST = 5, PQ_VST = 5;
constexpr uint32_t PQ_Q = 0;                        // two Q buffers x (Q_A, Q_B): 128 KB
constexpr uint32_t PQ_K = PQ_Q + 4 * TILE;
constexpr uint32_t PQ_V = PQ_K + PQ_KST * P2_KT;
constexpr uint32_t PQ_BAR = PQ_V + PQ_VST * P2_VT;
constexpr uint32_t PQ_SMEM_BYTES = PQ_BAR + 256 + 1024;
static_assert(PQ_SMEM_BYTES <= 232448, "persistent pair attention exceeds the 227 KB smem limit");

template <int kPoly8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PP_THREADS, 1)
    k_attn_pps(const __grid_constant__ AttnMapsP2 maps, int64_t rows, int64_t n0, int64_t n1, int heads,
               float scale_log2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PQ_BAR);
  uint64_t* q_full = bars + 0;              // [Q buffer] leader: both CTAs' Q tiles
  uint64_t* q_empty = q_full + 2;           // [Q buffer] each CTA: its two tiles' O stores have read it
  uint64_t* k_full = q_empty + 2;           // [PQ_KST] leader
  uint64_t* k_empty = k_full + PQ_KST;      // [PQ_KST] each CTA (multicast commit)
  uint64_t* v_full = k_empty + PQ_KST;      // [PQ_VST] leader
  uint64_t* v_empty = v_full + PQ_VST;      // [PQ_VST] each CTA
  uint64_t* s_full = v_empty + PQ_VST;      // [tile][buffer] each CTA
  uint64_t* p_full = s_full + 4;            // [tile][buffer] leader, 8 warp arrivals
  uint64_t* pv_done = p_full + 4;           // [tile] each CTA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);

  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const int cluster = static_cast<int>(blockIdx.x >> 1), nclusters = static_cast<int>(gridDim.x >> 1);
  const int t0 = static_cast<int>((n0 + PBK - 1) / PBK);
  const int t1 = static_cast<int>((n1 + PBK - 1) / PBK);
  const int T = t0 + t1;
  const int nquads = static_cast<int>((rows + 4 * BQ - 1) / (4 * BQ));
  const int items = nquads * heads;
  constexpr uint16_t kBoth = 0x3;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&maps.q);
    tc::tma_prefetch(&maps.k1);
    tc::tma_prefetch(&maps.v1);
    tc::tma_prefetch(&maps.o);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&q_full[b], 1);
      tc::mbar_init(&q_empty[b], 2);
    }
    for (int s = 0; s < PQ_KST; ++s) {
      tc::mbar_init(&k_full[s], 1);
      tc::mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < PQ_VST; ++s) {
      tc::mbar_init(&v_full[s], 1);
      tc::mbar_init(&v_empty[s], 1);
    }
    for (int i = 0; i < 4; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], 8);
    }
    tc::mbar_init(&pv_done[0], 1);
    tc::mbar_init(&pv_done[1], 1);
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
    // ---- TMA producer (both CTAs): own Q tiles, own K / V halves -> leader's barriers -------
    auto load_q = [&](int n, int item) {
      const int b = n & 1;
      tc::mbar_wait(&q_empty[b], ((n >> 1) & 1) ^ 1);
      const int quad = item % nquads, head = item / nquads;
      uint8_t* qd = smem + PQ_Q + b * 2 * TILE;
      const uint32_t lq = tc::mapa_shared(tc::smem_u32(&q_full[b]), 0);
      if (rank == 0) tc::mbar_arrive_expect_tx_elect(&q_full[b], 4 * TILE);
      for (int x = 0; x < 2; ++x) {
        const int qrow = quad * 4 * BQ + static_cast<int>(rank) * 2 * BQ + x * BQ;
        tc::tma_load_2d_cg2_elect(qd + x * TILE, &maps.q, lq, head * kDh, qrow);
        tc::tma_load_2d_cg2_elect(qd + x * TILE + HALF, &maps.q, lq, head * kDh + 64, qrow);
      }
    };
    int g = 0, n = 0;
    if (cluster < items) load_q(0, cluster);
    for (int item = cluster; item < items; item += nclusters, ++n) {
      const int head = item / nquads;
      for (int j = 0; j < T; ++j, ++g) {
        const bool seg0 = j < t0;
        const int row0 = (seg0 ? j : j - t0) * PBK;
        const int ks = g % PQ_KST, vs = g % PQ_VST;
        tc::mbar_wait_cluster(&k_empty[ks], ((g / PQ_KST) & 1) ^ 1);
        uint8_t* kd = smem + PQ_K + ks * P2_KT;
        const CUtensorMap* mk = seg0 ? &maps.k0 : &maps.k1;
        const uint32_t lk = tc::mapa_shared(tc::smem_u32(&k_full[ks]), 0);
        if (rank == 0) tc::mbar_arrive_expect_tx_elect(&k_full[ks], 2 * P2_KT);
        tc::tma_load_2d_cg2_elect(kd, mk, lk, head * kDh, row0 + static_cast<int>(rank) * 32);
        tc::tma_load_2d_cg2_elect(kd + P2_KH, mk, lk, head * kDh + 64, row0 + static_cast<int>(rank) * 32);
        tc::mbar_wait_cluster(&v_empty[vs], ((g / PQ_VST) & 1) ^ 1);
        uint8_t* vd = smem + PQ_V + vs * P2_VT;
        const CUtensorMap* mv = seg0 ? &maps.v0 : &maps.v1;
        const uint32_t lv = tc::mapa_shared(tc::smem_u32(&v_full[vs]), 0);
        if (rank == 0) tc::mbar_arrive_expect_tx_elect(&v_full[vs], 2 * P2_VT);
        tc::tma_load_2d_cg2_elect(vd, mv, lv, head * kDh + static_cast<int>(rank) * 64, row0);
        if (j == (T > 1 ? 1 : 0) && item + nclusters < items) load_q(n + 1, item + nclusters);
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      // ---- MMA issuer (leader) ---------------------------------------------------------------
      constexpr uint32_t idesc_s = tc::idesc_bf16(2 * BQ, PBK, 0, 0);  // Q x K^T, M256 N64
      constexpr uint32_t idesc_o = tc::idesc_bf16(2 * BQ, kDh, 0, 1);  // P (TMEM) x V, M256 N128
      int g = 0, n = 0;
      for (int item = cluster; item < items; item += nclusters, ++n) {
        const uint32_t q_base = tc::smem_u32(smem + PQ_Q + (n & 1) * 2 * TILE);
        auto qk_pair = [&](int gg) {  // S_x(gg) into buffer gg & 1 of both tiles
          tc::mbar_wait_cluster(&k_full[gg % PQ_KST], (gg / PQ_KST) & 1);
          tc::fence_after_sync();
          const uint32_t k_addr = tc::smem_u32(smem + PQ_K + (gg % PQ_KST) * P2_KT);
          for (int x = 0; x < 2; ++x) {
            const uint32_t d = tmem + static_cast<uint32_t>(x * 2 * PBK + (gg & 1) * PBK);
            tc::mma_ss_k128_cg2_elect<HALF / 16, P2_KH / 16>(d, tc::desc_sw128(q_base + x * TILE, 1024, 16),
                                                             tc::desc_sw128(k_addr, 1024, 16), idesc_s, 0u);
            tc::mma_commit_cg2_multicast_elect(&s_full[x * 2 + (gg & 1)], kBoth);
          }
          tc::mma_commit_cg2_multicast_elect(&k_empty[gg % PQ_KST], kBoth);
        };
        tc::mbar_wait_cluster(&q_full[n & 1], (n >> 1) & 1);
        tc::fence_after_sync();
        if (T > 0) qk_pair(g);
        if (T > 1) qk_pair(g + 1);
        for (int j = 0; j < T; ++j) {
          const int gg = g + j;
          tc::mbar_wait_cluster(&v_full[gg % PQ_VST], (gg / PQ_VST) & 1);
          const uint32_t v_addr = tc::smem_u32(smem + PQ_V + (gg % PQ_VST) * P2_VT);
          for (int x = 0; x < 2; ++x) {
            tc::mbar_wait_cluster(&p_full[x * 2 + (gg & 1)], (gg >> 1) & 1);
            tc::fence_after_sync();
            const uint32_t p_tm = tmem + static_cast<uint32_t>(x * 2 * PBK + (gg & 1) * PBK);
            tc::mma_ts_k64_cg2_elect<2048 / 16>(tmem + 256 + x * kDh, p_tm, tc::desc_sw128(v_addr, 1024, P2_VT),
                                                idesc_o, j > 0 ? 1u : 0u);
            tc::mma_commit_cg2_multicast_elect(&pv_done[x], kBoth);
          }
          tc::mma_commit_cg2_multicast_elect(&v_empty[gg % PQ_VST], kBoth);
          if (j + 2 < T) qk_pair(gg + 2);  // S buffer gg & 1 is free once PV(gg) is issued (in-order)
        }
        g += T;
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
    const int n0i = static_cast<int>(n0), n1i = static_cast<int>(n1);
    const uint32_t p_full_leader = tc::mapa_shared(tc::smem_u32(&p_full[x * 2]), 0);
    int g = 0, n = 0;
    for (int item = cluster; item < items; item += nclusters, ++n) {
      const int quad = item % nquads, head = item / nquads;
      float m_used = -INFINITY;
      float2 l2 = make_float2(0.f, 0.f);
      for (int j = 0; j < T; ++j) {
        const int gg = g + j;
        const int b = gg & 1;
        const bool seg0 = j < t0;
        const int row0 = (seg0 ? j : j - t0) * PBK;
        const int rem = (seg0 ? n0i : n1i) - row0;
        const uint32_t tm_s = tmem + lane_off + static_cast<uint32_t>(x * 2 * PBK + b * PBK);
        tc::mbar_wait_cluster(&s_full[x * 2 + b], (gg >> 1) & 1);
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
        // every PV completion is observed (one phase per step), so the parity
        // waits stay exact across items; O must hold PV(gg - 1) before it is
        // rescaled
        if (j >= 1) tc::mbar_wait_cluster(&pv_done[x], (gg - 1) & 1);
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
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(p_full_leader + static_cast<uint32_t>(b * 8));
      }
      g += T;
      if (T >= 1) {
        tc::mbar_wait_cluster(&pv_done[x], (g - 1) & 1);
        tc::fence_after_sync();
      }
      // O / l as bf16 into this item's Q buffer (its last QK^T completed
      // before the last PV), in the output map's 128B-swizzled layout, then
      // two TMA stores per tile; the buffer goes back to this CTA's producer
      // (q_empty) once the stores have read it
      const float inv_l = 1.f / (l2.x + l2.y);
      uint8_t* stage_o = smem + PQ_Q + (n & 1) * 2 * TILE + x * TILE;
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
        const int qrow = quad * 4 * BQ + static_cast<int>(rank) * 2 * BQ + x * BQ;
        tc::tma_store_2d(&maps.o, stage_o, head * kDh, qrow);
        tc::tma_store_2d(&maps.o, stage_o + HALF, head * kDh + 64, qrow);
        tc::bulk_commit_group();
        tc::bulk_wait_group_read<0>();
        tc::mbar_arrive(&q_empty[n & 1]);
      }
      // the next item's P arrives (after these TMEM reads completed) gate the
      // leader's first PV of that item, which overwrites O
      tc::fence_before_sync();
    }
    if (qq == 0 && lane == 0) tc::bulk_wait_group<0>();  // the O stores are complete before exit
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::cluster_sync();  // the peer's MMAs / arrivals / TMA into this CTA are done
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc_cg2<512>(tmem);
  }
}

