// Stage: device-resident ModelChunk + forward_chunk. See stage.hpp.
#include "stage.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

#include "kernels_bf16.cuh"
#include "kernels_simt.cuh"
#include "kernels_wan.cuh"
#include "schedule.hpp"

namespace bp {

namespace {

// Weight roles (model.cpp:17-24); the numeric values key the streams.
enum Role : uint64_t {
  kWq = 0, kWk, kWv, kWo, kCq, kCk, kCv, kCo, kW1, kW2,
  kLn1G, kLn1B, kLn2G, kLn2B, kLn3G, kLn3B,
  kPatchify = 100, kHead = 101
};
// Wan-block roles (oracle/wan_oracle.py): per layer, and global ones keyed by
// layer = L like kPatchify / kHead.
enum WanRole : uint64_t {
  kWanMod = 200, kWanQn, kWanKn, kWanCqn, kWanCkn,
  kWanT1 = 210, kWanTb1, kWanT2, kWanTb2, kWanTp, kWanTpb, kWanHmod
};

size_t align256(size_t n) { return (n + 255) & ~static_cast<size_t>(255); }

}  // namespace

Stage::Stage(int device, const bp_model_desc& m, uint64_t seed_model, uint64_t seed_context, int begin,
             int end, int precision, cudaStream_t stream)
    : device_(device), prec_(precision), m_(m), begin_(begin), end_(end), stream_(stream) {
  validate_model(m);
  if (begin < 0 || end > m.layers || begin >= end)
    fail(BP_ERR_CONFIG, "bad layer range [" + std::to_string(begin) + "," + std::to_string(end) +
                            ") for L=" + std::to_string(m.layers));
  if (prec_ < BP_PREC_F64 || prec_ > BP_PREC_BF16) fail(BP_ERR_CONFIG, "unknown precision");
  h_ = m.hidden;
  heads_ = m.heads;
  dh_ = h_ / heads_;
  F_ = ffn_width(m);
  C_ = m.channels;
  tpf_ = m.height * m.width;
  Lc_ = m.context_len;
  wan_ = m.block == BP_BLOCK_WAN;
  wan_rope_split(dh_, &wnt_, &wnh_);
  if (wan_ && prec_ == BP_PREC_BF16 && F_ < 2 * h_) fail(BP_ERR_CONFIG, "wan block on the bf16 path needs ffn >= 2 hidden");
  if (prec_ == BP_PREC_BF16) {
    if (h_ % 64 != 0 || F_ % 64 != 0) fail(BP_ERR_CONFIG, "bf16 path needs hidden and ffn multiples of 64");
    if (dh_ % 16 != 0 || dh_ > 256) fail(BP_ERR_CONFIG, "bf16 path needs head dim % 16 == 0 and <= 256");
  }
  BP_CUDA(cudaSetDevice(device_));
  if (!stream_) {
    BP_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    own_stream_ = true;
  }
  build_weights(seed_model, seed_context);
}

Stage::~Stage() {
  cudaSetDevice(device_);
  cudaStreamSynchronize(stream_);
  for (cudaEvent_t e : prof_pool_) cudaEventDestroy(e);
  if (own_stream_) cudaStreamDestroy(stream_);
}

size_t Stage::act_bytes() const { return prec_ == BP_PREC_F64 ? 8 : 4; }

void Stage::build_weights(uint64_t seed_model, uint64_t seed_context) {
  seed_model_ = seed_model;
  const int nl = end_ - begin_;
  const bool bf = prec_ == BP_PREC_BF16;
  const size_t te = prec_ == BP_PREC_F64 ? 8 : 4;  // SIMT element / fp32 side tensors
  const size_t me = bf ? 2 : te;                    // matrix element
  const size_t hh = static_cast<size_t>(h_) * h_;
  const size_t hF = static_cast<size_t>(h_) * F_;
  struct Off { size_t wqkv, wo, cq, co, w1, w2, ln, ctx_kv; };
  std::vector<Off> offs(static_cast<size_t>(nl));
  size_t at = 0;
  for (int l = 0; l < nl; ++l) {
    Off& o = offs[static_cast<size_t>(l)];
    o.wqkv = at; at += align256(3 * hh * me);
    o.wo = at; at += align256(hh * me);
    o.cq = at; at += align256(hh * me);
    o.co = at; at += align256(hh * me);
    o.w1 = at; at += align256(hF * me);
    o.w2 = at; at += align256(hF * me);
    o.ln = at; at += align256(6 * static_cast<size_t>(h_) * te);
    o.ctx_kv = at; at += align256(static_cast<size_t>(Lc_) * 2 * h_ * me);
  }
  size_t off_in = 0, off_out = 0;
  if (is_first()) { off_in = at; at += align256(static_cast<size_t>(C_) * h_ * 8); }
  if (is_last()) { off_out = at; at += align256(static_cast<size_t>(h_) * C_ * te); }
  // Wan block: per-layer vectors [nl][10h], the timestep MLP, the head modulation (T)
  const size_t H1 = static_cast<size_t>(h_);
  size_t off_wanv = 0, off_t1 = 0, off_tb1 = 0, off_t2 = 0, off_tb2 = 0, off_tp = 0, off_tpb = 0, off_hmod = 0;
  if (wan_) {
    off_wanv = at; at += align256(static_cast<size_t>(nl) * 10 * H1 * te);
    off_t1 = at; at += align256(kWanFreqDim * H1 * te);
    off_tb1 = at; at += align256(H1 * te);
    off_t2 = at; at += align256(H1 * H1 * te);
    off_tb2 = at; at += align256(H1 * te);
    off_tp = at; at += align256(6 * H1 * H1 * te);
    off_tpb = at; at += align256(6 * H1 * te);
    off_hmod = at; at += align256(2 * H1 * te);
  }
  weights_.alloc(at);
  char* base = weights_.as<char>();
  lw_.resize(static_cast<size_t>(nl));
  for (int l = 0; l < nl; ++l) {
    const Off& o = offs[static_cast<size_t>(l)];
    LayerW& w = lw_[static_cast<size_t>(l)];
    w.wqkv = base + o.wqkv; w.wo = base + o.wo; w.cq = base + o.cq; w.co = base + o.co;
    w.w1 = base + o.w1; w.w2 = base + o.w2; w.ln = base + o.ln; w.ctx_kv = base + o.ctx_kv;
  }
  if (is_first()) w_in_ = base + off_in;
  if (is_last()) w_out_ = base + off_out;
  if (wan_) {
    wanv_ = base + off_wanv;
    for (int l = 0; l < nl; ++l) lw_[static_cast<size_t>(l)].wan = base + off_wanv + static_cast<size_t>(l) * 10 * H1 * te;
    wg_ = WanGlobal{base + off_t1, base + off_tb1, base + off_t2, base + off_tb2, base + off_tp, base + off_tpb,
                    base + off_hmod};
  }

  // Scratch: fp64 draw buffer, context, and the cross K|V weights for hoisting.
  const size_t max_numel = std::max({hF, hh, static_cast<size_t>(Lc_) * h_,
                                     static_cast<size_t>(C_) * h_, wan_ ? 6 * hh : size_t{0}});
  DevBuf gen, ctx64;
  gen.alloc(max_numel * 8);
  ctx64.alloc(static_cast<size_t>(Lc_) * h_ * 8);
  double* g = gen.as<double>();
  cudaStream_t st = stream_;

  auto draw = [&](uint64_t layer, uint64_t role, int64_t numel, int64_t fan_in) {
    // draw (model.cpp:26-30): RandomSource(derive_seed(seed, {layer, role})), sigma 1/sqrt(fan_in)
    const uint64_t state = derive_seed2(seed_model, layer, role);
    launch_normal_fill(state, numel, 1.0 / std::sqrt(static_cast<double>(fan_in)), g, st);
  };
  // place an fp64 [rows, cols] draw into a matrix slot of this precision
  auto place_mat = [&](void* dst, int64_t rows, int64_t cols, int64_t ld, int64_t col_off, bool transposed_store) {
    if (bf) {
      // K-major weights: W^T [cols(out), rows(in)]; col_off counts output rows
      launch_place<bf16>(g, rows, cols, static_cast<bf16*>(dst) + col_off * rows, rows, 1, st);
    } else if (prec_ == BP_PREC_F64) {
      launch_place<double>(g, rows, cols, static_cast<double*>(dst) + col_off, ld, 0, st);
    } else {
      launch_place<float>(g, rows, cols, static_cast<float*>(dst) + col_off, ld, 0, st);
    }
    (void)transposed_store;
  };
  auto place_side = [&](void* dst, int64_t n, int64_t off) {  // fp32/fp64 vectors
    if (prec_ == BP_PREC_F64) launch_place<double>(g, 1, n, static_cast<double*>(dst) + off, n, 0, st);
    else launch_place<float>(g, 1, n, static_cast<float*>(dst) + off, n, 0, st);
  };

  // context (build_context, model.cpp:150-153): RandomSource(seed_context), sigma 1
  launch_normal_fill(seed_context, static_cast<int64_t>(Lc_) * h_, 1.0, ctx64.as<double>(), st);

  for (int l = 0; l < nl; ++l) {
    LayerW& w = lw_[static_cast<size_t>(l)];
    const uint64_t layer = static_cast<uint64_t>(begin_ + l);
    const int64_t H = h_;
    for (uint64_t r = kWq; r <= kWv; ++r) {
      draw(layer, r, H * H, H);
      place_mat(w.wqkv, H, H, 3 * H, static_cast<int64_t>(r) * H, true);
    }
    draw(layer, kWo, H * H, H); place_mat(w.wo, H, H, H, 0, true);
    draw(layer, kCq, H * H, H); place_mat(w.cq, H, H, H, 0, true);
    draw(layer, kCo, H * H, H); place_mat(w.co, H, H, H, 0, true);
    draw(layer, kW1, H * F_, H); place_mat(w.w1, H, F_, F_, 0, true);
    draw(layer, kW2, static_cast<int64_t>(F_) * H, F_); place_mat(w.w2, F_, H, H, 0, true);
    for (uint64_t r = kLn1G; r <= kLn3B; ++r) {
      draw(layer, r, H, H);
      place_side(w.ln, H, static_cast<int64_t>(r - kLn1G) * H);
    }
    if (wan_) {  // [mod 6h | gq | gk | gcq | gck]; RMSNorm gains are 1 + draw
      draw(layer, kWanMod, 6 * H, H);
      place_side(w.wan, 6 * H, 0);
      for (uint64_t r = kWanQn; r <= kWanCkn; ++r) {
        draw(layer, r, H, H);
        launch_elementwise(3, g, nullptr, H, 1.0, g, st);
        place_side(w.wan, H, (6 + static_cast<int64_t>(r - kWanQn)) * H);
      }
    }
  }
  if (wan_) {  // the per-frame timestep MLP (every stage computes it) and the head modulation
    const uint64_t L = static_cast<uint64_t>(m_.layers);
    const int64_t H = h_;
    draw(L, kWanT1, kWanFreqDim * H, kWanFreqDim); place_side(wg_.t1, kWanFreqDim * H, 0);
    draw(L, kWanTb1, H, kWanFreqDim); place_side(wg_.tb1, H, 0);
    draw(L, kWanT2, H * H, H); place_side(wg_.t2, H * H, 0);
    draw(L, kWanTb2, H, H); place_side(wg_.tb2, H, 0);
    draw(L, kWanTp, 6 * H * H, H); place_side(wg_.tp, 6 * H * H, 0);
    draw(L, kWanTpb, 6 * H, H); place_side(wg_.tpb, 6 * H, 0);
    draw(L, kWanHmod, 2 * H, H); place_side(wg_.hmod, 2 * H, 0);
    if (prec_ == BP_PREC_BF16) {  // static RoPE tables of the token grid: (cos, sin)(pos * 10000^(-j / nh))
      std::vector<float2> yt(static_cast<size_t>(m_.height) * wnh_), xt(static_cast<size_t>(m_.width) * wnh_);
      for (int p = 0; p < std::max(m_.height, m_.width); ++p)
        for (int j = 0; j < wnh_; ++j) {
          const double a = p * std::pow(10000.0, -static_cast<double>(j) / wnh_);
          const float2 cs = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
          if (p < m_.height) yt[static_cast<size_t>(p) * wnh_ + j] = cs;
          if (p < m_.width) xt[static_cast<size_t>(p) * wnh_ + j] = cs;
        }
      wytab_.alloc(std::max<size_t>(yt.size(), 1) * sizeof(float2));
      wxtab_.alloc(std::max<size_t>(xt.size(), 1) * sizeof(float2));
      BP_CUDA(cudaMemcpyAsync(wytab_.p, yt.data(), yt.size() * sizeof(float2), cudaMemcpyHostToDevice, st));
      BP_CUDA(cudaMemcpyAsync(wxtab_.p, xt.data(), xt.size() * sizeof(float2), cudaMemcpyHostToDevice, st));
      BP_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
    }
  }
  hoist_context(ctx64.as<double>());
  if (is_first()) {
    const uint64_t state = derive_seed2(seed_model, static_cast<uint64_t>(m_.layers), kPatchify);
    launch_normal_fill(state, static_cast<int64_t>(C_) * h_, 1.0 / std::sqrt(static_cast<double>(C_)),
                       static_cast<double*>(w_in_), st);
  }
  if (is_last()) {
    draw(static_cast<uint64_t>(m_.layers), kHead, static_cast<int64_t>(h_) * C_, h_);
    if (prec_ == BP_PREC_F64) launch_place<double>(g, h_, C_, static_cast<double*>(w_out_), C_, 0, st);
    else launch_place<float>(g, h_, C_, static_cast<float*>(w_out_), C_, 0, st);
  }
  // Embedding frequencies pow(10000, -2i/h) (model.cpp:158), computed with the
  // host libm so they match the reference bit-for-bit.
  std::vector<double> fr(static_cast<size_t>((h_ + 1) / 2));
  for (size_t i = 0; i < fr.size(); ++i) fr[i] = std::pow(10000.0, -2.0 * static_cast<double>(i) / h_);
  freq_.alloc(fr.size() * 8);
  BP_CUDA(cudaMemcpyAsync(freq_.p, fr.data(), fr.size() * 8, cudaMemcpyHostToDevice, st));
  if (is_first() && prec_ == BP_PREC_F32 && wan_) {
    winT_.alloc(static_cast<size_t>(C_) * h_ * 4);
    launch_convert<double, float>(static_cast<const double*>(w_in_), winT_.as<float>(), static_cast<int64_t>(C_) * h_, st);
  }
  if (is_first() && prec_ == BP_PREC_BF16) {
    w_in32_.alloc(static_cast<size_t>(C_) * h_ * 4);
    launch_convert<double, float>(static_cast<const double*>(w_in_), w_in32_.as<float>(),
                                  static_cast<int64_t>(C_) * h_, st);
    ttab_.alloc(static_cast<size_t>(tpf_) * (h_ / 2) * 16);
    launch_embed_table(freq_.as<double>(), h_, tpf_, ttab_.as<double>(), st);
  }
  BP_CUDA(cudaStreamSynchronize(st));
}

// Cross-attention K|V of the context, hoisted out of the per-pass loop
// (model.cpp:216-217 recomputes ctx@Ck, ctx@Cv every pass; it is constant).
// Ck/Cv are re-drawn from (seed, layer, role) so they need not stay resident.
void Stage::hoist_context(const double* ctx64) {
  const size_t te = prec_ == BP_PREC_F64 ? 8 : 4;
  const int64_t H = h_;
  const size_t hh = static_cast<size_t>(h_) * h_;
  DevBuf gen, ctxT, ckvT, kvT;
  gen.alloc(std::max(hh, static_cast<size_t>(Lc_) * 2 * h_) * 8);
  ctxT.alloc(static_cast<size_t>(Lc_) * h_ * te);
  ckvT.alloc(2 * hh * te);
  kvT.alloc(static_cast<size_t>(Lc_) * 2 * h_ * te);
  double* g = gen.as<double>();
  cudaStream_t st = stream_;
  if (prec_ == BP_PREC_F64) launch_place<double>(ctx64, Lc_, h_, ctxT.as<double>(), h_, 0, st);
  else launch_place<float>(ctx64, Lc_, h_, ctxT.as<float>(), h_, 0, st);
  for (int l = 0; l < end_ - begin_; ++l) {
    const LayerW& w = lw_[static_cast<size_t>(l)];
    for (uint64_t r = kCk; r <= kCv; ++r) {
      launch_normal_fill(derive_seed2(seed_model_, static_cast<uint64_t>(begin_ + l), r), H * H,
                         1.0 / std::sqrt(static_cast<double>(H)), g, st);
      const int64_t off = static_cast<int64_t>(r - kCk) * H;
      if (prec_ == BP_PREC_F64) launch_place<double>(g, H, H, ckvT.as<double>() + off, 2 * H, 0, st);
      else launch_place<float>(g, H, H, ckvT.as<float>() + off, 2 * H, 0, st);
    }
    // Wan block: the context keys are RMS-normalised (gain gck), no RoPE
    if (prec_ == BP_PREC_F64) {
      launch_matmul<double>(ctxT.as<double>(), H, ckvT.as<double>(), 2 * H, Lc_, 2 * h_, h_,
                            static_cast<double*>(w.ctx_kv), 2 * H, kEpiNone, nullptr, 0, st);
      if (wan_)
        launch_wan_qk<double>(static_cast<double*>(w.ctx_kv), 2 * H, Lc_, h_, heads_,
                              static_cast<const double*>(w.wan) + 9 * H, 1, 0, nullptr, 1, 1, 0, st);
    } else if (prec_ == BP_PREC_F32) {
      launch_matmul<float>(ctxT.as<float>(), H, ckvT.as<float>(), 2 * H, Lc_, 2 * h_, h_,
                           static_cast<float*>(w.ctx_kv), 2 * H, kEpiNone, nullptr, 0, st);
      if (wan_)
        launch_wan_qk<float>(static_cast<float*>(w.ctx_kv), 2 * H, Lc_, h_, heads_,
                             static_cast<const float*>(w.wan) + 9 * H, 1, 0, nullptr, 1, 1, 0, st);
    } else {
      launch_matmul<float>(ctxT.as<float>(), H, ckvT.as<float>(), 2 * H, Lc_, 2 * h_, h_, kvT.as<float>(), 2 * H,
                           kEpiNone, nullptr, 0, st);
      if (wan_)
        launch_wan_qk<float>(kvT.as<float>(), 2 * H, Lc_, h_, heads_, static_cast<const float*>(w.wan) + 9 * H, 1, 0,
                             nullptr, 1, 1, 0, st);
      launch_convert<float, double>(kvT.as<float>(), g, static_cast<int64_t>(Lc_) * 2 * H, st);
      launch_place<bf16>(g, Lc_, 2 * H, static_cast<bf16*>(w.ctx_kv), 2 * H, 0, st);
    }
  }
  BP_CUDA(cudaStreamSynchronize(st));
}

void Stage::set_context(const double* host, int64_t rows, int64_t cols) {
  if (rows != Lc_ || cols != h_) fail(BP_ERR_DIMENSION, "context must be [context_len, hidden]");
  BP_CUDA(cudaSetDevice(device_));
  DevBuf d;
  d.alloc(static_cast<size_t>(rows * cols) * 8);
  BP_CUDA(cudaMemcpyAsync(d.p, host, static_cast<size_t>(rows * cols) * 8, cudaMemcpyHostToDevice, stream_));
  hoist_context(d.as<double>());
}

// Host-provided prefix (reference KVCacheEntry / RecomputeEntry passed by the
// caller): fp64 on the device -> this stage's dtype, layer-major.
void Stage::load_host_prefix(int kind, const double* k64, const double* v64, int64_t rows) {
  const int nl = end_ - begin_;
  const size_t eb = prec_ == BP_PREC_F64 ? 8 : (prec_ == BP_PREC_F32 ? 4 : 2);
  const int64_t H = h_;
  host_rows_ = rows;
  host_kind_ = kind;
  if (kind == 3) {  // K|V per layer [rows][2h]
    hostpre_.reserve(static_cast<size_t>(nl) * rows * 2 * H * eb + 16);
    for (int l = 0; l < nl; ++l) {
      const int64_t base = static_cast<int64_t>(l) * rows * 2 * H;
      for (int kv = 0; kv < 2; ++kv) {
        const double* src = (kv ? v64 : k64) + static_cast<int64_t>(l) * rows * H;
        if (prec_ == BP_PREC_F64) launch_place<double>(src, rows, H, hostpre_.as<double>() + base + kv * H, 2 * H, 0, stream_);
        else if (prec_ == BP_PREC_F32) launch_place<float>(src, rows, H, hostpre_.as<float>() + base + kv * H, 2 * H, 0, stream_);
        else launch_place<bf16>(src, rows, H, hostpre_.as<bf16>() + base + kv * H, 2 * H, 0, stream_);
      }
    }
  } else {  // recorded layer inputs [rows][h] (fp32 on the bf16 path)
    const size_t xb = prec_ == BP_PREC_F64 ? 8 : 4;
    hostpre_.reserve(static_cast<size_t>(nl) * rows * H * xb + 16);
    if (prec_ == BP_PREC_F64) launch_place<double>(k64, nl * rows, H, hostpre_.as<double>(), H, 0, stream_);
    else launch_place<float>(k64, nl * rows, H, hostpre_.as<float>(), H, 0, stream_);
  }
  if (rows > cap_capture_) {
    kvp_.alloc(static_cast<size_t>(rows) * 2 * H * (prec_ == BP_PREC_BF16 ? 2 : eb));
    lnp_.alloc(static_cast<size_t>(rows) * H * (prec_ == BP_PREC_BF16 ? 2 : eb));
    cap_capture_ = rows;
  }
}

void Stage::recorded_rows(int layer, double* host_out) {
  if (!rec_.valid) fail(BP_ERR_CACHE, "no resident recording");
  if (layer < 0 || layer >= end_ - begin_) fail(BP_ERR_DIMENSION, "layer out of range");
  const int64_t n = rec_.tokens * h_;
  DevBuf d64;
  d64.alloc(static_cast<size_t>(n) * 8);
  if (prec_ == BP_PREC_F64) {
    BP_CUDA(cudaMemcpyAsync(d64.p, rec_.rec[static_cast<size_t>(layer)], static_cast<size_t>(n) * 8,
                            cudaMemcpyDeviceToDevice, stream_));
  } else {
    launch_convert<float, double>(static_cast<const float*>(rec_.rec[static_cast<size_t>(layer)]), d64.as<double>(), n, stream_);
  }
  BP_CUDA(cudaMemcpyAsync(host_out, d64.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, stream_));
  BP_CUDA(cudaStreamSynchronize(stream_));
}

void Stage::set_ring(int depth, int64_t max_tokens, const std::vector<void*>& x_slots,
                     const std::vector<void*>& eps_slots) {
  if (depth < 1 || depth > 3) fail(BP_ERR_CONFIG, "residual ring depth must be 1..3");
  BP_CUDA(cudaSetDevice(device_));
  BP_CUDA(cudaStreamSynchronize(stream_));
  const size_t te = prec_ == BP_PREC_F64 ? 8 : 4;
  xs_.assign(static_cast<size_t>(depth), nullptr);
  es_.assign(static_cast<size_t>(depth), nullptr);
  ring_external_ = !x_slots.empty();
  if (ring_external_ && (static_cast<int>(x_slots.size()) != depth ||
                         (is_last() && static_cast<int>(eps_slots.size()) != depth)))
    fail(BP_ERR_CONFIG, "ring slots must match the ring depth");
  for (int k = 0; k < depth; ++k) {
    if (ring_external_) {
      xs_[static_cast<size_t>(k)] = x_slots[static_cast<size_t>(k)];
      if (is_last()) es_[static_cast<size_t>(k)] = eps_slots[static_cast<size_t>(k)];
      continue;
    }
    xown_[k].reserve(static_cast<size_t>(max_tokens) * h_ * te);
    xs_[static_cast<size_t>(k)] = xown_[k].p;
    if (is_last()) {
      eown_[k].reserve(static_cast<size_t>(max_tokens) * C_ * te);
      es_[static_cast<size_t>(k)] = eown_[k].p;
    }
  }
  for (int k = depth; k < 3; ++k) { xown_[k].release(); eown_[k].release(); }
  ring_tokens_ = max_tokens;
}

void Stage::ensure_workspace(int64_t tokens, int64_t capture, bool new_cache, int use_prev) {
  const bool bf = prec_ == BP_PREC_BF16;
  const size_t te = prec_ == BP_PREC_F64 ? 8 : 4;
  const size_t me = bf ? 2 : te;
  const size_t S = static_cast<size_t>(tokens), P = static_cast<size_t>(capture);
  const size_t H = static_cast<size_t>(h_), nl = static_cast<size_t>(end_ - begin_);
  if (tokens > ring_tokens_) {
    if (ring_external_) fail(BP_ERR_DIMENSION, "pass exceeds the caller-supplied residual ring");
    set_ring(std::max<int>(1, ring_depth()), tokens);
  }
  if (tokens > cap_tokens_) {
    ln_.alloc(S * H * me);
    attn_.alloc(S * H * me);
    cq_.alloc(S * H * me);
    hmid_.alloc(S * static_cast<size_t>(F_) * me);
    if (bf && is_first()) {
      ftab_.alloc((S / static_cast<size_t>(tpf_) + 1) * static_cast<size_t>(h_ / 2) * 32);
      lat32_.alloc(S * static_cast<size_t>(C_) * 4);
    }
    cap_tokens_ = tokens;
  }
  qkv_.reserve(S * 3 * H * me);
  // the recording is written before the previous one is read: per parity
  if (capture > 0) recbuf_[parity_].reserve(nl * P * H * te);
  // The resident KV cache (read as the prefix when use_prev == 1) is read by
  // layer l's attention before this pass writes layer l's new capture. With an
  // equal capture size, layer l's new entry lands exactly on its old one, so
  // the entry is reused in place. A different size would shift the layer
  // offsets (layer 0's new entry could overwrite layer 1's old one before it
  // is read), so such a capture goes to the other buffer.
  if (new_cache) {
    if (use_prev == 1 && capture != cache_.tokens) cap_sel_ ^= 1;
    cap_[cap_sel_].reserve(nl * P * 2 * H * me);  // never the buffer being read (equal sizes need no growth)
  }
  if (capture > cap_capture_ || rec_.tokens > cap_capture_ || cache_.tokens > cap_capture_) {
    const int64_t p = std::max({capture, rec_.tokens, cache_.tokens, cap_capture_});
    kvp_.alloc(static_cast<size_t>(p) * 2 * H * me);
    lnp_.alloc(static_cast<size_t>(p) * H * me);
    cap_capture_ = p;
  }
}

// take_rows(k|v, capture rows) into the layer's cache entry (model.cpp:302-318,
// 321-322): after this layer's attention has read the previous entry, the
// captured K|V rows are copied out of the QKV buffer into [capture][2h].
// Runs of consecutive capture frames move with one launch.
void Stage::capture_kv(const StageInput& in, int li, const void* qkv, size_t eb, Entry* nc) {
  const int64_t H = h_, P = static_cast<int64_t>(in.capture_frames.size()) * tpf_;
  char* dst = cap_[cap_sel_].as<char>() + static_cast<int64_t>(li) * P * 2 * H * static_cast<int64_t>(eb);
  const char* src = static_cast<const char*>(qkv);
  const int64_t rs = 3 * H * static_cast<int64_t>(eb), rd = 2 * H * static_cast<int64_t>(eb);
  size_t f = 0;
  while (f < in.capture_frames.size()) {
    size_t g = f + 1;
    while (g < in.capture_frames.size() && in.capture_frames[g] == in.capture_frames[g - 1] + 1) ++g;
    launch_copy_rows(src + static_cast<int64_t>(in.capture_frames[f]) * tpf_ * rs + H * static_cast<int64_t>(eb), rs,
                     dst + static_cast<int64_t>(f) * tpf_ * rd, rd, static_cast<int64_t>(g - f) * tpf_, rd, stream_);
    f = g;
  }
  nc->k.push_back(dst);
  nc->v.push_back(dst + H * static_cast<int64_t>(eb));
  nc->ld = 2 * H;
}

void Stage::kv_prefix_from_recording(int li, const void* rec_rows, int64_t rows, void* kv_out) {
  const LayerW& w = lw_[static_cast<size_t>(li)];
  const int64_t H = h_;
  if (prec_ == BP_PREC_BF16) {
    const float* lnp = static_cast<const float*>(w.ln);
    launch_ln_bf16(static_cast<const float*>(rec_rows), H, lnp, lnp + H, rows, h_, lnp_.as<bf16>(), stream_);
    launch_gemm_bf16(lnp_.as<bf16>(), H, static_cast<const bf16*>(w.wqkv) + H * H, static_cast<int>(rows),
                     2 * h_, h_, kv_out, 2 * H, kGemmStoreBf16, stream_);
  } else if (prec_ == BP_PREC_F64) {
    const double* lnw = static_cast<const double*>(w.ln);
    launch_ln<double>(static_cast<const double*>(rec_rows), lnw, lnw + H, rows, h_, lnp_.as<double>(), stream_);
    launch_matmul<double>(lnp_.as<double>(), H, static_cast<const double*>(w.wqkv) + H, 3 * H,
                          static_cast<int>(rows), 2 * h_, h_, static_cast<double*>(kv_out), 2 * H,
                          kEpiNone, nullptr, 0, stream_);
  } else {
    const float* lnw = static_cast<const float*>(w.ln);
    launch_ln<float>(static_cast<const float*>(rec_rows), lnw, lnw + H, rows, h_, lnp_.as<float>(), stream_);
    launch_matmul<float>(lnp_.as<float>(), H, static_cast<const float*>(w.wqkv) + H, 3 * H,
                         static_cast<int>(rows), 2 * h_, h_, static_cast<float*>(kv_out), 2 * H,
                         kEpiNone, nullptr, 0, stream_);
  }
}

const void* Stage::forward(const StageInput& in) {
  BP_CUDA(cudaSetDevice(device_));
  const bool use_prefix = in.use_prev != 0;
  if (in.mode == BP_CACHE_DISABLED && use_prefix)
    fail(BP_ERR_CACHE, "cache supplied while caching is disabled");  // model.cpp:269-271
  if (in.use_prev == 1 && !cache_.valid) fail(BP_ERR_CACHE, "no resident captured K/V on this stage");
  if (in.use_prev == 2 && !rec_.valid) fail(BP_ERR_CACHE, "no resident recorded inputs on this stage");
  if ((in.use_prev == 3 || in.use_prev == 4) && host_kind_ != in.use_prev)
    fail(BP_ERR_CACHE, "host prefix not loaded");
  for (int f : in.capture_frames)
    if (f < 0 || f >= in.nframes) fail(BP_ERR_DIMENSION, "capture frame out of range");
  if (xs_.empty()) set_ring(1, in.tokens);
  if (in.slot < 0 || in.slot >= ring_depth()) fail(BP_ERR_INTERNAL, "residual ring slot out of range");
  if (in.out && !fuses_send()) fail(BP_ERR_INTERNAL, "fused send requested on a stage that cannot fuse it");
  if (wan_) {
    if (in.use_prev == 2 || in.use_prev == 4 || in.mode == BP_CACHE_RECOMPUTE || in.record_inputs)
      fail(BP_ERR_CONFIG, "wan block supports the resident K/V cache and no cache, not the recompute route");
    if (in.nframes > 0 && (!in.d_levels || !in.d_frame_ids))
      fail(BP_ERR_CONFIG, "wan block needs the pass's frame levels and ids on every stage");
    switch (prec_) {
      case BP_PREC_F64: return forward_wan_simt<double>(in);
      case BP_PREC_F32: return forward_wan_simt<float>(in);
      default: return forward_wan_bf16(in);
    }
  }
  switch (prec_) {
    case BP_PREC_F64: return forward_simt<double>(in);
    case BP_PREC_F32: return forward_simt<float>(in);
    default: return forward_bf16(in);
  }
}

// ---- optional Wan2.1-style block (bp_block WAN; oracle/wan_oracle.py) ----------------------
// Per pass: the timestep MLP for the pass's frames (e, e0 = SiLU(e) W_tp + b_tp)
// and the modulation tables modt[l][f] = mod_l + e0_f (1 + scale chunks), the
// head's hmt[f] = head_mod + e_f, and (bf16) the temporal RoPE table.
template <typename T>
void Stage::wan_pass_setup(const StageInput& in) {
  const int nf = in.nframes, nl = end_ - begin_;
  const int64_t H = h_;
  const size_t sz = sizeof(T);
  cudaStream_t st = stream_;
  wsin_.reserve(static_cast<size_t>(nf) * kWanFreqDim * sz + 16);
  wa_.reserve(static_cast<size_t>(nf) * H * sz + 16);
  we_.reserve(static_cast<size_t>(nf) * H * sz + 16);
  wes_.reserve(static_cast<size_t>(nf) * H * sz + 16);
  we0_.reserve(static_cast<size_t>(nf) * 6 * H * sz + 16);
  wmodt_.reserve(static_cast<size_t>(nl) * nf * 6 * H * sz + 16);
  launch_wan_sinus<T>(in.d_levels, nf, wsin_.as<T>(), st);
  launch_matmul<T>(wsin_.as<T>(), kWanFreqDim, static_cast<const T*>(wg_.t1), H, nf, h_, kWanFreqDim, wa_.as<T>(), H,
                   kEpiNone, nullptr, 0, st);
  launch_bias_act<T>(wa_.as<T>(), nf, h_, static_cast<const T*>(wg_.tb1), 1, nullptr, st);
  launch_matmul<T>(wa_.as<T>(), H, static_cast<const T*>(wg_.t2), H, nf, h_, h_, we_.as<T>(), H, kEpiNone, nullptr, 0,
                   st);
  launch_bias_act<T>(we_.as<T>(), nf, h_, static_cast<const T*>(wg_.tb2), 0, wes_.as<T>(), st);
  launch_matmul<T>(wes_.as<T>(), H, static_cast<const T*>(wg_.tp), 6 * H, nf, 6 * h_, h_, we0_.as<T>(), 6 * H,
                   kEpiNone, nullptr, 0, st);
  launch_bias_act<T>(we0_.as<T>(), nf, 6 * h_, static_cast<const T*>(wg_.tpb), 0, nullptr, st);
  launch_wan_modt<T>(static_cast<const T*>(wanv_), 10 * H, nl, we0_.as<T>(), 6 * H, nf, h_, 6, false,
                     wmodt_.as<T>(), st);
  if (is_last()) {
    whmt_.reserve(static_cast<size_t>(nf) * 2 * H * sz + 16);
    launch_wan_modt<T>(static_cast<const T*>(wg_.hmod), 0, 1, we_.as<T>(), H, nf, h_, 2, true, whmt_.as<T>(), st);
  }
  if (prec_ == BP_PREC_BF16) {
    wttab_.reserve(static_cast<size_t>(nf) * wnt_ * sizeof(float2) + 16);
    launch_wan_rope_frames(in.d_frame_ids, nf, wnt_, wttab_.as<float2>(), st);
  }
}

template <typename T>
const void* Stage::forward_wan_simt(const StageInput& in) {
  const int64_t S = in.tokens, H = h_;
  const int64_t P = static_cast<int64_t>(in.capture_frames.size()) * tpf_;
  const int nl = end_ - begin_, nf = in.nframes;
  const bool new_cache = P > 0 && in.mode == BP_CACHE_CACHED;
  ensure_workspace(S, P, new_cache, in.use_prev);
  cudaStream_t st = stream_;
  T* x = static_cast<T*>(xs_[static_cast<size_t>(in.slot)]);
  T* ln = ln_.as<T>();
  T* at = attn_.as<T>();
  T* tmp = cq_.as<T>();
  T* hm = hmid_.as<T>();
  if (is_first()) {  // x = latents W_in: positions enter through RoPE, time through the modulation
    const T* lat = static_cast<const T*>(in.payload);
    const T* win = static_cast<const T*>(w_in_);
    if (prec_ == BP_PREC_F32) {
      wlat_.reserve(static_cast<size_t>(S) * C_ * sizeof(T));
      launch_convert<double, T>(static_cast<const double*>(in.payload), wlat_.as<T>(), S * C_, st);
      lat = wlat_.as<T>();
      win = winT_.as<T>();
    }
    launch_matmul<T>(lat, C_, win, H, static_cast<int>(S), h_, C_, x, H, kEpiNone, nullptr, 0, st);
  } else if (in.payload != x) {
    BP_CUDA(cudaMemcpyAsync(x, in.payload, static_cast<size_t>(S * H) * sizeof(T), cudaMemcpyDeviceToDevice, st));
    ++input_copies_;
  }
  wan_pass_setup<T>(in);
  const int64_t mstride = 6 * H;  // modulation table: frame stride
  Entry nc;
  T* qkv = qkv_.as<T>();
  for (int li = 0; li < nl; ++li) {
    const LayerW& w = lw_[static_cast<size_t>(li)];
    const T* lnw = static_cast<const T*>(w.ln);
    const T* wv = static_cast<const T*>(w.wan);
    const T* mt = wmodt_.as<T>() + static_cast<int64_t>(li) * nf * mstride;
    launch_ln_mod<T>(x, H, mt + H, mt, tpf_, mstride, S, h_, kWanEps, ln, H, st);
    AttnArgs<T> a{};
    if (in.use_prev == 1) {
      a.k0 = static_cast<const T*>(cache_.k[static_cast<size_t>(li)]);
      a.v0 = static_cast<const T*>(cache_.v[static_cast<size_t>(li)]);
      a.ldk0 = a.ldv0 = cache_.ld;
      a.n0 = cache_.tokens;
    } else if (in.use_prev == 3) {
      a.k0 = hostpre_.as<T>() + static_cast<int64_t>(li) * host_rows_ * 2 * H;
      a.v0 = a.k0 + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = host_rows_;
    }
    launch_matmul<T>(ln, H, static_cast<const T*>(w.wqkv), 3 * H, static_cast<int>(S), 3 * h_, h_, qkv, 3 * H,
                     kEpiNone, nullptr, 0, st);
    launch_wan_qk<T>(qkv, 3 * H, S, h_, heads_, wv + 6 * H, 2, H, in.d_frame_ids, tpf_, m_.width, 1, st);
    a.q = qkv; a.ldq = 3 * H;
    a.k1 = qkv + H; a.ldk1 = 3 * H;
    a.v1 = qkv + 2 * H; a.ldv1 = 3 * H;
    a.n1 = S;
    a.out = at; a.ldo = H;
    a.dh = dh_;
    a.scale = static_cast<T>(1.0 / std::sqrt(static_cast<double>(dh_)));
    launch_attention<T>(a, S, heads_, st);
    if (new_cache) capture_kv(in, li, qkv, sizeof(T), &nc);
    launch_matmul<T>(at, H, static_cast<const T*>(w.wo), H, static_cast<int>(S), h_, h_, tmp, H, kEpiNone, nullptr, 0,
                     st);
    launch_gate_residual<T>(x, tmp, mt + 2 * H, tpf_, mstride, S, h_, st);
    launch_ln_mod<T>(x, H, lnw + 2 * H, lnw + 3 * H, 1, 0, S, h_, kWanEps, ln, H, st);
    launch_matmul<T>(ln, H, static_cast<const T*>(w.cq), H, static_cast<int>(S), h_, h_, tmp, H, kEpiNone, nullptr, 0,
                     st);
    launch_wan_qk<T>(tmp, H, S, h_, heads_, wv + 8 * H, 1, 0, nullptr, tpf_, m_.width, 0, st);
    AttnArgs<T> c{};
    c.q = tmp; c.ldq = H;
    c.k1 = static_cast<const T*>(w.ctx_kv); c.ldk1 = 2 * H;
    c.v1 = static_cast<const T*>(w.ctx_kv) + H; c.ldv1 = 2 * H;
    c.n1 = Lc_;
    c.out = at; c.ldo = H;
    c.dh = dh_;
    c.scale = a.scale;
    launch_attention<T>(c, S, heads_, st);
    launch_matmul<T>(at, H, static_cast<const T*>(w.co), H, static_cast<int>(S), h_, h_, x, H, kEpiResidual, x, H,
                     st);
    launch_ln_mod<T>(x, H, mt + 4 * H, mt + 3 * H, tpf_, mstride, S, h_, kWanEps, ln, H, st);
    launch_matmul<T>(ln, H, static_cast<const T*>(w.w1), F_, static_cast<int>(S), F_, h_, hm, F_, kEpiNone, nullptr,
                     0, st);
    launch_gelu_tanh<T>(hm, S * F_, st);
    launch_matmul<T>(hm, F_, static_cast<const T*>(w.w2), H, static_cast<int>(S), h_, F_, tmp, H, kEpiNone, nullptr,
                     0, st);
    launch_gate_residual<T>(x, tmp, mt + 5 * H, tpf_, mstride, S, h_, st);
  }
  cache_ = Entry{};
  if (new_cache) { nc.valid = true; nc.tokens = P; cache_ = std::move(nc); }
  rec_ = Entry{};
  parity_ ^= 1;
  (void)nf;
  if (is_last()) {
    const T* hmt = whmt_.as<T>();
    launch_ln_mod<T>(x, H, hmt + H, hmt, tpf_, 2 * H, S, h_, kWanEps, ln, H, st);
    T* eps = static_cast<T*>(es_[static_cast<size_t>(in.slot)]);
    launch_matmul<T>(ln, H, static_cast<const T*>(w_out_), C_, static_cast<int>(S), C_, h_, eps, C_, kEpiNone, nullptr,
                     0, st);
    return eps;
  }
  return x;
}

const void* Stage::forward_wan_bf16(const StageInput& in) {
  const int64_t S = in.tokens, H = h_;
  const int64_t P = static_cast<int64_t>(in.capture_frames.size()) * tpf_;
  const int nl = end_ - begin_, nf = in.nframes;
  const bool new_cache = P > 0 && in.mode == BP_CACHE_CACHED;
  ensure_workspace(S, P, new_cache, in.use_prev);
  cudaStream_t st = stream_;
  float* x = static_cast<float*>(xs_[static_cast<size_t>(in.slot)]);
  bf16* ln = ln_.as<bf16>();
  bf16* at = attn_.as<bf16>();
  bf16* cq = cq_.as<bf16>();
  bf16* hm = hmid_.as<bf16>();
  if (is_first()) {  // x = latents W_in (fp32): positions enter through RoPE, time through the modulation
    launch_convert<double, float>(static_cast<const double*>(in.payload), lat32_.as<float>(), S * C_, st);
    launch_gemm_f32_tile(lat32_.as<float>(), C_, w_in32_.as<float>(), H, static_cast<int>(S), h_, C_, x, H, false, st);
  } else if (in.payload != x) {
    BP_CUDA(cudaMemcpyAsync(x, in.payload, static_cast<size_t>(S * H) * 4, cudaMemcpyDeviceToDevice, st));
    ++input_copies_;
  }
  wan_pass_setup<float>(in);
  const int64_t mstride = 6 * H;
  const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(dh_)));
  const float eps_ln = static_cast<float>(kWanEps);
  const float2* tt = wttab_.as<float2>();
  const float2* yt = wytab_.as<float2>();
  const float2* xt = wxtab_.as<float2>();
  Entry nc;
  bf16* qkv = qkv_.as<bf16>();
  for (int li = 0; li < nl; ++li) {
    const LayerW& w = lw_[static_cast<size_t>(li)];
    const float* lnw = static_cast<const float*>(w.ln);
    const float* wv = static_cast<const float*>(w.wan);
    const float* mt = wmodt_.as<float>() + static_cast<int64_t>(li) * nf * mstride;
    prof_mark(3, true);
    launch_ln_bf16_grp(x, H, mt + H, mt, tpf_, mstride, eps_ln, S, h_, ln, st);  // LN(x) (1 + sc1) + sh1
    prof_mark(3, false);
    AttnBf16Args a{};
    if (in.use_prev == 1) {
      a.k0 = static_cast<const bf16*>(cache_.k[static_cast<size_t>(li)]);
      a.v0 = static_cast<const bf16*>(cache_.v[static_cast<size_t>(li)]);
      a.ldk0 = a.ldv0 = cache_.ld;
      a.n0 = cache_.tokens;
    } else if (in.use_prev == 3) {
      a.k0 = hostpre_.as<bf16>() + static_cast<int64_t>(li) * host_rows_ * 2 * H;
      a.v0 = a.k0 + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = host_rows_;
    }
    prof_mark(2, true);
    launch_gemm_bf16(ln, H, static_cast<const bf16*>(w.wqkv), static_cast<int>(S), 3 * h_, h_, qkv, 3 * H,
                     kGemmStoreBf16, st);
    prof_mark(2, false);
    prof_mark(3, true);
    launch_wan_qk_bf16(qkv, 3 * H, S, h_, heads_, wv + 6 * H, 2, H, tt, yt, xt, tpf_, m_.width, 1, st);
    prof_mark(3, false);
    a.q = qkv; a.ldq = 3 * H;
    a.k1 = qkv + H; a.ldk1 = 3 * H;
    a.v1 = qkv + 2 * H; a.ldv1 = 3 * H;
    a.n1 = S;
    a.out = at; a.ldo = H;
    a.heads = heads_; a.dh = dh_; a.scale = scale;
    prof_mark(0, true);
    launch_attn_bf16(a, S, st);
    prof_mark(0, false);
    if (new_cache) capture_kv(in, li, qkv, 2, &nc);
    prof_mark(2, true);
    launch_gemm_bf16(at, H, static_cast<const bf16*>(w.wo), static_cast<int>(S), h_, h_, x, H, kGemmResidualGatedF32,
                     st, GemmGate{mt + 2 * H, tpf_, mstride});
    prof_mark(2, false);
    prof_mark(3, true);
    launch_ln_bf16_grp(x, H, lnw + 2 * H, lnw + 3 * H, 1, 0, eps_ln, S, h_, ln, st);
    prof_mark(3, false);
    prof_mark(2, true);
    launch_gemm_bf16(ln, H, static_cast<const bf16*>(w.cq), static_cast<int>(S), h_, h_, cq, H, kGemmStoreBf16, st);
    prof_mark(2, false);
    prof_mark(3, true);
    launch_wan_qk_bf16(cq, H, S, h_, heads_, wv + 8 * H, 1, 0, tt, yt, xt, tpf_, m_.width, 0, st);
    prof_mark(3, false);
    AttnBf16Args c{};
    c.q = cq; c.ldq = H;
    c.k1 = static_cast<const bf16*>(w.ctx_kv); c.ldk1 = 2 * H;
    c.v1 = static_cast<const bf16*>(w.ctx_kv) + H; c.ldv1 = 2 * H;
    c.n1 = Lc_;
    c.out = at; c.ldo = H;
    c.heads = heads_; c.dh = dh_; c.scale = scale;
    prof_mark(1, true);
    launch_attn_bf16_cross(c, S, st);
    prof_mark(1, false);
    prof_mark(2, true);
    launch_gemm_bf16(at, H, static_cast<const bf16*>(w.co), static_cast<int>(S), h_, h_, x, H, kGemmResidualF32, st);
    prof_mark(2, false);
    prof_mark(3, true);
    launch_ln_bf16_grp(x, H, mt + 4 * H, mt + 3 * H, tpf_, mstride, eps_ln, S, h_, ln, st);  // LN(x) (1 + sc2) + sh2
    prof_mark(3, false);
    prof_mark(2, true);
    launch_gemm_bf16(ln, H, static_cast<const bf16*>(w.w1), static_cast<int>(S), F_, h_, hm, F_, kGemmGeluTanhBf16, st);
    launch_gemm_bf16(hm, F_, static_cast<const bf16*>(w.w2), static_cast<int>(S), h_, F_, x, H, kGemmResidualGatedF32,
                     st, GemmGate{mt + 5 * H, tpf_, mstride});
    prof_mark(2, false);
  }
  cache_ = Entry{};
  if (new_cache) { nc.valid = true; nc.tokens = P; cache_ = std::move(nc); }
  rec_ = Entry{};
  parity_ ^= 1;
  if (is_last()) {
    const float* hmt = whmt_.as<float>();
    float* hx = reinterpret_cast<float*>(hmid_.p);  // [S, h] fp32 fits the [S, F] bf16 buffer (F >= 2h)
    launch_ln_mod<float>(x, H, hmt + H, hmt, tpf_, 2 * H, S, h_, kWanEps, hx, H, st);
    float* eps = static_cast<float*>(es_[static_cast<size_t>(in.slot)]);
    launch_gemm_f32_tile(hx, H, static_cast<const float*>(w_out_), C_, static_cast<int>(S), C_, h_, eps, C_, false, st);
    return eps;
  }
  return x;
}

template <typename T>
const void* Stage::forward_simt(const StageInput& in) {
  const int64_t S = in.tokens, H = h_;
  const int64_t P = static_cast<int64_t>(in.capture_frames.size()) * tpf_;
  const int nl = end_ - begin_;
  const bool capturing = P > 0;
  const bool new_cache = capturing && in.mode == BP_CACHE_CACHED;
  const bool new_rec = capturing && (in.mode == BP_CACHE_RECOMPUTE || in.record_inputs);
  ensure_workspace(S, P, new_cache, in.use_prev);
  cudaStream_t st = stream_;
  T* x = static_cast<T*>(xs_[static_cast<size_t>(in.slot)]);
  T* ln = ln_.as<T>();
  T* at = attn_.as<T>();
  T* cq = cq_.as<T>();
  T* hm = hmid_.as<T>();
  if (is_first()) {
    launch_embed<T>(static_cast<const double*>(in.payload), static_cast<const double*>(w_in_),
                    freq_.as<double>(), in.d_levels, in.d_frame_ids, S, C_, h_, tpf_, x, st);
  } else {
    if (in.payload != x) {  // a receive that landed in the slot needs no copy
      BP_CUDA(cudaMemcpyAsync(x, in.payload, static_cast<size_t>(S * H) * sizeof(T), cudaMemcpyDeviceToDevice, st));
      ++input_copies_;
    }
  }
  Entry nc, nr;
  T* qkv = qkv_.as<T>();
  for (int li = 0; li < nl; ++li) {
    const LayerW& w = lw_[static_cast<size_t>(li)];
    const T* lnw = static_cast<const T*>(w.ln);
    if (new_rec) {  // recorded->layer_inputs += take_rows(x, capture_rows) (model.cpp:295)
      T* dst = recbuf_[parity_].as<T>() + static_cast<int64_t>(li) * P * H;
      for (size_t f = 0; f < in.capture_frames.size(); ++f)
        launch_copy_rows(x + static_cast<int64_t>(in.capture_frames[f]) * tpf_ * H, H * sizeof(T),
                         dst + static_cast<int64_t>(f) * tpf_ * H, H * sizeof(T), tpf_, H * sizeof(T), st);
      nr.rec.push_back(dst);
    }
    launch_ln<T>(x, lnw, lnw + H, S, h_, ln, st);
    AttnArgs<T> a{};
    if (in.use_prev == 1) {
      a.k0 = static_cast<const T*>(cache_.k[static_cast<size_t>(li)]);
      a.v0 = static_cast<const T*>(cache_.v[static_cast<size_t>(li)]);
      a.ldk0 = a.ldv0 = cache_.ld;
      a.n0 = cache_.tokens;
    } else if (in.use_prev == 2) {
      kv_prefix_from_recording(li, rec_.rec[static_cast<size_t>(li)], rec_.tokens, kvp_.p);
      a.k0 = kvp_.as<T>();
      a.v0 = kvp_.as<T>() + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = rec_.tokens;
    } else if (in.use_prev == 3) {
      a.k0 = hostpre_.as<T>() + static_cast<int64_t>(li) * host_rows_ * 2 * H;
      a.v0 = a.k0 + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = host_rows_;
    } else if (in.use_prev == 4) {
      kv_prefix_from_recording(li, hostpre_.as<T>() + static_cast<int64_t>(li) * host_rows_ * H, host_rows_, kvp_.p);
      a.k0 = kvp_.as<T>();
      a.v0 = kvp_.as<T>() + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = host_rows_;
    }
    launch_matmul<T>(ln, H, static_cast<const T*>(w.wqkv), 3 * H, static_cast<int>(S), 3 * h_, h_, qkv,
                     3 * H, kEpiNone, nullptr, 0, st);
    a.q = qkv; a.ldq = 3 * H;
    a.k1 = qkv + H; a.ldk1 = 3 * H;
    a.v1 = qkv + 2 * H; a.ldv1 = 3 * H;
    a.n1 = S;
    a.out = at; a.ldo = H;
    a.dh = dh_;
    a.scale = static_cast<T>(1.0 / std::sqrt(static_cast<double>(dh_)));
    launch_attention<T>(a, S, heads_, st);
    if (new_cache) capture_kv(in, li, qkv, sizeof(T), &nc);
    launch_matmul<T>(at, H, static_cast<const T*>(w.wo), H, static_cast<int>(S), h_, h_, x, H,
                     kEpiResidual, x, H, st);
    // cross-attention against the hoisted context K|V
    launch_ln<T>(x, lnw + 2 * H, lnw + 3 * H, S, h_, ln, st);
    launch_matmul<T>(ln, H, static_cast<const T*>(w.cq), H, static_cast<int>(S), h_, h_, cq, H, kEpiNone,
                     nullptr, 0, st);
    AttnArgs<T> c{};
    c.q = cq; c.ldq = H;
    c.k1 = static_cast<const T*>(w.ctx_kv); c.ldk1 = 2 * H;
    c.v1 = static_cast<const T*>(w.ctx_kv) + H; c.ldv1 = 2 * H;
    c.n1 = Lc_;
    c.out = at; c.ldo = H;
    c.dh = dh_;
    c.scale = a.scale;
    launch_attention<T>(c, S, heads_, st);
    launch_matmul<T>(at, H, static_cast<const T*>(w.co), H, static_cast<int>(S), h_, h_, x, H,
                     kEpiResidual, x, H, st);
    // FFN
    launch_ln<T>(x, lnw + 4 * H, lnw + 5 * H, S, h_, ln, st);
    launch_matmul<T>(ln, H, static_cast<const T*>(w.w1), F_, static_cast<int>(S), F_, h_, hm, F_,
                     kEpiGelu, nullptr, 0, st);
    launch_matmul<T>(hm, F_, static_cast<const T*>(w.w2), H, static_cast<int>(S), h_, F_, x, H,
                     kEpiResidual, x, H, st);
  }
  cache_ = Entry{};
  if (new_cache) { nc.valid = true; nc.tokens = P; cache_ = std::move(nc); }
  rec_ = Entry{};
  if (new_rec) { nr.valid = true; nr.tokens = P; rec_ = std::move(nr); }
  parity_ ^= 1;
  if (is_last()) {
    T* eps = static_cast<T*>(es_[static_cast<size_t>(in.slot)]);
    launch_matmul<T>(x, H, static_cast<const T*>(w_out_), C_, static_cast<int>(S), C_, h_, eps, C_, kEpiNone, nullptr,
                     0, st);
    return eps;
  }
  return x;
}

const void* Stage::forward_bf16(const StageInput& in) {
  const int64_t S = in.tokens, H = h_;
  const int64_t P = static_cast<int64_t>(in.capture_frames.size()) * tpf_;
  const int nl = end_ - begin_;
  const bool capturing = P > 0;
  const bool new_cache = capturing && in.mode == BP_CACHE_CACHED;
  const bool new_rec = capturing && (in.mode == BP_CACHE_RECOMPUTE || in.record_inputs);
  ensure_workspace(S, P, new_cache, in.use_prev);
  cudaStream_t st = stream_;
  float* x = static_cast<float*>(xs_[static_cast<size_t>(in.slot)]);
  bf16* ln = ln_.as<bf16>();
  bf16* at = attn_.as<bf16>();
  bf16* cq = cq_.as<bf16>();
  bf16* hm = hmid_.as<bf16>();
  if (is_first()) {
    launch_embed_fast(static_cast<const double*>(in.payload), w_in32_.as<float>(), freq_.as<double>(),
                      ttab_.as<double>(), ftab_.as<double>(), in.d_levels, in.d_frame_ids, S, C_, h_, tpf_,
                      lat32_.as<float>(), x, st);
  } else {
    if (in.payload != x) {  // a receive that landed in the slot needs no copy
      BP_CUDA(cudaMemcpyAsync(x, in.payload, static_cast<size_t>(S * H) * 4, cudaMemcpyDeviceToDevice, st));
      ++input_copies_;
    }
  }
  const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(dh_)));
  const bool fused = in.out != nullptr;

  Entry nc, nr;
  bf16* qkv = qkv_.as<bf16>();
  for (int li = 0; li < nl; ++li) {
    const LayerW& w = lw_[static_cast<size_t>(li)];
    const float* lnw = static_cast<const float*>(w.ln);
    if (new_rec) {
      float* dst = recbuf_[parity_].as<float>() + static_cast<int64_t>(li) * P * H;
      for (size_t f = 0; f < in.capture_frames.size(); ++f)
        launch_copy_rows(x + static_cast<int64_t>(in.capture_frames[f]) * tpf_ * H, H * 4,
                         dst + static_cast<int64_t>(f) * tpf_ * H, H * 4, tpf_, H * 4, st);
      nr.rec.push_back(dst);
    }
    nvtxRangePushA("self_attention_sublayer");  // model.cpp:201-211
    prof_mark(3, true);
    launch_ln_bf16(x, H, lnw, lnw + H, S, h_, ln, st);
    prof_mark(3, false);
    AttnBf16Args a{};
    if (in.use_prev == 1) {
      a.k0 = static_cast<const bf16*>(cache_.k[static_cast<size_t>(li)]);
      a.v0 = static_cast<const bf16*>(cache_.v[static_cast<size_t>(li)]);
      a.ldk0 = a.ldv0 = cache_.ld;
      a.n0 = cache_.tokens;
    } else if (in.use_prev == 2) {
      kv_prefix_from_recording(li, rec_.rec[static_cast<size_t>(li)], rec_.tokens, kvp_.p);
      a.k0 = kvp_.as<bf16>();
      a.v0 = kvp_.as<bf16>() + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = rec_.tokens;
    } else if (in.use_prev == 3) {
      a.k0 = hostpre_.as<bf16>() + static_cast<int64_t>(li) * host_rows_ * 2 * H;
      a.v0 = a.k0 + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = host_rows_;
    } else if (in.use_prev == 4) {
      kv_prefix_from_recording(li, hostpre_.as<float>() + static_cast<int64_t>(li) * host_rows_ * H, host_rows_, kvp_.p);
      a.k0 = kvp_.as<bf16>();
      a.v0 = kvp_.as<bf16>() + H;
      a.ldk0 = a.ldv0 = 2 * H;
      a.n0 = host_rows_;
    }
    prof_mark(2, true);
    launch_gemm_bf16(ln, H, static_cast<const bf16*>(w.wqkv), static_cast<int>(S), 3 * h_, h_, qkv, 3 * H,
                     kGemmStoreBf16, st);
    prof_mark(2, false);
    a.q = qkv; a.ldq = 3 * H;
    a.k1 = qkv + H; a.ldk1 = 3 * H;
    a.v1 = qkv + 2 * H; a.ldv1 = 3 * H;
    a.n1 = S;
    a.out = at; a.ldo = H;
    a.heads = heads_; a.dh = dh_; a.scale = scale;
    prof_mark(0, true);
    launch_attn_bf16(a, S, st);
    prof_mark(0, false);
    if (new_cache) capture_kv(in, li, qkv, 2, &nc);
    prof_mark(2, true);
    launch_gemm_bf16(at, H, static_cast<const bf16*>(w.wo), static_cast<int>(S), h_, h_, x, H,
                     kGemmResidualF32, st);
    prof_mark(2, false);
    nvtxRangePop();
    nvtxRangePushA("cross_attention_sublayer");  // model.cpp:213-219
    prof_mark(3, true);
    launch_ln_bf16(x, H, lnw + 2 * H, lnw + 3 * H, S, h_, ln, st);
    prof_mark(3, false);
    prof_mark(2, true);
    launch_gemm_bf16(ln, H, static_cast<const bf16*>(w.cq), static_cast<int>(S), h_, h_, cq, H,
                     kGemmStoreBf16, st);
    prof_mark(2, false);
    AttnBf16Args c{};
    c.q = cq; c.ldq = H;
    c.k1 = static_cast<const bf16*>(w.ctx_kv); c.ldk1 = 2 * H;
    c.v1 = static_cast<const bf16*>(w.ctx_kv) + H; c.ldv1 = 2 * H;
    c.n1 = Lc_;
    c.out = at; c.ldo = H;
    c.heads = heads_; c.dh = dh_; c.scale = scale;
    prof_mark(1, true);
    launch_attn_bf16_cross(c, S, st);
    prof_mark(1, false);
    prof_mark(2, true);
    launch_gemm_bf16(at, H, static_cast<const bf16*>(w.co), static_cast<int>(S), h_, h_, x, H,
                     kGemmResidualF32, st);
    prof_mark(2, false);
    nvtxRangePop();
    nvtxRangePushA("ffn_sublayer");  // model.cpp:221-225
    prof_mark(3, true);
    launch_ln_bf16(x, H, lnw + 4 * H, lnw + 5 * H, S, h_, ln, st);
    prof_mark(3, false);
    prof_mark(2, true);
    launch_gemm_bf16(ln, H, static_cast<const bf16*>(w.w1), static_cast<int>(S), F_, h_, hm, F_,
                     kGemmGeluBf16, st);
    if (fused && li == nl - 1) {  // x + FFN(x) written into the next rank's receive slot
      if (in.before_out) in.before_out(st, in.before_out_user);
      GemmGate g{};
      g.resid = x;
      g.ldr = H;
      launch_gemm_bf16(hm, F_, static_cast<const bf16*>(w.w2), static_cast<int>(S), h_, F_, in.out, H,
                       kGemmResidualOutF32, st, g);
    } else {
      launch_gemm_bf16(hm, F_, static_cast<const bf16*>(w.w2), static_cast<int>(S), h_, F_, x, H,
                       kGemmResidualF32, st);
    }
    prof_mark(2, false);
    nvtxRangePop();
  }
  cache_ = Entry{};
  if (new_cache) { nc.valid = true; nc.tokens = P; cache_ = std::move(nc); }
  rec_ = Entry{};
  if (new_rec) { nr.valid = true; nr.tokens = P; rec_ = std::move(nr); }
  parity_ ^= 1;
  if (is_last()) {
    float* eps = static_cast<float*>(es_[static_cast<size_t>(in.slot)]);
    launch_gemm_f32_tile(x, H, static_cast<const float*>(w_out_), C_, static_cast<int>(S), C_, h_, eps, C_, false, st);
    return eps;
  }
  return fused ? in.out : x;
}

void Stage::tag_entries(int64_t block_id, int level) {
  if (cache_.valid) { cache_.block_id = block_id; cache_.level = level; }
  if (rec_.valid) { rec_.block_id = block_id; rec_.level = level; }
}

void Stage::cache_rows(int layer, int which, double* host_out) {
  if (!cache_.valid) fail(BP_ERR_CACHE, "no resident cache");
  if (layer < 0 || layer >= end_ - begin_) fail(BP_ERR_DIMENSION, "layer out of range");
  const void* src = which ? cache_.v[static_cast<size_t>(layer)] : cache_.k[static_cast<size_t>(layer)];
  const int64_t rows = cache_.tokens, H = h_;
  const size_t eb = prec_ == BP_PREC_F64 ? 8 : (prec_ == BP_PREC_F32 ? 4 : 2);
  DevBuf tight, d64;
  tight.alloc(static_cast<size_t>(rows * H) * eb);
  launch_copy_rows(src, cache_.ld * static_cast<int64_t>(eb), tight.p, H * static_cast<int64_t>(eb), rows,
                   H * static_cast<int64_t>(eb), stream_);
  d64.alloc(static_cast<size_t>(rows * H) * 8);
  if (prec_ == BP_PREC_F64) {
    BP_CUDA(cudaMemcpyAsync(d64.p, tight.p, static_cast<size_t>(rows * H) * 8, cudaMemcpyDeviceToDevice, stream_));
  } else if (prec_ == BP_PREC_F32) {
    launch_convert<float, double>(tight.as<float>(), d64.as<double>(), rows * H, stream_);
  } else {
    std::vector<uint16_t> hb(static_cast<size_t>(rows * H));
    BP_CUDA(cudaMemcpyAsync(hb.data(), tight.p, hb.size() * 2, cudaMemcpyDeviceToHost, stream_));
    BP_CUDA(cudaStreamSynchronize(stream_));
    for (size_t i = 0; i < hb.size(); ++i) {
      const uint32_t u = static_cast<uint32_t>(hb[i]) << 16;
      float f;
      std::memcpy(&f, &u, 4);
      host_out[i] = f;
    }
    return;
  }
  BP_CUDA(cudaMemcpyAsync(host_out, d64.p, static_cast<size_t>(rows * H) * 8, cudaMemcpyDeviceToHost, stream_));
  BP_CUDA(cudaStreamSynchronize(stream_));
}

void Stage::bump_ulp(int layer, int which, int64_t index) {
  if (!cache_.valid) fail(BP_ERR_CACHE, "no resident cache");
  if (layer < 0 || layer >= end_ - begin_) fail(BP_ERR_DIMENSION, "layer out of range");
  if (index < 0 || index >= cache_.tokens * h_) fail(BP_ERR_DIMENSION, "index out of range");
  const size_t eb = prec_ == BP_PREC_F64 ? 8 : (prec_ == BP_PREC_F32 ? 4 : 2);
  const char* base = static_cast<const char*>(which ? cache_.v[static_cast<size_t>(layer)]
                                                    : cache_.k[static_cast<size_t>(layer)]);
  const int64_t r = index / h_, c = index % h_;
  void* p = const_cast<char*>(base) + (r * cache_.ld + c) * static_cast<int64_t>(eb);
  launch_bump_ulp(p, prec_ == BP_PREC_F64 ? 0 : (prec_ == BP_PREC_F32 ? 1 : 2), stream_);
}

std::string Stage::audit() {
  if (!cache_.valid || !rec_.valid) return "cache audit has no recording";
  if (cache_.block_id != rec_.block_id) return "cache and recording cover different blocks";
  const size_t eb = prec_ == BP_PREC_F64 ? 8 : (prec_ == BP_PREC_F32 ? 4 : 2);
  const int64_t rows = cache_.tokens, H = h_;
  scratch_.reserve(16 * static_cast<size_t>(end_ - begin_));
  auto* firsts = scratch_.as<unsigned long long>();
  const int nl = end_ - begin_;
  std::vector<unsigned long long> host(static_cast<size_t>(2 * nl));
  BP_CUDA(cudaMemsetAsync(firsts, 0xff, 16 * static_cast<size_t>(nl), stream_));
  for (int li = 0; li < nl; ++li) {
    kv_prefix_from_recording(li, rec_.rec[static_cast<size_t>(li)], rows, kvp_.p);
    const char* kv = kvp_.as<char>();
    if (eb == 2) {
      // compare in 16-bit units: rows of H bf16 = H/2 words; done as 4-byte
      // words first, the element index is refined on the host below
    }
    launch_first_diff(kv, 2 * H * eb, cache_.k[static_cast<size_t>(li)], cache_.ld * eb, rows, H * eb,
                      firsts + 2 * li, stream_);
    launch_first_diff(kv + H * eb, 2 * H * eb, cache_.v[static_cast<size_t>(li)], cache_.ld * eb, rows,
                      H * eb, firsts + 2 * li + 1, stream_);
  }
  BP_CUDA(cudaMemcpyAsync(host.data(), firsts, 16 * static_cast<size_t>(nl), cudaMemcpyDeviceToHost, stream_));
  BP_CUDA(cudaStreamSynchronize(stream_));
  const int64_t words_per_row = H * static_cast<int64_t>(eb) / 4;
  for (int li = 0; li < nl; ++li) {
    const unsigned long long fk = host[static_cast<size_t>(2 * li)], fv = host[static_cast<size_t>(2 * li + 1)];
    if (fk == ~0ULL && fv == ~0ULL) continue;
    // word index -> flat element index (first element covered by that word)
    auto elem = [&](unsigned long long wi) -> int64_t {
      const int64_t r = static_cast<int64_t>(wi) / words_per_row, wc = static_cast<int64_t>(wi) % words_per_row;
      return r * H + (wc * 4) / static_cast<int64_t>(eb);
    };
    const int64_t ek = fk == ~0ULL ? INT64_MAX : elem(fk);
    const int64_t ev = fv == ~0ULL ? INT64_MAX : elem(fv);
    const int layer = begin_ + li;
    if (ek <= ev) return "cached K diverges at layer " + std::to_string(layer) + " flat index " + std::to_string(ek);
    return "cached V diverges at layer " + std::to_string(layer) + " flat index " + std::to_string(ev);
  }
  return "";
}

void Stage::prof_mark(int cls, bool begin) {
  if (!prof_on_) return;
  if (prof_used_ == prof_pool_.size()) {
    cudaEvent_t e;
    BP_CUDA(cudaEventCreate(&e));
    prof_pool_.push_back(e);
  }
  cudaEvent_t e = prof_pool_[prof_used_++];
  BP_CUDA(cudaEventRecord(e, stream_));
  if (begin) {
    prof_open_ = e;
  } else {
    prof_marks_.push_back({cls, {prof_open_, e}});
  }
}

void Stage::prof_collect(double ms[4], int64_t launches[4]) {
  for (int i = 0; i < 4; ++i) { ms[i] = 0.0; launches[i] = 0; }
  if (!prof_marks_.empty()) BP_CUDA(cudaEventSynchronize(prof_marks_.back().second.second));
  for (const auto& m : prof_marks_) {
    float t = 0.f;
    BP_CUDA(cudaEventElapsedTime(&t, m.second.first, m.second.second));
    ms[m.first] += t;
    launches[m.first] += 1;
  }
  prof_marks_.clear();
  prof_used_ = 0;
}

template const void* Stage::forward_simt<double>(const StageInput&);
template const void* Stage::forward_simt<float>(const StageInput&);
template const void* Stage::forward_wan_simt<double>(const StageInput&);
template const void* Stage::forward_wan_simt<float>(const StageInput&);

}  // namespace bp
