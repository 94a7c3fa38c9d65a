// One pipeline stage on one GPU: the reference's ModelChunk (model.hpp:50-60)
// with device-resident weights, the per-device single-entry KV feature cache
// (KVCacheEntry / RecomputeEntry, model.hpp:82-101) kept in HBM and reused in
// place, and forward_chunk (model.cpp:227-336) as device kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "bp_cuda.h"
#include "device.cuh"

namespace bp {

struct StageInput {
  const void* payload = nullptr;       // device: fp64 latents [tokens, C] (first) or hidden [tokens, h]
  int64_t tokens = 0;
  int nframes = 0;
  const int32_t* d_levels = nullptr;   // device, nframes
  const int64_t* d_frame_ids = nullptr;
  std::vector<int> capture_frames;     // host
  bool record_inputs = false;
  int mode = BP_CACHE_DISABLED;
  int use_prev = 0;                    // 0 none, 1 resident cache, 2 resident recording
  int slot = 0;                        // residual-stream ring slot (see Stage::set_ring)
  // Fused send (bf16 reference block, not the last stage; see fuses_send()):
  // the last layer's FFN-down GEMM writes x + FFN(x) straight into out (the
  // next rank's receive slot, a peer mapping) instead of x, after
  // before_out(stream, user) has enqueued the wait for that slot to be free.
  void* out = nullptr;
  void (*before_out)(cudaStream_t, void*) = nullptr;
  void* before_out_user = nullptr;
};

class Stage {
 public:
  Stage(int device, const bp_model_desc& m, uint64_t seed_model, uint64_t seed_context, int begin,
        int end, int precision, cudaStream_t stream);
  ~Stage();

  // Runs forward_chunk; returns the device output pointer (hidden state in
  // the stage's activation dtype, or eps [tokens, C] on the last stage).
  const void* forward(const StageInput& in);

  bool is_first() const { return begin_ == 0; }
  bool is_last() const { return end_ == m_.layers; }
  // Whether forward() honours StageInput::out (the bf16 tensor-core path of
  // the reference block on a stage that sends a hidden state).
  bool fuses_send() const { return prec_ == BP_PREC_BF16 && !wan_ && !is_last() && end_ > begin_; }
  int precision() const { return prec_; }
  size_t act_bytes() const;  // bytes per hidden element (8 fp64, 4 fp32/bf16-path residual)
  size_t eps_bytes() const { return prec_ == BP_PREC_F64 ? 8 : 4; }
  int hidden() const { return m_.hidden; }
  int channels() const { return m_.channels; }
  int tokens_per_frame() const { return tpf_; }
  int local_layers() const { return end_ - begin_; }
  cudaStream_t stream() const { return stream_; }

  // Resident cache bookkeeping (DeviceWorker::cache_/recorded_, engine.cpp:215-216).
  bool cache_valid() const { return cache_.valid; }
  int64_t cache_block() const { return cache_.block_id; }
  int cache_level() const { return cache_.level; }
  int64_t cache_tokens() const { return cache_.tokens; }
  bool rec_valid() const { return rec_.valid; }
  int64_t rec_block() const { return rec_.block_id; }
  void tag_entries(int64_t block_id, int level);
  void cache_rows(int layer, int which, double* host_out);  // fp64 download
  void bump_ulp(int layer, int which, int64_t index);
  std::string audit();  // cache_mismatch_report (model.cpp:171-199)

  // Residual-stream ring for the multi-process executor: forward() runs in
  // place on ring slot `in.slot` (the hidden state [tokens, h] in the
  // activation dtype) and returns that slot (or eps slot `in.slot` on the
  // last stage). A payload that already IS the slot (a receive landed there)
  // is not copied, so a stage boundary costs no device copies: receive into
  // the slot, run the layers in place, send from the slot. Slots are either
  // the stage's own (depth slots of max_tokens rows) or supplied by the
  // caller (NCCL-registered / IPC-exported memory, >= max_tokens rows each).
  void set_ring(int depth, int64_t max_tokens, const std::vector<void*>& x_slots = {},
                const std::vector<void*>& eps_slots = {});
  void* x_slot(int k) const { return xs_[static_cast<size_t>(k)]; }
  void* eps_slot(int k) const { return es_[static_cast<size_t>(k)]; }
  int ring_depth() const { return static_cast<int>(xs_.size()); }
  int64_t input_copies() const { return input_copies_; }  // payloads copied into the ring (not received in place)

  void set_context(const double* host, int64_t rows, int64_t cols);
  // use_prev 3 (host K|V) / 4 (host recorded inputs), fp64 device arrays, layer-major
  void load_host_prefix(int kind, const double* k64, const double* v64, int64_t rows);
  void recorded_rows(int layer, double* host_out);
  int64_t rec_tokens() const { return rec_.tokens; }

  // Per-kernel-class device timing with CUDA events on this stage's stream:
  // class 0 self-attention, 1 cross-attention, 2 GEMMs, 3 LayerNorm.
  void set_profiling(bool on) { prof_on_ = on; }
  void prof_collect(double ms[4], int64_t launches[4]);

 private:
  void prof_mark(int cls, bool begin);
  bool prof_on_ = false;
  std::vector<cudaEvent_t> prof_pool_;
  size_t prof_used_ = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_marks_;
  cudaEvent_t prof_open_ = nullptr;

  struct LayerW {
    void* wqkv = nullptr;   // SIMT: [h, 3h] row-major; bf16: [3h, h] (K-major)
    void* wo = nullptr;
    void* cq = nullptr;
    void* co = nullptr;
    void* w1 = nullptr;     // SIMT: [h, F]; bf16: [F, h]
    void* w2 = nullptr;     // SIMT: [F, h]; bf16: [h, F]
    void* ln = nullptr;     // 6 x [h]: ln1 g,b ln2 g,b ln3 g,b (T; fp32 on bf16 path)
    void* ctx_kv = nullptr; // hoisted cross-attention K|V [Lc, 2h] (T; bf16 on bf16 path)
    void* wan = nullptr;    // Wan block: [mod 6h | gq h | gk h | gcq h | gck h] (T; fp32 on bf16 path)
  };
  struct Entry {  // resident KVCacheEntry or RecomputeEntry
    bool valid = false;
    int64_t block_id = -1;
    int level = -1;
    int64_t tokens = 0;
    std::vector<const void*> k, v, rec;  // per local layer
    int64_t ld = 0;                      // row stride of k/v in elements
  };

  template <typename T> const void* forward_simt(const StageInput& in);
  const void* forward_bf16(const StageInput& in);
  // Optional Wan2.1-style block (bp_block WAN, non-parity)
  template <typename T> void wan_pass_setup(const StageInput& in);
  template <typename T> const void* forward_wan_simt(const StageInput& in);
  const void* forward_wan_bf16(const StageInput& in);
  bool wan_ = false;
  int wnt_ = 0, wnh_ = 0;  // RoPE pairs per head: temporal, height (= width)
  void* wanv_ = nullptr;   // [L_local][10h] per-layer Wan vectors (LayerW::wan points into it)
  struct WanGlobal { void *t1, *tb1, *t2, *tb2, *tp, *tpb, *hmod; } wg_{};
  DevBuf wsin_, wa_, we_, wes_, we0_, wmodt_, whmt_, wttab_, wytab_, wxtab_, wlat_, winT_;
  void build_weights(uint64_t seed_model, uint64_t seed_context);
  void hoist_context(const double* ctx64_device);
  uint64_t seed_model_ = 0;
  DevBuf hostpre_;
  int64_t host_rows_ = 0;
  int host_kind_ = 0;
  void ensure_workspace(int64_t tokens, int64_t capture_tokens, bool new_cache = false, int use_prev = 0);
  void kv_prefix_from_recording(int li, const void* rec_rows, int64_t rows, void* kv_out);
  void capture_kv(const StageInput& in, int li, const void* qkv, size_t eb, Entry* nc);

  int device_, prec_;
  bp_model_desc m_;
  int begin_, end_;
  int h_, heads_, dh_, F_, C_, tpf_, Lc_;
  cudaStream_t stream_;
  bool own_stream_ = false;

  DevBuf weights_;
  std::vector<LayerW> lw_;
  void* w_in_ = nullptr;   // fp64 [C, h]
  void* w_out_ = nullptr;  // T [h, C] (fp32 on the bf16 path)
  DevBuf freq_;            // fp64 [h/2] embedding frequencies
  DevBuf w_in32_;          // fp32 [C, h] (bf16 path)
  DevBuf ttab_;            // (sin, cos)(t * f_k), [tpf][h/2] double2 (bf16 path)
  DevBuf ftab_, lat32_;    // per-pass frame terms / fp32 latents (bf16 path)

  // workspace
  int64_t cap_tokens_ = 0, cap_capture_ = 0;
  DevBuf ln_, attn_, cq_, hmid_, kvp_, lnp_;
  DevBuf xown_[3], eown_[3];       // own residual / eps ring slots
  std::vector<void*> xs_, es_;     // the ring in use (own or caller-supplied)
  bool ring_external_ = false;
  int64_t input_copies_ = 0;
  int64_t ring_tokens_ = 0;
  DevBuf qkv_;             // [tokens][3h], reused by every layer
  DevBuf recbuf_[2];       // [L_local][capture][h] per parity (written before the old one is read)
  DevBuf cap_[2];          // KV feature cache [L_local][capture][2h]; the second buffer
  int cap_sel_ = 0;        // takes a capture whose size differs from the resident entry's
  DevBuf scratch_;         // audit
  int parity_ = 0;
  Entry cache_, rec_;
};

}  // namespace bp
