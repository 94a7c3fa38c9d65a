// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference `blockpipe` library, compiled
// from the reference sources where they lie (/root/reference/proj/src, see
// oracle/Makefile) into oracle/_ref/libbp_ref.so. It lets the Python tests,
// the golden-vector generator and bench.py's reference/CPU-baseline arm drive
// the reference's own run_pipeline / forward_chunk / build_pool through ctypes.
// Nothing here re-implements reference logic: every call forwards to the
// reference function named in the comment.

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "blockpipe/engine.hpp"
#include "blockpipe/errors.hpp"
#include "blockpipe/model.hpp"
#include "blockpipe/noise.hpp"
#include "blockpipe/rng.hpp"

using namespace blockpipe;

namespace {

thread_local std::string g_err;
thread_local int g_err_kind = 0;

// Same numbering as the product's bp_status (include/bp_cuda.h).
int kind_of(const std::exception& e) {
  if (dynamic_cast<const PartitionError*>(&e)) return 7;
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const DimensionError*>(&e)) return 2;
  if (dynamic_cast<const CacheError*>(&e)) return 3;
  if (dynamic_cast<const SchedulerError*>(&e)) return 4;
  if (dynamic_cast<const QueueError*>(&e)) return 5;
  if (dynamic_cast<const SchedulingError*>(&e)) return 6;
  return 9;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    g_err_kind = 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_kind = kind_of(e);
    return g_err_kind;
  }
}

}  // namespace

extern "C" {

struct bpref_cfg {
  int32_t devices, order, cache_mode, threaded;
  int32_t num_b, num_c, steps, block_num, retain_clean_context;
  int32_t layers, hidden, heads, channels, height, width, context_len;
  int32_t strategy;
  uint64_t seed_model, seed_noise, seed_context;
  int32_t fault_inject_ulp, record_trace, check_cache;
};

const char* bpref_last_error(void) { return g_err.c_str(); }
int bpref_last_error_kind(void) { return g_err_kind; }

// ---- rng.hpp ----------------------------------------------------------------
uint64_t bpref_derive_seed(uint64_t base, const uint64_t* tags, int n) {
  uint64_t s = base;
  // derive_seed takes an initializer_list; fold one tag at a time, which is
  // exactly its loop (rng.cpp:51-60) applied incrementally.
  for (int i = 0; i < n; ++i) s = derive_seed(s, {tags[i]});
  return s;
}
void bpref_u64(uint64_t seed, int64_t n, uint64_t* out) {
  RandomSource rs(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rs.next_u64();
}
void bpref_normals(uint64_t seed, int64_t n, double sigma, double* out) {
  RandomSource rs(seed);
  Tensor t = rs.normal_tensor({n}, sigma);
  std::memcpy(out, t.data.data(), sizeof(double) * n);
}
void bpref_permutation(uint64_t seed, int n, int* out) {
  RandomSource rs(seed);
  std::vector<int> p = rs.permutation(n);
  std::memcpy(out, p.data(), sizeof(int) * n);
}
double bpref_log(double x) { return std::log(x); }
double bpref_cos(double x) { return std::cos(x); }

// ---- noise.hpp --------------------------------------------------------------
int bpref_pool(int num_b, int num_c, int64_t H, int64_t W, int64_t C, uint64_t seed,
               double* out) {
  return guard([&] {
    NoisePool p = build_pool(num_b, num_c, {H, W, C}, seed);
    const int64_t per = H * W * C;
    for (int i = 0; i < p.size(); ++i)
      std::memcpy(out + i * per, p.entries[i].data.data(), sizeof(double) * per);
  });
}

// ---- model.hpp --------------------------------------------------------------
static ModelConfig to_model(const bpref_cfg* c) {
  ModelConfig m;
  m.layers = c->layers;
  m.hidden = c->hidden;
  m.heads = c->heads;
  m.channels = c->channels;
  m.height = c->height;
  m.width = c->width;
  m.context_len = c->context_len;
  return m;
}

// Writes the 16 per-layer weight tensors (build_layer, model.cpp:87-107) back
// to back in Role order: wq wk wv wo cq ck cv co w1 w2 ln1g ln1b ln2g ln2b ln3g ln3b.
int bpref_build_layer(const bpref_cfg* c, uint64_t seed, int layer, double* out) {
  return guard([&] {
    LayerWeights w = build_layer(to_model(c), seed, layer);
    const Tensor* ts[] = {&w.wq, &w.wk, &w.wv, &w.wo, &w.cq, &w.ck, &w.cv, &w.co,
                          &w.w1, &w.w2, &w.ln1_g, &w.ln1_b, &w.ln2_g, &w.ln2_b,
                          &w.ln3_g, &w.ln3_b};
    for (const Tensor* t : ts) {
      std::memcpy(out, t->data.data(), sizeof(double) * t->numel());
      out += t->numel();
    }
  });
}
int bpref_build_context(const bpref_cfg* c, uint64_t seed, double* out) {
  return guard([&] {
    Tensor t = build_context(to_model(c), seed);
    std::memcpy(out, t.data.data(), sizeof(double) * t.numel());
  });
}

// A chunk plus the per-device single-entry cache a DeviceWorker keeps
// (engine.cpp:207-216), so tests can replay capture -> consume sequences.
struct bpref_chunk {
  ModelChunk chunk;
  Tensor context;
  std::optional<KVCacheEntry> cache;
  std::optional<RecomputeEntry> recorded;
};

void* bpref_chunk_create(const bpref_cfg* c, uint64_t seed, int begin, int end,
                         uint64_t context_seed) {
  bpref_chunk* h = nullptr;
  guard([&] {
    auto p = std::make_unique<bpref_chunk>();
    p->chunk = build_chunk(to_model(c), seed, begin, end);
    p->context = build_context(to_model(c), context_seed);
    h = p.release();
  });
  return h;
}
void bpref_chunk_destroy(void* h) { delete static_cast<bpref_chunk*>(h); }

// One forward_chunk (model.cpp:227-336). use_prev: 0 none, 1 the cache
// captured by the previous call, 2 the recording of the previous call.
// The previous call's capture/recording is replaced by this call's.
int bpref_chunk_forward(void* hv, const double* payload, int64_t rows, int64_t cols,
                        const int* levels, const int64_t* frame_ids, int nframes,
                        const int* capture, int ncap, int mode, int use_prev,
                        int record_inputs, double* out, int64_t* out_cols) {
  auto* h = static_cast<bpref_chunk*>(hv);
  return guard([&] {
    ChunkInput in;
    in.payload = Tensor({rows, cols}, std::vector<double>(payload, payload + rows * cols));
    in.frame_levels.assign(levels, levels + nframes);
    in.frame_ids.assign(frame_ids, frame_ids + nframes);
    in.capture_frames.assign(capture, capture + ncap);
    in.record_inputs = record_inputs != 0;
    const KVCacheEntry* cache = (use_prev == 1 && h->cache) ? &*h->cache : nullptr;
    const RecomputeEntry* rec = (use_prev == 2 && h->recorded) ? &*h->recorded : nullptr;
    ChunkOutput o = forward_chunk(h->chunk, in, h->context, static_cast<CacheMode>(mode),
                                  cache, rec);
    std::memcpy(out, o.payload.data.data(), sizeof(double) * o.payload.numel());
    *out_cols = o.payload.cols();
    h->cache = std::move(o.captured);
    h->recorded = std::move(o.recorded);
  });
}

// Captured K (or V when which=1) of layer li from the last call.
int bpref_chunk_cache(void* hv, int li, int which, double* out, int64_t* rows) {
  auto* h = static_cast<bpref_chunk*>(hv);
  return guard([&] {
    if (!h->cache) throw CacheError("no capture");
    const Tensor& t = which ? h->cache->per_layer[li].v : h->cache->per_layer[li].k;
    if (out) std::memcpy(out, t.data.data(), sizeof(double) * t.numel());
    *rows = t.rows();
  });
}

// ---- engine.hpp -------------------------------------------------------------
struct bpref_run_result {
  RunResult r;
  std::vector<int64_t> events;  // 6 per event
};

static PipelineConfig to_pipe(const bpref_cfg* c) {
  PipelineConfig p;
  p.devices = c->devices;
  p.order = static_cast<Order>(c->order);
  p.cache_mode = static_cast<CacheMode>(c->cache_mode);
  p.threaded = c->threaded != 0;
  p.queue.num_b = c->num_b;
  p.queue.num_c = c->num_c;
  p.queue.steps = c->steps;
  p.queue.block_num = c->block_num;
  p.queue.retain_clean_context = c->retain_clean_context != 0;
  p.model = to_model(c);
  p.strategy = static_cast<InitStrategy>(c->strategy);
  p.seed_model = c->seed_model;
  p.seed_noise = c->seed_noise;
  p.seed_context = c->seed_context;
  p.fault_inject_ulp = c->fault_inject_ulp != 0;
  p.record_trace = c->record_trace != 0;
  p.check_cache = c->check_cache != 0;
  return p;
}

// run_pipeline (engine.cpp:255) or serial_oracle (engine.cpp:499).
void* bpref_run(const bpref_cfg* c, int serial) {
  bpref_run_result* h = nullptr;
  guard([&] {
    auto p = std::make_unique<bpref_run_result>();
    p->r = serial ? serial_oracle(to_pipe(c)) : run_pipeline(to_pipe(c));
    for (const ScheduleEvent& e : p->r.log.events) {
      p->events.insert(p->events.end(), {e.slot, e.device, e.block_id, e.level,
                                         static_cast<int64_t>(e.phase), e.round});
    }
    h = p.release();
  });
  return h;
}
void bpref_run_free(void* h) { delete static_cast<bpref_run_result*>(h); }

int64_t bpref_run_rounds(void* h) { return static_cast<bpref_run_result*>(h)->r.rounds; }
int64_t bpref_run_nblocks(void* h) {
  return static_cast<int64_t>(static_cast<bpref_run_result*>(h)->r.blocks.size());
}
// Block i in emission order: id, frame count, noise-id count; then arrays.
void bpref_run_block_info(void* hv, int64_t i, int64_t* id, int64_t* frames, int64_t* nids) {
  const EmittedBlock& b = static_cast<bpref_run_result*>(hv)->r.blocks[i];
  *id = b.block_id;
  *frames = b.frames.shape[0];
  *nids = static_cast<int64_t>(b.noise_ids.size());
}
void bpref_run_block_data(void* hv, int64_t i, double* frames, int* noise_ids,
                          int64_t* frame_ids) {
  const EmittedBlock& b = static_cast<bpref_run_result*>(hv)->r.blocks[i];
  std::memcpy(frames, b.frames.data.data(), sizeof(double) * b.frames.numel());
  for (size_t k = 0; k < b.noise_ids.size(); ++k) noise_ids[k] = b.noise_ids[k];
  for (size_t k = 0; k < b.frame_ids.size(); ++k) frame_ids[k] = b.frame_ids[k];
}
int64_t bpref_run_nevents(void* h) {
  return static_cast<int64_t>(static_cast<bpref_run_result*>(h)->r.log.events.size());
}
void bpref_run_events(void* hv, int64_t* out) {
  auto* h = static_cast<bpref_run_result*>(hv);
  std::memcpy(out, h->events.data(), sizeof(int64_t) * h->events.size());
}
int64_t bpref_run_nledger(void* h) {
  return static_cast<int64_t>(static_cast<bpref_run_result*>(h)->r.ledger.entries.size());
}
void bpref_run_ledger(void* hv, int64_t i, char* channel, int64_t* round, int64_t* passes,
                      int64_t* scalars) {
  const LedgerEntry& e = static_cast<bpref_run_result*>(hv)->r.ledger.entries[i];
  std::strncpy(channel, e.channel.c_str(), 31);
  channel[31] = 0;
  *round = e.round;
  *passes = e.passes;
  *scalars = e.scalars;
}
int64_t bpref_run_nsnap(void* h) {
  return static_cast<int64_t>(static_cast<bpref_run_result*>(h)->r.queue_snapshots.size());
}
// Snapshot i: writes up to 64 (id, level) pairs; returns the count.
int bpref_run_snap(void* hv, int64_t i, int64_t* round, int64_t* ids, int* levels) {
  const QueueSnapshot& s = static_cast<bpref_run_result*>(hv)->r.queue_snapshots[i];
  *round = s.round;
  for (size_t k = 0; k < s.block_ids.size(); ++k) {
    ids[k] = s.block_ids[k];
    levels[k] = s.levels[k];
  }
  return static_cast<int>(s.block_ids.size());
}
int64_t bpref_run_ntrace(void* h) {
  return static_cast<int64_t>(static_cast<bpref_run_result*>(h)->r.trace.size());
}
void bpref_run_trace_info(void* hv, int64_t i, int64_t* round, int64_t* block, int64_t* rows,
                          int64_t* cols) {
  const TraceRecord& t = static_cast<bpref_run_result*>(hv)->r.trace[i];
  *round = t.round;
  *block = t.block_id;
  *rows = t.eps.rows();
  *cols = t.eps.cols();
}
void bpref_run_trace_data(void* hv, int64_t i, double* out) {
  const TraceRecord& t = static_cast<bpref_run_result*>(hv)->r.trace[i];
  std::memcpy(out, t.eps.data.data(), sizeof(double) * t.eps.numel());
}
// measure_bubbles (engine.cpp:505): first,last,busy,idle,warm,steady,cool; ratio.
void bpref_run_bubbles(void* hv, int64_t* out7, double* ratio) {
  BubbleStats st = measure_bubbles(static_cast<bpref_run_result*>(hv)->r.log);
  int64_t v[7] = {st.first_slot, st.last_slot, st.busy_per_device, st.idle_per_device,
                  st.warmup_idle, st.steady_idle, st.cooldown_idle};
  std::memcpy(out7, v, sizeof(v));
  *ratio = st.ratio;
}

}  // extern "C"

// ---- artifacts.hpp / run_config.hpp (operator surface, for byte-level goldens) ----
#include "blockpipe/artifacts.hpp"
#include "blockpipe/run_config.hpp"
extern "C" int bpref_write_artifacts(const char* config_json, const char* out_dir) {
  return guard([&] {
    RunConfig cfg = run_config_from_json_text(config_json);
    cfg.out_dir = out_dir;
    run_and_write_artifacts(cfg);
  });
}

// ---- analytics.hpp (closed-form formulas) and the noise-demo id walk ----------
#include "blockpipe/analytics.hpp"
extern "C" int bpref_bubble(int n, int t, int64_t blocks, int order, int64_t* size, double* ratio) {
  return guard([&] {
    const BubbleParams bp{n, t, blocks, order ? Order::kSequential : Order::kReverse};
    *size = bubble_size(bp);   // analytics.cpp:13-24
    *ratio = bubble_ratio(bp); // analytics.cpp:26-31
  });
}
// p = {frames,height,width,hidden,channels,layers,devices,num_b,num_c}; mem = {model_mem, kv_mem}
// out = {comm_scalars, comm_overlap, model_mem, kv_mem}
extern "C" int bpref_method_cost(const char* method, const int64_t* p, const double* mem, int ring,
                                 double* out) {
  return guard([&] {
    CostParams cp;
    cp.frames = p[0]; cp.height = p[1]; cp.width = p[2]; cp.hidden = p[3]; cp.channels = p[4];
    cp.layers = p[5]; cp.devices = p[6]; cp.num_b = p[7]; cp.num_c = p[8];
    cp.model_mem = mem[0]; cp.kv_mem = mem[1]; cp.ring_refinement = ring != 0;
    const MethodCost c = method_cost(parse_method(method), cp);  // analytics.cpp:67-117
    out[0] = c.comm_scalars; out[1] = c.comm_overlap ? 1.0 : 0.0; out[2] = c.model_mem; out[3] = c.kv_mem;
  });
}
// Noise ids of the first block and `appends` appends, drawn by the reference's
// draw_first_block / draw_next_block exactly as cli.cpp:499-529 drives them.
// ids is a row-major [appends+1][cap_per] array (-1 padded); counts per block.
extern "C" int bpref_noise_walk(const char* strategy, int appends, int num_b, int num_c, uint64_t seed,
                                int cap_per, int* ids, int* counts) {
  return guard([&] {
    const InitStrategy s = parse_strategy(strategy);
    NoisePool pool = build_pool(num_b, num_c, {2, 2, 1}, seed);
    RandomSource rng(derive_seed(seed, {1}));
    NoiseDraw cur = draw_first_block(s, pool, rng);
    auto put = [&](int row, const std::vector<int>& v) {
      counts[row] = static_cast<int>(v.size());
      for (int k = 0; k < cap_per; ++k) ids[row * cap_per + k] = k < static_cast<int>(v.size()) ? v[k] : -1;
    };
    put(0, cur.noise_ids);
    for (int i = 1; i <= appends; ++i) {
      std::vector<int> window;
      const int w = num_c / 2;
      if (w > 0 && static_cast<int>(cur.noise_ids.size()) >= w) window.assign(cur.noise_ids.end() - w, cur.noise_ids.end());
      cur = draw_next_block(s, pool, window, rng);
      put(i, cur.noise_ids);
    }
  });
}

// draw_first_block then `appends` draw_next_block calls (the engine's window
// rule, engine.cpp:301-324) over a pool of frame_shape; frames of every draw
// concatenated into frames_out (capacity (appends + 1) * M * H*W*C), ids as
// bpref_noise_walk.
extern "C" int bpref_noise_walk_frames(const char* strategy, int appends, int num_b, int num_c, const int64_t* shape,
                                       uint64_t seed, int cap_per, int* ids, int* counts, double* frames_out,
                                       int64_t* nvals) {
  return guard([&] {
    const InitStrategy s = parse_strategy(strategy);
    NoisePool pool = build_pool(num_b, num_c, {shape[0], shape[1], shape[2]}, seed);
    RandomSource rng(derive_seed(seed, {1}));
    int64_t at = 0;
    auto put = [&](int row, const NoiseDraw& d) {
      counts[row] = static_cast<int>(d.noise_ids.size());
      for (int k = 0; k < cap_per; ++k)
        ids[row * cap_per + k] = k < static_cast<int>(d.noise_ids.size()) ? d.noise_ids[static_cast<size_t>(k)] : -1;
      for (double v : d.frames.data) frames_out[at++] = v;
    };
    NoiseDraw cur = draw_first_block(s, pool, rng);
    put(0, cur);
    for (int i = 1; i <= appends; ++i) {
      std::vector<int> window;
      const int w = num_c / 2;
      if (w > 0 && static_cast<int>(cur.noise_ids.size()) >= w) window.assign(cur.noise_ids.end() - w, cur.noise_ids.end());
      cur = draw_next_block(s, pool, window, rng);
      put(i, cur);
    }
    *nvals = at;
  });
}
