// C++ mirror of the reference blockpipe API over the B200 C-ABI.
// See include/blockpipe/blockpipe_b200.hpp.
#include "blockpipe/blockpipe_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

#include "bp_cuda.h"

namespace blockpipe {

namespace {

[[noreturn]] void rethrow(bp_status s) {
  const std::string m = bp_last_error();
  switch (s) {
    case BP_ERR_CONFIG: throw ConfigError(m);
    case BP_ERR_DIMENSION: throw DimensionError(m);
    case BP_ERR_CACHE: throw CacheError(m);
    case BP_ERR_SCHEDULER: throw SchedulerError(m);
    case BP_ERR_QUEUE: throw QueueError(m);
    case BP_ERR_SCHEDULING: throw SchedulingError(m);
    case BP_ERR_PARTITION: throw PartitionError(m);
    case BP_ERR_IO: throw IoError(m);
    default: throw DeviceError(m);
  }
}
void ck(bp_status s) {
  if (s != BP_OK) rethrow(s);
}

int64_t product(const std::vector<int64_t>& s) {
  int64_t n = 1;
  for (int64_t d : s) n *= d;
  return n;
}

bp_model_desc desc_of(const ModelConfig& c) {
  bp_model_desc d{};
  d.layers = c.layers;
  d.hidden = c.hidden;
  d.heads = c.heads;
  d.channels = c.channels;
  d.height = c.height;
  d.width = c.width;
  d.context_len = c.context_len;
  d.ffn = c.ffn;
  d.block = c.wan_block ? BP_BLOCK_WAN : BP_BLOCK_REFERENCE;
  return d;
}

uint64_t fnv(const Tensor& t) {
  uint64_t h = 0xCBF29CE484222325ULL;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(t.data.data());
  for (size_t i = 0; i < t.data.size() * sizeof(double); ++i) h = (h ^ p[i]) * 0x100000001B3ULL;
  return h ^ static_cast<uint64_t>(t.rows() * 1315423911u);
}

}  // namespace

// ---------------------------------------------------------------- Tensor
Tensor::Tensor(std::vector<int64_t> s) : shape(std::move(s)) {
  for (int64_t d : shape)
    if (d < 0) throw DimensionError("negative dimension");
  data.assign(static_cast<size_t>(product(shape)), 0.0);
}
Tensor::Tensor(std::vector<int64_t> s, std::vector<double> d) : shape(std::move(s)), data(std::move(d)) {
  if (product(shape) != static_cast<int64_t>(data.size())) throw DimensionError("data length does not match shape");
}
int64_t Tensor::cols() const {
  if (shape.empty()) return 0;
  int64_t c = 1;
  for (size_t i = 1; i < shape.size(); ++i) c *= shape[i];
  return c;
}
bool Tensor::bitwise_equal(const Tensor& o) const {
  return shape == o.shape && (data.empty() || std::memcmp(data.data(), o.data.data(), data.size() * 8) == 0);
}
bool Tensor::all_finite() const {
  return std::all_of(data.begin(), data.end(), [](double v) { return std::isfinite(v); });
}
Tensor Tensor::reshaped(std::vector<int64_t> s) const {
  if (product(s) != numel()) throw DimensionError("reshape changes the element count");
  return Tensor(std::move(s), data);
}

// ---------------------------------------------------------------- rng
uint64_t RandomSource::next_u64() {
  state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
double RandomSource::next_uniform() { return static_cast<double>(next_u64() >> 11) * (1.0 / 9007199254740992.0); }
double RandomSource::next_normal() {
  double v = 0.0;
  uint64_t fin = 0;
  ck(bp_normals(0, state, 1, 1.0, &v, 0, &fin));
  state = fin;
  return v;
}
Tensor RandomSource::normal_tensor(std::vector<int64_t> shape, double sigma) {
  Tensor t(std::move(shape));
  uint64_t fin = state;
  if (t.numel() > 0) ck(bp_normals(0, state, t.numel(), sigma, t.data.data(), 0, &fin));
  state = fin;
  return t;
}
std::vector<int> RandomSource::permutation(int n) {
  std::vector<int> p(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) p[static_cast<size_t>(i)] = i;
  for (int i = n - 1; i > 0; --i) std::swap(p[static_cast<size_t>(i)], p[next_below(static_cast<uint64_t>(i) + 1)]);
  return p;
}
uint64_t derive_seed(uint64_t base, std::initializer_list<uint64_t> tags) {
  std::vector<uint64_t> t(tags);
  return bp_derive_seed(base, t.data(), static_cast<int32_t>(t.size()));
}

// ---------------------------------------------------------------- model
void ModelConfig::validate() const {
  if (layers < 1) throw ConfigError("layers must be >= 1");
  if (hidden < 2) throw ConfigError("hidden must be >= 2");
  if (heads < 1 || hidden % heads != 0) throw ConfigError("heads must divide hidden");
  if (channels < 1) throw ConfigError("channels must be >= 1");
  if (height < 1 || width < 1) throw ConfigError("token grid must be at least 1x1");
  if (context_len < 1) throw ConfigError("context_len must be >= 1");
}

ModelChunk build_chunk(const ModelConfig& cfg, uint64_t seed, int begin, int end) {
  cfg.validate();
  if (begin < 0 || end > cfg.layers || begin >= end) throw ConfigError("bad layer range");
  ModelChunk c;
  c.cfg = cfg;
  c.seed = seed;
  c.begin = begin;
  c.end = end;
  const bp_model_desc d = desc_of(cfg);
  bp_stage* s = nullptr;
  // the context is loaded on first use by forward_chunk (seed 0 placeholder)
  ck(bp_stage_create(cfg.device, &d, seed, 0, begin, end, static_cast<int32_t>(cfg.precision), &s));
  c.stage = std::shared_ptr<bp_stage>(s, [](bp_stage* p) { bp_stage_destroy(p); });
  c.context_tag = std::make_shared<uint64_t>(0);
  return c;
}
ModelChunk build_model(const ModelConfig& cfg, uint64_t seed) { return build_chunk(cfg, seed, 0, cfg.layers); }

std::vector<ModelChunk> partition(const ModelConfig& cfg, uint64_t seed, int devices) {
  cfg.validate();
  if (devices < 1) throw PartitionError("device count must be >= 1");
  if (cfg.layers % devices != 0)
    throw PartitionError("layers " + std::to_string(cfg.layers) + " not divisible by devices " + std::to_string(devices));
  std::vector<ModelChunk> out;
  const int per = cfg.layers / devices;
  for (int j = 0; j < devices; ++j) out.push_back(build_chunk(cfg, seed, j * per, (j + 1) * per));
  return out;
}

Tensor build_context(const ModelConfig& cfg, uint64_t context_seed) {
  RandomSource rs(context_seed);
  return rs.normal_tensor({cfg.context_len, cfg.hidden});
}

Tensor position_embedding(int64_t pos, int hidden) {
  Tensor e({1, hidden});
  for (int i = 0; 2 * i < hidden; ++i) {
    const double f = std::pow(10000.0, -2.0 * i / hidden);
    e.data[static_cast<size_t>(2 * i)] = std::sin(pos * f);
    if (2 * i + 1 < hidden) e.data[static_cast<size_t>(2 * i + 1)] = std::cos(pos * f);
  }
  return e;
}
Tensor timestep_embedding(int level, int hidden) { return position_embedding(static_cast<int64_t>(level) + 1000000, hidden); }

ChunkOutput forward_chunk(const ModelChunk& chunk, const ChunkInput& in, const Tensor& context, CacheMode mode,
                          const KVCacheEntry* cache, const RecomputeEntry* recorded) {
  const ModelConfig& cfg = chunk.cfg;
  const int tpf = cfg.tokens_per_frame();
  const int64_t frames = static_cast<int64_t>(in.frame_levels.size());
  if (in.frame_ids.size() != in.frame_levels.size()) throw DimensionError("frame_ids and frame_levels disagree");
  const int64_t want_cols = chunk.is_first() ? cfg.channels : cfg.hidden;
  if (in.payload.rows() != frames * tpf || in.payload.cols() != want_cols)
    throw DimensionError(chunk.is_first() ? "chunk 0 expects [tokens, C] latents"
                                          : "interior chunk expects [tokens, h] hidden state");
  const bool use_prefix = cache != nullptr || recorded != nullptr;
  if (mode == CacheMode::kDisabled && use_prefix) throw CacheError("cache supplied while caching is disabled");
  const size_t nl = static_cast<size_t>(chunk.end - chunk.begin);
  if (cache && cache->per_layer.size() != nl) throw CacheError("cache layer count mismatch");
  if (recorded && recorded->layer_inputs.size() != nl) throw CacheError("recorded layer count mismatch");

  const uint64_t tag = fnv(context);
  if (*chunk.context_tag != tag) {
    ck(bp_stage_set_context(chunk.stage.get(), context.data.data(), context.rows(), context.cols()));
    *chunk.context_tag = tag;
  }
  std::vector<int32_t> levels(in.frame_levels.begin(), in.frame_levels.end());
  std::vector<int32_t> cap(in.capture_frames.begin(), in.capture_frames.end());
  std::vector<double> pk, pv;
  bp_chunk_in ci{};
  ci.payload = in.payload.data.data();
  ci.rows = in.payload.rows();
  ci.cols = in.payload.cols();
  ci.frame_levels = levels.data();
  ci.frame_ids = in.frame_ids.data();
  ci.nframes = static_cast<int32_t>(frames);
  ci.capture_frames = cap.data();
  ci.ncapture = static_cast<int32_t>(cap.size());
  ci.record_inputs = in.record_inputs ? 1 : 0;
  ci.mode = static_cast<int32_t>(mode);
  if (cache) {
    const int64_t rows = cache->captured_tokens;
    for (const LayerKV& kv : cache->per_layer) {
      if (kv.k.rows() != rows || kv.k.cols() != cfg.hidden) throw CacheError("cached kv geometry mismatch");
      pk.insert(pk.end(), kv.k.data.begin(), kv.k.data.end());
      pv.insert(pv.end(), kv.v.data.begin(), kv.v.data.end());
    }
    ci.use_prev = 3;
    ci.prefix_k = pk.data();
    ci.prefix_v = pv.data();
    ci.prefix_rows = rows;
  } else if (recorded) {
    for (const Tensor& t : recorded->layer_inputs) pk.insert(pk.end(), t.data.begin(), t.data.end());
    ci.use_prev = 4;
    ci.prefix_k = pk.data();
    ci.prefix_rows = recorded->captured_tokens;
  }
  ChunkOutput out;
  const int64_t out_cols = chunk.is_last() ? cfg.channels : cfg.hidden;
  out.payload = Tensor({in.payload.rows(), out_cols});
  bp_chunk_out co{};
  co.payload = out.payload.data.data();
  co.payload_capacity = out.payload.numel();
  ck(bp_forward_chunk(chunk.stage.get(), &ci, &co));
  if (co.captured) {
    KVCacheEntry e;
    e.captured_tokens = co.captured_tokens;
    for (size_t l = 0; l < nl; ++l) {
      LayerKV kv{Tensor({e.captured_tokens, cfg.hidden}), Tensor({e.captured_tokens, cfg.hidden})};
      int64_t rows = 0;
      ck(bp_stage_cache_rows(chunk.stage.get(), static_cast<int32_t>(l), 0, kv.k.data.data(), &rows));
      ck(bp_stage_cache_rows(chunk.stage.get(), static_cast<int32_t>(l), 1, kv.v.data.data(), &rows));
      e.per_layer.push_back(std::move(kv));
    }
    out.captured = std::move(e);
  }
  if (co.recorded) {
    RecomputeEntry r;
    int64_t rows = 0;
    ck(bp_stage_recorded_rows(chunk.stage.get(), 0, nullptr, &rows));
    r.captured_tokens = rows;
    for (size_t l = 0; l < nl; ++l) {
      Tensor t({rows, cfg.hidden});
      ck(bp_stage_recorded_rows(chunk.stage.get(), static_cast<int32_t>(l), t.data.data(), &rows));
      r.layer_inputs.push_back(std::move(t));
    }
    out.recorded = std::move(r);
  }
  return out;
}

Tensor scheduler_step(const Tensor& x_t, const Tensor& eps_t, int level, int steps) {
  if (!x_t.same_shape(eps_t)) throw SchedulerError("x and eps shapes disagree");
  if (level < 1 || level > steps)
    throw SchedulerError("level " + std::to_string(level) + " outside 1.." + std::to_string(steps));
  Tensor out(x_t.shape);
  ck(bp_scheduler_step(0, x_t.data.data(), eps_t.data.data(), x_t.numel(), level, steps, out.data.data()));
  return out;
}

// ---------------------------------------------------------------- queue / noise
NoisePool build_pool(int num_b, int num_c, std::vector<int64_t> frame_shape, uint64_t noise_seed) {
  if (frame_shape.size() != 3) throw DimensionError("frame_shape must be [H, W, C]");
  NoisePool p;
  p.num_b = num_b;
  p.num_c = num_c;
  p.frame_shape = frame_shape;
  const int m = num_b + num_c / 2;
  const int64_t per = product(frame_shape);
  std::vector<double> all(static_cast<size_t>(std::max(0, m) * per));
  ck(bp_noise_pool(0, num_b, num_c, frame_shape.data(), noise_seed, all.data(), 0));
  for (int i = 0; i < m; ++i)
    p.entries.emplace_back(frame_shape, std::vector<double>(all.begin() + i * per, all.begin() + (i + 1) * per));
  return p;
}

InitStrategy parse_strategy(const std::string& n) {
  if (n == "coordinated") return InitStrategy::kCoordinated;
  if (n == "complete-shuffle") return InitStrategy::kCompleteShuffle;
  if (n == "subset") return InitStrategy::kSubset;
  if (n == "fresh") return InitStrategy::kFresh;
  if (n == "repeat") return InitStrategy::kRepeat;
  throw ConfigError("unknown noise strategy: " + n);
}
std::string strategy_name(InitStrategy s) {
  static const char* names[] = {"coordinated", "complete-shuffle", "subset", "fresh", "repeat"};
  return names[static_cast<int>(s)];
}

// ---------------------------------------------------------------- engine
void PipelineConfig::validate() const {
  model.validate();
  queue.validate();
  if (devices < 1) throw ConfigError("devices must be >= 1");
  if (transport != Transport::kLoopback && world > 1) {
    if (world != devices) throw ConfigError("multi-process transports need world == devices (one stage per process)");
    if (rank < 0 || rank >= world) throw ConfigError("rank outside [0, world)");
    if (bootstrap_dir.empty()) throw ConfigError("multi-process transports need a bootstrap_dir");
  } else if (world != 1 || rank != 0) {
    throw ConfigError("rank / world apply to the multi-process transports (nccl, ipc) only");
  }
  if (model.layers % devices != 0 && !uneven_split)
    throw ConfigError("layers " + std::to_string(model.layers) + " not divisible by devices " + std::to_string(devices));
}

std::string phase_name(Phase p) {
  switch (p) {
    case Phase::kWarmup: return "warmup";
    case Phase::kSteady: return "steady";
    default: return "cooldown";
  }
}

namespace {
bp_pipeline_desc pipe_desc(const PipelineConfig& c) {
  bp_pipeline_desc d{};
  d.devices = c.devices;
  d.order = static_cast<int32_t>(c.order);
  d.cache_mode = static_cast<int32_t>(c.cache_mode);
  d.num_b = c.queue.num_b;
  d.num_c = c.queue.num_c;
  d.steps = c.queue.steps;
  d.block_num = c.queue.block_num;
  d.retain_clean_context = c.queue.retain_clean_context ? 1 : 0;
  d.strategy = static_cast<int32_t>(c.strategy);
  d.model = desc_of(c.model);
  d.seed_model = c.seed_model;
  d.seed_noise = c.seed_noise;
  d.seed_context = c.seed_context;
  d.fault_inject_ulp = c.fault_inject_ulp;
  d.record_trace = c.record_trace;
  d.check_cache = c.check_cache;
  d.precision = static_cast<int32_t>(c.model.precision);
  d.transport = c.devices > 1 && c.world > 1 ? static_cast<int32_t>(c.transport) : BP_TRANSPORT_LOOPBACK;
  d.uneven_split = c.uneven_split;
  return d;
}

struct Collector {
  std::vector<EmittedBlock>* blocks;
  std::vector<int64_t> shape;
};
void on_emit(void* user, int64_t block_id, int64_t frames, const double* data, const int32_t* ids, int32_t nids,
             const int64_t* fids) {
  auto* c = static_cast<Collector*>(user);
  EmittedBlock b;
  b.block_id = block_id;
  std::vector<int64_t> s = c->shape;
  s.insert(s.begin(), frames);
  b.frames = Tensor(s, std::vector<double>(data, data + frames * product(c->shape)));
  b.noise_ids.assign(ids, ids + nids);
  b.frame_ids.assign(fids, fids + frames);
  c->blocks->push_back(std::move(b));
}
}  // namespace

namespace {
// Everything in a RunResult that the data-independent schedule determines
// (event log, ledger, rounds, queue snapshots) -- engine.cpp:343-414 (D6).
void load_schedule(const bp_schedule* s, const PipelineConfig& cfg, RunResult& r) {
  r.rounds = bp_schedule_rounds(s);
  r.log.devices = cfg.devices;
  std::vector<int64_t> ev(static_cast<size_t>(bp_schedule_nevents(s)) * 6);
  bp_schedule_events(s, ev.data());
  for (size_t i = 0; i < ev.size(); i += 6)
    r.log.events.push_back({ev[i], static_cast<int>(ev[i + 1]), ev[i + 2], static_cast<int>(ev[i + 3]),
                            static_cast<Phase>(ev[i + 4]), ev[i + 5]});
  for (int64_t i = 0; i < bp_schedule_nledger(s); ++i) {
    char ch[32];
    LedgerEntry e;
    bp_schedule_ledger(s, i, ch, &e.round, &e.passes, &e.scalars);
    e.channel = ch;
    r.ledger.entries.push_back(e);
  }
  for (int64_t i = 0; i < bp_schedule_nsnapshots(s); ++i) {
    QueueSnapshot q;
    const int32_t n = bp_schedule_snapshot(s, i, &q.round, nullptr, nullptr);
    q.block_ids.resize(static_cast<size_t>(n));
    std::vector<int32_t> lv(static_cast<size_t>(n));
    bp_schedule_snapshot(s, i, &q.round, q.block_ids.data(), lv.data());
    q.levels.assign(lv.begin(), lv.end());
    r.queue_snapshots.push_back(std::move(q));
  }
}

using ScheduleGuard = std::unique_ptr<bp_schedule, void (*)(bp_schedule*)>;
ScheduleGuard make_schedule(const bp_pipeline_desc& d) {
  bp_schedule* s = nullptr;
  ck(bp_schedule_create(&d, &s));
  return ScheduleGuard(s, bp_schedule_destroy);
}
}  // namespace

RunResult run_pipeline(const PipelineConfig& cfg) {
  cfg.validate();
  const bp_pipeline_desc d = pipe_desc(cfg);
  RunResult r;
  ScheduleGuard s = make_schedule(d);
  bp_pipeline* p = nullptr;
  const bool multi = d.transport != BP_TRANSPORT_LOOPBACK;
  std::vector<uint8_t> ids;
  if (multi && d.transport == BP_TRANSPORT_NCCL) {
    ids.resize(static_cast<size_t>(cfg.world) * 128);
    ck(bp_bootstrap_nccl_ids(cfg.bootstrap_dir.c_str(), cfg.rank, cfg.world, cfg.bootstrap_timeout_ms, ids.data()));
  }
  ck(bp_pipeline_create(&d, multi ? cfg.rank : 0, multi ? cfg.world : 1, cfg.model.device,
                        ids.empty() ? nullptr : ids.data(), &p));
  std::unique_ptr<bp_pipeline, bp_status (*)(bp_pipeline*)> pg(p, bp_pipeline_destroy);
  if (multi && d.transport == BP_TRANSPORT_IPC)
    ck(bp_bootstrap_ipc(p, cfg.bootstrap_dir.c_str(), cfg.rank, cfg.world, cfg.bootstrap_timeout_ms));
  Collector col{&r.blocks, {cfg.model.height, cfg.model.width, cfg.model.channels}};
  ck(bp_pipeline_run(p, on_emit, &col));
  bp_pipeline_stats st{};
  ck(bp_pipeline_get_stats(p, &st));
  r.gpu_ms = st.gpu_ms;
  load_schedule(s.get(), cfg, r);
  for (int64_t i = 0; i < bp_pipeline_ntrace(p); ++i) {
    TraceRecord t;
    int64_t rows = 0, cols = 0;
    ck(bp_pipeline_trace(p, i, &t.round, &t.block_id, &rows, &cols, nullptr));
    t.eps = Tensor({rows, cols});
    ck(bp_pipeline_trace(p, i, &t.round, &t.block_id, &rows, &cols, t.eps.data.data()));
    r.trace.push_back(std::move(t));
  }
  return r;
}

RunResult plan_pipeline(const PipelineConfig& cfg) {
  cfg.validate();
  const bp_pipeline_desc d = pipe_desc(cfg);
  RunResult r;
  ScheduleGuard s = make_schedule(d);
  load_schedule(s.get(), cfg, r);
  for (int64_t i = 0; i < bp_schedule_nblocks(s.get()); ++i) {
    EmittedBlock b;
    int64_t frames = 0;
    const int32_t nids = bp_schedule_block(s.get(), i, &b.block_id, &frames, nullptr, nullptr);
    b.noise_ids.resize(static_cast<size_t>(nids));
    b.frame_ids.resize(static_cast<size_t>(frames));
    bp_schedule_block(s.get(), i, &b.block_id, &frames, b.noise_ids.data(), b.frame_ids.data());
    b.frames.shape = {frames, cfg.model.height, cfg.model.width, cfg.model.channels};
    r.blocks.push_back(std::move(b));
  }
  return r;
}

RunResult serial_oracle(PipelineConfig cfg) {
  cfg.devices = 1;
  cfg.threaded = false;
  cfg.uneven_split = false;
  return run_pipeline(cfg);
}

BubbleStats measure_bubbles(const EventLog& log) {
  BubbleStats st;
  if (log.events.empty()) return st;
  if (log.devices < 1) throw SchedulingError("malformed event log: no devices");
  std::vector<std::vector<const ScheduleEvent*>> per(static_cast<size_t>(log.devices));
  int64_t first = log.events.front().slot, last = first;
  for (const ScheduleEvent& e : log.events) {
    if (e.device < 0 || e.device >= log.devices) throw SchedulingError("malformed event log: device out of range");
    per[static_cast<size_t>(e.device)].push_back(&e);
    first = std::min(first, e.slot);
    last = std::max(last, e.slot);
  }
  const int64_t busy = static_cast<int64_t>(per[0].size());
  for (const auto& v : per) {
    if (static_cast<int64_t>(v.size()) != busy) throw SchedulingError("malformed event log: devices saw different pass counts");
    for (size_t i = 1; i < v.size(); ++i)
      if (v[i]->slot <= v[i - 1]->slot) throw SchedulingError("malformed event log: duplicate slot on one device");
  }
  st.first_slot = first;
  st.last_slot = last;
  st.busy_per_device = busy;
  st.idle_per_device = (last - first + 1) - busy;
  for (const auto& v : per) {
    size_t k = 0;
    for (int64_t s = first; s <= last; ++s) {
      while (k < v.size() && v[k]->slot < s) ++k;
      if (k < v.size() && v[k]->slot == s) continue;
      const Phase p = k < v.size() ? v[k]->phase : Phase::kCooldown;
      (p == Phase::kWarmup ? st.warmup_idle : p == Phase::kSteady ? st.steady_idle : st.cooldown_idle)++;
    }
  }
  const double idle = static_cast<double>(st.idle_per_device) * log.devices;
  st.ratio = idle <= 0 ? 0.0 : idle / (idle + static_cast<double>(busy) * log.devices);
  return st;
}

std::vector<ScheduleEvent> schedule_grid(const EventLog& log) {
  std::vector<ScheduleEvent> grid;
  if (log.events.empty()) return grid;
  int64_t first = log.events.front().slot, last = first;
  for (const ScheduleEvent& e : log.events) {
    first = std::min(first, e.slot);
    last = std::max(last, e.slot);
  }
  for (int64_t s = first; s <= last; ++s) {
    for (int d = 0; d < log.devices; ++d) {
      const ScheduleEvent* hit = nullptr;
      const ScheduleEvent* next = nullptr;
      for (const ScheduleEvent& e : log.events) {
        if (e.device != d) continue;
        if (e.slot == s) hit = &e;
        if (e.slot >= s && (!next || e.slot < next->slot)) next = &e;
      }
      if (hit) grid.push_back(*hit);
      else grid.push_back({s, d, -1, -1, next ? next->phase : Phase::kCooldown, 0});
    }
  }
  return grid;
}

bool blocks_bitwise_equal(const std::vector<EmittedBlock>& a, const std::vector<EmittedBlock>& b, std::string* diff) {
  auto fail = [&](const std::string& m) { if (diff) *diff = m; return false; };
  if (a.size() != b.size()) return fail("emitted block counts differ");
  for (size_t i = 0; i < a.size(); ++i) {
    if (a[i].block_id != b[i].block_id) return fail("block id mismatch at position " + std::to_string(i));
    if (!a[i].frames.bitwise_equal(b[i].frames)) return fail("block " + std::to_string(a[i].block_id) + " differs");
  }
  return true;
}

bool traces_bitwise_equal(const std::vector<TraceRecord>& a, const std::vector<TraceRecord>& b, std::string* diff) {
  auto fail = [&](const std::string& m) { if (diff) *diff = m; return false; };
  if (a.size() != b.size()) return fail("trace lengths differ");
  for (size_t i = 0; i < a.size(); ++i) {
    if (a[i].round != b[i].round || a[i].block_id != b[i].block_id) return fail("trace order diverges");
    if (!a[i].eps.bitwise_equal(b[i].eps)) return fail("pass output differs at round " + std::to_string(a[i].round));
  }
  return true;
}

}  // namespace blockpipe
