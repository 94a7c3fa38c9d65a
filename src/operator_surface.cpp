// Operator surface over the B200 engine: closed-form analytics, the flat JSON
// run config and the four byte-deterministic artifacts.
//
// Parity anchors:
//   bubble_size / bubble_ratio        P/src/analytics.cpp:13-31
//   method_cost (+ sweeps)            P/src/analytics.cpp:67-141
//   run_config_from_json_text / _to_  P/src/run_config.cpp:48-141
//   write_latents .. write_summary    P/src/artifacts.cpp:25-128
// JSON goes through nlohmann::ordered_json -- the library the reference uses --
// so number formatting (shortest round-trip doubles, "x.0" for integral
// doubles) and the dump(2) layout are identical by construction. The goldens in
// tests/golden/artifacts/ were written by the reference itself.
#include "blockpipe/operator.hpp"

#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>

#include <nlohmann/json.hpp>

namespace blockpipe {

using ojson = nlohmann::ordered_json;

// ============================================================== analytics
void BubbleParams::validate() const {
  if (devices < 1) throw ConfigError("devices must be >= 1");
  if (steps < 1) throw ConfigError("steps must be >= 1");
  if (block_num < 1) throw ConfigError("block_num must be >= 1");
}

int64_t bubble_size(const BubbleParams& bp) {
  bp.validate();
  const int64_t n = bp.devices, t = bp.steps, b = bp.block_num;
  if (n == 1) return 0;                           // one device never waits
  if (bp.order == Order::kSequential) return n * n - 1;
  if (b >= n) return n * (n - 1) - 1;             // warm-up + cool-down only (Eq. 4)
  const int64_t idle = b * (n - t) + n * (t - 2) + 1;  // few blocks: gaps every step (Eq. 5)
  if (idle < 0) throw ConfigError("bubble size negative; parameters out of regime");
  return idle;
}

double bubble_ratio(const BubbleParams& bp) {
  const int64_t idle = bubble_size(bp);
  if (idle == 0) return 0.0;
  const double busy = static_cast<double>(bp.steps) * static_cast<double>(bp.block_num);
  return static_cast<double>(idle) / (static_cast<double>(idle) + busy);
}

void CostParams::validate() const {
  for (int64_t v : {frames, height, width, hidden, channels, layers, devices, num_b})
    if (v < 1) throw ConfigError("cost parameters must be positive");
  if (num_c < 0) throw ConfigError("num_c must be >= 0");
  if (model_mem < 0 || kv_mem < 0) throw ConfigError("memory units must be >= 0");
  if (bytes_per_scalar < 0) throw ConfigError("bytes_per_scalar must be >= 0");
}

namespace {
const std::pair<Method, const char*> kMethods[] = {
    {Method::kRingAttention, "ring-attention"}, {Method::kUlysses, "ulysses"},
    {Method::kVideoInfinity, "video-infinity"}, {Method::kFifo, "fifo"},
    {Method::kDualParal, "dualparal"}};
}  // namespace

Method parse_method(const std::string& name) {
  for (const auto& m : kMethods)
    if (name == m.second) return m.first;
  throw ConfigError("unknown method: " + name);
}

std::string method_name(Method m) {
  for (const auto& e : kMethods)
    if (e.first == m) return e.second;
  throw ConfigError("unreachable method");
}

std::vector<Method> all_methods() {
  std::vector<Method> v;
  for (const auto& m : kMethods) v.push_back(m.first);
  return v;
}

MethodCost method_cost(Method m, const CostParams& cp) {
  cp.validate();
  // Same operand order as the reference so every double is bit-identical.
  const double p = static_cast<double>(cp.seq_len());
  const double h = static_cast<double>(cp.hidden), l = static_cast<double>(cp.layers);
  const double n = static_cast<double>(cp.devices), f = static_cast<double>(cp.frames);
  const double hw = static_cast<double>(cp.height * cp.width), c = static_cast<double>(cp.channels);
  const double nb = static_cast<double>(cp.num_b), nc = static_cast<double>(cp.num_c);
  MethodCost r;
  r.method = m;
  r.model_mem = cp.model_mem;
  switch (m) {
    case Method::kRingAttention:  // K/V ring per layer, overlappable
      r.comm_scalars = 2.0 * p * h * l;
      if (cp.ring_refinement) r.comm_scalars *= (n - 1.0) / n;
      r.comm_overlap = true;
      r.kv_mem = (f / n) * cp.kv_mem;
      break;
    case Method::kUlysses:  // two all-to-alls per attention
      r.comm_scalars = (4.0 / n) * p * h * l;
      r.kv_mem = (f / n) * cp.kv_mem;
      break;
    case Method::kVideoInfinity:  // context frames' activations per layer
      r.comm_scalars = 2.0 * nc * hw * h * l;
      r.kv_mem = (f / n + nc) * cp.kv_mem;
      break;
    case Method::kFifo:  // raw latents (token grid == latent grid)
      r.comm_scalars = 2.0 * (nb + nc) * hw * c;
      r.comm_overlap = true;
      r.kv_mem = (nb + nc) * cp.kv_mem;
      break;
    case Method::kDualParal:  // one block's boundary activations, pipelined
      r.comm_scalars = 2.0 * (nb + nc / 2.0) * hw * h;
      r.comm_overlap = true;
      r.model_mem = cp.model_mem / n;
      r.kv_mem = (nb + nc) * cp.kv_mem;
      break;
  }
  r.comm_bytes = r.comm_scalars * static_cast<double>(cp.bytes_per_scalar);
  return r;
}

namespace {
std::vector<SweepPoint> sweep(const CostParams& cp, const std::vector<Method>& ms,
                              const std::vector<int64_t>& axis_values, const char* axis) {
  if (axis_values.empty()) throw ConfigError("empty sweep axis");
  std::vector<SweepPoint> out;
  for (int64_t v : axis_values) {
    CostParams p = cp;
    (axis[0] == 'N' ? p.devices : p.frames) = v;
    for (Method m : ms) out.push_back({axis, v, method_cost(m, p)});
  }
  return out;
}
}  // namespace

std::vector<SweepPoint> sweep_devices(const CostParams& cp, const std::vector<Method>& ms,
                                      const std::vector<int64_t>& device_counts) {
  return sweep(cp, ms, device_counts, "N");
}
std::vector<SweepPoint> sweep_frames(const CostParams& cp, const std::vector<Method>& ms,
                                     const std::vector<int64_t>& frame_counts) {
  return sweep(cp, ms, frame_counts, "F");
}

TrafficReport traffic_report(const TransferLedger& ledger, Precision p, int64_t measured_bytes) {
  // Only device->device channels cross a GPU boundary; host->dev0 latents and
  // the eps return stay on rank 0 (loopback) or are counted separately. The
  // bf16 path ships its fp32 residual stream, so N stages == 1 stage bitwise.
  const int64_t elem = p == Precision::kF64 ? 8 : 4;
  TrafficReport r;
  for (const LedgerEntry& e : ledger.entries)
    if (e.channel.rfind("dev", 0) == 0 && e.channel.find("->dev") != std::string::npos)
      r.ledger_scalars += e.scalars;
  r.predicted_bytes = r.ledger_scalars * elem;
  r.measured_bytes = measured_bytes;
  return r;
}

// ============================================================== run config
void RunConfig::validate() const {
  pipe.validate();
  if (format != "json" && format != "text" && format != "csv")
    throw ConfigError("format must be json, text or csv");
}

std::string order_token(Order o) { return o == Order::kReverse ? "reverse" : "sequential"; }

Order parse_order(const std::string& s) {
  if (s == "reverse") return Order::kReverse;
  if (s == "sequential") return Order::kSequential;
  throw ConfigError("order must be reverse or sequential, got " + s);
}

std::string cache_token(CacheMode m) {
  return m == CacheMode::kDisabled ? "off" : m == CacheMode::kCached ? "on" : "recompute";
}

CacheMode parse_cache(const std::string& s) {
  if (s == "off") return CacheMode::kDisabled;
  if (s == "on") return CacheMode::kCached;
  if (s == "recompute") return CacheMode::kRecompute;
  throw ConfigError("cache must be on, off or recompute, got " + s);
}

namespace {
const char* precision_token(Precision p) {
  return p == Precision::kF64 ? "f64" : p == Precision::kF32 ? "f32" : "bf16";
}
Precision parse_precision(const std::string& s) {
  if (s == "f64") return Precision::kF64;
  if (s == "f32") return Precision::kF32;
  if (s == "bf16") return Precision::kBF16;
  throw ConfigError("precision must be f64, f32 or bf16, got " + s);
}
bool parse_mode(const std::string& m) {
  if (m == "threaded") return true;
  if (m == "single") return false;
  throw ConfigError("mode must be threaded or single");
}

// Key -> setter table; the JSON value's own conversion rules (nlohmann get<>)
// decide what is accepted, exactly as in the reference.
using Setter = void (*)(RunConfig&, const ojson&);
const std::map<std::string, Setter>& setters() {
  static const std::map<std::string, Setter> t = {
      {"devices", [](RunConfig& c, const ojson& v) { c.pipe.devices = v.get<int>(); }},
      {"order", [](RunConfig& c, const ojson& v) { c.pipe.order = parse_order(v.get<std::string>()); }},
      {"cache", [](RunConfig& c, const ojson& v) { c.pipe.cache_mode = parse_cache(v.get<std::string>()); }},
      {"mode", [](RunConfig& c, const ojson& v) { c.pipe.threaded = parse_mode(v.get<std::string>()); }},
      {"num_b", [](RunConfig& c, const ojson& v) { c.pipe.queue.num_b = v.get<int>(); }},
      {"num_c", [](RunConfig& c, const ojson& v) { c.pipe.queue.num_c = v.get<int>(); }},
      {"steps", [](RunConfig& c, const ojson& v) { c.pipe.queue.steps = v.get<int>(); }},
      {"blocks", [](RunConfig& c, const ojson& v) { c.pipe.queue.block_num = v.get<int>(); }},
      {"retain_clean_context",
       [](RunConfig& c, const ojson& v) { c.pipe.queue.retain_clean_context = v.get<bool>(); }},
      {"layers", [](RunConfig& c, const ojson& v) { c.pipe.model.layers = v.get<int>(); }},
      {"hidden", [](RunConfig& c, const ojson& v) { c.pipe.model.hidden = v.get<int>(); }},
      {"heads", [](RunConfig& c, const ojson& v) { c.pipe.model.heads = v.get<int>(); }},
      {"channels", [](RunConfig& c, const ojson& v) { c.pipe.model.channels = v.get<int>(); }},
      {"height", [](RunConfig& c, const ojson& v) { c.pipe.model.height = v.get<int>(); }},
      {"width", [](RunConfig& c, const ojson& v) { c.pipe.model.width = v.get<int>(); }},
      {"context_len", [](RunConfig& c, const ojson& v) { c.pipe.model.context_len = v.get<int>(); }},
      {"strategy", [](RunConfig& c, const ojson& v) { c.pipe.strategy = parse_strategy(v.get<std::string>()); }},
      {"seed_model", [](RunConfig& c, const ojson& v) { c.pipe.seed_model = v.get<uint64_t>(); }},
      {"seed_noise", [](RunConfig& c, const ojson& v) { c.pipe.seed_noise = v.get<uint64_t>(); }},
      {"seed_context", [](RunConfig& c, const ojson& v) { c.pipe.seed_context = v.get<uint64_t>(); }},
      {"fault_inject", [](RunConfig& c, const ojson& v) { c.pipe.fault_inject_ulp = v.get<bool>(); }},
      {"out_dir", [](RunConfig& c, const ojson& v) { c.out_dir = v.get<std::string>(); }},
      {"emit_first_surplus", [](RunConfig& c, const ojson& v) { c.emit_first_surplus = v.get<bool>(); }},
      {"format", [](RunConfig& c, const ojson& v) { c.format = v.get<std::string>(); }},
      // B200 extensions (precision of the tensor-core path)
      {"precision", [](RunConfig& c, const ojson& v) { c.pipe.model.precision = parse_precision(v.get<std::string>()); }},
      {"ffn", [](RunConfig& c, const ojson& v) { c.pipe.model.ffn = v.get<int>(); }},
      {"block", [](RunConfig& c, const ojson& v) {
         const std::string b = v.get<std::string>();
         if (b != "reference" && b != "wan") throw ConfigError("block must be reference or wan");
         c.pipe.model.wan_block = b == "wan";
       }},
      {"uneven_split", [](RunConfig& c, const ojson& v) { c.pipe.uneven_split = v.get<bool>(); }},
  };
  return t;
}
}  // namespace

RunConfig run_config_from_json_text(const std::string& text) {
  ojson j;
  try {
    j = ojson::parse(text);
  } catch (const ojson::parse_error& e) {
    throw ConfigError(std::string("config parse error: ") + e.what());
  }
  RunConfig cfg;
  if (const char* env = std::getenv("BLOCKPIPE_SEED")) {  // default seeds S, S+1, S+2
    const uint64_t s = std::strtoull(env, nullptr, 10);
    cfg.pipe.seed_model = s;
    cfg.pipe.seed_noise = s + 1;
    cfg.pipe.seed_context = s + 2;
  }
  for (auto it = j.begin(); it != j.end(); ++it) {
    const auto found = setters().find(it.key());
    if (found == setters().end()) throw ConfigError("unknown config key: " + it.key());
    try {
      found->second(cfg, it.value());
    } catch (const ojson::exception& e) {
      throw ConfigError("bad value for key '" + it.key() + "': " + e.what());
    }
  }
  return cfg;
}

RunConfig load_run_config(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open config file: " + path);
  std::ostringstream text;
  text << in.rdbuf();
  return run_config_from_json_text(text.str());
}

namespace {
ojson config_object(const RunConfig& cfg) {
  const PipelineConfig& p = cfg.pipe;
  ojson j;
  j["devices"] = p.devices;
  j["order"] = order_token(p.order);
  j["cache"] = cache_token(p.cache_mode);
  j["mode"] = p.threaded ? "threaded" : "single";
  j["num_b"] = p.queue.num_b;
  j["num_c"] = p.queue.num_c;
  j["steps"] = p.queue.steps;
  j["blocks"] = p.queue.block_num;
  j["retain_clean_context"] = p.queue.retain_clean_context;
  j["layers"] = p.model.layers;
  j["hidden"] = p.model.hidden;
  j["heads"] = p.model.heads;
  j["channels"] = p.model.channels;
  j["height"] = p.model.height;
  j["width"] = p.model.width;
  j["context_len"] = p.model.context_len;
  j["strategy"] = strategy_name(p.strategy);
  j["seed_model"] = p.seed_model;
  j["seed_noise"] = p.seed_noise;
  j["seed_context"] = p.seed_context;
  j["fault_inject"] = p.fault_inject_ulp;
  j["out_dir"] = cfg.out_dir;
  j["emit_first_surplus"] = cfg.emit_first_surplus;
  j["format"] = cfg.format;
  if (p.model.precision != Precision::kF64) j["precision"] = precision_token(p.model.precision);
  if (p.model.ffn != 0) j["ffn"] = p.model.ffn;
  if (p.model.wan_block) j["block"] = "wan";
  if (p.uneven_split) j["uneven_split"] = true;
  return j;
}

std::ofstream open_for_write(const std::string& path, bool binary = false) {
  std::ofstream f(path, binary ? std::ios::out | std::ios::binary : std::ios::out);
  if (!f) throw IoError("cannot write " + path);
  return f;
}
void finish(std::ofstream& f, const std::string& path) {
  f.flush();
  if (!f) throw IoError("short write to " + path);
}
}  // namespace

std::string run_config_to_json(const RunConfig& cfg) { return config_object(cfg).dump(2); }

// ============================================================== artifacts
void write_latents(const std::string& path, const RunResult& result, const RunConfig& cfg) {
  std::ofstream f = open_for_write(path, true);
  const ModelConfig& m = cfg.pipe.model;
  f << "blockpipe-latents v1\n"
    << "shape " << m.height << " " << m.width << " " << m.channels << "\n";
  const int64_t frame_elems = static_cast<int64_t>(m.height) * m.width * m.channels;
  const int64_t surplus = cfg.pipe.queue.num_c / 2;
  for (const EmittedBlock& b : result.blocks) {
    const int64_t frames = b.frames.shape.empty() ? 0 : b.frames.shape[0];
    // --trim-first-surplus drops the first block's built-in context frames.
    const int64_t skip = (!cfg.emit_first_surplus && b.block_id == 1 && frames > surplus) ? surplus : 0;
    const int64_t kept = frames - skip;
    if (static_cast<int64_t>(b.frames.data.size()) != frames * frame_elems)
      throw IoError("block " + std::to_string(b.block_id) + " has no latents to write");
    f << "block " << b.block_id << " " << kept << "\n";
    f.write(reinterpret_cast<const char*>(b.frames.data.data() + skip * frame_elems),
            static_cast<std::streamsize>(kept * frame_elems * static_cast<int64_t>(sizeof(double))));
  }
  finish(f, path);
}

void write_schedule_csv(const std::string& path, const EventLog& log, const RunConfig& cfg) {
  std::ofstream f = open_for_write(path);
  f << "# config " << config_object(cfg).dump() << "\n";
  f << "slot,device,block_id,level,phase\n";
  for (const ScheduleEvent& e : schedule_grid(log)) {
    f << e.slot << ',' << e.device << ',';
    if (e.block_id < 0)
      f << "IDLE,,";
    else
      f << e.block_id << ',' << e.level << ',';
    f << phase_name(e.phase) << '\n';
  }
  finish(f, path);
}

void write_transfers_json(const std::string& path, const TransferLedger& ledger, const RunConfig& cfg) {
  ojson entries = ojson::array();
  for (const LedgerEntry& e : ledger.entries)
    entries.push_back({{"channel", e.channel}, {"round", e.round}, {"passes", e.passes}, {"scalars", e.scalars}});
  ojson j;
  j["config"] = config_object(cfg);
  j["entries"] = std::move(entries);
  std::ofstream f = open_for_write(path);
  f << j.dump(2) << "\n";
  finish(f, path);
}

void write_summary_json(const std::string& path, const RunConfig& cfg, const RunResult& result) {
  const BubbleStats st = measure_bubbles(result.log);
  const BubbleParams bp{cfg.pipe.devices, cfg.pipe.queue.steps, cfg.pipe.queue.block_num, cfg.pipe.order};
  ojson j;
  j["config"] = config_object(cfg);
  j["rounds"] = result.rounds;
  ojson measured;
  measured["busy_per_device"] = st.busy_per_device;
  measured["idle_per_device"] = st.idle_per_device;
  measured["warmup_idle"] = st.warmup_idle;
  measured["steady_idle"] = st.steady_idle;
  measured["cooldown_idle"] = st.cooldown_idle;
  measured["ratio"] = st.ratio;
  ojson formula;
  formula["size"] = bubble_size(bp);
  formula["ratio"] = bubble_ratio(bp);
  j["bubbles"]["measured"] = std::move(measured);
  j["bubbles"]["formula"] = std::move(formula);
  ojson emitted = ojson::array();
  for (const EmittedBlock& b : result.blocks) {
    ojson e;
    e["block_id"] = b.block_id;
    e["frames"] = b.frames.shape.empty() ? 0 : b.frames.shape[0];
    e["noise_ids"] = b.noise_ids;
    e["frame_ids"] = b.frame_ids;
    emitted.push_back(std::move(e));
  }
  j["emitted"] = std::move(emitted);
  ojson totals = ojson::object();  // channel -> scalars, first-appearance order
  for (const LedgerEntry& e : result.ledger.entries) {
    const int64_t prev = totals.contains(e.channel) ? totals[e.channel].get<int64_t>() : 0;
    totals[e.channel] = prev + e.scalars;
  }
  j["transfer_totals"] = std::move(totals);
  ojson queue = ojson::array();
  for (const QueueSnapshot& s : result.queue_snapshots) {
    ojson q;
    q["round"] = s.round;
    q["block_ids"] = s.block_ids;
    q["levels"] = s.levels;
    queue.push_back(std::move(q));
  }
  j["queue"] = std::move(queue);
  std::ofstream f = open_for_write(path);
  f << j.dump(2) << "\n";
  finish(f, path);
}

namespace {
std::string prepare_out_dir(const RunConfig& cfg) {
  cfg.validate();
  std::error_code ec;
  std::filesystem::create_directories(cfg.out_dir, ec);
  if (ec) throw IoError("cannot create output directory " + cfg.out_dir);
  return cfg.out_dir + "/";
}
}  // namespace

std::string run_and_write_artifacts(const RunConfig& cfg) {
  const std::string dir = prepare_out_dir(cfg);
  const RunResult r = run_pipeline(cfg.pipe);
  write_latents(dir + "latents.bin", r, cfg);
  write_schedule_csv(dir + "schedule.csv", r.log, cfg);
  write_transfers_json(dir + "transfers.json", r.ledger, cfg);
  write_summary_json(dir + "summary.json", cfg, r);
  return dir + "summary.json";
}

std::string plan_and_write_artifacts(const RunConfig& cfg) {
  const std::string dir = prepare_out_dir(cfg);
  const RunResult r = plan_pipeline(cfg.pipe);
  write_schedule_csv(dir + "schedule.csv", r.log, cfg);
  write_transfers_json(dir + "transfers.json", r.ledger, cfg);
  write_summary_json(dir + "summary.json", cfg, r);
  return dir + "summary.json";
}

}  // namespace blockpipe
