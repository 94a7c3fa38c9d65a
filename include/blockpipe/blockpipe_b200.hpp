// blockpipe_b200.hpp — the reference blockpipe C++ API for the block-wise
// denoising path, served by the B200 C-ABI (bp_cuda.h, libbp_cuda.so).
//
// Same namespace, type names, function names and argument meaning as the
// reference headers (P = /root/reference/proj/include/blockpipe): errors.hpp,
// tensor.hpp, rng.hpp, model.hpp, noise.hpp, block_queue.hpp, engine.hpp, so
// a caller recompiles against this header and links libblockpipe_b200.so.
// Host containers (Tensor, RunResult, ...) are plain C++; all model math,
// noise and the pipeline run on the GPU. Extensions are defaulted so that a
// reference-default config behaves like the reference (fp64 parity mode).
#pragma once

#include <cstdint>
#include <deque>
#include <initializer_list>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

struct bp_stage;

namespace blockpipe {

// ---------------------------------------------------------------- errors (P/errors.hpp)
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DimensionError : std::runtime_error { using std::runtime_error::runtime_error; };
struct PartitionError : ConfigError { using ConfigError::ConfigError; };
struct CacheError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SchedulerError : std::runtime_error { using std::runtime_error::runtime_error; };
struct QueueError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SchedulingError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };  // CUDA / NCCL

// ---------------------------------------------------------------- tensor (P/tensor.hpp)
// Host row-major fp64 container used at the API boundary.
struct Tensor {
  std::vector<int64_t> shape;
  std::vector<double> data;
  Tensor() = default;
  explicit Tensor(std::vector<int64_t> s);
  Tensor(std::vector<int64_t> s, std::vector<double> d);
  int64_t numel() const { return static_cast<int64_t>(data.size()); }
  int64_t rows() const { return shape.empty() ? 0 : shape[0]; }
  int64_t cols() const;
  double& at(int64_t r, int64_t c) { return data[static_cast<size_t>(r * cols() + c)]; }
  double at(int64_t r, int64_t c) const { return data[static_cast<size_t>(r * cols() + c)]; }
  bool same_shape(const Tensor& o) const { return shape == o.shape; }
  bool bitwise_equal(const Tensor& o) const;
  bool all_finite() const;
  Tensor reshaped(std::vector<int64_t> s) const;
};

// Free functions of P/tensor.hpp:36-57. matmul / softmax_rows / layer_norm /
// add / sub / scale run on the GPU (bp_matmul, bp_softmax_rows,
// bp_layer_norm, bp_elementwise: the reference's operation order, so results
// are bitwise or within 1e-13 of the reference's); vcat_rows / slice_rows /
// take_rows are row copies of the host container. Same shape checks and
// DimensionError messages as tensor.cpp.
Tensor matmul(const Tensor& a, const Tensor& b);
Tensor softmax_rows(const Tensor& x);
Tensor layer_norm(const Tensor& x, double eps);
Tensor add(const Tensor& a, const Tensor& b);
Tensor sub(const Tensor& a, const Tensor& b);
Tensor scale(const Tensor& a, double s);
Tensor vcat_rows(const Tensor& a, const Tensor& b);
Tensor slice_rows(const Tensor& x, int64_t begin, int64_t end);
Tensor take_rows(const Tensor& x, const std::vector<int64_t>& idx);

// ---------------------------------------------------------------- rng (P/rng.hpp)
// The integer stream runs on the host; normal_tensor draws on the GPU (bit-exact).
struct RandomSource {
  uint64_t state;
  explicit RandomSource(uint64_t seed) : state(seed) {}
  uint64_t next_u64();
  double next_uniform();
  double next_normal();
  uint64_t next_below(uint64_t n) { return next_u64() % n; }
  Tensor normal_tensor(std::vector<int64_t> shape, double sigma = 1.0);
  std::vector<int> permutation(int n);
};
uint64_t derive_seed(uint64_t base, std::initializer_list<uint64_t> tags);

// ---------------------------------------------------------------- model (P/model.hpp)
enum class Precision { kF64 = 0, kF32 = 1, kBF16 = 2 };

struct ModelConfig {
  int layers = 4, hidden = 16, heads = 2, channels = 2, height = 2, width = 2, context_len = 4;
  int ffn = 0;                        // extension: 0 => 4 * hidden
  bool wan_block = false;             // extension: the optional non-parity Wan2.1-style block (bp_block WAN)
  Precision precision = Precision::kF64;  // extension
  int device = 0;                     // extension
  int tokens_per_frame() const { return height * width; }
  void validate() const;
};

// A contiguous layer range resident on one GPU (weights regenerated on the
// device from derive_seed(seed, {layer, role}); they never live on the host).
struct ModelChunk {
  ModelConfig cfg;
  uint64_t seed = 0;
  int begin = 0, end = 0;
  std::shared_ptr<bp_stage> stage;
  std::shared_ptr<uint64_t> context_tag;  // hash of the context last loaded
  bool is_first() const { return begin == 0; }
  bool is_last() const { return end == cfg.layers; }
};

ModelChunk build_chunk(const ModelConfig& cfg, uint64_t seed, int begin, int end);
ModelChunk build_model(const ModelConfig& cfg, uint64_t seed);
std::vector<ModelChunk> partition(const ModelConfig& cfg, uint64_t seed, int devices);
Tensor build_context(const ModelConfig& cfg, uint64_t context_seed);
Tensor position_embedding(int64_t pos, int hidden);
Tensor timestep_embedding(int level, int hidden);

struct LayerKV { Tensor k, v; };
struct KVCacheEntry {
  int64_t block_id = -1;
  int level = -1;
  int64_t captured_tokens = 0;
  std::vector<LayerKV> per_layer;
};
struct RecomputeEntry {
  int64_t block_id = -1;
  int level = -1;
  int64_t captured_tokens = 0;
  std::vector<Tensor> layer_inputs;
};
enum class CacheMode { kDisabled, kCached, kRecompute };

struct ChunkInput {
  Tensor payload;
  std::vector<int> frame_levels;
  std::vector<int64_t> frame_ids;
  std::vector<int> capture_frames;
  bool record_inputs = false;
};
struct ChunkOutput {
  Tensor payload;
  std::optional<KVCacheEntry> captured;
  std::optional<RecomputeEntry> recorded;
};

ChunkOutput forward_chunk(const ModelChunk& chunk, const ChunkInput& in, const Tensor& context, CacheMode mode,
                          const KVCacheEntry* cache, const RecomputeEntry* recorded);
Tensor scheduler_step(const Tensor& x_t, const Tensor& eps_t, int level, int steps);

// ---------------------------------------------------------------- queue / noise (P/block_queue.hpp, P/noise.hpp)
enum class Order { kReverse, kSequential };
struct QueueParams {
  int num_b = 2, num_c = 4, steps = 8, block_num = 6;
  bool retain_clean_context = true;
  void validate() const;
};
struct NoisePool {
  int num_b = 0, num_c = 0;
  std::vector<int64_t> frame_shape;
  std::vector<Tensor> entries;
  int size() const { return static_cast<int>(entries.size()); }
};
NoisePool build_pool(int num_b, int num_c, std::vector<int64_t> frame_shape, uint64_t noise_seed);
enum class InitStrategy { kCoordinated, kCompleteShuffle, kSubset, kFresh, kRepeat };
InitStrategy parse_strategy(const std::string& name);
std::string strategy_name(InitStrategy s);

// P/noise.hpp:40-68. Ids come from the host integer stream of `rng` (advanced
// exactly as the reference advances it); frames are stacked from the pool on
// the GPU (bp_gather_block / bp_noise_draw), fresh normals drawn on the GPU.
struct NoiseDraw {
  Tensor frames;               // [f, H, W, C]
  std::vector<int> noise_ids;  // pool ids per frame; empty for kFresh
};
NoiseDraw init_first_block(const NoisePool& pool, RandomSource& rng);
NoiseDraw init_next_block(const NoisePool& pool, const std::vector<int>& tail_window_ids, RandomSource& rng);
NoiseDraw init_baseline(InitStrategy variant, const NoisePool& pool, RandomSource& rng);
NoiseDraw draw_first_block(InitStrategy s, const NoisePool& pool, RandomSource& rng);
NoiseDraw draw_next_block(InitStrategy s, const NoisePool& pool, const std::vector<int>& tail_window_ids,
                          RandomSource& rng);

// P/block_queue.hpp:13-102: the FIFO of latent blocks on the host (the engine
// itself replays the same lifecycle from its static schedule, schedule.cpp).
struct LatentBlock {
  int64_t block_id = 0;
  Tensor frames;                      // current state [f, H, W, C]
  std::optional<Tensor> prev_frames;  // state before the last update
  int level = 0;
  int updates = 0;
  std::vector<int> noise_ids;
  std::vector<int64_t> frame_ids;
  int64_t frame_count() const { return frames.rows() == 0 ? 0 : frames.shape[0]; }
};
struct RetainedContext {
  int64_t source_block_id = 0;
  Tensor frames;  // [num_c/2, H, W, C], level 0
  std::vector<int64_t> frame_ids;
};
struct QueueState {
  QueueParams params;
  std::deque<LatentBlock> blocks;  // head first
  int64_t appended_count = 0;
  std::optional<RetainedContext> retained;
  std::vector<int64_t> popped_ids;
  const LatentBlock* find(int64_t block_id) const;
  LatentBlock* find(int64_t block_id);
  int context_frames() const { return params.num_c / 2; }
};
struct ExtendedBlock {
  enum class CtxSource { kNone, kInQueue, kRetained };
  int64_t center_id = 0;
  CtxSource source = CtxSource::kNone;
  int64_t ctx_block_id = 0;
  Tensor explicit_frames;
  std::vector<int> explicit_levels;
  std::vector<int64_t> explicit_frame_ids;
  std::optional<int64_t> cached_context_id;
};
void apply_update(QueueState& q, int64_t block_id, Tensor frames);
QueueState advance(QueueState q, std::optional<LatentBlock> new_block);
std::vector<int64_t> processing_order(const QueueState& q, Order order);
ExtendedBlock assemble_extended(const QueueState& q, int64_t block_id, Order order);
bool levels_are_unit_ladder(const QueueState& q);

// ---------------------------------------------------------------- engine (P/engine.hpp)
enum class Transport { kLoopback = 0, kNccl = 1, kIpc = 2 };  // bp_transport
struct PipelineConfig {
  int devices = 2;
  Order order = Order::kReverse;
  CacheMode cache_mode = CacheMode::kCached;
  bool threaded = true;  // accepted; the GPU engine is stream-ordered
  QueueParams queue;
  ModelConfig model;
  InitStrategy strategy = InitStrategy::kCoordinated;
  uint64_t seed_model = 1, seed_noise = 2, seed_context = 3;
  bool fault_inject_ulp = false, record_trace = false, check_cache = false;
  Transport transport = Transport::kLoopback;  // extension
  bool uneven_split = false;                   // extension
  // Extension, multi-process transports (kNccl / kIpc, one process per
  // stage): this process's rank in [0, world), world == devices; the ranks
  // rendezvous through files in bootstrap_dir (a fresh directory every rank
  // sees). run_pipeline then returns the blocks on rank 0 only (the other
  // ranks' RunResult carries the schedule, no frames). kLoopback runs every
  // stage in this process on model.device.
  int rank = 0, world = 1;
  std::string bootstrap_dir;
  int bootstrap_timeout_ms = 120000;
  void validate() const;
};

enum class Phase { kWarmup, kSteady, kCooldown };
std::string phase_name(Phase p);
struct ScheduleEvent {
  int64_t slot = 0;
  int device = 0;
  int64_t block_id = 0;
  int level = 0;
  Phase phase = Phase::kWarmup;
  int64_t round = 0;
};
struct EventLog { int devices = 1; std::vector<ScheduleEvent> events; };
struct LedgerEntry { std::string channel; int64_t round = 0, passes = 0, scalars = 0; };
struct TransferLedger { std::vector<LedgerEntry> entries; };
struct EmittedBlock { int64_t block_id = 0; Tensor frames; std::vector<int> noise_ids; std::vector<int64_t> frame_ids; };
struct TraceRecord { int64_t round = 0, block_id = 0; Tensor eps; };
struct QueueSnapshot { int64_t round = 0; std::vector<int64_t> block_ids; std::vector<int> levels; };
struct RunResult {
  std::vector<EmittedBlock> blocks;
  EventLog log;
  TransferLedger ledger;
  int64_t rounds = 0;
  std::vector<TraceRecord> trace;
  std::vector<QueueSnapshot> queue_snapshots;
  double gpu_ms = 0.0;  // extension: device time of the run
};

RunResult run_pipeline(const PipelineConfig& cfg);
RunResult serial_oracle(PipelineConfig cfg);
// Extension: the RunResult the static schedule determines -- event log,
// ledger, rounds, queue snapshots and each emitted block's ids and frame
// shape -- without any device work (frames carry a shape but no data).
RunResult plan_pipeline(const PipelineConfig& cfg);

struct BubbleStats {
  int64_t first_slot = 0, last_slot = 0, busy_per_device = 0, idle_per_device = 0;
  int64_t warmup_idle = 0, steady_idle = 0, cooldown_idle = 0;
  double ratio = 0.0;
};
BubbleStats measure_bubbles(const EventLog& log);
std::vector<ScheduleEvent> schedule_grid(const EventLog& log);
bool blocks_bitwise_equal(const std::vector<EmittedBlock>& a, const std::vector<EmittedBlock>& b,
                          std::string* first_diff = nullptr);
bool traces_bitwise_equal(const std::vector<TraceRecord>& a, const std::vector<TraceRecord>& b,
                          std::string* first_diff = nullptr);

}  // namespace blockpipe
