// Operator surface of the B200 blockpipe: closed-form analytics, the flat
// JSON run config, the four artifact writers and the CLI.
// Mirrors P/include/blockpipe/{analytics,run_config,artifacts,cli}.hpp so a
// reference user finds the same names; every run goes through the GPU engine
// (run_pipeline in blockpipe_b200.hpp).
#pragma once

#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "blockpipe/blockpipe_b200.hpp"

namespace blockpipe {

// ---------------------------------------------------------------- analytics (P/analytics.hpp:15-75)
struct BubbleParams {
  int devices = 1;       // N
  int steps = 1;         // T
  int64_t block_num = 1;
  Order order = Order::kReverse;
  void validate() const;
};
int64_t bubble_size(const BubbleParams& bp);   // analytics.cpp:13-24
double bubble_ratio(const BubbleParams& bp);   // analytics.cpp:26-31

struct CostParams {
  int64_t frames = 16, height = 4, width = 4, hidden = 8, channels = 4, layers = 8, devices = 2;
  int64_t num_b = 8, num_c = 8;
  double model_mem = 1.0, kv_mem = 1.0;
  bool ring_refinement = false;
  // Extension ("analytics in bytes"): bytes per communicated scalar
  // (8 fp64, 4 fp32, 2 bf16); 0 leaves comm_bytes unset.
  int bytes_per_scalar = 0;
  int64_t seq_len() const { return frames * height * width; }
  void validate() const;
};

enum class Method { kRingAttention, kUlysses, kVideoInfinity, kFifo, kDualParal };
Method parse_method(const std::string& name);
std::string method_name(Method m);
std::vector<Method> all_methods();

struct MethodCost {
  Method method = Method::kDualParal;
  double comm_scalars = 0.0;
  bool comm_overlap = false;
  double model_mem = 0.0;
  double kv_mem = 0.0;
  double comm_bytes = 0.0;  // extension: comm_scalars * bytes_per_scalar
};
MethodCost method_cost(Method m, const CostParams& cp);  // analytics.cpp:67-117

struct SweepPoint {
  std::string axis;  // "N" or "F"
  int64_t value = 0;
  MethodCost cost;
};
std::vector<SweepPoint> sweep_devices(const CostParams& cp, const std::vector<Method>& ms,
                                      const std::vector<int64_t>& device_counts);
std::vector<SweepPoint> sweep_frames(const CostParams& cp, const std::vector<Method>& ms,
                                     const std::vector<int64_t>& frame_counts);

// Extension: predicted boundary traffic of one whole run in bytes, from the
// transfer ledger (scalars x boundary element size: 8 for f64, 4 for f32 and
// for bf16, whose residual stream crosses stages in fp32), next to
// what the engine actually moved (bp_pipeline_stats.boundary_bytes).
struct TrafficReport {
  int64_t ledger_scalars = 0;
  int64_t predicted_bytes = 0;
  int64_t measured_bytes = -1;  // -1: not measured (plan only)
};
TrafficReport traffic_report(const TransferLedger& ledger, Precision p, int64_t measured_bytes = -1);

// ---------------------------------------------------------------- run config (P/run_config.hpp:14-31)
struct RunConfig {
  PipelineConfig pipe;
  std::string out_dir = "out";
  bool emit_first_surplus = true;
  std::string format = "text";
  void validate() const;
};
std::string order_token(Order o);
Order parse_order(const std::string& s);
std::string cache_token(CacheMode m);
CacheMode parse_cache(const std::string& s);
RunConfig load_run_config(const std::string& path);
RunConfig run_config_from_json_text(const std::string& text);
// Reference keys in reference order, dumped with indent 2. B200 extension
// keys (precision, ffn, uneven_split) appear only when set away from their
// defaults, so a reference-valid config echoes byte-identically.
std::string run_config_to_json(const RunConfig& cfg);

// ---------------------------------------------------------------- artifacts (P/artifacts.hpp:20-38)
void write_latents(const std::string& path, const RunResult& result, const RunConfig& cfg);
void write_schedule_csv(const std::string& path, const EventLog& log, const RunConfig& cfg);
void write_transfers_json(const std::string& path, const TransferLedger& ledger, const RunConfig& cfg);
void write_summary_json(const std::string& path, const RunConfig& cfg, const RunResult& result);
// Runs the GPU pipeline and writes the four artifacts; returns the summary path.
std::string run_and_write_artifacts(const RunConfig& cfg);
// Extension: schedule.csv, transfers.json and summary.json from plan_pipeline
// (no device work, no latents.bin). Returns the summary path.
std::string plan_and_write_artifacts(const RunConfig& cfg);

// ---------------------------------------------------------------- CLI (P/cli.hpp:13)
// Subcommands run / verify / analyze {bubble,costs,sweep} / noise-demo (+ plan).
// Exit codes: 0 ok, 1 failure, 2 usage or config error, 3 I/O error.
int cli_main(const std::vector<std::string>& args, std::ostream& out, std::ostream& err);

}  // namespace blockpipe
