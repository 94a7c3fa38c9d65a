// C-ABI wrappers of the operator surface (include/bp_operator.h).
#include "bp_operator.h"

#include <cstring>
#include <sstream>
#include <string>

#include "blockpipe/operator.hpp"

namespace {
thread_local std::string g_err;

template <typename F>
int32_t guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const blockpipe::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const blockpipe::IoError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void copy_out(const std::string& s, char* out, int64_t cap) {
  if (!out || cap <= 0) return;
  const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
  std::memcpy(out, s.data(), n);
  out[n] = '\0';
}

blockpipe::CostParams from_c(const bp_cost_params& c) {
  blockpipe::CostParams p;
  p.frames = c.frames;
  p.height = c.height;
  p.width = c.width;
  p.hidden = c.hidden;
  p.channels = c.channels;
  p.layers = c.layers;
  p.devices = c.devices;
  p.num_b = c.num_b;
  p.num_c = c.num_c;
  p.model_mem = c.model_mem;
  p.kv_mem = c.kv_mem;
  p.ring_refinement = c.ring_refinement != 0;
  p.bytes_per_scalar = c.bytes_per_scalar;
  return p;
}
}  // namespace

extern "C" {

const char* bp_operator_last_error(void) { return g_err.c_str(); }

int32_t bp_cli_main(int32_t argc, const char* const* argv, bp_text_sink sink, void* user) {
  std::vector<std::string> args;
  for (int32_t i = 0; i < argc; ++i) args.emplace_back(argv[i]);
  std::ostringstream out, err;
  const int code = blockpipe::cli_main(args, out, err);
  if (sink) {
    const std::string o = out.str(), e = err.str();
    sink(user, 1, o.data(), static_cast<int64_t>(o.size()));
    sink(user, 2, e.data(), static_cast<int64_t>(e.size()));
  }
  return code;
}

int32_t bp_write_artifacts(const char* config_json, int32_t plan_only, char* summary_path, int64_t cap) {
  return guarded([&] {
    const blockpipe::RunConfig cfg = blockpipe::run_config_from_json_text(config_json ? config_json : "{}");
    copy_out(plan_only ? blockpipe::plan_and_write_artifacts(cfg) : blockpipe::run_and_write_artifacts(cfg),
             summary_path, cap);
  });
}

int64_t bp_config_echo(const char* config_json, char* out, int64_t cap) {
  std::string s;
  if (guarded([&] { s = blockpipe::run_config_to_json(blockpipe::run_config_from_json_text(config_json)); }) != 0)
    return -1;
  copy_out(s, out, cap);
  return static_cast<int64_t>(s.size());
}

int32_t bp_bubble(int32_t devices, int32_t steps, int64_t block_num, int32_t order, int64_t* size, double* ratio) {
  return guarded([&] {
    const blockpipe::BubbleParams bp{devices, steps, block_num,
                                     order == BP_ORDER_SEQUENTIAL ? blockpipe::Order::kSequential
                                                                  : blockpipe::Order::kReverse};
    if (size) *size = blockpipe::bubble_size(bp);
    if (ratio) *ratio = blockpipe::bubble_ratio(bp);
  });
}

void bp_cost_defaults(bp_cost_params* cp) {
  const blockpipe::CostParams d;
  *cp = bp_cost_params{d.frames, d.height, d.width, d.hidden, d.channels, d.layers, d.devices, d.num_b, d.num_c,
                       d.model_mem, d.kv_mem, d.ring_refinement ? 1 : 0, d.bytes_per_scalar};
}

int32_t bp_method_cost(const char* method, const bp_cost_params* cp, bp_cost_row* out) {
  return guarded([&] {
    const blockpipe::MethodCost c = blockpipe::method_cost(blockpipe::parse_method(method), from_c(*cp));
    *out = bp_cost_row{c.comm_scalars, c.comm_overlap ? 1 : 0, c.model_mem, c.kv_mem, c.comm_bytes};
  });
}

}  // extern "C"
