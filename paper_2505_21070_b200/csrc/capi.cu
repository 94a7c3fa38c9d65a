// C-ABI entry points for rng / noise / stage / scheduler_step (bp_cuda.h).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "device.cuh"
#include "kernels_simt.cuh"
#include "schedule.hpp"
#include "stage.hpp"

namespace bp {

std::atomic<int64_t> g_launches{0};
std::atomic<int64_t> g_dev_bytes{0}, g_dev_peak{0};

namespace {
thread_local std::string t_last_error;

void require_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    fail(BP_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
  if (device < 0 || device >= n) fail(BP_ERR_CUDA, "device index out of range");
  BP_CUDA(cudaSetDevice(device));
}
}  // namespace

void set_last_error(const std::string& m) { t_last_error = m; }

void set_smem_attr_impl(const void* fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  BP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (!done.insert({fn, dev}).second) return;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) {
    done.erase({fn, dev});
    fail(BP_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  }
}

}  // namespace bp

struct bp_stage {
  std::unique_ptr<bp::Stage> s;
  int device = 0;
  bp::DevBuf payload, levels, ids;
};

extern "C" {

const char* bp_last_error(void) { return bp::t_last_error.c_str(); }
const char* bp_version(void) { return "blockpipe-b200 0.1 (sm_100a)"; }

uint64_t bp_derive_seed(uint64_t base, const uint64_t* tags, int32_t ntags) {
  return bp::derive_seed(base, tags, ntags);
}

bp_status bp_normals(int32_t device, uint64_t state, int64_t n, double sigma, double* out,
                     int32_t out_is_device, uint64_t* final_state) {
  return bp::guarded([&] {
    if (n < 0) bp::fail(BP_ERR_DIMENSION, "negative count");
    bp::require_device(device);
    bp::DevBuf tmp;
    double* dst = out;
    if (!out_is_device) {
      tmp.alloc(static_cast<size_t>(n) * 8);
      dst = tmp.as<double>();
    }
    bp::launch_normal_fill(state, n, sigma, dst, nullptr);
    if (!out_is_device) BP_CUDA(cudaMemcpy(out, dst, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
    BP_CUDA(cudaDeviceSynchronize());
    if (final_state) *final_state = state + bp::kGolden * static_cast<uint64_t>(2 * n);
  });
}

bp_status bp_noise_pool(int32_t device, int32_t num_b, int32_t num_c, const int64_t frame_shape[3],
                        uint64_t noise_seed, double* out, int32_t out_is_device) {
  return bp::guarded([&] {
    // build_pool argument checks (noise.cpp:28-29)
    if (num_b < 1) bp::fail(BP_ERR_CONFIG, "num_b must be >= 1");
    if (num_c < 0 || num_c % 2 != 0) bp::fail(BP_ERR_CONFIG, "num_c must be even and >= 0");
    bp::require_device(device);
    const int m = num_b + num_c / 2;
    const int64_t per = frame_shape[0] * frame_shape[1] * frame_shape[2];
    bp::DevBuf tmp, flags;
    double* dst = out;
    if (!out_is_device) {
      tmp.alloc(static_cast<size_t>(m * per) * 8);
      dst = tmp.as<double>();
    }
    bp::launch_normal_fill(noise_seed, m * per, 1.0, dst, nullptr);
    if (m > 1) {
      flags.alloc(static_cast<size_t>(m) * m * 4);
      BP_CUDA(cudaMemset(flags.p, 0, static_cast<size_t>(m) * m * 4));
      bp::launch_pool_differs(dst, m, per, flags.as<int>(), nullptr);
      std::vector<int> f(static_cast<size_t>(m) * m);
      BP_CUDA(cudaMemcpy(f.data(), flags.p, f.size() * 4, cudaMemcpyDeviceToHost));
      for (int i = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j)
          if (!f[static_cast<size_t>(i) * m + j])
            bp::fail(BP_ERR_CONFIG, "noise pool entries collided; change the noise seed");
    }
    if (!out_is_device) BP_CUDA(cudaMemcpy(out, dst, static_cast<size_t>(m * per) * 8, cudaMemcpyDeviceToHost));
    BP_CUDA(cudaDeviceSynchronize());
  });
}

namespace {
// Frames of one block from the pool by id, on the device; host or device I/O.
void gather_block(const double* pool, int32_t pool_size, int64_t per, const std::vector<int32_t>& ids, double* out,
                  bool on_device) {
  for (int32_t id : ids)
    if (id < 0 || id >= pool_size) bp::fail(BP_ERR_QUEUE, "noise id out of pool range");
  const int n = static_cast<int>(ids.size());
  bp::DevBuf dids, dpool, dout;
  dids.alloc(static_cast<size_t>(n) * 4 + 4);
  if (n > 0) BP_CUDA(cudaMemcpy(dids.p, ids.data(), static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice));
  const double* src = pool;
  double* dst = out;
  if (!on_device) {
    dpool.alloc(static_cast<size_t>(pool_size) * per * 8 + 8);
    BP_CUDA(cudaMemcpy(dpool.p, pool, static_cast<size_t>(pool_size) * per * 8, cudaMemcpyHostToDevice));
    src = dpool.as<double>();
    dout.alloc(static_cast<size_t>(n) * per * 8 + 8);
    dst = dout.as<double>();
  }
  bp::launch_gather_ids(src, per, dids.as<int32_t>(), n, dst, nullptr);
  BP_CUDA(cudaDeviceSynchronize());
  if (!on_device && n > 0) BP_CUDA(cudaMemcpy(out, dst, static_cast<size_t>(n) * per * 8, cudaMemcpyDeviceToHost));
}
}  // namespace

bp_status bp_gather_block(int32_t device, const double* pool, int32_t pool_size, int64_t frame_elems,
                          const int32_t* ids, int32_t nids, double* out, int32_t io_on_device) {
  return bp::guarded([&] {
    if (pool_size < 0 || frame_elems < 0 || nids < 0) bp::fail(BP_ERR_DIMENSION, "negative size");
    if ((nids > 0 && (!ids || !out)) || (pool_size > 0 && !pool)) bp::fail(BP_ERR_CONFIG, "null argument");
    bp::require_device(device);
    gather_block(pool, pool_size, frame_elems, std::vector<int32_t>(ids, ids + nids), out, io_on_device != 0);
  });
}

bp_status bp_noise_draw(int32_t device, int32_t strategy, int32_t first, int32_t num_b, int32_t num_c,
                        const int64_t frame_shape[3], const double* pool, int32_t pool_size,
                        const int32_t* tail_window_ids, int32_t ntail, uint64_t* rng_state, double* out_frames,
                        int32_t* out_ids, int32_t* out_frames_count, int32_t* out_nids, int32_t io_on_device) {
  return bp::guarded([&] {
    if (!frame_shape || !rng_state || !out_frames_count || !out_nids) bp::fail(BP_ERR_CONFIG, "null argument");
    if (strategy < BP_INIT_COORDINATED || strategy > BP_INIT_REPEAT) bp::fail(BP_ERR_CONFIG, "unknown noise strategy");
    if (num_b < 1) bp::fail(BP_ERR_CONFIG, "num_b must be >= 1");
    if (num_c < 0 || num_c % 2 != 0) bp::fail(BP_ERR_CONFIG, "num_c must be even and >= 0");
    if (pool_size != num_b + num_c / 2) bp::fail(BP_ERR_CONFIG, "pool must hold num_b + num_c/2 entries");
    if (ntail < 0 || (ntail > 0 && !tail_window_ids)) bp::fail(BP_ERR_CONFIG, "bad tail window");
    const int64_t per = frame_shape[0] * frame_shape[1] * frame_shape[2];
    if (per < 0) bp::fail(BP_ERR_DIMENSION, "negative frame shape");
    bp::require_device(device);
    bp::HostRng rng(*rng_state);
    const std::vector<int> window(tail_window_ids, tail_window_ids + ntail);
    bp::NoiseIds n = bp::draw_noise_ids(strategy, first != 0, num_b, num_c, window, per, rng);
    const int64_t count = static_cast<int64_t>(n.frames) * per;
    if (n.fresh) {  // rng.normal_tensor({frames, H, W, C}) (noise.cpp:118-122, 142-148)
      bp::DevBuf tmp;
      double* dst = out_frames;
      if (!io_on_device) {
        tmp.alloc(static_cast<size_t>(count) * 8 + 8);
        dst = tmp.as<double>();
      }
      bp::launch_normal_fill(n.fresh_state, count, 1.0, dst, nullptr);
      BP_CUDA(cudaDeviceSynchronize());
      if (!io_on_device && count > 0)
        BP_CUDA(cudaMemcpy(out_frames, dst, static_cast<size_t>(count) * 8, cudaMemcpyDeviceToHost));
    } else {
      if (!pool) bp::fail(BP_ERR_CONFIG, "null pool");
      gather_block(pool, pool_size, per, std::vector<int32_t>(n.ids.begin(), n.ids.end()), out_frames,
                   io_on_device != 0);
    }
    if (out_ids)
      for (size_t i = 0; i < n.ids.size(); ++i) out_ids[i] = n.ids[i];
    *out_frames_count = n.frames;
    *out_nids = static_cast<int32_t>(n.ids.size());
    *rng_state = rng.state;
  });
}

bp_status bp_stage_create(int32_t device, const bp_model_desc* model, uint64_t seed_model,
                          uint64_t seed_context, int32_t layer_begin, int32_t layer_end, int32_t precision,
                          bp_stage** out) {
  return bp::guarded([&] {
    if (!model || !out) bp::fail(BP_ERR_CONFIG, "null argument");
    bp::validate_model(*model);
    bp::require_device(device);
    auto h = std::make_unique<bp_stage>();
    h->device = device;
    h->s = std::make_unique<bp::Stage>(device, *model, seed_model, seed_context, layer_begin, layer_end,
                                       precision, nullptr);
    *out = h.release();
  });
}

bp_status bp_stage_destroy(bp_stage* stage) {
  return bp::guarded([&] { delete stage; });
}

bp_status bp_forward_chunk(bp_stage* h, const bp_chunk_in* in, bp_chunk_out* out) {
  return bp::guarded([&] {
    if (!h || !in || !out) bp::fail(BP_ERR_CONFIG, "null argument");
    bp::Stage& s = *h->s;
    BP_CUDA(cudaSetDevice(h->device));
    const int64_t frames = in->nframes;
    // forward_chunk's shape checks (model.cpp:230-266), before anything is uploaded
    if (frames < 0 || in->rows < 0 || in->ncapture < 0) bp::fail(BP_ERR_DIMENSION, "negative size");
    if (in->rows != frames * s.tokens_per_frame())
      bp::fail(BP_ERR_DIMENSION, "payload rows do not match frames * tokens_per_frame");
    if (frames > 0 && (!in->frame_levels || !in->frame_ids || !in->payload)) bp::fail(BP_ERR_CONFIG, "null argument");
    if (in->ncapture > 0 && !in->capture_frames) bp::fail(BP_ERR_CONFIG, "null argument");
    for (int32_t c = 0; c < in->ncapture; ++c)
      if (in->capture_frames[c] < 0 || in->capture_frames[c] >= frames)
        bp::fail(BP_ERR_DIMENSION, "capture frame out of range");
    if (in->mode < BP_CACHE_DISABLED || in->mode > BP_CACHE_RECOMPUTE) bp::fail(BP_ERR_CONFIG, "unknown cache mode");
    if (in->use_prev < 0 || in->use_prev > 4) bp::fail(BP_ERR_CONFIG, "unknown use_prev");
    bp::StageInput si;
    // tokens = frames * tokens_per_frame, checked against the payload rows
    si.nframes = in->nframes;
    si.tokens = in->rows;
    si.capture_frames.assign(in->capture_frames, in->capture_frames + in->ncapture);
    si.record_inputs = in->record_inputs != 0;
    si.mode = in->mode;
    si.use_prev = in->use_prev;
    const int64_t want_cols = s.is_first() ? s.channels() : s.hidden();
    if (in->cols != want_cols)
      bp::fail(BP_ERR_DIMENSION, s.is_first() ? "chunk 0 expects [tokens, C] latents"
                                              : "interior chunk expects [tokens, h] hidden state");
    // upload payload (fp64 host -> device, in the stage's activation dtype)
    const size_t n = static_cast<size_t>(in->rows * in->cols);
    h->payload.reserve(n * 8 + 8);
    h->levels.reserve(static_cast<size_t>(frames) * 4 + 4);
    h->ids.reserve(static_cast<size_t>(frames) * 8 + 8);
    cudaStream_t st = s.stream();
    BP_CUDA(cudaMemcpyAsync(h->payload.p, in->payload, n * 8, cudaMemcpyHostToDevice, st));
    if (!s.is_first() && s.act_bytes() == 4) {
      bp::DevBuf f;
      f.alloc(n * 4);
      bp::launch_convert<double, float>(h->payload.as<double>(), f.as<float>(), static_cast<int64_t>(n), st);
      BP_CUDA(cudaMemcpyAsync(h->payload.p, f.p, n * 4, cudaMemcpyDeviceToDevice, st));
      BP_CUDA(cudaStreamSynchronize(st));
    }
    if (frames > 0) {
      BP_CUDA(cudaMemcpyAsync(h->levels.p, in->frame_levels, static_cast<size_t>(frames) * 4, cudaMemcpyHostToDevice, st));
      BP_CUDA(cudaMemcpyAsync(h->ids.p, in->frame_ids, static_cast<size_t>(frames) * 8, cudaMemcpyHostToDevice, st));
    }
    if (in->use_prev == 3 || in->use_prev == 4) {
      // host KVCacheEntry / RecomputeEntry (model.hpp:86-101) for this call
      const int nl = s.local_layers();
      const size_t n1 = static_cast<size_t>(nl) * in->prefix_rows * s.hidden();
      if (!in->prefix_k || (in->use_prev == 3 && !in->prefix_v)) bp::fail(BP_ERR_CACHE, "missing host prefix");
      bp::DevBuf dk, dv;
      dk.alloc(n1 * 8 + 8);
      BP_CUDA(cudaMemcpyAsync(dk.p, in->prefix_k, n1 * 8, cudaMemcpyHostToDevice, st));
      if (in->use_prev == 3) {
        dv.alloc(n1 * 8 + 8);
        BP_CUDA(cudaMemcpyAsync(dv.p, in->prefix_v, n1 * 8, cudaMemcpyHostToDevice, st));
      }
      s.load_host_prefix(in->use_prev, dk.as<double>(), dv.as<double>(), in->prefix_rows);
      BP_CUDA(cudaStreamSynchronize(st));
    }
    si.payload = h->payload.p;
    si.d_levels = h->levels.as<int32_t>();
    si.d_frame_ids = h->ids.as<int64_t>();
    const void* res = s.forward(si);
    const int64_t out_cols = s.is_last() ? s.channels() : s.hidden();
    const size_t on = static_cast<size_t>(in->rows * out_cols);
    if (out->payload_capacity < static_cast<int64_t>(on)) bp::fail(BP_ERR_DIMENSION, "output buffer too small");
    if (s.is_last() ? s.eps_bytes() == 8 : s.act_bytes() == 8) {
      BP_CUDA(cudaMemcpyAsync(out->payload, res, on * 8, cudaMemcpyDeviceToHost, st));
    } else {
      std::vector<float> f(on);
      BP_CUDA(cudaMemcpyAsync(f.data(), res, on * 4, cudaMemcpyDeviceToHost, st));
      BP_CUDA(cudaStreamSynchronize(st));
      for (size_t i = 0; i < on; ++i) out->payload[i] = f[i];
    }
    BP_CUDA(cudaStreamSynchronize(st));
    out->rows = in->rows;
    out->cols = out_cols;
    out->captured = s.cache_valid() ? 1 : 0;
    out->recorded = s.rec_valid() ? 1 : 0;
    out->captured_tokens = s.cache_valid() ? s.cache_tokens() : 0;
  });
}

bp_status bp_stage_cache_rows(bp_stage* h, int32_t layer, int32_t which, double* out, int64_t* rows) {
  return bp::guarded([&] {
    if (!h->s->cache_valid()) bp::fail(BP_ERR_CACHE, "no resident cache");
    if (rows) *rows = h->s->cache_tokens();
    if (out) h->s->cache_rows(layer, which, out);
  });
}

bp_status bp_stage_recorded_rows(bp_stage* h, int32_t layer, double* out, int64_t* rows) {
  return bp::guarded([&] {
    if (!h->s->rec_valid()) bp::fail(BP_ERR_CACHE, "no resident recording");
    if (rows) *rows = h->s->rec_tokens();
    if (out) h->s->recorded_rows(layer, out);
  });
}

bp_status bp_stage_set_context(bp_stage* h, const double* context, int64_t rows, int64_t cols) {
  return bp::guarded([&] { h->s->set_context(context, rows, cols); });
}

bp_status bp_stage_cache_bump_ulp(bp_stage* h, int32_t layer, int32_t which, int64_t index) {
  return bp::guarded([&] {
    h->s->bump_ulp(layer, which, index);
    BP_CUDA(cudaStreamSynchronize(h->s->stream()));
  });
}

bp_status bp_stage_cache_audit(bp_stage* h, char* report, int32_t report_len) {
  return bp::guarded([&] {
    const std::string r = h->s->audit();
    if (report && report_len > 0) {
      std::strncpy(report, r.c_str(), static_cast<size_t>(report_len) - 1);
      report[report_len - 1] = 0;
    }
  });
}

bp_status bp_scheduler_step(int32_t device, const double* x, const double* eps, int64_t n, int32_t level,
                            int32_t steps, double* out) {
  return bp::guarded([&] {
    // scheduler_step's range check (model.cpp:339-343)
    if (level < 1 || level > steps)
      bp::fail(BP_ERR_SCHEDULER, "level " + std::to_string(level) + " outside 1.." + std::to_string(steps));
    bp::require_device(device);
    bp::DevBuf dx, de, dout;
    dx.alloc(static_cast<size_t>(n) * 8 + 8);
    de.alloc(static_cast<size_t>(n) * 8 + 8);
    dout.alloc(static_cast<size_t>(n) * 8 + 8);
    BP_CUDA(cudaMemcpy(dx.p, x, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(de.p, eps, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice));
    bp::launch_scheduler_step<double>(dx.as<double>(), de.as<double>(), n, steps, dout.as<double>(), nullptr);
    BP_CUDA(cudaMemcpy(out, dout.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
  });
}

namespace {
// Host-buffer round trip for the tensor primitives: copy in, launch, copy out.
struct HostOp {
  std::vector<bp::DevBuf> bufs;
  double* in(const double* h, int64_t n) {
    bufs.emplace_back();
    bufs.back().alloc(static_cast<size_t>(n) * 8 + 8);
    if (n > 0) BP_CUDA(cudaMemcpy(bufs.back().p, h, static_cast<size_t>(n) * 8, cudaMemcpyHostToDevice));
    return bufs.back().as<double>();
  }
  double* scratch(int64_t n) {
    bufs.emplace_back();
    bufs.back().alloc(static_cast<size_t>(n) * 8 + 8);
    return bufs.back().as<double>();
  }
  static void out(double* h, const double* d, int64_t n) {
    BP_CUDA(cudaDeviceSynchronize());
    if (n > 0) BP_CUDA(cudaMemcpy(h, d, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
  }
};
void require_2d(int64_t rows, int64_t cols, const char* what) {
  if (rows < 0 || cols < 0) bp::fail(BP_ERR_DIMENSION, std::string(what) + ": negative extent");
  if (rows > INT32_MAX || cols > INT32_MAX) bp::fail(BP_ERR_DIMENSION, std::string(what) + ": extent too large");
}
}  // namespace

bp_status bp_matmul(int32_t device, const double* a, const double* b, int64_t m, int64_t k, int64_t n,
                    double* out) {
  return bp::guarded([&] {
    require_2d(m, k, "matmul");
    require_2d(k, n, "matmul");
    bp::require_device(device);
    HostOp op;
    const double* da = op.in(a, m * k);
    const double* db = op.in(b, k * n);
    double* dc = op.scratch(m * n);
    if (m > 0 && n > 0) {
      if (k == 0) BP_CUDA(cudaMemset(dc, 0, static_cast<size_t>(m * n) * 8));
      else bp::launch_matmul<double>(da, k, db, n, static_cast<int>(m), static_cast<int>(n), static_cast<int>(k),
                                     dc, n, bp::kEpiNone, nullptr, 0, nullptr);
    }
    HostOp::out(out, dc, m * n);
  });
}

bp_status bp_elementwise(int32_t device, int32_t op, const double* a, const double* b, int64_t n, double s,
                         double* out) {
  return bp::guarded([&] {
    if (op < 0 || op > 2) bp::fail(BP_ERR_CONFIG, "elementwise op must be 0 (add), 1 (sub) or 2 (scale)");
    if (n < 0) bp::fail(BP_ERR_DIMENSION, "negative count");
    bp::require_device(device);
    HostOp o;
    const double* da = o.in(a, n);
    const double* db = op == 2 ? nullptr : o.in(b, n);
    double* dc = o.scratch(n);
    bp::launch_elementwise(op, da, db, n, s, dc, nullptr);
    HostOp::out(out, dc, n);
  });
}

bp_status bp_softmax_rows(int32_t device, const double* x, int64_t rows, int64_t cols, double* out) {
  return bp::guarded([&] {
    require_2d(rows, cols, "softmax_rows");
    bp::require_device(device);
    HostOp op;
    const double* dx = op.in(x, rows * cols);
    double* dy = op.scratch(rows * cols);
    bp::launch_softmax_rows(dx, rows, cols, dy, nullptr);
    HostOp::out(out, dy, rows * cols);
  });
}

bp_status bp_layer_norm(int32_t device, const double* x, int64_t rows, int64_t cols, double eps, double* out) {
  return bp::guarded([&] {
    require_2d(rows, cols, "layer_norm");
    if (cols < 1) bp::fail(BP_ERR_DIMENSION, "layer_norm needs at least one column");
    bp::require_device(device);
    HostOp op;
    const double* dx = op.in(x, rows * cols);
    double* dy = op.scratch(rows * cols);
    bp::launch_layer_norm(dx, rows, static_cast<int>(cols), eps, dy, nullptr);
    HostOp::out(out, dy, rows * cols);
  });
}

}  // extern "C"
