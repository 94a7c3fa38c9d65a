// C++ mirror, continued: the tensor.hpp free functions, the noise draws of
// noise.hpp and the block queue of block_queue.hpp over the B200 C-ABI.
// Arithmetic (matmul, softmax, layer norm, add / sub / scale) and noise
// frames run on the GPU; what remains on the host is row bookkeeping of the
// host containers (the reference's own Tensor is a host vector as well).
#include <algorithm>
#include <cstring>
#include <string>

#include "blockpipe/blockpipe_b200.hpp"
#include "bp_cuda.h"

namespace blockpipe {

namespace {

[[noreturn]] void raise(bp_status s) {
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
void check(bp_status s) {
  if (s != BP_OK) raise(s);
}

// "[2x3]" -- the reference's shape spelling in error messages (tensor.cpp:19-26)
std::string dims(const std::vector<int64_t>& s) {
  std::string o = "[";
  for (size_t i = 0; i < s.size(); ++i) o += (i ? "x" : "") + std::to_string(s[i]);
  return o + "]";
}

Tensor elementwise(int op, const Tensor& a, const Tensor* b, double s) {
  Tensor out(a.shape);
  if (a.numel() > 0)
    check(bp_elementwise(0, op, a.data.data(), b ? b->data.data() : nullptr, a.numel(), s, out.data.data()));
  return out;
}

// The frames of `ids` stacked from the pool on the GPU ([n, H, W, C]).
Tensor stack(const NoisePool& pool, const std::vector<int>& ids) {
  std::vector<int64_t> shape = pool.frame_shape;
  shape.insert(shape.begin(), static_cast<int64_t>(ids.size()));
  Tensor out(shape);
  if (ids.empty()) return out;
  const int64_t per = pool.entries.empty() ? 0 : pool.entries.front().numel();
  std::vector<double> flat(static_cast<size_t>(pool.size() * per));
  for (int i = 0; i < pool.size(); ++i)
    std::copy(pool.entries[static_cast<size_t>(i)].data.begin(), pool.entries[static_cast<size_t>(i)].data.end(),
              flat.begin() + i * per);
  check(bp_gather_block(0, flat.data(), pool.size(), per, ids.data(), static_cast<int32_t>(ids.size()),
                        out.data.data(), 0));
  return out;
}

// One engine-style draw through bp_noise_draw (ids on the host stream, frames
// on the GPU); pool.size() must be num_b + num_c/2 as build_pool makes it.
NoiseDraw engine_draw(InitStrategy s, bool first, const NoisePool& pool, const std::vector<int>& window,
                      RandomSource& rng) {
  if (pool.frame_shape.size() != 3) throw DimensionError("noise pool frame_shape must be [H, W, C]");
  const int64_t per = pool.frame_shape[0] * pool.frame_shape[1] * pool.frame_shape[2];
  const int cap = first ? pool.size() : pool.num_b;
  std::vector<double> flat(static_cast<size_t>(pool.size() * per));
  for (int i = 0; i < pool.size(); ++i)
    std::copy(pool.entries[static_cast<size_t>(i)].data.begin(), pool.entries[static_cast<size_t>(i)].data.end(),
              flat.begin() + i * per);
  std::vector<double> frames(static_cast<size_t>(std::max(cap, 0) * per) + 1);
  std::vector<int32_t> ids(static_cast<size_t>(std::max(cap, 0)) + 1);
  int32_t nframes = 0, nids = 0;
  check(bp_noise_draw(0, static_cast<int32_t>(s), first ? 1 : 0, pool.num_b, pool.num_c, pool.frame_shape.data(),
                      flat.data(), pool.size(), window.data(), static_cast<int32_t>(window.size()), &rng.state,
                      frames.data(), ids.data(), &nframes, &nids, 0));
  NoiseDraw d;
  std::vector<int64_t> shape = pool.frame_shape;
  shape.insert(shape.begin(), nframes);
  frames.resize(static_cast<size_t>(nframes * per));
  d.frames = Tensor(shape, std::move(frames));
  d.noise_ids.assign(ids.begin(), ids.begin() + nids);
  return d;
}

Tensor frame_rows(const Tensor& frames, int64_t begin, int64_t end) {  // frames [begin, end) keeping [H, W, C]
  const int64_t f = frames.shape[0];
  std::vector<int64_t> shape = frames.shape;
  shape[0] = end - begin;
  return slice_rows(frames.reshaped({f, frames.numel() / f}), begin, end).reshaped(shape);
}

}  // namespace

// ---------------------------------------------------------------- tensor.hpp
Tensor matmul(const Tensor& a, const Tensor& b) {
  if (a.shape.size() != 2 || b.shape.size() != 2)
    throw DimensionError("matmul expects 2-d operands, got " + dims(a.shape) + " and " + dims(b.shape));
  if (a.shape[1] != b.shape[0])
    throw DimensionError("matmul inner dimensions disagree: " + dims(a.shape) + " vs " + dims(b.shape));
  Tensor out({a.shape[0], b.shape[1]});
  if (out.numel() > 0)
    check(bp_matmul(0, a.data.data(), b.data.data(), a.shape[0], a.shape[1], b.shape[1], out.data.data()));
  return out;
}

Tensor softmax_rows(const Tensor& x) {
  Tensor out({x.rows(), x.cols()});
  if (out.numel() > 0) check(bp_softmax_rows(0, x.data.data(), x.rows(), x.cols(), out.data.data()));
  return out;
}

Tensor layer_norm(const Tensor& x, double eps) {
  if (x.cols() < 1) throw DimensionError("layer_norm needs at least one column");
  Tensor out({x.rows(), x.cols()});
  if (out.numel() > 0) check(bp_layer_norm(0, x.data.data(), x.rows(), x.cols(), eps, out.data.data()));
  return out;
}

Tensor add(const Tensor& a, const Tensor& b) {
  if (!a.same_shape(b)) throw DimensionError("add shape mismatch " + dims(a.shape) + " vs " + dims(b.shape));
  return elementwise(0, a, &b, 0.0);
}

Tensor sub(const Tensor& a, const Tensor& b) {
  if (!a.same_shape(b)) throw DimensionError("sub shape mismatch " + dims(a.shape) + " vs " + dims(b.shape));
  return elementwise(1, a, &b, 0.0);
}

Tensor scale(const Tensor& a, double s) { return elementwise(2, a, nullptr, s); }

Tensor vcat_rows(const Tensor& a, const Tensor& b) {
  if (a.numel() == 0) return b;
  if (b.numel() == 0) return a;
  if (a.cols() != b.cols())
    throw DimensionError("vcat_rows column mismatch " + dims(a.shape) + " vs " + dims(b.shape));
  std::vector<double> d(a.data);
  d.insert(d.end(), b.data.begin(), b.data.end());
  return Tensor({a.rows() + b.rows(), a.cols()}, std::move(d));
}

Tensor slice_rows(const Tensor& x, int64_t begin, int64_t end) {
  if (begin < 0 || end < begin || end > x.rows())
    throw DimensionError("slice_rows [" + std::to_string(begin) + "," + std::to_string(end) +
                         ") out of range for " + dims(x.shape));
  const int64_t c = x.cols();
  return Tensor({end - begin, c}, std::vector<double>(x.data.begin() + begin * c, x.data.begin() + end * c));
}

Tensor take_rows(const Tensor& x, const std::vector<int64_t>& idx) {
  const int64_t c = x.cols();
  std::vector<double> d;
  d.reserve(idx.size() * static_cast<size_t>(c));
  for (int64_t r : idx) {
    if (r < 0 || r >= x.rows())
      throw DimensionError("take_rows index " + std::to_string(r) + " out of range for " + dims(x.shape));
    d.insert(d.end(), x.data.begin() + r * c, x.data.begin() + (r + 1) * c);
  }
  return Tensor({static_cast<int64_t>(idx.size()), c}, std::move(d));
}

// ---------------------------------------------------------------- noise.hpp
NoiseDraw init_first_block(const NoisePool& pool, RandomSource& rng) {
  NoiseDraw d;
  d.noise_ids = rng.permutation(pool.size());  // noise.cpp:70-75
  d.frames = stack(pool, d.noise_ids);
  return d;
}

NoiseDraw init_next_block(const NoisePool& pool, const std::vector<int>& tail_window_ids, RandomSource& rng) {
  return engine_draw(InitStrategy::kCoordinated, false, pool, tail_window_ids, rng);  // noise.cpp:77-101
}

NoiseDraw init_baseline(InitStrategy variant, const NoisePool& pool, RandomSource& rng) {
  NoiseDraw d;
  switch (variant) {  // noise.cpp:103-133
    case InitStrategy::kCompleteShuffle:
      d.noise_ids = rng.permutation(pool.size());
      break;
    case InitStrategy::kSubset: {
      const std::vector<int> p = rng.permutation(pool.size());
      d.noise_ids.assign(p.begin(), p.begin() + pool.num_b);
      break;
    }
    case InitStrategy::kFresh: {
      std::vector<int64_t> shape = pool.frame_shape;
      shape.insert(shape.begin(), pool.num_b);
      d.frames = rng.normal_tensor(shape);
      return d;
    }
    case InitStrategy::kRepeat:
      for (int i = 0; i < pool.size(); ++i) d.noise_ids.push_back(i);
      break;
    case InitStrategy::kCoordinated:
      throw ConfigError("coordinated is not a baseline variant");
  }
  d.frames = stack(pool, d.noise_ids);
  return d;
}

NoiseDraw draw_first_block(InitStrategy s, const NoisePool& pool, RandomSource& rng) {
  return engine_draw(s, true, pool, {}, rng);
}

NoiseDraw draw_next_block(InitStrategy s, const NoisePool& pool, const std::vector<int>& tail_window_ids,
                          RandomSource& rng) {
  return engine_draw(s, false, pool, tail_window_ids, rng);
}

// ---------------------------------------------------------------- block_queue.hpp
void QueueParams::validate() const {
  if (num_b < 1) throw ConfigError("num_b must be >= 1");
  if (num_c < 0 || num_c % 2 != 0) throw ConfigError("num_c must be even and >= 0");
  if (num_c / 2 > num_b) throw ConfigError("num_c/2 must not exceed num_b (context cannot outgrow a block)");
  if (steps < 1) throw ConfigError("steps must be >= 1");
  if (block_num < 1) throw ConfigError("block_num must be >= 1");
}

const LatentBlock* QueueState::find(int64_t block_id) const {
  auto it = std::find_if(blocks.begin(), blocks.end(), [&](const LatentBlock& b) { return b.block_id == block_id; });
  return it == blocks.end() ? nullptr : &*it;
}

LatentBlock* QueueState::find(int64_t block_id) {
  auto it = std::find_if(blocks.begin(), blocks.end(), [&](const LatentBlock& b) { return b.block_id == block_id; });
  return it == blocks.end() ? nullptr : &*it;
}

void apply_update(QueueState& q, int64_t block_id, Tensor frames) {  // block_queue.cpp:34-42
  LatentBlock* b = q.find(block_id);
  if (!b) throw QueueError("update for unknown block " + std::to_string(block_id));
  if (b->level < 1) throw QueueError("block " + std::to_string(block_id) + " already clean");
  b->prev_frames = std::move(b->frames);
  b->frames = std::move(frames);
  --b->level;
  ++b->updates;
}

QueueState advance(QueueState q, std::optional<LatentBlock> new_block) {  // block_queue.cpp:44-78
  q.params.validate();
  if (!q.blocks.empty() && q.blocks.front().level == 0) {
    const LatentBlock& head = q.blocks.front();
    const int ctx = q.context_frames();
    if (q.params.retain_clean_context && ctx > 0) {
      const int64_t f = head.frame_count();
      RetainedContext r;
      r.source_block_id = head.block_id;
      r.frames = frame_rows(head.frames, f - ctx, f);
      r.frame_ids.assign(head.frame_ids.end() - ctx, head.frame_ids.end());
      q.retained = std::move(r);
    }
    q.popped_ids.push_back(head.block_id);
    q.blocks.pop_front();
  }
  if (new_block) {
    if (q.appended_count >= q.params.block_num)
      throw QueueError("append after block_num=" + std::to_string(q.params.block_num) +
                       " blocks were already appended");
    new_block->level = q.params.steps;
    new_block->updates = 0;
    q.blocks.push_back(std::move(*new_block));
    ++q.appended_count;
  }
  if (static_cast<int>(q.blocks.size()) > q.params.steps)
    throw QueueError("queue exceeded steps=" + std::to_string(q.params.steps));
  return q;
}

std::vector<int64_t> processing_order(const QueueState& q, Order order) {  // block_queue.cpp:80-86
  std::vector<int64_t> ids;
  for (const LatentBlock& b : q.blocks) ids.push_back(b.block_id);
  if (order == Order::kReverse) std::reverse(ids.begin(), ids.end());
  return ids;
}

ExtendedBlock assemble_extended(const QueueState& q, int64_t block_id, Order order) {  // block_queue.cpp:88-138
  const LatentBlock* center = q.find(block_id);
  if (!center) throw QueueError("assemble_extended: unknown block " + std::to_string(block_id));
  ExtendedBlock e;
  e.center_id = block_id;
  const int ctx = q.context_frames();
  const LatentBlock* earlier = q.find(block_id - 1);
  if (ctx > 0 && earlier) {
    // the neighbour's state at the centre's update count (its latest state is
    // one pass ahead of a pipelined pass, so round-atomic drivers read prev)
    const Tensor* src = nullptr;
    if (earlier->updates == center->updates) src = &earlier->frames;
    else if (earlier->updates == center->updates + 1 && earlier->prev_frames) src = &*earlier->prev_frames;
    else
      throw QueueError("context state for block " + std::to_string(block_id) + " unavailable (neighbor updates " +
                       std::to_string(earlier->updates) + ", center " + std::to_string(center->updates) + ")");
    const int64_t f = earlier->frame_count();
    e.explicit_frames = frame_rows(*src, f - ctx, f);
    e.explicit_levels.assign(static_cast<size_t>(ctx), center->level);
    e.explicit_frame_ids.assign(earlier->frame_ids.end() - ctx, earlier->frame_ids.end());
    e.source = ExtendedBlock::CtxSource::kInQueue;
    e.ctx_block_id = block_id - 1;
  } else if (ctx > 0 && q.retained && q.retained->source_block_id == block_id - 1) {
    e.explicit_frames = q.retained->frames;
    e.explicit_levels.assign(static_cast<size_t>(ctx), 0);
    e.explicit_frame_ids = q.retained->frame_ids;
    e.source = ExtendedBlock::CtxSource::kRetained;
    e.ctx_block_id = block_id - 1;
  }
  if (order == Order::kReverse && ctx > 0 && q.find(block_id + 1)) e.cached_context_id = block_id + 1;
  return e;
}

bool levels_are_unit_ladder(const QueueState& q) {  // block_queue.cpp:140-145
  for (size_t i = 1; i < q.blocks.size(); ++i)
    if (q.blocks[i].level != q.blocks[i - 1].level + 1) return false;
  return true;
}

}  // namespace blockpipe
