// Host schedule builder + its C-ABI accessors. See schedule.hpp.
#include "schedule.hpp"

#include <algorithm>
#include <cstring>
#include <deque>
#include <map>
#include <set>

#include "common.hpp"

namespace bp {

NoiseIds draw_noise_ids(int strategy, bool first, int num_b, int num_c, const std::vector<int>& tail_window,
                        int64_t frame_elems, HostRng& rng) {
  const int M = num_b + num_c / 2, ctx = num_c / 2;
  NoiseIds n;
  n.frames = first ? M : num_b;
  if (strategy == BP_INIT_FRESH) {  // fresh Gaussians from the append stream
    n.fresh = true;
    n.fresh_state = rng.state;
    rng.skip_normals(static_cast<int64_t>(n.frames) * frame_elems);
    return n;
  }
  if (first) {  // draw_first_block (noise.cpp:135-152)
    if (strategy == BP_INIT_REPEAT) {
      for (int i = 0; i < M; ++i) n.ids.push_back(i);
    } else {
      n.ids = rng.permutation(M);
    }
    return n;
  }
  switch (strategy) {  // draw_next_block (noise.cpp:154-178)
    case BP_INIT_COORDINATED: {  // init_next_block (noise.cpp:77-101)
      if (static_cast<int>(tail_window.size()) != ctx) fail(BP_ERR_QUEUE, "tail window must hold num_c/2 ids");
      std::set<int> excluded(tail_window.begin(), tail_window.end());
      if (static_cast<int>(excluded.size()) != ctx) fail(BP_ERR_QUEUE, "tail window ids must be distinct");
      for (int e : excluded)
        if (e < 0 || e >= M) fail(BP_ERR_QUEUE, "tail window id out of pool range");
      std::vector<int> remaining;
      for (int i = 0; i < M; ++i)
        if (!excluded.count(i)) remaining.push_back(i);
      for (int p : rng.permutation(static_cast<int>(remaining.size())))
        n.ids.push_back(remaining[static_cast<size_t>(p)]);
      break;
    }
    case BP_INIT_COMPLETE_SHUFFLE:
    case BP_INIT_SUBSET: {
      const std::vector<int> perm = rng.permutation(M);
      n.ids.assign(perm.begin(), perm.begin() + num_b);
      break;
    }
    case BP_INIT_REPEAT:
      for (int i = M - num_b; i < M; ++i) n.ids.push_back(i);
      break;
    default:
      fail(BP_ERR_CONFIG, "unknown noise strategy");
  }
  return n;
}


int ffn_width(const bp_model_desc& m) { return m.ffn > 0 ? m.ffn : 4 * m.hidden; }

// ModelConfig::validate (model.cpp:76-85).
void validate_model(const bp_model_desc& m) {
  if (m.layers < 1) fail(BP_ERR_CONFIG, "layers must be >= 1");
  if (m.hidden < 2) fail(BP_ERR_CONFIG, "hidden must be >= 2");
  if (m.heads < 1 || m.hidden % m.heads != 0)
    fail(BP_ERR_CONFIG, "heads must divide hidden (" + std::to_string(m.hidden) + "/" +
                            std::to_string(m.heads) + ")");
  if (m.channels < 1) fail(BP_ERR_CONFIG, "channels must be >= 1");
  if (m.height < 1 || m.width < 1) fail(BP_ERR_CONFIG, "token grid must be at least 1x1");
  if (m.context_len < 1) fail(BP_ERR_CONFIG, "context_len must be >= 1");
  if (m.ffn < 0) fail(BP_ERR_CONFIG, "ffn must be >= 0");
  if (m.block != BP_BLOCK_REFERENCE && m.block != BP_BLOCK_WAN) fail(BP_ERR_CONFIG, "block must be reference or wan");
  if (m.block == BP_BLOCK_WAN && ((m.hidden / m.heads) < 6 || (m.hidden / m.heads) % 2 != 0))
    fail(BP_ERR_CONFIG, "wan block needs an even head dim of at least 6 (3D RoPE)");
}

namespace {

// QueueParams::validate (block_queue.cpp:10-18).
void validate_queue(const bp_pipeline_desc& d) {
  if (d.num_b < 1) fail(BP_ERR_CONFIG, "num_b must be >= 1");
  if (d.num_c < 0 || d.num_c % 2 != 0) fail(BP_ERR_CONFIG, "num_c must be even and >= 0");
  if (d.num_c / 2 > d.num_b)
    fail(BP_ERR_CONFIG, "num_c/2 must not exceed num_b (context cannot outgrow a block)");
  if (d.steps < 1) fail(BP_ERR_CONFIG, "steps must be >= 1");
  if (d.block_num < 1) fail(BP_ERR_CONFIG, "block_num must be >= 1");
}

// Queue entry as the host tracks it: only integer state, no frames.
struct QBlock {
  int64_t id;
  int frames;
  int level;
  int updates;
};

}  // namespace

void partition_layers(const bp_pipeline_desc& d, std::vector<int>* begins, std::vector<int>* ends) {
  const int L = d.model.layers, N = d.devices;
  begins->clear();
  ends->clear();
  bool explicit_split = false;
  for (int j = 0; j < N && j < 64; ++j) explicit_split |= d.layer_split[j] != 0;
  if (explicit_split) {
    if (N > 64) fail(BP_ERR_PARTITION, "explicit split supports at most 64 stages");
    int at = 0;
    for (int j = 0; j < N; ++j) {
      if (d.layer_split[j] < 1) fail(BP_ERR_PARTITION, "every stage needs >= 1 layer");
      begins->push_back(at);
      at += d.layer_split[j];
      ends->push_back(at);
    }
    if (at != L) fail(BP_ERR_PARTITION, "layer_split does not sum to layers");
    return;
  }
  if (L % N != 0 && !d.uneven_split) {
    fail(BP_ERR_PARTITION,
         "layers " + std::to_string(L) + " not divisible by devices " + std::to_string(N));
  }
  if (N > L) fail(BP_ERR_PARTITION, "more stages than layers");
  // Contiguous; the first L % N stages take one extra layer.
  int at = 0;
  for (int j = 0; j < N; ++j) {
    const int n = L / N + (j < L % N ? 1 : 0);
    begins->push_back(at);
    at += n;
    ends->push_back(at);
  }
}

Schedule build_schedule(const bp_pipeline_desc& d) {
  // PipelineConfig::validate (engine.cpp:245-253).
  validate_model(d.model);
  validate_queue(d);
  if (d.devices < 1) fail(BP_ERR_CONFIG, "devices must be >= 1");
  if (d.model.layers % d.devices != 0 && !d.uneven_split) {
    bool explicit_split = false;
    for (int j = 0; j < d.devices && j < 64; ++j) explicit_split |= d.layer_split[j] != 0;
    if (!explicit_split)
      fail(BP_ERR_CONFIG, "layers " + std::to_string(d.model.layers) +
                              " not divisible by devices " + std::to_string(d.devices));
  }
  if (d.strategy < 0 || d.strategy > 4) fail(BP_ERR_CONFIG, "unknown noise strategy");
  if (d.order != BP_ORDER_REVERSE && d.order != BP_ORDER_SEQUENTIAL)
    fail(BP_ERR_CONFIG, "unknown order");
  if (d.cache_mode < 0 || d.cache_mode > 2) fail(BP_ERR_CONFIG, "unknown cache mode");
  if (d.model.block == BP_BLOCK_WAN && (d.cache_mode == BP_CACHE_RECOMPUTE || d.check_cache))
    fail(BP_ERR_CONFIG, "wan block supports cache modes on / off without the recompute audit");

  Schedule s;
  s.desc = d;
  s.devices = d.devices;
  partition_layers(d, &s.begins, &s.ends);

  const int N = d.devices;
  const int T = d.steps;
  const int B = d.block_num;
  const int ctx = d.num_c / 2;
  const int64_t tpf = static_cast<int64_t>(d.model.height) * d.model.width;
  const int64_t hwc = tpf * d.model.channels;
  const bool reverse = d.order == BP_ORDER_REVERSE;
  const bool caching = d.cache_mode != BP_CACHE_DISABLED;
  s.rounds = static_cast<int64_t>(T) + B - 1;  // total_rounds (engine.cpp:222)
  const int64_t q_max = std::min<int64_t>(T, B);

  // append_rng = RandomSource(derive_seed(seed_noise, {1})) (engine.cpp:291).
  const uint64_t tag1 = 1;
  HostRng append_rng(derive_seed(d.seed_noise, &tag1, 1));

  std::deque<QBlock> q;
  int64_t appended = 0, next_frame_id = 0;
  int64_t retained_src = 0;  // block id whose clean tail is retained (0 = none)
  std::map<std::pair<int64_t, int64_t>, int64_t> completion;
  std::vector<int64_t> next_free(static_cast<size_t>(N), 1);
  std::vector<std::map<int64_t, std::pair<int64_t, int64_t>>> counters(static_cast<size_t>(N) + 1);
  std::vector<std::vector<SchedEvent>> dev_events(static_cast<size_t>(N));

  auto find = [&](int64_t id) -> QBlock* {
    for (QBlock& b : q)
      if (b.id == id) return &b;
    return nullptr;
  };

  // make_block (engine.cpp:301-324) with draw_first_block / draw_next_block
  // (noise.cpp:135-178): integer ids on the host.
  auto make_block = [&](int64_t id) {
    SchedBlock b;
    b.id = id;
    std::vector<int> window;
    if (id > 1 && ctx > 0) {
      const SchedBlock& tail = s.blocks[static_cast<size_t>(q.back().id - 1)];
      if (static_cast<int>(tail.noise_ids.size()) >= ctx) {
        window.assign(tail.noise_ids.end() - ctx, tail.noise_ids.end());
      } else if (d.strategy == BP_INIT_COORDINATED) {
        fail(BP_ERR_QUEUE, "tail block lacks noise ids for the exclusion window");
      }
    }
    NoiseIds n = draw_noise_ids(d.strategy, id == 1, d.num_b, d.num_c, window, hwc, append_rng);
    b.noise_ids = std::move(n.ids);
    b.frames = n.frames;
    b.fresh = n.fresh;
    b.fresh_state = n.fresh_state;
    for (int k = 0; k < b.frames; ++k) b.frame_ids.push_back(next_frame_id++);
    return b;
  };

  // emit_if_clean + advance (engine.cpp:326-331, block_queue.cpp:44-78).
  auto emit_and_advance = [&](bool with_new, int64_t new_id) {
    if (!q.empty() && q.front().level == 0) {
      const QBlock head = q.front();
      s.emission.push_back(head.id);
      if (d.retain_clean_context && ctx > 0) retained_src = head.id;
      q.pop_front();
    }
    if (with_new) {
      if (appended >= B)
        fail(BP_ERR_QUEUE, "append after block_num=" + std::to_string(B) +
                               " blocks were already appended");
      q.push_back({new_id, s.blocks[static_cast<size_t>(new_id - 1)].frames, T, 0});
      appended += 1;
    }
    if (static_cast<int>(q.size()) > T) fail(BP_ERR_QUEUE, "queue exceeded steps=" + std::to_string(T));
  };

  int64_t next_block = 1;
  for (int64_t r = 1; r <= s.rounds; ++r) {
    bool with_new = false;
    int64_t new_id = 0;
    if (next_block <= B) {
      new_id = next_block++;
      s.blocks.push_back(make_block(new_id));
      s.blocks.back().append_round = r;
      with_new = true;
    }
    emit_and_advance(with_new, new_id);
    for (size_t i = 1; i < q.size(); ++i)  // levels_are_unit_ladder (block_queue.cpp:140-145)
      if (q[i].level != q[i - 1].level + 1) fail(BP_ERR_QUEUE, "level ladder violated");

    SchedSnapshot snap;
    snap.round = r;
    for (const QBlock& b : q) {
      snap.ids.push_back(b.id);
      snap.levels.push_back(b.level);
    }
    s.snapshots.push_back(std::move(snap));

    // round_phase (engine.cpp:224-232)
    const int phase = r < q_max ? 0 : (r > s.rounds - q_max + 1 ? 2 : 1);

    std::vector<int64_t> order;
    for (const QBlock& b : q) order.push_back(b.id);
    if (reverse) std::reverse(order.begin(), order.end());

    for (int64_t id : order) {
      const QBlock& blk = *find(id);
      SchedPass p;
      p.index = static_cast<int64_t>(s.passes.size());
      p.round = r;
      p.block = id;
      p.level = blk.level;
      p.phase = phase;
      p.version = blk.updates;
      p.center_frames = blk.frames;

      // assemble_extended (block_queue.cpp:88-138)
      const QBlock* earlier = find(id - 1);
      if (ctx > 0 && earlier != nullptr) {
        if (!(earlier->updates == blk.updates ||
              (earlier->updates == blk.updates + 1 && earlier->updates >= 1))) {
          fail(BP_ERR_QUEUE, "context state for block " + std::to_string(id) + " unavailable");
        }
        p.ctx = CtxSrc::InQueue;
        p.ctx_block = id - 1;
        p.ctx_frames = ctx;
        p.ctx_version = blk.updates;
        p.ctx_first_frame = earlier->frames - ctx;
        const SchedBlock& eb = s.blocks[static_cast<size_t>(id - 2)];
        for (int k = 0; k < ctx; ++k) {
          p.frame_levels.push_back(blk.level);
          p.frame_ids.push_back(eb.frame_ids[static_cast<size_t>(eb.frames - ctx + k)]);
        }
      } else if (ctx > 0 && retained_src != 0 && retained_src == id - 1) {
        const SchedBlock& eb = s.blocks[static_cast<size_t>(id - 2)];
        p.ctx = CtxSrc::Retained;
        p.ctx_block = id - 1;
        p.ctx_frames = ctx;
        p.ctx_version = T;  // the popped block's final (clean) state
        p.ctx_first_frame = eb.frames - ctx;
        for (int k = 0; k < ctx; ++k) {
          p.frame_levels.push_back(0);
          p.frame_ids.push_back(eb.frame_ids[static_cast<size_t>(eb.frames - ctx + k)]);
        }
      }
      const SchedBlock& cb = s.blocks[static_cast<size_t>(id - 1)];
      for (int k = 0; k < blk.frames; ++k) {
        p.frame_levels.push_back(blk.level);
        p.frame_ids.push_back(cb.frame_ids[static_cast<size_t>(k)]);
      }
      if (caching && reverse && ctx > 0 && find(id + 1) != nullptr) p.cached_context_id = id + 1;
      // capture the center's leading frames (engine.cpp:392-396)
      if (caching && reverse && ctx > 0 && find(id - 1) != nullptr) {
        for (int k = 0; k < ctx; ++k) p.capture_frames.push_back(p.ctx_frames + k);
      }
      p.tokens = static_cast<int64_t>(p.frame_levels.size()) * tpf;
      p.center_tokens = static_cast<int64_t>(blk.frames) * tpf;
      s.max_tokens = std::max(s.max_tokens, p.tokens);

      // logical clock (engine.cpp:402-410)
      int64_t earliest = 1;
      auto dep = [&](int64_t b, int64_t rr) {
        auto it = completion.find({b, rr});
        if (it != completion.end()) earliest = std::max(earliest, it->second + 1);
      };
      if (blk.updates > 0) dep(id, r - 1);
      if (p.ctx == CtxSrc::InQueue) dep(p.ctx_block, r - 2);
      if (p.ctx == CtxSrc::Retained) dep(p.ctx_block, r - 1);
      p.earliest = earliest;

      // ledger: host->dev0 push (engine.cpp:412)
      auto& hc = counters[0][r];
      hc.first += 1;
      hc.second += p.tokens * d.model.channels;
      int64_t at = earliest;
      for (int j = 0; j < N; ++j) {  // DeviceWorker::process (engine.cpp:138-205)
        const int64_t slot = std::max(at, next_free[static_cast<size_t>(j)]);
        next_free[static_cast<size_t>(j)] = slot + 1;
        p.slots.push_back(slot);
        dev_events[static_cast<size_t>(j)].push_back({slot, j, id, p.level, phase, r});
        at = slot + 1;
        auto& c = counters[static_cast<size_t>(j) + 1][r];
        c.first += 1;
        c.second += p.tokens * (j + 1 < N ? d.model.hidden : d.model.channels);
      }
      p.completion = p.slots.back();
      p.finishes_block = (blk.level == 1);
      s.passes.push_back(std::move(p));
    }
    // collect + apply_update (engine.cpp:418-447)
    const size_t first = s.passes.size() - order.size();
    for (size_t i = first; i < s.passes.size(); ++i) {
      QBlock* b = find(s.passes[i].block);
      if (b->level < 1) fail(BP_ERR_QUEUE, "block already clean");
      b->level -= 1;
      b->updates += 1;
      completion[{s.passes[i].block, r}] = s.passes[i].completion;
    }
    for (auto it = completion.begin(); it != completion.end();)
      it = it->first.second < r - 1 ? completion.erase(it) : ++it;
  }
  emit_and_advance(false, 0);
  if (!q.empty()) fail(BP_ERR_QUEUE, "queue not empty after the final round");

  for (const SchedBlock& b : s.blocks) s.max_block_frames = std::max(s.max_block_frames, b.frames);
  for (auto& v : dev_events) s.events.insert(s.events.end(), v.begin(), v.end());
  std::sort(s.events.begin(), s.events.end(), [](const SchedEvent& a, const SchedEvent& b) {
    return a.slot != b.slot ? a.slot < b.slot : a.device < b.device;
  });
  auto emit_counter = [&](const std::string& name, const std::map<int64_t, std::pair<int64_t, int64_t>>& c) {
    for (const auto& [round, pr] : c) s.ledger.push_back({name, round, pr.first, pr.second});
  };
  emit_counter("host->dev0", counters[0]);
  for (int j = 0; j < N; ++j) {
    const std::string name = (j + 1 < N) ? "dev" + std::to_string(j) + "->dev" + std::to_string(j + 1)
                                         : "dev" + std::to_string(j) + "->host";
    emit_counter(name, counters[static_cast<size_t>(j) + 1]);
  }
  return s;
}

std::vector<RankOp> rank_program(const Schedule& s, int rank) {
  std::vector<RankOp> ops;
  if (rank != 0) {
    for (const SchedPass& p : s.passes) ops.push_back({0, p.index});
    return ops;
  }
  struct Timed { double t; RankOp op; };
  std::vector<Timed> v;
  for (const SchedPass& p : s.passes) {
    v.push_back({static_cast<double>(p.slots[0]), {0, p.index}});
    v.push_back({static_cast<double>(p.completion) + 0.5, {1, p.index}});
  }
  std::stable_sort(v.begin(), v.end(), [](const Timed& a, const Timed& b) { return a.t < b.t; });
  for (const Timed& t : v) ops.push_back(t.op);
  return ops;
}

}  // namespace bp

// ---- C-ABI accessors ---------------------------------------------------------
struct bp_schedule {
  bp::Schedule s;
};

extern "C" {

bp_status bp_schedule_create(const bp_pipeline_desc* desc, bp_schedule** out) {
  return bp::guarded([&] {
    if (!desc || !out) bp::fail(BP_ERR_CONFIG, "null argument");
    auto* h = new bp_schedule{bp::build_schedule(*desc)};
    *out = h;
  });
}
void bp_schedule_destroy(bp_schedule* s) { delete s; }
int64_t bp_schedule_rounds(const bp_schedule* s) { return s->s.rounds; }
int64_t bp_schedule_npasses(const bp_schedule* s) { return static_cast<int64_t>(s->s.passes.size()); }
int64_t bp_schedule_nevents(const bp_schedule* s) { return static_cast<int64_t>(s->s.events.size()); }
void bp_schedule_events(const bp_schedule* s, int64_t* out) {
  for (const bp::SchedEvent& e : s->s.events) {
    *out++ = e.slot;
    *out++ = e.device;
    *out++ = e.block;
    *out++ = e.level;
    *out++ = e.phase;
    *out++ = e.round;
  }
}
int64_t bp_schedule_nledger(const bp_schedule* s) { return static_cast<int64_t>(s->s.ledger.size()); }
void bp_schedule_ledger(const bp_schedule* s, int64_t i, char* channel, int64_t* round,
                        int64_t* passes, int64_t* scalars) {
  const bp::SchedLedger& e = s->s.ledger[static_cast<size_t>(i)];
  std::strncpy(channel, e.channel.c_str(), 31);
  channel[31] = 0;
  *round = e.round;
  *passes = e.passes;
  *scalars = e.scalars;
}
int64_t bp_schedule_nsnapshots(const bp_schedule* s) {
  return static_cast<int64_t>(s->s.snapshots.size());
}
int32_t bp_schedule_snapshot(const bp_schedule* s, int64_t i, int64_t* round, int64_t* ids,
                             int32_t* levels) {
  const bp::SchedSnapshot& sn = s->s.snapshots[static_cast<size_t>(i)];
  *round = sn.round;
  for (size_t k = 0; k < sn.ids.size(); ++k) {
    if (ids) ids[k] = sn.ids[k];
    if (levels) levels[k] = sn.levels[k];
  }
  return static_cast<int32_t>(sn.ids.size());
}
int64_t bp_schedule_nblocks(const bp_schedule* s) { return static_cast<int64_t>(s->s.emission.size()); }
int32_t bp_schedule_block(const bp_schedule* s, int64_t i, int64_t* block_id, int64_t* frames,
                          int32_t* noise_ids, int64_t* frame_ids) {
  const bp::SchedBlock& b = s->s.blocks[static_cast<size_t>(s->s.emission[static_cast<size_t>(i)] - 1)];
  *block_id = b.id;
  *frames = b.frames;
  for (size_t k = 0; k < b.noise_ids.size(); ++k)
    if (noise_ids) noise_ids[k] = b.noise_ids[k];
  for (size_t k = 0; k < b.frame_ids.size(); ++k)
    if (frame_ids) frame_ids[k] = b.frame_ids[k];
  return static_cast<int32_t>(b.noise_ids.size());
}
int64_t bp_schedule_rank_program(const bp_schedule* s, int32_t rank, int64_t* out, int64_t cap) {
  const std::vector<bp::RankOp> ops = bp::rank_program(s->s, rank);
  for (size_t i = 0; i < ops.size() && static_cast<int64_t>(i) < cap && out; ++i) {
    out[2 * i] = ops[i].kind;
    out[2 * i + 1] = ops[i].pass;
  }
  return static_cast<int64_t>(ops.size());
}

int32_t bp_schedule_pass(const bp_schedule* s, int64_t i, int64_t* rec, int32_t* levels, int64_t* frame_ids,
                         int32_t* capture) {
  const bp::SchedPass& p = s->s.passes[static_cast<size_t>(i)];
  const int64_t v[20] = {p.round, p.block, p.level, p.version, static_cast<int64_t>(p.ctx), p.ctx_block,
                         p.ctx_frames, p.ctx_version, p.ctx_first_frame, p.center_frames, p.tokens,
                         p.center_tokens, p.cached_context_id, static_cast<int64_t>(p.capture_frames.size()),
                         p.earliest, p.slots.empty() ? 0 : p.slots[0], p.completion, p.finishes_block ? 1 : 0,
                         p.phase, static_cast<int64_t>(p.frame_levels.size())};
  if (rec) std::memcpy(rec, v, sizeof(v));
  for (size_t k = 0; k < p.frame_levels.size(); ++k) {
    if (levels) levels[k] = p.frame_levels[k];
    if (frame_ids) frame_ids[k] = p.frame_ids[k];
  }
  for (size_t k = 0; k < p.capture_frames.size(); ++k)
    if (capture) capture[k] = p.capture_frames[k];
  return static_cast<int32_t>(p.frame_levels.size());
}

void bp_schedule_block_meta(const bp_schedule* s, int64_t block_id, int64_t* rec4) {
  const bp::SchedBlock& b = s->s.blocks[static_cast<size_t>(block_id - 1)];
  rec4[0] = b.frames;
  rec4[1] = b.append_round;
  rec4[2] = b.fresh ? 1 : 0;
  rec4[3] = static_cast<int64_t>(b.fresh_state);
}

void bp_schedule_partition(const bp_schedule* s, int32_t* begins, int32_t* ends) {
  for (size_t j = 0; j < s->s.begins.size(); ++j) {
    begins[j] = s->s.begins[j];
    ends[j] = s->s.ends[j];
  }
}

}  // extern "C"
