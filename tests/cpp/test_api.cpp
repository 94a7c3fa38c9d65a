// The reference's own C++ test cases (P/tests/test_model.cpp, test_engine.cpp,
// test_tensor.cpp, test_rng.cpp, test_noise.cpp, test_queue.cpp) re-run
// against the B200 mirror of the blockpipe API. doctest is not vendored
// in this image, so a minimal CHECK harness stands in for it. Exit code =
// number of failed checks; the last line prints the cfg-1 latents FNV.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <map>
#include <set>
#include <string>

#include "blockpipe/block_queue.hpp"
#include "blockpipe/engine.hpp"
#include "blockpipe/model.hpp"
#include "blockpipe/noise.hpp"
#include "blockpipe/rng.hpp"
#include "blockpipe/tensor.hpp"

using namespace blockpipe;

static int g_fail = 0, g_pass = 0;
#define CHECK(c) do { if (c) ++g_pass; else { ++g_fail; std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); } } while (0)
template <class E, class F> bool throws(F&& f) { try { f(); } catch (const E&) { return true; } catch (...) { return false; } return false; }

static ModelConfig tiny_cfg() {
  ModelConfig c;
  c.layers = 2; c.hidden = 8; c.heads = 2; c.channels = 2; c.height = 1; c.width = 1; c.context_len = 3;
  return c;
}
static PipelineConfig cfg_small(int devices, int steps, int blocks) {
  PipelineConfig p;
  p.devices = devices; p.threaded = false;
  p.model.layers = 4; p.model.hidden = 8; p.model.heads = 2; p.model.channels = 2; p.model.height = 2;
  p.model.width = 2; p.model.context_len = 3;
  p.queue.num_b = 2; p.queue.num_c = 4; p.queue.steps = steps; p.queue.block_num = blocks;
  return p;
}

static bool near(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(std::abs(a), std::abs(b)); }

// ---- test_tensor.cpp ------------------------------------------------------------
static void tensor_cases() {
  Tensor eye({2, 2}, {1, 0, 0, 1}), b22({2, 2}, {3, 4, 5, 6});
  CHECK(matmul(eye, b22).bitwise_equal(b22));
  Tensor c = matmul(Tensor({1, 2}, {1, 2}), Tensor({2, 1}, {3, 4}));
  CHECK(c.shape == std::vector<int64_t>({1, 1}) && c.data[0] == 11.0);
  {  // bitwise equal to an ascending-k triple loop
    RandomSource rs(42);
    Tensor a = rs.normal_tensor({5, 7}), bb = rs.normal_tensor({7, 3});
    Tensor want({5, 3});
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 3; ++j) {
        volatile double acc = 0.0;
        for (int t = 0; t < 7; ++t) {
          volatile double prod = a.data[static_cast<size_t>(i * 7 + t)] * bb.data[static_cast<size_t>(t * 3 + j)];
          acc = acc + prod;
        }
        want.data[static_cast<size_t>(i * 3 + j)] = acc;
      }
    CHECK(matmul(a, bb).bitwise_equal(want));
  }
  CHECK(throws<DimensionError>([] { matmul(Tensor({2, 3}), Tensor({2, 3})); }));
  Tensor s = softmax_rows(Tensor({1, 2}, {0, 0}));
  CHECK(s.data[0] == 0.5 && s.data[1] == 0.5);
  Tensor sb = softmax_rows(Tensor({1, 2}, {1000, 1000}));
  CHECK(sb.data[0] == 0.5 && sb.data[1] == 0.5 && sb.all_finite());
  Tensor sl = softmax_rows(Tensor({1, 2}, {0.0, std::log(3.0)}));
  CHECK(near(sl.data[0], 0.25, 1e-12) && near(sl.data[1], 0.75, 1e-12));
  {
    RandomSource rs(7);
    Tensor p = softmax_rows(rs.normal_tensor({6, 9}));
    for (int i = 0; i < 6; ++i) {
      double sum = 0.0;
      for (int j = 0; j < 9; ++j) { CHECK(p.at(i, j) >= 0.0); sum += p.at(i, j); }
      CHECK(near(sum, 1.0, 1e-12));
    }
  }
  for (double v : layer_norm(Tensor({1, 4}, {5, 5, 5, 5}), 1e-5).data) CHECK(v == 0.0);
  Tensor ln = layer_norm(Tensor({1, 2}, {1, -1}), 1e-5);
  CHECK(near(ln.data[0], 1.0, 1e-4) && near(ln.data[1], -1.0, 1e-4));
  {  // two-pass oracle and output moments
    RandomSource rs(3);
    Tensor x = rs.normal_tensor({4, 11});
    Tensor y = layer_norm(x, 1e-5);
    for (int i = 0; i < 4; ++i) {
      double mean = 0.0, var = 0.0, om = 0.0, ov = 0.0;
      for (int j = 0; j < 11; ++j) mean += x.at(i, j);
      mean /= 11.0;
      for (int j = 0; j < 11; ++j) var += (x.at(i, j) - mean) * (x.at(i, j) - mean);
      var /= 11.0;
      for (int j = 0; j < 11; ++j) {
        CHECK(std::abs(y.at(i, j) - (x.at(i, j) - mean) / std::sqrt(var + 1e-5)) <= 1e-12);
        om += y.at(i, j);
        ov += y.at(i, j) * y.at(i, j);
      }
      CHECK(std::abs(om / 11.0) <= 1e-10 && near(ov / 11.0, 1.0, 1e-4));
    }
  }
  Tensor a({2, 3}, {1, 2, 3, 4, 5, 6}), r({1, 3}, {7, 8, 9});
  Tensor v = vcat_rows(a, r);
  CHECK(v.shape == std::vector<int64_t>({3, 3}) && v.at(2, 0) == 7.0);
  CHECK(slice_rows(v, 1, 3).at(0, 2) == 6.0);
  Tensor t = take_rows(v, {2, 0});
  CHECK(t.at(0, 1) == 8.0 && t.at(1, 0) == 1.0);
  CHECK(throws<DimensionError>([&] { slice_rows(v, 0, 4); }));
  CHECK(throws<DimensionError>([&] { take_rows(v, {3}); }));
  CHECK(add(a, a).at(1, 2) == 12.0 && sub(a, a).at(1, 2) == 0.0 && scale(a, 0.5).at(0, 1) == 1.0);
  CHECK(throws<DimensionError>([&] { add(a, r); }));
  {  // purity and finiteness
    RandomSource rs(11);
    Tensor x = rs.normal_tensor({3, 5}), w = rs.normal_tensor({5, 2});
    CHECK(matmul(x, w).bitwise_equal(matmul(x, w)));
    CHECK(softmax_rows(x).bitwise_equal(softmax_rows(x)));
    CHECK(layer_norm(x, 1e-5).bitwise_equal(layer_norm(x, 1e-5)));
    RandomSource rs5(5);
    Tensor q = rs5.normal_tensor({8, 8});
    CHECK(matmul(q, q).all_finite() && softmax_rows(scale(q, 500.0)).all_finite() && layer_norm(q, 1e-5).all_finite());
  }
}

// ---- test_rng.cpp ---------------------------------------------------------------
static void rng_cases() {
  {
    RandomSource a(123), b(123);
    Tensor ta = a.normal_tensor({10000}), tb = b.normal_tensor({10000});
    CHECK(ta.bitwise_equal(tb));
  }
  {
    RandomSource rs(2024);
    Tensor x = rs.normal_tensor({100000});
    double sum = 0, sq = 0;
    for (double d : x.data) { sum += d; sq += d * d; }
    const double mean = sum / 1e5, var = sq / 1e5 - mean * mean;
    CHECK(std::abs(mean) < 0.02 && std::abs(var - 1.0) < 0.02);
  }
  {
    RandomSource a(77), b(78);
    bool diverged = false;
    for (int i = 0; i < 16 && !diverged; ++i) diverged = a.next_normal() != b.next_normal();
    CHECK(diverged);
  }
  {  // placement independence: k + k == 2k, and single draws == tensor draws
    RandomSource whole(9), split(9), single(9);
    Tensor all = whole.normal_tensor({64});
    Tensor p1 = split.normal_tensor({32}), p2 = split.normal_tensor({32});
    bool same = true;
    for (int i = 0; i < 32; ++i) same = same && all.data[static_cast<size_t>(i)] == p1.data[static_cast<size_t>(i)] &&
                                        all.data[static_cast<size_t>(32 + i)] == p2.data[static_cast<size_t>(i)];
    CHECK(same);
    for (int i = 0; i < 4; ++i) CHECK(single.next_normal() == all.data[static_cast<size_t>(i)]);
  }
  {
    RandomSource rs(31337);
    bool ok = true;
    for (int i = 0; i < 1000; ++i) {
      const double u = rs.next_uniform();
      ok = ok && u >= 0.0 && u < 1.0;
    }
    CHECK(ok && rs.normal_tensor({1000}).all_finite());
  }
  {
    RandomSource a(5), b(5);
    const std::vector<int> p = a.permutation(12);
    CHECK(p == b.permutation(12));
    std::set<int> seen(p.begin(), p.end());
    CHECK(seen.size() == 12 && *seen.begin() == 0 && *seen.rbegin() == 11);
  }
  CHECK(derive_seed(99, {0, 1}) != derive_seed(99, {1, 0}));
  CHECK(derive_seed(99, {0}) != derive_seed(99, {1}));
  CHECK(derive_seed(99, {3, 7}) == derive_seed(99, {3, 7}));
}

// ---- test_noise.cpp -------------------------------------------------------------
static void noise_cases() {
  const std::vector<int64_t> fr = {2, 2, 1};
  CHECK(build_pool(8, 8, fr, 1).size() == 12 && build_pool(4, 0, fr, 1).size() == 4);
  {
    NoisePool pool = build_pool(8, 8, fr, 2);
    RandomSource r1(5), r2(5);
    NoiseDraw d = init_first_block(pool, r1), d2 = init_first_block(pool, r2);
    std::set<int> ids(d.noise_ids.begin(), d.noise_ids.end());
    CHECK(d.frames.shape[0] == 12 && ids.size() == 12 && *ids.begin() == 0 && *ids.rbegin() == 11);
    CHECK(d.noise_ids == d2.noise_ids && d.frames.bitwise_equal(d2.frames));
    // the stacked frames are the pool entries of the drawn ids
    bool stacked = true;
    for (size_t i = 0; i < d.noise_ids.size(); ++i)
      for (int k = 0; k < 4; ++k)
        stacked = stacked && d.frames.data[i * 4 + static_cast<size_t>(k)] ==
                                 pool.entries[static_cast<size_t>(d.noise_ids[i])].data[static_cast<size_t>(k)];
    CHECK(stacked);
  }
  {
    NoisePool pool = build_pool(6, 0, fr, 3);
    RandomSource rng(1);
    CHECK(init_first_block(pool, rng).frames.shape[0] == 6);
    NoiseDraw next = init_next_block(pool, {}, rng);
    CHECK(std::set<int>(next.noise_ids.begin(), next.noise_ids.end()).size() == 6);
  }
  {
    NoisePool pool = build_pool(8, 8, fr, 4);
    RandomSource rng(9);
    NoiseDraw d = init_next_block(pool, {8, 9, 10, 11}, rng);
    CHECK(d.noise_ids.size() == 8 && std::set<int>(d.noise_ids.begin(), d.noise_ids.end()).size() == 8);
    for (int id : d.noise_ids) CHECK(id < 8);
    CHECK(throws<QueueError>([&] { init_next_block(pool, {1, 1, 2, 3}, rng); }));
    CHECK(throws<QueueError>([&] { init_next_block(pool, {1, 2, 3}, rng); }));
    CHECK(throws<QueueError>([&] { init_next_block(pool, {1, 2, 3, 99}, rng); }));
  }
  {
    NoisePool pool = build_pool(5, 6, fr, 11);  // m = 8, window 3
    for (uint64_t seed = 0; seed < 50; ++seed) {
      RandomSource rng(seed);
      const std::vector<int> perm = rng.permutation(pool.size());
      std::vector<int> window(perm.begin(), perm.begin() + 3);
      NoiseDraw d = init_next_block(pool, window, rng);
      std::set<int> all(window.begin(), window.end());
      bool disjoint = true;
      for (int id : d.noise_ids) disjoint = all.insert(id).second && disjoint;
      CHECK(disjoint && static_cast<int>(all.size()) == pool.size());
    }
  }
  {
    NoisePool pool = build_pool(4, 4, fr, 6);
    RandomSource rng(2);
    NoiseDraw a = init_baseline(InitStrategy::kRepeat, pool, rng), b = init_baseline(InitStrategy::kRepeat, pool, rng);
    CHECK(a.frames.bitwise_equal(b.frames) && a.noise_ids == b.noise_ids);
    NoiseDraw f1 = init_baseline(InitStrategy::kFresh, pool, rng), f2 = init_baseline(InitStrategy::kFresh, pool, rng);
    CHECK(f1.noise_ids.empty() && f2.noise_ids.empty() && !f1.frames.bitwise_equal(f2.frames));
    CHECK(throws<ConfigError>([&] { init_baseline(InitStrategy::kCoordinated, pool, rng); }));
  }
  {
    NoisePool pool = build_pool(6, 0, fr, 7);
    RandomSource rng(3);
    NoiseDraw sub = init_baseline(InitStrategy::kSubset, pool, rng);
    CHECK(sub.noise_ids.size() == 6 && std::set<int>(sub.noise_ids.begin(), sub.noise_ids.end()).size() == 6);
  }
  {  // 1000 coordinated appends keep the window invariant
    NoisePool pool = build_pool(8, 8, fr, 12);
    RandomSource rng(13);
    NoiseDraw cur = init_first_block(pool, rng);
    bool ok = true;
    for (int i = 0; i < 1000; ++i) {
      std::vector<int> window(cur.noise_ids.end() - 4, cur.noise_ids.end());
      NoiseDraw next = init_next_block(pool, window, rng);
      std::set<int> seen(window.begin(), window.end());
      for (int id : next.noise_ids) ok = seen.insert(id).second && ok;
      ok = ok && static_cast<int>(seen.size()) == pool.size();
      cur = std::move(next);
    }
    CHECK(ok);
  }
  {  // repeat overlaps the tail window on every append
    NoisePool pool = build_pool(8, 8, fr, 14);
    RandomSource rng(15);
    NoiseDraw cur = draw_first_block(InitStrategy::kRepeat, pool, rng);
    bool ok = true;
    for (int i = 0; i < 100; ++i) {
      std::vector<int> window(cur.noise_ids.end() - 4, cur.noise_ids.end());
      NoiseDraw next = draw_next_block(InitStrategy::kRepeat, pool, window, rng);
      int overlap = 0;
      for (int id : next.noise_ids) overlap += static_cast<int>(std::count(window.begin(), window.end(), id));
      ok = ok && overlap > 0;
      cur = std::move(next);
    }
    CHECK(ok);
  }
  {  // engine draws: first block M frames for every strategy, fresh draws bit-exact normals
    NoisePool pool = build_pool(4, 4, fr, 21);
    for (InitStrategy st : {InitStrategy::kCoordinated, InitStrategy::kCompleteShuffle, InitStrategy::kSubset,
                            InitStrategy::kFresh, InitStrategy::kRepeat}) {
      RandomSource rng(8);
      NoiseDraw d = draw_first_block(st, pool, rng);
      CHECK(d.frames.shape[0] == 6);
      std::vector<int> window = st == InitStrategy::kFresh ? std::vector<int>{} :
                                std::vector<int>(d.noise_ids.end() - 2, d.noise_ids.end());
      CHECK(draw_next_block(st, pool, window, rng).frames.shape[0] == 4);
    }
    RandomSource a(8), b(8);
    NoiseDraw fresh = draw_first_block(InitStrategy::kFresh, pool, a);
    CHECK(fresh.frames.bitwise_equal(b.normal_tensor({6, 2, 2, 1})) && a.state == b.state);
  }
  for (InitStrategy st : {InitStrategy::kCoordinated, InitStrategy::kCompleteShuffle, InitStrategy::kSubset,
                          InitStrategy::kFresh, InitStrategy::kRepeat})
    CHECK(parse_strategy(strategy_name(st)) == st);
  CHECK(throws<ConfigError>([] { parse_strategy("bogus"); }));
}

// ---- test_queue.cpp -------------------------------------------------------------
static QueueParams qparams(int num_b, int num_c, int steps, int block_num) {
  QueueParams p;
  p.num_b = num_b; p.num_c = num_c; p.steps = steps; p.block_num = block_num;
  return p;
}
static Tensor qframes(int64_t id, int64_t count) {
  Tensor t({count, 1, 1, 1});
  for (int64_t i = 0; i < count; ++i) t.data[static_cast<size_t>(i)] = 100.0 * static_cast<double>(id) + static_cast<double>(i);
  return t;
}
static LatentBlock qblock(const QueueParams& p, int64_t id, int64_t* next_frame) {
  LatentBlock b;
  b.block_id = id;
  const int64_t f = id == 1 ? p.num_b + p.num_c / 2 : p.num_b;
  b.frames = qframes(id, f);
  for (int64_t i = 0; i < f; ++i) {
    b.noise_ids.push_back(static_cast<int>(i));
    b.frame_ids.push_back((*next_frame)++);
  }
  return b;
}
static void update_all(QueueState& q, Order order) {
  for (int64_t id : processing_order(q, order)) apply_update(q, id, qframes(id, q.find(id)->frame_count()));
}

static void queue_cases() {
  {
    QueueParams p = qparams(2, 4, 3, 4);
    QueueState q;
    q.params = p;
    int64_t nf = 0;
    q = advance(std::move(q), qblock(p, 1, &nf));
    CHECK(q.blocks.size() == 1 && q.blocks[0].level == 3 && q.blocks[0].frame_count() == 4);
  }
  {  // steady: pop the clean head, append at T, retain the clean tail
    QueueParams p = qparams(2, 2, 3, 4);
    QueueState q;
    q.params = p;
    int64_t nf = 0, nb = 1;
    for (int r = 1; r <= 3; ++r) {
      q = advance(std::move(q), qblock(p, nb++, &nf));
      update_all(q, Order::kSequential);
    }
    CHECK(q.blocks.size() == 3 && q.blocks[0].level == 0 && q.blocks[1].level == 1 && q.blocks[2].level == 2);
    q = advance(std::move(q), qblock(p, nb++, &nf));
    CHECK(q.blocks.size() == 3 && q.blocks[0].block_id == 2 && q.blocks[0].level == 1 && q.blocks[2].level == 3);
    CHECK(q.popped_ids == std::vector<int64_t>({1}));
    CHECK(q.retained.has_value() && q.retained->source_block_id == 1 && q.retained->frames.shape[0] == 1);
  }
  {  // cool-down
    QueueParams p = qparams(2, 2, 4, 2);
    QueueState q;
    q.params = p;
    int64_t nf = 0;
    q = advance(std::move(q), qblock(p, 1, &nf));
    q = advance(std::move(q), qblock(p, 2, &nf));
    CHECK(throws<QueueError>([&] { advance(QueueState(q), qblock(p, 3, &nf)); }));
    for (int r = 0; r < 4; ++r) {
      update_all(q, Order::kSequential);
      if (r < 3) q = advance(std::move(q), std::nullopt);
    }
    CHECK(q.blocks.front().level == 0);
    q = advance(std::move(q), std::nullopt);
    CHECK(q.blocks.size() == 1 && q.blocks[0].block_id == 2);
  }
  {  // processing order
    QueueParams p = qparams(2, 2, 3, 3);
    QueueState q;
    q.params = p;
    int64_t nf = 0;
    for (int64_t id = 1; id <= 3; ++id) {
      q = advance(std::move(q), qblock(p, id, &nf));
      if (id < 3) update_all(q, Order::kReverse);
    }
    CHECK(processing_order(q, Order::kReverse) == std::vector<int64_t>({3, 2, 1}));
    CHECK(processing_order(q, Order::kSequential) == std::vector<int64_t>({1, 2, 3}));
  }
  {  // assemble_extended boundaries
    QueueParams p = qparams(2, 4, 3, 3);
    QueueState q;
    q.params = p;
    int64_t nf = 0;
    for (int64_t id = 1; id <= 3; ++id) {
      q = advance(std::move(q), qblock(p, id, &nf));
      if (id < 3) update_all(q, Order::kReverse);
    }
    ExtendedBlock tail = assemble_extended(q, 3, Order::kReverse);
    CHECK(!tail.cached_context_id && tail.source == ExtendedBlock::CtxSource::kInQueue);
    ExtendedBlock mid = assemble_extended(q, 2, Order::kReverse);
    CHECK(mid.cached_context_id && *mid.cached_context_id == 3 && mid.explicit_frames.shape[0] == 2);
    CHECK(mid.explicit_frame_ids == std::vector<int64_t>({2, 3}));
    ExtendedBlock head = assemble_extended(q, 1, Order::kReverse);
    CHECK(head.source == ExtendedBlock::CtxSource::kNone && head.explicit_frames.numel() == 0 &&
          head.cached_context_id && *head.cached_context_id == 2);
    CHECK(!assemble_extended(q, 2, Order::kSequential).cached_context_id);
    CHECK(throws<QueueError>([&] { assemble_extended(q, 99, Order::kReverse); }));
  }
  {  // the neighbour's state at the centre's update count
    QueueParams p = qparams(2, 2, 4, 3);
    QueueState q;
    q.params = p;
    int64_t nf = 0;
    q = advance(std::move(q), qblock(p, 1, &nf));
    apply_update(q, 1, qframes(10, 3));
    q = advance(std::move(q), qblock(p, 2, &nf));
    ExtendedBlock e = assemble_extended(q, 2, Order::kReverse);
    CHECK(e.explicit_frames.shape[0] == 1 && e.explicit_frames.data[0] == 102.0 && e.explicit_levels == std::vector<int>({4}));
    apply_update(q, 2, qframes(20, 2));
    CHECK(assemble_extended(q, 2, Order::kReverse).explicit_frames.data[0] == 1002.0);
    apply_update(q, 2, qframes(21, 2));
    CHECK(throws<QueueError>([&] { assemble_extended(q, 2, Order::kReverse); }));
  }
  for (bool retain : {true, false}) {  // round-atomic lifecycle: ladder, conservation, FIFO emission
    for (Order order : {Order::kReverse, Order::kSequential}) {
      QueueParams p = retain ? qparams(2, 4, 4, 6) : qparams(2, 2, 2, 3);
      p.retain_clean_context = retain;
      QueueState q;
      q.params = p;
      int64_t nf = 0, nb = 1;
      const int64_t rounds = p.steps + p.block_num - 1;
      std::vector<int64_t> emitted;
      std::map<int64_t, int> passes;
      bool ladder = true;
      for (int64_t r = 1; r <= rounds + 1; ++r) {
        std::optional<LatentBlock> blk;
        if (r <= rounds && nb <= p.block_num) blk = qblock(p, nb++, &nf);
        if (!q.blocks.empty() && q.blocks.front().level == 0) emitted.push_back(q.blocks.front().block_id);
        q = advance(std::move(q), std::move(blk));
        if (r > rounds) break;
        ladder = ladder && levels_are_unit_ladder(q) && static_cast<int>(q.blocks.size()) <= p.steps;
        for (int64_t id : processing_order(q, order)) (void)assemble_extended(q, id, order);
        std::vector<int64_t> ids;
        for (const LatentBlock& b : q.blocks) ids.push_back(b.block_id);
        for (int64_t id : ids) {
          apply_update(q, id, qframes(id, q.find(id)->frame_count()));
          passes[id] += 1;
        }
      }
      CHECK(ladder && q.blocks.empty());
      std::vector<int64_t> want;
      for (int64_t i = 1; i <= p.block_num; ++i) want.push_back(i);
      CHECK(emitted == want && static_cast<int>(passes.size()) == p.block_num);
      for (const auto& kv : passes) CHECK(kv.second == p.steps);
    }
  }
}

int main() {
  tensor_cases();
  rng_cases();
  noise_cases();
  queue_cases();
  {  // cached path equals explicit recompute oracle (test_model.cpp:178-223)
    ModelConfig cfg = tiny_cfg();
    ModelChunk model = build_model(cfg, 17);
    Tensor context = build_context(cfg, 19);
    RandomSource rs(23);
    ChunkInput prev;
    prev.payload = rs.normal_tensor({2, cfg.channels});
    prev.frame_levels = {5, 5};
    prev.frame_ids = {4, 5};
    prev.capture_frames = {0};
    ChunkOutput cap = forward_chunk(model, prev, context, CacheMode::kCached, nullptr, nullptr);
    CHECK(cap.captured.has_value());
    ChunkOutput rec = forward_chunk(model, prev, context, CacheMode::kRecompute, nullptr, nullptr);
    CHECK(rec.recorded.has_value());
    CHECK(cap.payload.bitwise_equal(rec.payload));
    ChunkInput cur;
    cur.payload = rs.normal_tensor({3, cfg.channels});
    cur.frame_levels = {4, 4, 4};
    cur.frame_ids = {1, 2, 3};
    ChunkOutput via_cache = forward_chunk(model, cur, context, CacheMode::kCached, &*cap.captured, nullptr);
    ChunkOutput via_rec = forward_chunk(model, cur, context, CacheMode::kRecompute, nullptr, &*rec.recorded);
    CHECK(via_cache.payload.bitwise_equal(via_rec.payload));
    ChunkOutput cap2 = forward_chunk(model, prev, context, CacheMode::kCached, nullptr, nullptr);
    for (size_t l = 0; l < cap.captured->per_layer.size(); ++l) {
      CHECK(cap.captured->per_layer[l].k.bitwise_equal(cap2.captured->per_layer[l].k));
      CHECK(cap.captured->per_layer[l].v.bitwise_equal(cap2.captured->per_layer[l].v));
    }
    KVCacheEntry tampered = *cap.captured;
    double& v0 = tampered.per_layer[0].v.data[0];
    v0 = std::nextafter(v0, 1e308);
    ChunkOutput via_t = forward_chunk(model, cur, context, CacheMode::kCached, &tampered, nullptr);
    CHECK(!via_t.payload.bitwise_equal(via_cache.payload));
    CHECK(throws<CacheError>([&] { forward_chunk(model, cur, context, CacheMode::kDisabled, &*cap.captured, nullptr); }));
  }
  {  // chunked forward equals monolithic forward (test_model.cpp:155-176)
    ModelConfig cfg = tiny_cfg();
    cfg.layers = 4;
    ModelChunk mono = build_model(cfg, 9);
    std::vector<ModelChunk> parts = partition(cfg, 9, 2);
    Tensor context = build_context(cfg, 13);
    RandomSource rs(33);
    ChunkInput in;
    in.payload = rs.normal_tensor({3, cfg.channels});
    in.frame_levels = {2, 2, 2};
    in.frame_ids = {5, 6, 7};
    ChunkOutput whole = forward_chunk(mono, in, context, CacheMode::kDisabled, nullptr, nullptr);
    ChunkOutput first = forward_chunk(parts[0], in, context, CacheMode::kDisabled, nullptr, nullptr);
    ChunkInput second = in;
    second.payload = first.payload;
    ChunkOutput last = forward_chunk(parts[1], second, context, CacheMode::kDisabled, nullptr, nullptr);
    CHECK(last.payload.bitwise_equal(whole.payload));
    cfg.layers = 6;
    CHECK(throws<PartitionError>([&] { partition(cfg, 1, 4); }));
  }
  {  // scheduler (test_model.cpp:270-298)
    Tensor x({2, 2}, {1, 2, 3, 4});
    CHECK(scheduler_step(x, Tensor({2, 2}), 3, 8).bitwise_equal(x));
    RandomSource rs(71);
    Tensor a = rs.normal_tensor({2, 3}), e = rs.normal_tensor({2, 3});
    Tensor got = scheduler_step(a, e, 25, 50);
    for (size_t i = 0; i < a.data.size(); ++i) CHECK(got.data[i] == a.data[i] - 0.02 * e.data[i]);
    CHECK(throws<SchedulerError>([&] { scheduler_step(x, x, 0, 8); }));
  }
  {  // pipeline == serial oracle for N in {2,4} x cache on/off (test_engine.cpp:66-78)
    for (int n : {2, 4}) {
      for (CacheMode m : {CacheMode::kDisabled, CacheMode::kCached}) {
        PipelineConfig p = cfg_small(n, 4, 4);
        p.cache_mode = m;
        std::string diff;
        CHECK(blocks_bitwise_equal(run_pipeline(p).blocks, serial_oracle(p).blocks, &diff));
      }
    }
    PipelineConfig p = cfg_small(2, 4, 5);  // emission order + first-block surplus (:80-91)
    RunResult r = run_pipeline(p);
    CHECK(r.blocks.size() == 5);
    for (size_t i = 0; i < r.blocks.size(); ++i) CHECK(r.blocks[i].block_id == static_cast<int64_t>(i + 1));
    CHECK(r.blocks[0].frames.shape[0] == 4 && r.blocks[1].frames.shape[0] == 2);
    BubbleStats st = measure_bubbles(run_pipeline(cfg_small(1, 4, 4)).log);
    CHECK(st.idle_per_device == 0 && st.busy_per_device == 16);
  }
  {  // cached == recompute (+ trace); 1-ulp fault caught (test_engine.cpp:129-150)
    PipelineConfig p = cfg_small(2, 6, 5);
    p.model.hidden = 16;
    p.record_trace = true;
    RunResult cached = run_pipeline(p);
    p.cache_mode = CacheMode::kRecompute;
    RunResult recomputed = run_pipeline(p);
    std::string diff;
    CHECK(blocks_bitwise_equal(cached.blocks, recomputed.blocks, &diff));
    CHECK(traces_bitwise_equal(cached.trace, recomputed.trace, &diff));
    p.cache_mode = CacheMode::kCached;
    p.fault_inject_ulp = true;
    p.check_cache = true;
    CHECK(throws<CacheError>([&] { run_pipeline(p); }));
    p.fault_inject_ulp = false;
    CHECK(blocks_bitwise_equal(run_pipeline(p).blocks, cached.blocks, &diff));
    CHECK(throws<ConfigError>([&] { run_pipeline(cfg_small(3, 4, 4)); }));
  }
  // BASELINE configs[0]: latents FNV-1a-64 in emission order (compared by the pytest wrapper)
  PipelineConfig c1;
  c1.devices = 1; c1.model.layers = 2; c1.model.hidden = 128; c1.model.heads = 4;
  c1.queue.steps = 10; c1.queue.block_num = 4;
  RunResult r1 = run_pipeline(c1);
  uint64_t h = 0xCBF29CE484222325ULL;
  double sumsq = 0;
  for (const EmittedBlock& b : r1.blocks)
    for (double v : b.frames.data) {
      sumsq += v * v;
      const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
      for (int k = 0; k < 8; ++k) h = (h ^ p[k]) * 0x100000001B3ULL;
    }
  std::printf("passed %d failed %d\ncfg1 sumsq %.17g fnv %016llx\n", g_pass, g_fail, sumsq, static_cast<unsigned long long>(h));
  return g_fail;
}
