// Static, data-independent schedule of one block-wise denoising run.
//
// Everything run_pipeline decides (engine.cpp:255-497) except the tensor
// values is a pure function of the config: queue lifecycle
// (block_queue.cpp:34-145), processing order, explicit-context sources,
// cache ids, noise ids (noise.cpp:70-178, drawn on the host with the
// reference's integer stream), the logical slot clock (engine.cpp:139-140,
// 398-410), the transfer ledger and queue snapshots. We compute it once on
// the host, identically on every rank, and the GPU executor replays it.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "bp_cuda.h"

namespace bp {

enum class CtxSrc : int { None = 0, InQueue = 1, Retained = 2 };

struct SchedBlock {
  int64_t id = 0;
  int frames = 0;
  std::vector<int> noise_ids;
  std::vector<int64_t> frame_ids;
  bool fresh = false;          // kFresh: frames are normals of append_rng at fresh_state
  uint64_t fresh_state = 0;
  int64_t append_round = 0;
};

// draw_first_block / draw_next_block (noise.cpp:135-178) on the host integer
// stream: the pool ids of one block, or (kFresh) the stream position of its
// frames * frame_elems fresh normals, which the stream then skips. A first
// block has num_b + num_c/2 frames, later blocks num_b.
struct NoiseIds {
  std::vector<int> ids;
  int frames = 0;
  bool fresh = false;
  uint64_t fresh_state = 0;
};
struct HostRng;
NoiseIds draw_noise_ids(int strategy, bool first, int num_b, int num_c, const std::vector<int>& tail_window,
                        int64_t frame_elems, HostRng& rng);

struct SchedPass {
  int64_t index = 0, round = 0, block = 0;
  int level = 0, phase = 0;
  int version = 0;             // updates applied to the center so far (state read)
  int center_frames = 0;
  CtxSrc ctx = CtxSrc::None;
  int64_t ctx_block = 0;
  int ctx_frames = 0;          // explicit context frames prepended
  int ctx_version = 0;         // state version of the context source read
  int ctx_first_frame = 0;     // first frame index inside the context block
  std::vector<int> frame_levels;
  std::vector<int64_t> frame_ids;
  std::vector<int> capture_frames;
  int64_t cached_context_id = -1;  // video-later neighbour whose K/V is the prefix
  int64_t tokens = 0, center_tokens = 0;
  int64_t earliest = 1;
  std::vector<int64_t> slots;  // per device
  int64_t completion = 0;
  bool finishes_block = false; // this pass's update brings the block to level 0
};

struct SchedEvent {
  int64_t slot, device, block, level, phase, round;
};
struct SchedLedger {
  std::string channel;
  int64_t round, passes, scalars;
};
struct SchedSnapshot {
  int64_t round;
  std::vector<int64_t> ids;
  std::vector<int> levels;
};

struct Schedule {
  bp_pipeline_desc desc{};
  int devices = 1;
  std::vector<int> begins, ends;   // per stage layer range
  int64_t rounds = 0;
  int64_t max_tokens = 0;
  int max_block_frames = 0;
  std::vector<SchedBlock> blocks;  // index = id - 1
  std::vector<SchedPass> passes;   // issue order (round by round, processing order)
  std::vector<int64_t> emission;   // block ids in emission order
  std::vector<SchedEvent> events;  // sorted by (slot, device)
  std::vector<SchedLedger> ledger;
  std::vector<SchedSnapshot> snapshots;
};

// One rank's ordered program for the one-process-per-GPU pipeline:
// kind 0 = stage forward of a pass (rank 0 also appends due blocks and
// assembles the payload; every rank then sends its output downstream),
// kind 1 = rank 0 receives a pass's eps and applies the Euler update.
// Rank 0 merges both kinds by the logical slot clock (forward at slot_0(p),
// update at completion(p) + 0.5); other ranks run forwards in pass order.
struct RankOp {
  int kind;
  int64_t pass;
};
std::vector<RankOp> rank_program(const Schedule& s, int rank);

int ffn_width(const bp_model_desc& m);
void validate_model(const bp_model_desc& m);
// Stage layer ranges: the reference's even split (model.cpp:134-148), or the
// opt-in uneven / explicit contiguous split.
void partition_layers(const bp_pipeline_desc& d, std::vector<int>* begins, std::vector<int>* ends);
Schedule build_schedule(const bp_pipeline_desc& d);

}  // namespace bp
