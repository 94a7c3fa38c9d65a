// run_pipeline (engine.cpp:255-497) on B200s: the host replays the static
// schedule (schedule.cpp); rank 0 owns the block latents, the noise pool
// and the Euler updates; stage j runs on rank j (NCCL transport, one process
// per GPU; NCCL or CUDA-IPC transport) or all stages share one GPU
// (loopback). Hidden states move between stages on dedicated streams from and
// into a 3-slot residual ring (no boundary copies), event-chained to compute,
// so transfers overlap the next pass.
#include <cuda.h>
#include <cuda_runtime.h>
#include "nccl_dl.hpp"

#include <algorithm>
#include <string>
#include <unistd.h>
#include <thread>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "device.cuh"
#include "kernels_bf16.cuh"
#include "kernels_simt.cuh"
#include "schedule.hpp"
#include "stage.hpp"

#define BP_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess)                                                             \
      ::bp::fail(BP_ERR_NCCL, std::string(#call) + ": " + bp::nccl().GetErrorString(r_));     \
  } while (0)

namespace bp {

class Pipeline {
 public:
  Pipeline(const bp_pipeline_desc& d, int rank, int world, int device, const uint8_t* ids);
  ~Pipeline();
  void run(bp_emit_fn emit, void* user);
  Schedule sched;
  bp_pipeline_stats stats{};
  std::vector<std::vector<double>> trace;  // host eps per pass (record_trace)
  std::vector<int64_t> trace_rows;
  std::vector<const double*> block_dev;    // emitted blocks' device latents (rank 0)
  std::vector<int64_t> block_count;
  bool profiling = false;
  const double* host_pool = nullptr;       // borrowed caller pool (bp_pipeline_set_pool)

 private:
  void run_rank0_loopback(bp_emit_fn emit, void* user);
  void run_nccl(bp_emit_fn emit, void* user);
  void build_pool_and_check(cudaStream_t st);
  void append_block(const SchedBlock& b, cudaStream_t st);
  void assemble(const SchedPass& p, cudaStream_t st);
  void step(const SchedPass& p, const void* eps, cudaStream_t st);
  void emit_block(const SchedBlock& b, cudaStream_t st, bool to_host);
  StageInput stage_input(const SchedPass& p, int stage, const void* payload, bool* use_cache_checked);
  void before_stage(const SchedPass& p, int stage, Stage& s, StageInput* in);
  void after_stage(const SchedPass& p, int stage, Stage& s);
  double* version_ptr(int64_t block, int version) const;

  bp_pipeline_desc d_;
  int rank_, world_, device_;
  int64_t tpf_, C_, hwc_;
  std::vector<std::unique_ptr<Stage>> stages_;  // index = stage id (only local ones non-null)
  cudaStream_t st_ = nullptr;
  // rank 0 state
  DevBuf pool_, latents_, payload_, pass_levels_, pass_ids_, flags_;
  std::vector<int64_t> block_off_;             // element offset of each block's 3 versions
  std::vector<int64_t> pass_off_;              // offset into pass_levels_/pass_ids_
  std::vector<double*> pinned_;                // emission buffers
  bool fault_pending_ = false;
  bool failed_ = false;  // a multi-process run threw (see ~Pipeline)
  int64_t launches_at_start_ = 0;
  // NCCL
  ncclComm_t comm_prev_ = nullptr, comm_next_ = nullptr, comm_eps_ = nullptr;
  cudaStream_t s_recv_ = nullptr, s_send_ = nullptr, s_eps_ = nullptr;
  DevBuf ebuf_[2];
  // Stage-boundary ring (multi-process): the local stage's residual stream
  // has kRing slots; a pass receives into its slot, runs every layer in place
  // and is sent from the same slot, so no device copies sit on the boundary.
  // NCCL: slots from ncclMemAlloc, registered with the channels' comms where
  // NCCL accepts it (zero-copy P2P over NVLink); IPC: the slots of ranks > 0
  // ARE the exported receive ring the predecessor's peer copies land in.
  static constexpr int kRing = 3;
  void* alloc_ring_buffer(size_t bytes);
  void register_buffer(ncclComm_t comm, void* p, size_t bytes);
  std::vector<DevBuf> own_ring_;
  std::vector<void*> nccl_mem_;
  std::vector<std::pair<ncclComm_t, void*>> nccl_regs_;
  int64_t registered_ = 0;

 public:
  // IPC transport: this rank's exported block = [hidden ring: kRing slots]
  // [eps ring: 2 slots][counters]; the same layout on every rank.
  //   cnt[0] hidden passes delivered into my ring (written by rank - 1)
  //   cnt[1] eps passes delivered into my eps ring (rank 0; written by N - 1)
  //   cnt[2] my outgoing hidden passes consumed (written by rank + 1)
  //   cnt[3] my outgoing eps passes consumed (rank N - 1; written by rank 0)
  // Counters grow monotonically across runs (ipc_epoch_ passes per run).
  void ipc_handle(uint8_t out[64]);
  void ipc_connect(const uint8_t* handles);
  void ipc_counters(uint32_t out[4]);

 private:
  bool multi() const { return d_.transport != BP_TRANSPORT_LOOPBACK && d_.devices > 1; }
  bool ipc() const { return d_.transport == BP_TRANSPORT_IPC && d_.devices > 1; }
  // hidden ring: kRing slots (slot i % kRing); eps ring: 2 slots (i & 1)
  char* ipc_slot(char* block, int which, int64_t i) const {
    return which == 0 ? block + (i % kRing) * ipc_hid_ : block + kRing * ipc_hid_ + (i & 1) * ipc_eps_;
  }
  uint32_t* ipc_cnt(char* block, int k) const {
    return reinterpret_cast<uint32_t*>(block + kRing * ipc_hid_ + 2 * ipc_eps_) + k;
  }
  void ipc_send(char* peer, int which, int64_t i, const void* src, size_t bytes, cudaStream_t s);
  void ipc_wait_delivered(int which, int64_t i, cudaStream_t s);
  void ipc_release(char* peer, int which, int64_t i, cudaStream_t s);
  DevBuf ipc_block_;
  size_t ipc_hid_ = 0, ipc_eps_ = 0;
  char* peer_next_ = nullptr;  // rank + 1's block (my hidden sends land there)
  char* peer_prev_ = nullptr;  // rank - 1's block (I release its hidden sends)
  char* peer_eps_ = nullptr;   // rank 0 <-> rank N - 1 (eps return)
  std::vector<char*> opened_;
  bool ipc_ready_ = false;
  uint32_t ipc_epoch_ = 0;
};

__device__ __forceinline__ uint64_t tc_globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Stream-ordered wait until *addr >= v (wrap-safe). A one-warp polling kernel
// rather than cuStreamWaitValue32: a channel parked in a semaphore acquire is
// not switched out under time-slicing, so two processes sharing one GPU
// deadlock on each other's counters (observed on B200), while a polling
// kernel is preempted like any other. Traps after 20 s instead of hanging.
__device__ unsigned long long g_ipc_timeouts[4];  // diagnostics: count, last addr, last wanted, last seen
__global__ void k_wait_geq(const uint32_t* addr, uint32_t v, int soft) {
  if (threadIdx.x != 0) return;
  const uint64_t t0 = tc_globaltimer();
  for (;;) {
    uint32_t cur;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(cur) : "l"(addr) : "memory");
    if (static_cast<int32_t>(cur - v) >= 0) break;
    __nanosleep(256);
    if (tc_globaltimer() - t0 > (soft ? 3000000000ULL : 20000000000ULL)) {
      if (!soft) __trap();
      atomicAdd(&g_ipc_timeouts[0], 1ULL);
      g_ipc_timeouts[1] = reinterpret_cast<unsigned long long>(addr);
      g_ipc_timeouts[2] = v;
      g_ipc_timeouts[3] = cur;
      break;
    }
  }
}
static const bool g_ipc_soft = std::getenv("BP_IPC_SOFT") != nullptr;
// BP_IPC_FUSED_SEND=0: send hidden states with a peer copy after the forward
// instead of from the last GEMM's epilogue (A/B and tests)
static const bool g_ipc_fused = [] {
  const char* e = std::getenv("BP_IPC_FUSED_SEND");
  return !(e && e[0] == '0');
}();
void stream_wait_geq(cudaStream_t s, const uint32_t* addr, uint32_t v) {
  k_wait_geq<<<1, 32, 0, s>>>(addr, v, g_ipc_soft ? 1 : 0);
  BP_CUDA(cudaGetLastError());
}
// Stream-ordered release store of a counter (possibly in a peer process's
// memory): everything the stream did before is visible before the value.
__global__ void k_write_release(uint32_t* addr, uint32_t v) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
  }
}
void stream_write(cudaStream_t s, uint32_t* addr, uint32_t v) {
  k_write_release<<<1, 32, 0, s>>>(addr, v);
  BP_CUDA(cudaGetLastError());
}

extern std::atomic<int64_t> g_launches;

Pipeline::Pipeline(const bp_pipeline_desc& d, int rank, int world, int device, const uint8_t* ids)
    : sched(build_schedule(d)), d_(d), rank_(rank), world_(world), device_(device) {
  const int N = d.devices;
  if (d.transport == BP_TRANSPORT_NCCL || d.transport == BP_TRANSPORT_IPC) {
    if (world != N) fail(BP_ERR_CONFIG, "multi-process transports need world == devices (one stage per process)");
    if (rank < 0 || rank >= world) fail(BP_ERR_CONFIG, "bad rank");
    if (d.transport == BP_TRANSPORT_NCCL && N > 1 && ids == nullptr) fail(BP_ERR_CONFIG, "NCCL transport needs unique ids");
  } else {
    if (world != 1 || rank != 0) fail(BP_ERR_CONFIG, "loopback runs as a single process");
  }
  BP_CUDA(cudaSetDevice(device_));
  BP_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  tpf_ = static_cast<int64_t>(d.model.height) * d.model.width;
  C_ = d.model.channels;
  hwc_ = tpf_ * C_;
  stages_.resize(static_cast<size_t>(N));
  for (int j = 0; j < N; ++j) {
    const bool local = d.transport == BP_TRANSPORT_LOOPBACK || j == rank;
    if (!local) continue;
    stages_[static_cast<size_t>(j)] = std::make_unique<Stage>(
        device_, d.model, d.seed_model, d.seed_context, sched.begins[static_cast<size_t>(j)],
        sched.ends[static_cast<size_t>(j)], d.precision, st_);
  }
  {  // per-pass frame levels / ids (static schedule): rank 0 embeds with them; with the
     // Wan block every stage needs them (modulation, RoPE)
    std::vector<int32_t> lv;
    std::vector<int64_t> fi;
    for (const SchedPass& p : sched.passes) {
      pass_off_.push_back(static_cast<int64_t>(lv.size()));
      lv.insert(lv.end(), p.frame_levels.begin(), p.frame_levels.end());
      fi.insert(fi.end(), p.frame_ids.begin(), p.frame_ids.end());
    }
    pass_levels_.alloc(std::max<size_t>(lv.size(), 1) * 4);
    pass_ids_.alloc(std::max<size_t>(fi.size(), 1) * 8);
    BP_CUDA(cudaMemcpy(pass_levels_.p, lv.data(), lv.size() * 4, cudaMemcpyHostToDevice));
    BP_CUDA(cudaMemcpy(pass_ids_.p, fi.data(), fi.size() * 8, cudaMemcpyHostToDevice));
  }
  if (rank_ == 0) {
    const int M = d.num_b + d.num_c / 2;
    pool_.alloc(static_cast<size_t>(M) * hwc_ * 8);
    flags_.alloc(static_cast<size_t>(M) * M * 4);
    int64_t at = 0;
    for (const SchedBlock& b : sched.blocks) {
      block_off_.push_back(at);
      at += 3 * b.frames * hwc_;  // three state versions (current, previous, one older)
    }
    latents_.alloc(static_cast<size_t>(at) * 8);
    payload_.alloc(static_cast<size_t>(sched.max_tokens) * C_ * 8);
    for (int64_t id : sched.emission) {
      double* h = nullptr;
      const size_t n = static_cast<size_t>(sched.blocks[static_cast<size_t>(id - 1)].frames * hwc_);
      BP_CUDA(cudaMallocHost(&h, n * 8));
      pinned_.push_back(h);
    }
  }
  if (d.transport == BP_TRANSPORT_NCCL && N > 1) {
    // NCCL's p2p kernels (a send, a receive, rank 0's eps receive) need SMs
    // the persistent GEMMs do not hold (BP_SM_RESERVE overrides the 4)
    const char* res = std::getenv("BP_SM_RESERVE");
    set_sm_reserve(res ? std::atoi(res) : 4);
    auto id_of = [&](int k) {
      ncclUniqueId u;
      std::memcpy(&u, ids + 128 * k, sizeof(u));
      return u;
    };
    // pair (j, j+1) uses id j; the eps return (N-1 -> 0) uses id N-1.
    if (rank_ > 0) BP_NCCL(bp::nccl().CommInitRank(&comm_prev_, 2, id_of(rank_ - 1), 1));
    if (rank_ + 1 < N) BP_NCCL(bp::nccl().CommInitRank(&comm_next_, 2, id_of(rank_), 0));
    if (rank_ == N - 1) BP_NCCL(bp::nccl().CommInitRank(&comm_eps_, 2, id_of(N - 1), 0));
    if (rank_ == 0) BP_NCCL(bp::nccl().CommInitRank(&comm_eps_, 2, id_of(N - 1), 1));
    BP_CUDA(cudaStreamCreateWithFlags(&s_recv_, cudaStreamNonBlocking));
    BP_CUDA(cudaStreamCreateWithFlags(&s_send_, cudaStreamNonBlocking));
    BP_CUDA(cudaStreamCreateWithFlags(&s_eps_, cudaStreamNonBlocking));
    Stage& s = *stages_[static_cast<size_t>(rank_)];
    const size_t hid = static_cast<size_t>(sched.max_tokens) * d.model.hidden * s.act_bytes();
    const size_t eps = static_cast<size_t>(sched.max_tokens) * C_ * s.eps_bytes();
    std::vector<void*> xs, es;
    for (int k = 0; k < kRing; ++k) {
      xs.push_back(alloc_ring_buffer(hid));
      if (comm_prev_) register_buffer(comm_prev_, xs.back(), hid);  // receives land here
      if (comm_next_) register_buffer(comm_next_, xs.back(), hid);  // and are sent on from here
      if (s.is_last()) {
        es.push_back(alloc_ring_buffer(eps));
        register_buffer(comm_eps_, es.back(), eps);
      }
    }
    s.set_ring(kRing, sched.max_tokens, xs, es);
    if (rank_ == 0) {
      for (int k = 0; k < 2; ++k) {
        ebuf_[k].alloc(eps);
        register_buffer(comm_eps_, ebuf_[k].p, eps);
      }
    }
    // Connect every channel now, in an order with no cycle. NCCL connects a
    // point-to-point pair lazily at its first operation and blocks until the
    // peer takes part; the run's first operations are receives on BOTH ends
    // of the ring (rank 0 posts its eps receives before its first send, the
    // last rank posts its hidden receive before its first eps send), which
    // would wait on each other forever. Here each stage first receives from
    // its predecessor, then sends to its successor; the eps return goes last.
    DevBuf tiny;
    tiny.alloc(256);
    if (rank_ > 0) {
      BP_NCCL(bp::nccl().Recv(tiny.p, 1, ncclFloat32, 0, comm_prev_, s_recv_));
      BP_CUDA(cudaStreamSynchronize(s_recv_));
    }
    if (rank_ + 1 < N) {
      BP_NCCL(bp::nccl().Send(tiny.p, 1, ncclFloat32, 1, comm_next_, s_send_));
      BP_CUDA(cudaStreamSynchronize(s_send_));
    }
    if (rank_ == N - 1) {
      BP_NCCL(bp::nccl().Send(tiny.p, 1, ncclFloat32, 1, comm_eps_, s_send_));
      BP_CUDA(cudaStreamSynchronize(s_send_));
    }
    if (rank_ == 0) {
      BP_NCCL(bp::nccl().Recv(tiny.p, 1, ncclFloat32, 0, comm_eps_, s_eps_));
      BP_CUDA(cudaStreamSynchronize(s_eps_));
    }
  }
  if (d.transport == BP_TRANSPORT_IPC && N > 1) {
    BP_CUDA(cudaStreamCreateWithFlags(&s_recv_, cudaStreamNonBlocking));
    BP_CUDA(cudaStreamCreateWithFlags(&s_send_, cudaStreamNonBlocking));
    BP_CUDA(cudaStreamCreateWithFlags(&s_eps_, cudaStreamNonBlocking));
    Stage& s = *stages_[static_cast<size_t>(rank_)];
    auto align256 = [](size_t n) { return (n + 255) & ~static_cast<size_t>(255); };
    ipc_hid_ = align256(static_cast<size_t>(sched.max_tokens) * d.model.hidden * s.act_bytes());
    ipc_eps_ = align256(static_cast<size_t>(sched.max_tokens) * C_ * s.eps_bytes());
    ipc_block_.alloc(kRing * ipc_hid_ + 2 * ipc_eps_ + 256);
    BP_CUDA(cudaMemset(ipc_cnt(ipc_block_.as<char>(), 0), 0, 256));
    std::vector<void*> xs, es;
    for (int k = 0; k < kRing; ++k) {
      // ranks > 0 run their layers in the receive slots themselves; rank 0
      // (whose input is the embedding) keeps its own residual ring
      xs.push_back(rank_ > 0 ? static_cast<void*>(ipc_slot(ipc_block_.as<char>(), 0, k))
                             : alloc_ring_buffer(ipc_hid_));
      if (s.is_last()) es.push_back(alloc_ring_buffer(ipc_eps_));
    }
    stages_[static_cast<size_t>(rank_)]->set_ring(kRing, sched.max_tokens, xs, es);
  }
  BP_CUDA(cudaDeviceSynchronize());
}

Pipeline::~Pipeline() {
  cudaSetDevice(device_);
  if (failed_) {
    // a run failed part-way (a peer may be gone): abort the communicators
    // first, so NCCL kernels still waiting on a peer return, and never touch
    // the aborted handles again (ncclCommAbort on error)
    for (ncclComm_t* c : {&comm_prev_, &comm_next_, &comm_eps_}) {
      if (*c && bp::nccl().CommAbort) bp::nccl().CommAbort(*c);
      if (bp::nccl().CommAbort) *c = nullptr;
    }
    nccl_regs_.clear();
  }
  cudaDeviceSynchronize();
  if (d_.transport == BP_TRANSPORT_NCCL && d_.devices > 1) set_sm_reserve(0);
  for (char* q : opened_) cudaIpcCloseMemHandle(q);
  for (double* h : pinned_) cudaFreeHost(h);
  stages_.clear();  // the stages' rings may live in the buffers released below
  for (auto& r : nccl_regs_) bp::nccl().CommDeregister(r.first, r.second);
  for (void* q : nccl_mem_) bp::nccl().MemFree(q);
  own_ring_.clear();
  if (comm_prev_) bp::nccl().CommDestroy(comm_prev_);
  if (comm_next_) bp::nccl().CommDestroy(comm_next_);
  if (comm_eps_) bp::nccl().CommDestroy(comm_eps_);
  stages_.clear();
  if (s_recv_) cudaStreamDestroy(s_recv_);
  if (s_send_) cudaStreamDestroy(s_send_);
  if (s_eps_) cudaStreamDestroy(s_eps_);
  if (st_) cudaStreamDestroy(st_);
}

double* Pipeline::version_ptr(int64_t block, int version) const {
  const SchedBlock& b = sched.blocks[static_cast<size_t>(block - 1)];
  return latents_.as<double>() + block_off_[static_cast<size_t>(block - 1)] + (version % 3) * b.frames * hwc_;
}

// build_pool (noise.cpp:26-48) on the device, plus its collision check.
void Pipeline::build_pool_and_check(cudaStream_t st) {
  const int M = d_.num_b + d_.num_c / 2;
  const uint64_t tag0 = 0;
  if (host_pool) {
    BP_CUDA(cudaMemcpyAsync(pool_.p, host_pool, static_cast<size_t>(M * hwc_) * 8, cudaMemcpyHostToDevice, st));
    stats.h2d_bytes += M * hwc_ * 8;
  } else {
    launch_normal_fill(derive_seed(d_.seed_noise, &tag0, 1), M * hwc_, 1.0, pool_.as<double>(), st);
  }
  if (M > 1) {
    BP_CUDA(cudaMemsetAsync(flags_.p, 0, static_cast<size_t>(M) * M * 4, st));
    launch_pool_differs(pool_.as<double>(), M, hwc_, flags_.as<int>(), st);
    std::vector<int> f(static_cast<size_t>(M) * M);
    BP_CUDA(cudaMemcpyAsync(f.data(), flags_.p, f.size() * 4, cudaMemcpyDeviceToHost, st));
    BP_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < M; ++i)
      for (int j = i + 1; j < M; ++j)
        if (!f[static_cast<size_t>(i) * M + j]) fail(BP_ERR_CONFIG, "noise pool entries collided; change the noise seed");
  }
}

// make_block's frames: stack_entries of the pool (noise.cpp:12-22) or fresh normals.
void Pipeline::append_block(const SchedBlock& b, cudaStream_t st) {
  double* dst = version_ptr(b.id, 0);
  if (b.fresh) {
    launch_normal_fill(b.fresh_state, b.frames * hwc_, 1.0, dst, st);
    return;
  }
  // at most 4 segments per launch
  for (size_t i = 0; i < b.noise_ids.size(); i += 4) {
    GatherSegs g;
    for (size_t k = i; k < b.noise_ids.size() && k < i + 4; ++k)
      g.add(pool_.as<double>() + static_cast<int64_t>(b.noise_ids[k]) * hwc_, 1);
    launch_gather_rows(g, hwc_, dst + static_cast<int64_t>(i) * hwc_, st);
  }
}

// vcat(explicit context frames, center frames) (engine.cpp:373-383).
void Pipeline::assemble(const SchedPass& p, cudaStream_t st) {
  GatherSegs g;
  if (p.ctx != CtxSrc::None)
    g.add(version_ptr(p.ctx_block, p.ctx_version) + static_cast<int64_t>(p.ctx_first_frame) * hwc_,
          p.ctx_frames * tpf_);
  g.add(version_ptr(p.block, p.version), p.center_tokens);
  launch_gather_rows(g, C_, payload_.as<double>(), st);
}

// scheduler_step on the center rows + apply_update (engine.cpp:440-445).
void Pipeline::step(const SchedPass& p, const void* eps, cudaStream_t st) {
  const int64_t off = (p.tokens - p.center_tokens) * C_;
  const int64_t n = p.center_tokens * C_;
  double* x = version_ptr(p.block, p.version);
  double* out = version_ptr(p.block, p.version + 1);
  if (p.level < 1 || p.level > d_.steps) fail(BP_ERR_SCHEDULER, "level outside 1..T");
  if (d_.precision == BP_PREC_F64)
    launch_scheduler_step<double>(x, static_cast<const double*>(eps) + off, n, d_.steps, out, st);
  else
    launch_scheduler_step<float>(x, static_cast<const float*>(eps) + off, n, d_.steps, out, st);
  if (d_.record_trace) {
    std::vector<double> h(static_cast<size_t>(p.tokens * C_));
    if (d_.precision == BP_PREC_F64) {
      BP_CUDA(cudaMemcpyAsync(h.data(), eps, h.size() * 8, cudaMemcpyDeviceToHost, st));
      BP_CUDA(cudaStreamSynchronize(st));
    } else {
      std::vector<float> f(h.size());
      BP_CUDA(cudaMemcpyAsync(f.data(), eps, f.size() * 4, cudaMemcpyDeviceToHost, st));
      BP_CUDA(cudaStreamSynchronize(st));
      for (size_t i = 0; i < f.size(); ++i) h[i] = f[i];
    }
    trace.push_back(std::move(h));
    trace_rows.push_back(p.tokens);
  }
}

void Pipeline::emit_block(const SchedBlock& b, cudaStream_t st, bool to_host) {
  const size_t k = block_dev.size();
  const double* src = version_ptr(b.id, d_.steps);
  block_dev.push_back(src);
  block_count.push_back(b.frames * hwc_);
  if (to_host) {
    BP_CUDA(cudaMemcpyAsync(pinned_[k], src, static_cast<size_t>(b.frames * hwc_) * 8, cudaMemcpyDeviceToHost, st));
    stats.d2h_bytes += b.frames * hwc_ * 8;
  }
}

// DeviceWorker::process cache checks (engine.cpp:142-171) before the forward.
void Pipeline::before_stage(const SchedPass& p, int j, Stage& s, StageInput* in) {
  in->tokens = p.tokens;
  in->nframes = static_cast<int>(p.frame_levels.size());
  in->d_levels = pass_levels_.as<int32_t>() + pass_off_[static_cast<size_t>(p.index)];
  in->d_frame_ids = pass_ids_.as<int64_t>() + pass_off_[static_cast<size_t>(p.index)];
  in->capture_frames = p.capture_frames;
  in->mode = d_.cache_mode;
  in->record_inputs = d_.check_cache && d_.cache_mode == BP_CACHE_CACHED;
  in->use_prev = 0;
  if (p.cached_context_id >= 0 && d_.cache_mode != BP_CACHE_DISABLED) {
    if (d_.cache_mode == BP_CACHE_CACHED) {
      if (!s.cache_valid() || s.cache_block() != p.cached_context_id)
        fail(BP_ERR_CACHE, "device " + std::to_string(j) + " expected cache of block " +
                               std::to_string(p.cached_context_id));
      if (s.cache_level() != p.level + 1)
        fail(BP_ERR_CACHE, "cache level " + std::to_string(s.cache_level()) +
                               " does not precede pass level " + std::to_string(p.level));
      if (d_.check_cache) {
        if (!s.rec_valid() || s.rec_block() != s.cache_block())
          fail(BP_ERR_CACHE, "cache audit has no recording for block " + std::to_string(s.cache_block()));
        const std::string report = s.audit();
        if (!report.empty()) fail(BP_ERR_CACHE, report);
      }
      in->use_prev = 1;
    } else {
      if (!s.rec_valid() || s.rec_block() != p.cached_context_id)
        fail(BP_ERR_CACHE, "device " + std::to_string(j) + " expected recorded rows of block " +
                               std::to_string(p.cached_context_id));
      in->use_prev = 2;
    }
  }
}

void Pipeline::after_stage(const SchedPass& p, int j, Stage& s) {
  s.tag_entries(p.block, p.level);
  // fault injection: one cached V value on device 0, once (engine.cpp:185-189)
  if (fault_pending_ && j == 0 && s.cache_valid() && !p.capture_frames.empty() &&
      d_.cache_mode == BP_CACHE_CACHED) {
    s.bump_ulp(0, 1, 0);
    fault_pending_ = false;
  }
}

void Pipeline::ipc_handle(uint8_t out[64]) {
  if (!ipc()) fail(BP_ERR_CONFIG, "pipeline does not use the IPC transport");
  cudaIpcMemHandle_t h;
  BP_CUDA(cudaIpcGetMemHandle(&h, ipc_block_.p));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  std::memcpy(out, &h, 64);
}

void Pipeline::ipc_connect(const uint8_t* handles) {
  if (!ipc()) fail(BP_ERR_CONFIG, "pipeline does not use the IPC transport");
  if (ipc_ready_) fail(BP_ERR_CONFIG, "IPC transport already connected");
  BP_CUDA(cudaSetDevice(device_));
  const int N = d_.devices;
  std::vector<char*> mapped(static_cast<size_t>(N), nullptr);
  auto open = [&](int r) {
    if (r == rank_) fail(BP_ERR_INTERNAL, "IPC: a rank does not map its own block");
    if (!mapped[static_cast<size_t>(r)]) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * r, 64);
      void* q = nullptr;
      BP_CUDA(cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess));
      mapped[static_cast<size_t>(r)] = static_cast<char*>(q);
      opened_.push_back(static_cast<char*>(q));
    }
    return mapped[static_cast<size_t>(r)];
  };
  if (rank_ + 1 < N) peer_next_ = open(rank_ + 1);
  if (rank_ > 0) peer_prev_ = open(rank_ - 1);
  if (rank_ == 0) peer_eps_ = open(N - 1);
  if (rank_ == N - 1) peer_eps_ = open(0);
  ipc_ready_ = true;
}

// Diagnostic: this rank's four counters, read on a private stream (works
// while the pipeline's streams are blocked in stream waits).
void Pipeline::ipc_counters(uint32_t out[4]) {
  if (!ipc()) fail(BP_ERR_CONFIG, "pipeline does not use the IPC transport");
  cudaStream_t s;
  BP_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  BP_CUDA(cudaMemcpyAsync(out, ipc_cnt(ipc_block_.as<char>(), 0), 16, cudaMemcpyDeviceToHost, s));
  BP_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
}

// Sender side of one ring: wait until the receiver consumed pass i - 2 (its
// slot i & 1 is free), copy into the receiver's slot, publish delivery.
static const bool g_ipc_trace = std::getenv("BP_IPC_TRACE") != nullptr;
static_assert(sizeof(long long) == 8, "");
void Pipeline::ipc_send(char* peer, int which, int64_t i, const void* src, size_t bytes, cudaStream_t s) {
  if (g_ipc_trace) std::fprintf(stderr, "[rank %d] send ch%d pass %lld (%zu B)\n", rank_, which, static_cast<long long>(i), bytes);
  // the slot of pass i is free once pass i - R is released (R = kRing hidden
  // slots, 2 eps slots); the first R passes of a run wait until every pass of
  // the previous run is released (the receiver may still be finishing it)
  const uint32_t base = ipc_epoch_;
  const int64_t R = which == 0 ? kRing : 2;
  stream_wait_geq(s, ipc_cnt(ipc_block_.as<char>(), which == 0 ? 2 : 3),
                  i >= R ? base + static_cast<uint32_t>(i - R + 1) : base);
  BP_CUDA(cudaMemcpyAsync(ipc_slot(peer, which, i), src, bytes, cudaMemcpyDeviceToDevice, s));
  stream_write(s, ipc_cnt(peer, which == 0 ? 0 : 1), base + static_cast<uint32_t>(i + 1));
}
// Receiver side: pass i has landed in my slot of it.
void Pipeline::ipc_wait_delivered(int which, int64_t i, cudaStream_t s) {
  if (g_ipc_trace) std::fprintf(stderr, "[rank %d] recv ch%d pass %lld\n", rank_, which, static_cast<long long>(i));
  stream_wait_geq(s, ipc_cnt(ipc_block_.as<char>(), which == 0 ? 0 : 1), ipc_epoch_ + static_cast<uint32_t>(i + 1));
}
// Receiver side: pass i's slot has been consumed (stream-ordered after its use).
void Pipeline::ipc_release(char* peer, int which, int64_t i, cudaStream_t s) {
  stream_write(s, ipc_cnt(peer, which == 0 ? 2 : 3), ipc_epoch_ + static_cast<uint32_t>(i + 1));
}

void Pipeline::run(bp_emit_fn emit, void* user) {
  BP_CUDA(cudaSetDevice(device_));
  trace.clear();
  trace_rows.clear();
  block_dev.clear();
  block_count.clear();
  fault_pending_ = d_.fault_inject_ulp != 0;
  launches_at_start_ = g_launches.load();
  stats.h2d_bytes = stats.d2h_bytes = 0;
  for (auto& s : stages_)
    if (s) s->set_profiling(profiling);
  if (ipc() && !ipc_ready_) fail(BP_ERR_CONFIG, "IPC transport: bp_ipc_connect has not been called");
  {
    NvtxRange range("run_pipeline");
    if (multi()) {
      try {
        run_nccl(emit, user);
      } catch (...) {
        failed_ = true;  // the destructor aborts the NCCL communicators instead of destroying them
        throw;
      }
    } else {
      run_rank0_loopback(emit, user);
    }
  }
  stats.attn_ms = stats.gemm_ms = stats.cross_ms = stats.ln_ms = 0.0;
  stats.attn_launches = stats.gemm_launches = stats.cross_launches = stats.ln_launches = 0;
  for (auto& s : stages_) {
    if (!s) continue;
    double ms[4];
    int64_t n[4];
    s->prof_collect(ms, n);
    stats.attn_ms += ms[0]; stats.cross_ms += ms[1]; stats.gemm_ms += ms[2]; stats.ln_ms += ms[3];
    stats.attn_launches += n[0]; stats.cross_launches += n[1]; stats.gemm_launches += n[2];
    stats.ln_launches += n[3];
  }
  stats.passes = static_cast<int64_t>(sched.passes.size());
  stats.kernel_launches = g_launches.load() - launches_at_start_;
  stats.peak_bytes = g_dev_peak.load();
}

void Pipeline::run_rank0_loopback(bp_emit_fn emit, void* user) {
  cudaStream_t st = st_;
  auto copies = [&] {
    int64_t c = 0;
    for (auto& sp : stages_) c += sp ? sp->input_copies() : 0;
    return c;
  };
  const int64_t copies_at_start = copies();
  cudaEvent_t e0, e1;
  BP_CUDA(cudaEventCreate(&e0));
  BP_CUDA(cudaEventCreate(&e1));
  BP_CUDA(cudaEventRecord(e0, st));
  build_pool_and_check(st);
  size_t next_append = 0;
  size_t next_emit = 0;
  const int N = d_.devices;
  int64_t boundary = 0;
  for (const SchedPass& p : sched.passes) {
    while (next_append < sched.blocks.size() && sched.blocks[next_append].append_round <= p.round)
      append_block(sched.blocks[next_append++], st);
    assemble(p, st);
    const void* cur = payload_.p;
    for (int j = 0; j < N; ++j) {
      Stage& s = *stages_[static_cast<size_t>(j)];
      StageInput in;
      before_stage(p, j, s, &in);
      in.payload = cur;
      {
        char name[48];
        std::snprintf(name, sizeof name, "pass %lld stage %d", static_cast<long long>(p.index), j);
        NvtxRange range(name);
        cur = s.forward(in);
      }
      after_stage(p, j, s);
      if (j + 1 < N) boundary += p.tokens * d_.model.hidden * static_cast<int64_t>(s.act_bytes());
    }
    step(p, cur, st);
    if (p.finishes_block) {
      const SchedBlock& b = sched.blocks[static_cast<size_t>(p.block - 1)];
      emit_block(b, st, emit != nullptr);
      ++next_emit;
    }
  }
  BP_CUDA(cudaEventRecord(e1, st));
  BP_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  BP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  stats.gpu_ms = ms;
  stats.boundary_bytes = boundary;
  stats.boundary_copies = copies() - copies_at_start;
  stats.registered_buffers = 0;
  stats.fused_sends = 0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (emit) {
    for (size_t k = 0; k < sched.emission.size(); ++k) {
      const SchedBlock& b = sched.blocks[static_cast<size_t>(sched.emission[k] - 1)];
      emit(user, b.id, b.frames, pinned_[k], b.noise_ids.data(), static_cast<int32_t>(b.noise_ids.size()),
           b.frame_ids.data());
    }
  }
}

void* Pipeline::alloc_ring_buffer(size_t bytes) {
  if (d_.transport == BP_TRANSPORT_NCCL && bp::nccl().MemAlloc && bp::nccl().MemFree) {
    void* q = nullptr;
    if (bp::nccl().MemAlloc(&q, bytes) == ncclSuccess && q) {
      nccl_mem_.push_back(q);
      const int64_t now = g_dev_bytes.fetch_add(static_cast<int64_t>(bytes)) + static_cast<int64_t>(bytes);
      int64_t peak = g_dev_peak.load();
      while (now > peak && !g_dev_peak.compare_exchange_weak(peak, now)) {}
      return q;
    }
  }
  own_ring_.emplace_back();
  own_ring_.back().alloc(bytes);
  return own_ring_.back().p;
}

// Best effort: NCCL registers user buffers for zero-copy transfers where its
// transport supports it (NVLink P2P); elsewhere (e.g. the socket transport of
// the one-GPU tests) the call fails and the transfer goes through NCCL's own
// staging, with identical results.
void Pipeline::register_buffer(ncclComm_t comm, void* p, size_t bytes) {
  if (!comm || !p || d_.transport != BP_TRANSPORT_NCCL || !bp::nccl().CommRegister) return;
  if (std::find(nccl_mem_.begin(), nccl_mem_.end(), p) == nccl_mem_.end())
    return;  // only cuMem (ncclMemAlloc) buffers qualify for NVLink zero-copy
  void* h = nullptr;
  if (bp::nccl().CommRegister(comm, p, bytes, &h) == ncclSuccess && h) {
    nccl_regs_.push_back({comm, h});
    ++registered_;
  }
}

// One process per GPU. Stream layout per rank: st_ (compute), s_recv_
// (hidden state from rank-1), s_send_ (hidden state to rank+1), s_eps_
// (eps return N-1 -> 0); every cross-stream edge is an event. The local
// stage's residual stream is a kRing-slot ring (see kRing): pass i receives
// into slot i % kRing, runs its layers in place and is sent from that slot,
// so the boundary has no device-to-device copies. A slot is reused by pass
// i + kRing once pass i's send (or, on the last rank, its forward) is done.
// Rank 0 orders its compute stream by the logical slot clock so the data
// dependencies of the ideal schedule are never inverted.
void Pipeline::run_nccl(bp_emit_fn emit, void* user) {
  const int N = d_.devices;
  const int j = rank_;
  Stage& s = *stages_[static_cast<size_t>(j)];
  const int64_t P = static_cast<int64_t>(sched.passes.size());
  const size_t abytes = s.act_bytes(), ebytes = s.eps_bytes();
  const ncclDataType_t adt = abytes == 8 ? ncclFloat64 : ncclFloat32;
  const ncclDataType_t edt = ebytes == 8 ? ncclFloat64 : ncclFloat32;
  const int H = d_.model.hidden;
  const bool last = s.is_last();
  std::vector<cudaEvent_t> ev_fwd(P), ev_recv(P), ev_sent(P), ev_used(P);
  for (int64_t i = 0; i < P; ++i) {
    BP_CUDA(cudaEventCreateWithFlags(&ev_fwd[i], cudaEventDisableTiming));
    BP_CUDA(cudaEventCreateWithFlags(&ev_recv[i], cudaEventDisableTiming));
    BP_CUDA(cudaEventCreateWithFlags(&ev_sent[i], cudaEventDisableTiming));
    BP_CUDA(cudaEventCreateWithFlags(&ev_used[i], cudaEventDisableTiming));
  }
  cudaEvent_t e0, e1;
  BP_CUDA(cudaEventCreate(&e0));
  BP_CUDA(cudaEventCreate(&e1));
  BP_CUDA(cudaEventRecord(e0, st_));
  const int64_t copies_at_start = s.input_copies();
  int64_t boundary = 0, fused_sends = 0;
  const bool use_ipc = ipc();
  // the event after which pass i's ring slot may be overwritten: its send
  // (the slot holds the outgoing hidden state, or the last rank's eps), and
  // on the last rank also its forward (the x slot is not sent from there)
  auto slot_free = [&](int64_t i) { return ev_sent[i]; };

  // Fused send (IPC, bf16): the last layer's FFN-down GEMM writes x + FFN(x)
  // straight into the next rank's receive slot; the slot-free wait moves onto
  // the compute stream right before that GEMM, and the send only publishes.
  const bool fused_send = use_ipc && !last && s.fuses_send() && g_ipc_fused;
  struct SlotWait { const uint32_t* addr; uint32_t v; };
  auto forward_pass = [&](const SchedPass& p, const void* payload) {
    StageInput in;
    before_stage(p, j, s, &in);
    in.payload = payload;
    in.slot = static_cast<int>(p.index % kRing);
    const int64_t i = p.index;
    SlotWait sw{};
    if (fused_send) {
      sw.addr = ipc_cnt(ipc_block_.as<char>(), 2);
      sw.v = i >= kRing ? ipc_epoch_ + static_cast<uint32_t>(i - kRing + 1) : ipc_epoch_;
      in.out = ipc_slot(peer_next_, 0, i);
      in.before_out = [](cudaStream_t st, void* u) {
        const SlotWait* w = static_cast<const SlotWait*>(u);
        stream_wait_geq(st, w->addr, w->v);
      };
      in.before_out_user = &sw;
    }
    if (i >= kRing && (j == 0 || last)) BP_CUDA(cudaStreamWaitEvent(st_, slot_free(i - kRing), 0));
    char name[48];
    std::snprintf(name, sizeof name, "pass %lld stage %d", static_cast<long long>(i), j);
    NvtxRange range(name);
    const void* out = s.forward(in);
    after_stage(p, j, s);
    BP_CUDA(cudaEventRecord(ev_fwd[i], st_));
    return out;
  };
  // channel 0: hidden state j -> j+1; channel 1: eps N-1 -> 0
  auto send_to = [&](ncclComm_t comm, cudaStream_t ss, const SchedPass& p, const void* buf, int peer,
                     size_t count, ncclDataType_t dt) {
    BP_CUDA(cudaStreamWaitEvent(ss, ev_fwd[p.index], 0));
    if (use_ipc && fused_send && peer >= 0) {
      stream_write(ss, ipc_cnt(peer_next_, 0), ipc_epoch_ + static_cast<uint32_t>(p.index + 1));
      ++fused_sends;
    } else if (use_ipc) {
      const bool eps_ch = peer < 0;
      ipc_send(eps_ch ? peer_eps_ : peer_next_, eps_ch ? 1 : 0, p.index, buf,
               count * (dt == ncclFloat64 ? 8 : 4), ss);
    } else {
      BP_NCCL(bp::nccl().Send(buf, count, dt, peer, comm, ss));
    }
    BP_CUDA(cudaEventRecord(ev_sent[p.index], ss));
  };
  auto eps_buf = [&](int64_t i) -> void* {
    return use_ipc ? static_cast<void*>(ipc_slot(ipc_block_.as<char>(), 1, i)) : ebuf_[i & 1].p;
  };

  if (j == 0) {
    build_pool_and_check(st_);
    // stage-0 passes and eps updates merged by the logical slot clock
    const std::vector<RankOp> ops = rank_program(sched, 0);
    // eps receives are posted in pass order; receive i reuses the ring slot
    // of receive i-2, so it is posted right after STEP(i-2) is enqueued
    // (an event must be recorded before another stream can wait on it).
    auto post_eps_recv = [&](int64_t i) {
      if (i >= P) return;
      const SchedPass& p = sched.passes[static_cast<size_t>(i)];
      if (use_ipc) {
        if (i >= 2) {  // give slot i & 1 back once STEP(i - 2) has read it
          BP_CUDA(cudaStreamWaitEvent(s_eps_, ev_used[i - 2], 0));
          ipc_release(peer_eps_, 1, i - 2, s_eps_);
        }
        ipc_wait_delivered(1, i, s_eps_);
      } else {
        if (i >= 2) BP_CUDA(cudaStreamWaitEvent(s_eps_, ev_used[i - 2], 0));
        BP_NCCL(bp::nccl().Recv(ebuf_[i & 1].p, static_cast<size_t>(p.tokens) * C_, edt, 0, comm_eps_, s_eps_));
      }
      BP_CUDA(cudaEventRecord(ev_recv[i], s_eps_));
    };
    post_eps_recv(0);
    post_eps_recv(1);
    size_t next_append = 0;
    for (const RankOp& op : ops) {
      const SchedPass& p = sched.passes[static_cast<size_t>(op.pass)];
      if (op.kind == 0) {
        while (next_append < sched.blocks.size() && sched.blocks[next_append].append_round <= p.round)
          append_block(sched.blocks[next_append++], st_);
        assemble(p, st_);
        const void* out = forward_pass(p, payload_.p);
        send_to(comm_next_, s_send_, p, out, 1, static_cast<size_t>(p.tokens) * H, adt);
        boundary += p.tokens * H * static_cast<int64_t>(abytes);
      } else {
        BP_CUDA(cudaStreamWaitEvent(st_, ev_recv[p.index], 0));
        step(p, eps_buf(p.index), st_);
        BP_CUDA(cudaEventRecord(ev_used[p.index], st_));
        post_eps_recv(p.index + 2);
        if (p.finishes_block) emit_block(sched.blocks[static_cast<size_t>(p.block - 1)], st_, emit != nullptr);
      }
    }
  } else {
    // receive i lands in ring slot i % kRing once pass i - kRing left it:
    // sent on (middle ranks) or consumed by the forward (last rank, whose
    // output is the eps slot)
    auto x_free = [&](int64_t i) { return last ? ev_fwd[i] : ev_sent[i]; };
    auto post_recv = [&](int64_t i) {
      if (i >= P) return;
      const SchedPass& p = sched.passes[static_cast<size_t>(i)];
      if (use_ipc) {
        if (i >= kRing) {  // give slot i % kRing back to the sender
          BP_CUDA(cudaStreamWaitEvent(s_recv_, x_free(i - kRing), 0));
          ipc_release(peer_prev_, 0, i - kRing, s_recv_);
        }
        ipc_wait_delivered(0, i, s_recv_);
      } else {
        if (i >= kRing) BP_CUDA(cudaStreamWaitEvent(s_recv_, x_free(i - kRing), 0));
        BP_NCCL(bp::nccl().Recv(s.x_slot(static_cast<int>(i % kRing)), static_cast<size_t>(p.tokens) * H, adt, 0,
                                comm_prev_, s_recv_));
      }
      BP_CUDA(cudaEventRecord(ev_recv[i], s_recv_));
    };
    // a receive is posted once the event it waits on has been recorded: pass
    // i + kRing - 1's receive right after pass i - 1's send / forward
    for (int64_t i = 0; i < std::min<int64_t>(kRing - 1, P); ++i) post_recv(i);
    for (int64_t i = 0; i < P; ++i) {
      const SchedPass& p = sched.passes[static_cast<size_t>(i)];
      BP_CUDA(cudaStreamWaitEvent(st_, ev_recv[i], 0));
      const void* out = forward_pass(p, s.x_slot(static_cast<int>(i % kRing)));
      BP_CUDA(cudaEventRecord(ev_used[i], st_));
      if (!last) {
        send_to(comm_next_, s_send_, p, out, 1, static_cast<size_t>(p.tokens) * H, adt);
        boundary += p.tokens * H * static_cast<int64_t>(abytes);
      } else {
        send_to(comm_eps_, s_send_, p, out, use_ipc ? -1 : 1, static_cast<size_t>(p.tokens) * C_, edt);
      }
      post_recv(i + kRing - 1);
    }
  }
  if (use_ipc) {  // release the last slots so the counters line up for the next run
    if (j == 0) {
      for (int64_t i = std::max<int64_t>(0, P - 2); i < P; ++i) {
        BP_CUDA(cudaStreamWaitEvent(s_eps_, ev_used[i], 0));
        ipc_release(peer_eps_, 1, i, s_eps_);
      }
    } else {
      for (int64_t i = std::max<int64_t>(0, P - kRing); i < P; ++i) {
        BP_CUDA(cudaStreamWaitEvent(s_recv_, last ? ev_fwd[i] : ev_sent[i], 0));
        ipc_release(peer_prev_, 0, i, s_recv_);
      }
    }
  }
  BP_CUDA(cudaStreamSynchronize(s_send_));
  if (s_eps_) BP_CUDA(cudaStreamSynchronize(s_eps_));
  BP_CUDA(cudaStreamSynchronize(s_recv_));
  if (use_ipc) ipc_epoch_ += static_cast<uint32_t>(P);
  if (use_ipc && g_ipc_soft) {
    unsigned long long t[4];
    BP_CUDA(cudaMemcpyFromSymbol(t, g_ipc_timeouts, sizeof t));
    uint32_t c[4];
    BP_CUDA(cudaMemcpy(c, ipc_cnt(ipc_block_.as<char>(), 0), 16, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, "[rank %d] ipc timeouts %llu (addr off %lld want %llu seen %llu) counters %u %u %u %u epoch %u\n",
                 rank_, t[0], static_cast<long long>(t[1]) - reinterpret_cast<long long>(ipc_block_.p), t[2], t[3],
                 c[0], c[1], c[2], c[3], ipc_epoch_);
  }
  BP_CUDA(cudaEventRecord(e1, st_));
  BP_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  BP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  stats.gpu_ms = ms;
  stats.boundary_bytes = boundary;
  stats.boundary_copies = s.input_copies() - copies_at_start;
  stats.registered_buffers = registered_;
  stats.fused_sends = fused_sends;
  for (int64_t i = 0; i < P; ++i) {
    cudaEventDestroy(ev_fwd[i]); cudaEventDestroy(ev_recv[i]);
    cudaEventDestroy(ev_sent[i]); cudaEventDestroy(ev_used[i]);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (j == 0 && emit) {
    for (size_t k = 0; k < sched.emission.size(); ++k) {
      const SchedBlock& b = sched.blocks[static_cast<size_t>(sched.emission[k] - 1)];
      emit(user, b.id, b.frames, pinned_[k], b.noise_ids.data(), static_cast<int32_t>(b.noise_ids.size()),
           b.frame_ids.data());
    }
  }
}

}  // namespace bp

// ---- C-ABI -------------------------------------------------------------------------
struct bp_pipeline {
  std::unique_ptr<bp::Pipeline> p;
};

extern "C" {

bp_status bp_nccl_unique_id(uint8_t out[128]) {
  return bp::guarded([&] {
    ncclUniqueId u;
    BP_NCCL(bp::nccl().GetUniqueId(&u));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    std::memcpy(out, &u, 128);
  });
}

bp_status bp_pipeline_create(const bp_pipeline_desc* desc, int32_t rank, int32_t world, int32_t device,
                             const uint8_t* nccl_ids, bp_pipeline** out) {
  return bp::guarded([&] {
    if (!desc || !out) bp::fail(BP_ERR_CONFIG, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) bp::fail(BP_ERR_CUDA, "no CUDA device");
    auto h = std::make_unique<bp_pipeline>();
    h->p = std::make_unique<bp::Pipeline>(*desc, rank, world, device, nccl_ids);
    *out = h.release();
  });
}

}  // extern "C"

namespace {
// File rendezvous for the multi-process transports: `name` appears in `dir`
// atomically (written to a private temporary, then renamed), readers poll.
void publish_file(const std::string& dir, const std::string& name, const void* data, size_t n) {
  const std::string tmp = dir + "/." + name + ".tmp." + std::to_string(static_cast<long>(getpid()));
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) bp::fail(BP_ERR_IO, "bootstrap: cannot write " + tmp);
  const bool ok = std::fwrite(data, 1, n, f) == n;
  std::fclose(f);
  if (!ok || std::rename(tmp.c_str(), (dir + "/" + name).c_str()) != 0)
    bp::fail(BP_ERR_IO, "bootstrap: cannot publish " + dir + "/" + name);
}
void await_file(const std::string& dir, const std::string& name, void* data, size_t n, int32_t timeout_ms) {
  const std::string path = dir + "/" + name;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (f) {
      const size_t got = std::fread(data, 1, n, f);
      std::fclose(f);
      if (got == n) return;
    }
    if (std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(timeout_ms))
      bp::fail(BP_ERR_IO, "bootstrap: timed out waiting for " + path);
    std::this_thread::sleep_for(std::chrono::milliseconds(5));
  }
}
}  // namespace

extern "C" {

bp_status bp_bootstrap_nccl_ids(const char* dir, int32_t rank, int32_t world, int32_t timeout_ms,
                                uint8_t* ids_out) {
  return bp::guarded([&] {
    if (!dir || !ids_out) bp::fail(BP_ERR_CONFIG, "null argument");
    if (world < 1 || rank < 0 || rank >= world) bp::fail(BP_ERR_CONFIG, "bad rank / world");
    const size_t n = static_cast<size_t>(world) * 128;
    if (rank == 0) {
      std::vector<uint8_t> ids(n);
      for (int k = 0; k < world; ++k) {
        ncclUniqueId u;
        BP_NCCL(bp::nccl().GetUniqueId(&u));
        std::memcpy(ids.data() + 128 * k, &u, 128);
      }
      publish_file(dir, "nccl_ids", ids.data(), n);
    }
    await_file(dir, "nccl_ids", ids_out, n, timeout_ms);
  });
}

bp_status bp_bootstrap_ipc(bp_pipeline* p, const char* dir, int32_t rank, int32_t world, int32_t timeout_ms) {
  return bp::guarded([&] {
    if (!p || !dir) bp::fail(BP_ERR_CONFIG, "null argument");
    if (world < 1 || rank < 0 || rank >= world) bp::fail(BP_ERR_CONFIG, "bad rank / world");
    uint8_t mine[64];
    p->p->ipc_handle(mine);
    publish_file(dir, "ipc." + std::to_string(rank), mine, 64);
    std::vector<uint8_t> all(static_cast<size_t>(world) * 64);
    for (int r = 0; r < world; ++r) await_file(dir, "ipc." + std::to_string(r), all.data() + 64 * r, 64, timeout_ms);
    p->p->ipc_connect(all.data());
  });
}

bp_status bp_ipc_handle(bp_pipeline* p, uint8_t out[64]) {
  return bp::guarded([&] {
    if (!p || !out) bp::fail(BP_ERR_CONFIG, "null argument");
    p->p->ipc_handle(out);
  });
}

bp_status bp_ipc_counters(bp_pipeline* p, uint32_t out[4]) {
  return bp::guarded([&] { p->p->ipc_counters(out); });
}

bp_status bp_ipc_connect(bp_pipeline* p, const uint8_t* handles) {
  return bp::guarded([&] {
    if (!p || !handles) bp::fail(BP_ERR_CONFIG, "null argument");
    p->p->ipc_connect(handles);
  });
}

bp_status bp_pipeline_destroy(bp_pipeline* p) {
  return bp::guarded([&] { delete p; });
}

bp_status bp_pipeline_run(bp_pipeline* p, bp_emit_fn emit, void* user) {
  return bp::guarded([&] { p->p->run(emit, user); });
}

bp_status bp_pipeline_get_stats(bp_pipeline* p, bp_pipeline_stats* out) {
  return bp::guarded([&] { *out = p->p->stats; });
}

bp_status bp_pipeline_set_profiling(bp_pipeline* p, int32_t on) {
  return bp::guarded([&] { p->p->profiling = on != 0; });
}

int64_t bp_pipeline_ntrace(bp_pipeline* p) { return static_cast<int64_t>(p->p->trace.size()); }

bp_status bp_pipeline_trace(bp_pipeline* p, int64_t i, int64_t* round, int64_t* block_id, int64_t* rows,
                            int64_t* cols, double* eps) {
  return bp::guarded([&] {
    if (i < 0 || i >= static_cast<int64_t>(p->p->trace.size())) bp::fail(BP_ERR_DIMENSION, "trace index");
    const bp::SchedPass& ps = p->p->sched.passes[static_cast<size_t>(i)];
    *round = ps.round;
    *block_id = ps.block;
    *rows = p->p->trace_rows[static_cast<size_t>(i)];
    *cols = p->p->sched.desc.model.channels;
    if (eps) std::memcpy(eps, p->p->trace[static_cast<size_t>(i)].data(), p->p->trace[static_cast<size_t>(i)].size() * 8);
  });
}

bp_status bp_pipeline_set_pool(bp_pipeline* p, const double* host_pool, int64_t count) {
  return bp::guarded([&] {
    if (!p) bp::fail(BP_ERR_CONFIG, "null pipeline");
    const bp_pipeline_desc& d = p->p->sched.desc;
    const int64_t want = static_cast<int64_t>(d.num_b + d.num_c / 2) * d.model.height * d.model.width *
                         d.model.channels;
    if (host_pool && count != want)
      bp::fail(BP_ERR_DIMENSION, "pool holds " + std::to_string(count) + " values, the queue needs " +
                                     std::to_string(want) + " (M = num_b + num_c/2 entries)");
    p->p->host_pool = host_pool;
  });
}

bp_status bp_host_alloc(int64_t bytes, void** out) {
  return bp::guarded([&] {
    if (!out || bytes < 0) bp::fail(BP_ERR_CONFIG, "bad host allocation request");
    BP_CUDA(cudaMallocHost(out, static_cast<size_t>(bytes > 0 ? bytes : 1)));
  });
}

bp_status bp_host_free(void* ptr) {
  return bp::guarded([&] { if (ptr) BP_CUDA(cudaFreeHost(ptr)); });
}

bp_status bp_pipeline_block(bp_pipeline* p, int64_t i, const double** dev_data, int64_t* count) {
  return bp::guarded([&] {
    if (i < 0 || i >= static_cast<int64_t>(p->p->block_dev.size())) bp::fail(BP_ERR_DIMENSION, "block index");
    *dev_data = p->p->block_dev[static_cast<size_t>(i)];
    *count = p->p->block_count[static_cast<size_t>(i)];
  });
}

}  // extern "C"
