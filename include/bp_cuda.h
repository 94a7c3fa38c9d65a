/* bp_cuda.h — C-ABI boundary of the B200-native block-wise denoising path.
 *
 * Drop-in for the reference `blockpipe` hot path (/root/reference/proj). The
 * reference has no FFI of its own; its operator API is the C++ headers, and
 * every entry point here replaces one of those functions (cited per entry).
 * The C++ mirror in include/blockpipe/ (*.hpp) and the Python mirror in
 * paper_2505_21070_b200/ both call through this header.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the boundary.
 *  - Every call returns a bp_status that maps 1:1 onto the reference's
 *    exception taxonomy (errors.hpp:11-41); bp_last_error() returns the
 *    thread-local message of the last failure on the calling thread.
 *  - Buffers are caller-owned. Arguments flagged *_is_device take device
 *    pointers; all others are host memory.
 *  - Handles are thread-affine (one host thread per stage, like one
 *    DeviceWorker thread per device in engine.cpp:280-285).
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    returns BP_ERR_CUDA. Host-only entries (schedule, seeds) work anywhere.
 */
#ifndef BP_CUDA_H_
#define BP_CUDA_H_

#include <stdint.h>

/* Only the C-ABI is exported; everything else in libbp_cuda.so is hidden. */
#if defined(__GNUC__)
#define BP_API __attribute__((visibility("default")))
#else
#define BP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.hpp:11-41) ------------------------------------ */
typedef enum {
  BP_OK = 0,
  BP_ERR_CONFIG = 1,      /* ConfigError     */
  BP_ERR_DIMENSION = 2,   /* DimensionError  */
  BP_ERR_CACHE = 3,       /* CacheError      */
  BP_ERR_SCHEDULER = 4,   /* SchedulerError  */
  BP_ERR_QUEUE = 5,       /* QueueError      */
  BP_ERR_SCHEDULING = 6,  /* SchedulingError */
  BP_ERR_PARTITION = 7,   /* PartitionError (a ConfigError) */
  BP_ERR_IO = 8,          /* IoError         */
  BP_ERR_CUDA = 9,        /* CUDA runtime / no device */
  BP_ERR_NCCL = 10,       /* NCCL transport  */
  BP_ERR_INTERNAL = 11
} bp_status;

BP_API const char* bp_last_error(void);
BP_API const char* bp_version(void);

/* ---- enums mirroring the reference ---------------------------------------- */
typedef enum { BP_ORDER_REVERSE = 0, BP_ORDER_SEQUENTIAL = 1 } bp_order; /* block_queue.hpp:13 */
typedef enum { BP_CACHE_DISABLED = 0, BP_CACHE_CACHED = 1, BP_CACHE_RECOMPUTE = 2 } bp_cache_mode; /* model.hpp:103 */
typedef enum {
  BP_INIT_COORDINATED = 0, BP_INIT_COMPLETE_SHUFFLE = 1, BP_INIT_SUBSET = 2,
  BP_INIT_FRESH = 3, BP_INIT_REPEAT = 4
} bp_init_strategy; /* noise.hpp:29-35 */
typedef enum {
  BP_PREC_F64 = 0,   /* reference-order fp64 SIMT kernels (parity mode)         */
  BP_PREC_F32 = 1,   /* fp32 verification mode (rel-L2 <= 1e-4)                  */
  BP_PREC_BF16 = 2   /* tcgen05 bf16 tensor-core path, fp32 residual (<= 2e-2)  */
} bp_precision;
/* LOOPBACK: every stage on one GPU in one process. NCCL: one process per GPU,
 * ncclSend/ncclRecv between consecutive stages. IPC: one process per GPU (or
 * several processes on one GPU), each stage writes the next stage's receive
 * ring directly through CUDA IPC memory (peer copies over NVLink between
 * GPUs) and signals through counters in the receiver's and sender's memory,
 * written and polled by one-warp stream-ordered kernels. */
typedef enum { BP_TRANSPORT_LOOPBACK = 0, BP_TRANSPORT_NCCL = 1, BP_TRANSPORT_IPC = 2 } bp_transport;

/* Block variant. REFERENCE is the reference's block (LayerNorm + ln_affine,
 * additive sinusoidal position / timestep embeddings, model.cpp:32-43,
 * 155-169, 227-336) and the only one parity is judged on. WAN is an opt-in,
 * non-parity extension: the Wan2.1 DiT block north_star names (adaLN
 * modulation from a per-frame timestep MLP, gated residuals, RMS-normalised
 * Q/K with 3D RoPE, tanh-GELU FFN, oracle/wan_oracle.py).
 * WAN supports the resident K/V cache and no cache, not the recompute route. */
typedef enum { BP_BLOCK_REFERENCE = 0, BP_BLOCK_WAN = 1 } bp_block;

/* ModelConfig (model.hpp:21-32) + the defaulted FFN width extension. */
typedef struct {
  int32_t layers, hidden, heads, channels, height, width, context_len;
  int32_t ffn;   /* 0 => 4*hidden, the reference's fixed width (model.cpp:98-99) */
  int32_t block; /* bp_block; 0 = the reference block */
} bp_model_desc;

/* PipelineConfig (engine.hpp:24-38) + QueueParams (block_queue.hpp:36-43). */
typedef struct {
  int32_t devices;                 /* N pipeline stages */
  int32_t order;                   /* bp_order */
  int32_t cache_mode;              /* bp_cache_mode */
  int32_t num_b, num_c, steps, block_num, retain_clean_context;
  int32_t strategy;                /* bp_init_strategy */
  bp_model_desc model;
  uint64_t seed_model, seed_noise, seed_context;
  int32_t fault_inject_ulp, record_trace, check_cache;
  /* extensions */
  int32_t precision;               /* bp_precision */
  int32_t transport;               /* bp_transport */
  int32_t uneven_split;            /* 1: allow L % N != 0 (contiguous, larger stages first) */
  int32_t layer_split[64];         /* explicit per-stage layer counts; all 0 => automatic */
} bp_pipeline_desc;

/* ---- rng.hpp ---------------------------------------------------------------- */
/* derive_seed (rng.cpp:51-60). Host-only. */
BP_API uint64_t bp_derive_seed(uint64_t base, const uint64_t* tags, int32_t ntags);
/* RandomSource(state).normal_tensor({n}, sigma) (rng.cpp:35-39) on the GPU,
 * bit-exact (glibc log/cos port). Writes n doubles; returns the final state. */
BP_API bp_status bp_normals(int32_t device, uint64_t state, int64_t n, double sigma, double* out,
                     int32_t out_is_device, uint64_t* final_state);

/* ---- noise.hpp -------------------------------------------------------------- */
/* build_pool (noise.cpp:26-48): M = num_b + num_c/2 entries of H*W*C normals,
 * drawn on the GPU. out holds M*H*W*C doubles (entry-major). */
BP_API bp_status bp_noise_pool(int32_t device, int32_t num_b, int32_t num_c, const int64_t frame_shape[3],
                        uint64_t noise_seed, double* out, int32_t out_is_device);

/* stack_entries (noise.cpp:12-22): out[i] = pool entry ids[i], each entry
 * frame_elems = H*W*C doubles; ids must lie in [0, pool_size). Host buffers,
 * or device buffers when io_on_device != 0. */
BP_API bp_status bp_gather_block(int32_t device, const double* pool, int32_t pool_size, int64_t frame_elems,
                                 const int32_t* ids, int32_t nids, double* out, int32_t io_on_device);

/* draw_first_block (first != 0) / draw_next_block (noise.cpp:135-178) with
 * strategy bp_init_strategy: the pool ids on the host from *rng_state (the
 * append RandomSource's state, advanced in place exactly as the reference
 * advances it), the frames on the GPU -- pool entries stacked by id, or for
 * BP_INIT_FRESH fresh normals of the same stream (bit-exact). pool holds
 * pool_size = num_b + num_c/2 entries of H*W*C doubles (build_pool's layout);
 * tail_window_ids (ntail = num_c/2 ids) is the coordinated exclusion window,
 * ignored by the baselines. out_frames needs (first ? pool_size : num_b) *
 * H*W*C doubles, out_ids as many ints; *out_frames_count / *out_nids receive
 * the frame count and the number of ids (0 for fresh). Host buffers, or
 * device buffers (pool, out_frames) when io_on_device != 0. */
BP_API bp_status bp_noise_draw(int32_t device, int32_t strategy, int32_t first, int32_t num_b, int32_t num_c,
                               const int64_t frame_shape[3], const double* pool, int32_t pool_size,
                               const int32_t* tail_window_ids, int32_t ntail, uint64_t* rng_state,
                               double* out_frames, int32_t* out_ids, int32_t* out_frames_count, int32_t* out_nids,
                               int32_t io_on_device);

/* ---- model.hpp: one pipeline stage (ModelChunk) -------------------------------- */
typedef struct bp_stage bp_stage;

/* build_chunk (model.cpp:109-128) + build_context (model.cpp:150-153): the
 * stage's weights are generated on the device from (seed_model, layer, role). */
BP_API bp_status bp_stage_create(int32_t device, const bp_model_desc* model, uint64_t seed_model,
                          uint64_t seed_context, int32_t layer_begin, int32_t layer_end,
                          int32_t precision, bp_stage** out);
BP_API bp_status bp_stage_destroy(bp_stage* stage);

/* ChunkInput (model.hpp:106-112), host fp64 payload. */
typedef struct {
  const double* payload;           /* chunk 0: [rows=tokens, cols=C]; else [tokens, h] */
  int64_t rows, cols;
  const int32_t* frame_levels;     /* nframes */
  const int64_t* frame_ids;        /* nframes */
  int32_t nframes;
  const int32_t* capture_frames;   /* ncapture frame positions to snapshot */
  int32_t ncapture;
  int32_t record_inputs;
  int32_t mode;                    /* bp_cache_mode */
  int32_t use_prev;                /* 0: no prefix; 1: the stage's resident captured
                                      K/V (KVCacheEntry); 2: its recorded inputs;
                                      3: host K/V below; 4: host recorded inputs below */
  /* use_prev 3: a host KVCacheEntry, per local layer [prefix_rows, h] K then V,
   * layer-major (prefix_k[l*rows*h ...]). use_prev 4: a host RecomputeEntry,
   * per local layer [prefix_rows, h] layer inputs in prefix_k. */
  const double* prefix_k;
  const double* prefix_v;
  int64_t prefix_rows;
} bp_chunk_in;

/* ChunkOutput (model.hpp:114-118). payload is a caller buffer of
 * payload_capacity doubles; rows/cols/captured/recorded are filled in. */
typedef struct {
  double* payload;
  int64_t payload_capacity;
  int64_t rows, cols;
  int32_t captured, recorded;
  int64_t captured_tokens;
} bp_chunk_out;

/* forward_chunk (model.cpp:227-336). The captured K/V / recorded inputs stay
 * resident on the device and replace the stage's previous entry, like
 * DeviceWorker::cache_ (engine.cpp:195-196). */
BP_API bp_status bp_forward_chunk(bp_stage* stage, const bp_chunk_in* in, bp_chunk_out* out);
/* Downloads the resident captured K (which=0) or V (which=1) rows of one local
 * layer as fp64 [rows, h]; out may be NULL to query rows. */
BP_API bp_status bp_stage_cache_rows(bp_stage* stage, int32_t layer, int32_t which, double* out,
                              int64_t* rows);
/* Downloads the resident recorded layer inputs of one local layer as fp64
 * [rows, h] (RecomputeEntry::layer_inputs); out may be NULL to query rows. */
BP_API bp_status bp_stage_recorded_rows(bp_stage* stage, int32_t layer, double* out, int64_t* rows);
/* Replaces the cross-attention context [rows = context_len, cols = h] (host
 * fp64) and re-derives the hoisted context K/V (model.cpp:216-217). */
BP_API bp_status bp_stage_set_context(bp_stage* stage, const double* context, int64_t rows, int64_t cols);
/* Bumps one resident cached value by one ulp towards +inf (engine.cpp:185-189). */
BP_API bp_status bp_stage_cache_bump_ulp(bp_stage* stage, int32_t layer, int32_t which, int64_t index);
/* cache_mismatch_report (model.cpp:171-199) on the resident cache vs the
 * resident recording; report gets "" when they agree bitwise. */
BP_API bp_status bp_stage_cache_audit(bp_stage* stage, char* report, int32_t report_len);

/* scheduler_step (model.cpp:338-345): out = x - eps*(1/steps), n doubles, host. */
BP_API bp_status bp_scheduler_step(int32_t device, const double* x, const double* eps, int64_t n,
                            int32_t level, int32_t steps, double* out);

/* ---- tensor.hpp primitives on the GPU (fp64, host buffers, row-major) ---------- */
/* matmul (tensor.cpp:84-109): out[m,n] = a[m,k] @ b[k,n]; ascending-k accumulation. */
BP_API bp_status bp_matmul(int32_t device, const double* a, const double* b, int64_t m, int64_t k, int64_t n,
                           double* out);
/* add / sub / scale (tensor.cpp:148-172) over n doubles: op 0 out = a + b,
 * op 1 out = a - b, op 2 out = a * s (b unused). One IEEE operation per
 * element, bitwise the reference's. */
BP_API bp_status bp_elementwise(int32_t device, int32_t op, const double* a, const double* b, int64_t n, double s,
                                double* out);
/* softmax_rows (tensor.cpp:111-126) over [rows, cols]. */
BP_API bp_status bp_softmax_rows(int32_t device, const double* x, int64_t rows, int64_t cols, double* out);
/* layer_norm (tensor.cpp:128-146), no affine, over [rows, cols]. */
BP_API bp_status bp_layer_norm(int32_t device, const double* x, int64_t rows, int64_t cols, double eps,
                               double* out);

/* ---- engine.hpp: static schedule (host-only; no GPU needed) -------------------- */
typedef struct bp_schedule bp_schedule;
/* Builds the data-independent schedule of run_pipeline (engine.cpp:255-497):
 * queue states, pass order, noise ids, logical slots, ledger. */
BP_API bp_status bp_schedule_create(const bp_pipeline_desc* desc, bp_schedule** out);
BP_API void bp_schedule_destroy(bp_schedule* s);
BP_API int64_t bp_schedule_rounds(const bp_schedule* s);
BP_API int64_t bp_schedule_npasses(const bp_schedule* s);
/* ScheduleEvent list (engine.hpp:46-58) sorted by (slot, device):
 * 6 int64 per event: slot, device, block_id, level, phase, round. */
BP_API int64_t bp_schedule_nevents(const bp_schedule* s);
BP_API void bp_schedule_events(const bp_schedule* s, int64_t* out);
/* TransferLedger (engine.hpp:62-71): channel name (<=31 chars), round, passes, scalars. */
BP_API int64_t bp_schedule_nledger(const bp_schedule* s);
BP_API void bp_schedule_ledger(const bp_schedule* s, int64_t i, char* channel, int64_t* round,
                        int64_t* passes, int64_t* scalars);
/* QueueSnapshot per round (engine.hpp:90-94); returns the block count. */
BP_API int64_t bp_schedule_nsnapshots(const bp_schedule* s);
BP_API int32_t bp_schedule_snapshot(const bp_schedule* s, int64_t i, int64_t* round, int64_t* ids,
                             int32_t* levels);
/* Emitted blocks in emission order: id, frame count, noise ids (<= frames). */
BP_API int64_t bp_schedule_nblocks(const bp_schedule* s);
BP_API int32_t bp_schedule_block(const bp_schedule* s, int64_t i, int64_t* block_id, int64_t* frames,
                          int32_t* noise_ids, int64_t* frame_ids);
/* One rank's ordered program for the NCCL pipeline (2 int64 per op: kind,
 * pass): kind 0 = stage forward (+ send downstream), kind 1 = rank 0's eps
 * receive + Euler update. Returns the op count; out may be NULL. */
BP_API int64_t bp_schedule_rank_program(const bp_schedule* s, int32_t rank, int64_t* out, int64_t cap);
/* Pass record i (issue order), 20 int64: round, block, level, version, ctx
 * source (0 none, 1 in-queue, 2 retained), ctx block, ctx frames, ctx version,
 * ctx first frame, centre frames, tokens, centre tokens, cached-context id (-1),
 * capture count, earliest slot, slot on device 0, completion slot,
 * finishes-block, phase, frame count; plus per-frame levels / ids and the
 * capture frame positions. Returns the frame count. */
BP_API int32_t bp_schedule_pass(const bp_schedule* s, int64_t i, int64_t* rec, int32_t* levels, int64_t* frame_ids,
                         int32_t* capture);
/* Block meta by id: frames, append round, fresh (0/1), fresh RNG state bits. */
BP_API void bp_schedule_block_meta(const bp_schedule* s, int64_t block_id, int64_t* rec4);
/* Stage layer ranges actually used: begins[N], ends[N]. */
BP_API void bp_schedule_partition(const bp_schedule* s, int32_t* begins, int32_t* ends);

/* ---- engine.hpp: the pipeline ------------------------------------------------ */
typedef struct bp_pipeline bp_pipeline;

/* NCCL unique id for the transport (128 bytes). */
BP_API bp_status bp_nccl_unique_id(uint8_t out[128]);
/* Loopback: rank=0, world=1, all N stages on `device`, nccl_ids NULL.
 * NCCL: one process per GPU, rank j owns stage j, world = N; nccl_ids holds
 * N unique ids made by rank 0 and shared by the caller (128 bytes each). */
BP_API bp_status bp_pipeline_create(const bp_pipeline_desc* desc, int32_t rank, int32_t world,
                             int32_t device, const uint8_t* nccl_ids, bp_pipeline** out);
BP_API bp_status bp_pipeline_destroy(bp_pipeline* p);
/* File rendezvous for the multi-process transports, no MPI / PyTorch needed:
 * every rank passes the same fresh directory (on a filesystem all ranks
 * see). bp_bootstrap_nccl_ids: rank 0 creates the `world` NCCL unique ids
 * (ncclGetUniqueId) and publishes them; every rank receives them in ids_out
 * (world x 128 bytes) for bp_pipeline_create. bp_bootstrap_ipc: publishes
 * this rank's IPC handle, waits for every rank's and connects (the
 * bp_ipc_handle + bp_ipc_connect exchange). Both block up to timeout_ms and
 * fail with BP_ERR_IO. */
BP_API bp_status bp_bootstrap_nccl_ids(const char* dir, int32_t rank, int32_t world, int32_t timeout_ms,
                                       uint8_t* ids_out);
BP_API bp_status bp_bootstrap_ipc(bp_pipeline* p, const char* dir, int32_t rank, int32_t world, int32_t timeout_ms);
/* IPC transport handshake: each rank exports the handle of its receive block
 * (64 bytes), the caller all-gathers them in rank order, then every rank
 * connects before its first run. */
BP_API bp_status bp_ipc_handle(bp_pipeline* p, uint8_t out[64]);
BP_API bp_status bp_ipc_connect(bp_pipeline* p, const uint8_t* handles /* world x 64 bytes */);
/* Diagnostic: this rank's ring counters (delivered hidden, delivered eps,
 * consumed hidden-out, consumed eps-out). */
BP_API bp_status bp_ipc_counters(bp_pipeline* p, uint32_t out[4]);

/* EmittedBlock (engine.hpp:73-78) callback, rank 0 only, emission order. */
typedef void (*bp_emit_fn)(void* user, int64_t block_id, int64_t frames, const double* data,
                           const int32_t* noise_ids, int32_t nids, const int64_t* frame_ids);

/* run_pipeline (engine.cpp:255-497): one whole generation. emit may be NULL:
 * the emitted latents then stay on the device (no device->host copies;
 * bp_pipeline_block returns their device pointers). */
BP_API bp_status bp_pipeline_run(bp_pipeline* p, bp_emit_fn emit, void* user);

typedef struct {
  double gpu_ms;            /* device time of the last run (CUDA events) */
  int64_t passes;
  int64_t kernel_launches;  /* our kernels launched by the last run */
  int64_t peak_bytes;       /* device memory high-water mark of this pipeline */
  int64_t boundary_bytes;   /* bytes moved across stage boundaries */
  double attn_ms, gemm_ms;  /* per-class device time when profiling is enabled */
  double cross_ms;          /* cross-attention device time (profiling)             */
  int64_t attn_launches, gemm_launches, cross_launches;
  double ln_ms;             /* LayerNorm device time (profiling)                   */
  int64_t ln_launches;
  int64_t h2d_bytes;        /* host->device bytes of the last run (host-supplied pool) */
  int64_t d2h_bytes;        /* device->host bytes of the last run (emitted latents)   */
  int64_t boundary_copies;  /* device copies of hidden states at stage boundaries in the last
                               run (0 for the multi-process transports: received in place) */
  int64_t registered_buffers; /* stage-boundary buffers NCCL accepted for registration */
  int64_t fused_sends;      /* hidden states this rank wrote into the next rank's receive slot
                               from the last layer's residual GEMM epilogue (IPC, bf16) */
} bp_pipeline_stats;
BP_API bp_status bp_pipeline_get_stats(bp_pipeline* p, bp_pipeline_stats* out);
/* Per-kernel-class timing with CUDA events on the launching stream (0/1). */
BP_API bp_status bp_pipeline_set_profiling(bp_pipeline* p, int32_t on);
/* TraceRecord (engine.hpp:83-87) of pass i when record_trace is set. */
BP_API int64_t bp_pipeline_ntrace(bp_pipeline* p);
BP_API bp_status bp_pipeline_trace(bp_pipeline* p, int64_t i, int64_t* round, int64_t* block_id,
                            int64_t* rows, int64_t* cols, double* eps /* may be NULL */);
/* Host-supplied noise pool: replaces build_pool(seed_noise) (noise.cpp:26-48,
 * engine.cpp:288-290) with M = num_b + num_c/2 caller entries of
 * height*width*channels fp64 values in id order (the layout bp_noise_pool
 * writes). The buffer is borrowed: it must stay valid for every later run,
 * which uploads it host->device and applies the reference's pairwise
 * collision check. NULL restores the seeded device pool. Rank 0 only. */
BP_API bp_status bp_pipeline_set_pool(bp_pipeline* p, const double* host_pool, int64_t count);
/* Page-locked host memory for pools and emission buffers (cudaMallocHost). */
BP_API bp_status bp_host_alloc(int64_t bytes, void** out);
BP_API bp_status bp_host_free(void* p);
/* Device pointer + element count of emitted block i's latents (fp64). */
BP_API bp_status bp_pipeline_block(bp_pipeline* p, int64_t i, const double** dev_data, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* BP_CUDA_H_ */
