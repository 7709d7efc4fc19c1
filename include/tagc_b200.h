/*
 * tagc_b200.h — C-ABI of the B200-native TAGC compressed gradient-exchange
 * path (libtagc_b200.so). Plain pointers and sizes only; no torch types.
 *
 * This boundary replaces the reference's per-shard exchange
 *   tagc::tagc_reduce_shard       (reference proj/include/tagc/hook.hpp:76-80,
 *                                  proj/src/hook.cpp:98-200)
 *   tagc::baseline_reduce_shard   (hook.hpp:84-86, hook.cpp:90-96)
 * and the per-layer codec calls it is built from:
 *   tagc::sparsify / apply_accumulator        (sparsify.hpp:23-38)
 *   tagc::Index::create / merge_indices / presence (index.hpp:26,36,50)
 *   tagc::CountSketch::compress / sketch_add  (sketch.hpp:44-46,65)
 *   tagc::peeling_decompress / estimation_decompress (decode.hpp:25-32)
 * plus the host-side policy/config/model calls (config.hpp:16-35,
 * layers.hpp:35-50, hook.hpp:42-43,98-104, sketch.hpp:21-28).
 *
 * Conventions (mirroring the reference):
 *  - Status: TAGC_OK (0); TAGC_INVALID (2) wherever the reference throws
 *    std::invalid_argument; TAGC_RUNTIME (1) for any other failure (CUDA,
 *    NCCL, allocation). tagc_last_error() returns a thread-local message.
 *    The CLI mapping 0/1/2 follows reference cli.cpp:375-382.
 *  - Buffers marked "dev" are caller-owned device pointers; the accumulator
 *    is in/out and persists across steps (reference train.cpp:249-252).
 *  - Work is enqueued on the context's stream. Calls that return statistics
 *    (a non-NULL stats/tau/count out-pointer) synchronise that stream once at
 *    the end; with NULL stats pointers nothing blocks the host.
 *  - There is no CPU fallback: every compute entry point runs sm_100a CUDA
 *    kernels and fails with TAGC_RUNTIME when no device is usable.
 */
#ifndef TAGC_B200_H
#define TAGC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define TAGC_B200_ABI_VERSION 1

enum tagc_status { TAGC_OK = 0, TAGC_RUNTIME = 1, TAGC_INVALID = 2 };

/* reference config.hpp:10 */
enum tagc_policy {
  TAGC_POLICY_ALL_LAYERS = 0,
  TAGC_POLICY_NON_ATTENTION_LINEAR = 1,
  TAGC_POLICY_NONE = 2
};

/* reference layers.hpp:12-22 */
enum tagc_layer_kind {
  TAGC_KIND_EMBEDDING = 0,
  TAGC_KIND_POSITIONAL_EMBEDDING = 1,
  TAGC_KIND_ATTENTION_QKV = 2,
  TAGC_KIND_ATTENTION_OUT_PROJ = 3,
  TAGC_KIND_FEED_FORWARD = 4,
  TAGC_KIND_LM_HEAD = 5,
  TAGC_KIND_NORM = 6,
  TAGC_KIND_BIAS = 7,
  TAGC_KIND_OTHER = 8
};

/* reference CompressionConfig, config.hpp:16-35 (same fields, same defaults
 * via tagc_config_default). */
typedef struct tagc_config {
  double theta;                  /* sparsification threshold, percent */
  uint32_t ratio;                /* 1 = codec bypass, else one of {2,4,10} */
  uint32_t index_width;          /* 1 or 4 */
  int32_t policy;                /* enum tagc_policy */
  int32_t include_out_proj;      /* bool */
  uint64_t seed;                 /* hash seed, one per exchange */
  uint32_t sketch_rows;          /* k, default 3 */
  int32_t allow_low_theta;       /* bool */
  uint64_t min_compress_segment; /* default 1024 */
} tagc_config;

/* reference LayerSegment, hook.hpp:21-28 (global flat coordinates) */
typedef struct tagc_segment {
  int32_t kind; /* enum tagc_layer_kind */
  uint64_t begin, end;
  const char* name; /* ledger tag component; may be NULL ("seg<i>") */
} tagc_segment;

/* reference ShardSpec, hook.hpp:30-38 */
typedef struct tagc_shard {
  uint32_t id, owner;
  uint64_t begin, end;
  const tagc_segment* segments;
  uint32_t num_segments;
} tagc_shard;

/* reference PeelStats, hook.hpp:45-59. index_lost / index_spurious are
 * TAGC_STAT_UNAVAILABLE when a 1-bit-index split exchange (_begin / _end)
 * was not given the ranks' support blocks (tagc_reduce_shards_support). */
#define TAGC_STAT_UNAVAILABLE UINT64_MAX
typedef struct tagc_peel_stats {
  uint64_t presence, peeled, unresolved, index_lost, index_spurious, compressed_segments,
      baseline_segments;
} tagc_peel_stats;

/* reference SketchGeometry, sketch.hpp:21-28 */
typedef struct tagc_sketch_geom {
  uint32_t n, ratio, rows, buckets_per_row;
} tagc_sketch_geom;

/* reference CommVolume, hook.hpp:88-93 */
typedef struct tagc_comm_volume {
  double index_bits, sketch_bits, total_bits, factor;
} tagc_comm_volume;

/* reference LayerSpec, layers.hpp:27-31 */
typedef struct tagc_layer_spec {
  const char* name;
  int32_t kind;
  uint64_t param_count;
} tagc_layer_spec;

/* ------------------------------------------------------------ errors / misc */
const char* tagc_last_error(void);
int tagc_abi_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int tagc_device_count(void);

/* -------------------------------------------------- host policy and models */
void tagc_config_default(tagc_config* out);
/* CompressionConfig::validate_for_world (config.cpp:53-59) */
int tagc_config_validate(const tagc_config* cfg, uint32_t world_size);
/* CompressionConfig::theta_floor (config.cpp:27-35) */
int tagc_theta_floor(uint32_t ratio, double* out);
/* kind_compressible (layers.cpp:42-65): returns 0/1, or -1 for a bad enum */
int tagc_kind_compressible(int32_t kind, int32_t policy, int32_t include_out_proj);
/* sketch_geometry (sketch.cpp:11-27) */
int tagc_sketch_geometry(uint32_t n, uint32_t ratio, uint32_t rows, tagc_sketch_geom* out);
/* words_needed (index.cpp:17-20) */
uint32_t tagc_index_words(uint32_t n, uint32_t width);
/* comm_volume_model / lhc_comm_volume_model (hook.cpp:202-236); n == 0 means
 * "no explicit length" (the asymptotic 32/ratio payload). */
int tagc_comm_volume_model(const tagc_config* cfg, uint32_t world_size, uint64_t n,
                           tagc_comm_volume* out);
int tagc_lhc_comm_volume_model(const tagc_config* cfg, uint32_t world_size, uint64_t n,
                               tagc_comm_volume* out);

/* make_shards (hook.cpp:30-61). The returned set owns its segments; segment
 * names point into the set ("pad" for the alignment tail). */
typedef struct tagc_shard_set tagc_shard_set;
int tagc_make_shards(const tagc_layer_spec* layers, uint32_t n_layers, uint32_t shard_count,
                     uint32_t world_size, tagc_shard_set** out);
uint32_t tagc_shard_set_count(const tagc_shard_set* set);
/* Fills *out with shard i; pointers stay valid until tagc_shard_set_destroy. */
int tagc_shard_set_get(const tagc_shard_set* set, uint32_t i, tagc_shard* out);
void tagc_shard_set_destroy(tagc_shard_set* set);

/* ---------------------------------------------------------------- context */
typedef struct tagc_ctx tagc_ctx;
/* world_size/rank describe the caller's process in a real multi-GPU world
 * (nccl_comm = an ncclComm_t, or NULL and call tagc_ctx_init_nccl). For the
 * simulated-world entry points (suffix _sim) the context may be created with
 * world_size = 1, rank = 0; the simulated W comes from the call.
 * stream: a cudaStream_t (cudaStreamLegacy = (void*)1 for the legacy default
 * stream) or NULL for a context-owned non-blocking stream. */
int tagc_ctx_create(const tagc_config* cfg, uint32_t world_size, uint32_t rank, int device,
                    void* nccl_comm, void* cuda_stream, tagc_ctx** out);
void tagc_ctx_destroy(tagc_ctx* ctx);
/* Replace the compression config (validated against the ctx world). */
int tagc_ctx_set_config(tagc_ctx* ctx, const tagc_config* cfg);
void* tagc_ctx_stream(tagc_ctx* ctx);
/* NCCL bootstrap helpers (the 128-byte ncclUniqueId is exchanged by the
 * caller, e.g. torch.distributed.broadcast_object_list). */
int tagc_nccl_unique_id(uint8_t out[128]);
int tagc_ctx_init_nccl(tagc_ctx* ctx, const uint8_t unique_id[128]);
/* Traffic ledger as CSV in the reference's format (collectives.cpp:70-78). */
int tagc_ctx_ledger_csv(tagc_ctx* ctx, char* buf, size_t len, size_t* needed);
int tagc_ctx_ledger_reset(tagc_ctx* ctx);

/* ------------------------------------------------- traffic ledger (§8f row 3)
 * tagc::TrafficLedger (collectives.hpp:60-81, collectives.cpp:37-93): the
 * declared cost model, All-Reduce charged 2x, others 1x. A context records
 * into its own ledger (tagc_ctx_ledger, borrowed, valid while the context
 * lives) at every exchange with the reference's tags; a standalone ledger is
 * host-only. op: 0 all_reduce, 1 reduce, 2 reduce_scatter, 3 all_gather.
 * _csv / _json write the reference's to_csv / to_json().dump() text (NUL
 * terminated, truncated to len; *needed = full size + 1). */
typedef struct tagc_ledger tagc_ledger;
tagc_ledger* tagc_ledger_create(void);
void tagc_ledger_destroy(tagc_ledger* l);
int tagc_ledger_record(tagc_ledger* l, int32_t op, const char* tag, uint64_t payload_bits, uint64_t params);
int tagc_ledger_csv(tagc_ledger* l, char* buf, size_t len, size_t* needed);
int tagc_ledger_json(tagc_ledger* l, char* buf, size_t len, size_t* needed);
/* bits_per_param_per_rank over the rows whose tag starts with prefix
 * (collectives.cpp:60-68); prefix NULL or "" = all rows. */
int tagc_ledger_bits_per_param(tagc_ledger* l, const char* prefix, double* out);
int tagc_ledger_clear(tagc_ledger* l);
/* TrafficLedger::rows() (collectives.hpp:67, ordered by (op, tag)): the row
 * count, and row i's fields (tag NUL-terminated, truncated to tag_len; any
 * output pointer may be NULL). A reference-side adapter replays a call's rows
 * into the reference World's ledger with these. */
int tagc_ledger_row_count(tagc_ledger* l, uint32_t* out);
int tagc_ledger_row(tagc_ledger* l, uint32_t i, int32_t* op, char* tag, size_t tag_len, uint64_t* calls,
                    uint64_t* payload_bits, uint64_t* charged_bits, uint64_t* params);
tagc_ledger* tagc_ctx_ledger(tagc_ctx* ctx);
/* Bytes this context actually handed to the transport (NCCL or peer pulls)
 * since creation: measured, beside the ledger's modelled bits. */
int tagc_ctx_wire_bytes(tagc_ctx* ctx, uint64_t* out);
/* Index::to_bytes / CountSketch::to_bytes (index.cpp:59-69, sketch.cpp:77-89):
 * the wire format is the little-endian u32 / f32 word layout the device
 * buffers already hold (index words, sketch rows, and the send / receive
 * blocks of tagc_plan_exchange), so this is a stream-ordered copy of n_words
 * words to host_out (4 * n_words bytes). */
int tagc_wire_bytes_from_device(tagc_ctx* ctx, const void* dev, uint64_t n_words, uint8_t* host_out);
/* Device bytes the context currently holds in workspaces. */
uint64_t tagc_ctx_workspace_bytes(const tagc_ctx* ctx);
/* Optional per-stage device timing of the last fused call (ms): prep
 * (descriptor uploads, sketch zeroing), the sampled select + fused
 * split/encode pass, select finish (exact tau, fix-up), exchange, decode.
 * Enabled by tagc_ctx_set_timing(ctx, 1). */
int tagc_ctx_set_timing(tagc_ctx* ctx, int enabled);
int tagc_ctx_last_timing(tagc_ctx* ctx, float out_ms[5]);
/* Timing mode: device execution spans (ms) of the last fused call's two
 * dominant kernel chains, stamped by the kernels themselves (%globaltimer):
 * out_ms[0] = the fused select/split/encode pass (k_fused start to end),
 * out_ms[1] = decode (k_count start to k_final end). */
int tagc_ctx_last_kernel_spans(tagc_ctx* ctx, float out_ms[2]);
/* CUDA-graph replay of tagc_reduce_shards / _host (default on; the
 * environment variable TAGC_GRAPHS=0 turns it off): a call whose shard
 * layout, config and buffer pointers repeat is captured on its second
 * occurrence and replayed with one graph launch afterwards. Calls with stats,
 * timing mode, or a 1-bit index over several ranks always run eagerly. */
int tagc_ctx_set_graphs(tagc_ctx* ctx, int enabled);
/* Kernel launches enqueued by the last fused call. */
uint64_t tagc_ctx_last_launches(const tagc_ctx* ctx);
/* Synchronise the context stream and surface deferred device errors (a NaN
 * input found by an asynchronous call without stats returns TAGC_INVALID). */
int tagc_ctx_sync(tagc_ctx* ctx);
/* Peel rounds of the last fused call that returned stats:
 * out[0] = grid-wide rounds, out[1] = single-CTA tail rounds. */
int tagc_ctx_last_peel_rounds(tagc_ctx* ctx, uint32_t out[2]);

/* -------------------------------------------- fused exchange: simulated world
 * tagc_reduce_shard (hook.cpp:98-200) with W logical ranks on this GPU.
 * grads[r], accs[r]: dev, shard.size() floats each (accs mutated for
 * compressed segments only); out: dev, shard.size() floats (the owner's
 * decoded shard). stats may be NULL. */
int tagc_reduce_shard_sim(tagc_ctx* ctx, const tagc_shard* shard, uint32_t world,
                          const float* const* grads, float* const* accs, float* out,
                          tagc_peel_stats* stats);
/* tagc_reduce_shard(..., collect_audit = true) (hook.cpp:98-200): as
 * tagc_reduce_shard_sim, plus audit (dev, shard.size() floats) =
 * ShardReduceResult::audit_exchanged_sum (hook.hpp:61-68, hook.cpp:191-195):
 * the ascending-rank sum of the exchanged (post-sparsify) vectors over
 * compressed segments, zeros over raw segments. */
int tagc_reduce_shard_sim_audit(tagc_ctx* ctx, const tagc_shard* shard, uint32_t world,
                                const float* const* grads, float* const* accs, float* out,
                                tagc_peel_stats* stats, float* audit);
/* baseline_reduce_shard (hook.cpp:90-96): ascending-rank fp32 sum. */
int tagc_baseline_reduce_shard_sim(tagc_ctx* ctx, const tagc_shard* shard, uint32_t world,
                                   const float* const* grads, float* out);

/* ---------------------------------------------- fused exchange: NCCL world
 * One process per GPU. grad/acc: dev, this rank's flat buffers covering every
 * shard (shards[i].begin .. end index into them). out: dev, the concatenation
 * (in shard order) of the shards this rank owns. The index and sketch (and
 * raw segments) of all shards are exchanged in one grouped NCCL
 * reduce-scatter. stats (may be NULL) covers this rank's owned shards. */
int tagc_reduce_shards(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                       const float* grad, float* acc, float* out, tagc_peel_stats* stats);
/* Single-shard form of the above (reference tagc_reduce_shard call shape);
 * out is written on the owner rank only. */
int tagc_reduce_shard(tagc_ctx* ctx, const tagc_shard* shard, const float* grad, float* acc,
                      float* out, tagc_peel_stats* stats);
/* Host-buffer form of tagc_reduce_shards: the call a user makes when the
 * gradient lives in host memory (the reference's tagc_reduce_shard takes host
 * std::vector<float> slices, hook.hpp:76-80). host_grad: host, max(shard.end)
 * floats; acc: dev (engine-side error-feedback state, in/out); host_out: host,
 * the owned shards' decoded values (as `out` above). Page-locked host buffers
 * give full overlap: the gradient is copied in on one copy stream into one of
 * two device buffers and the result copied out on another, so consecutive
 * calls overlap D2H(k), H2D(k+1) and the exchange. The call is asynchronous
 * unless stats != NULL; host_out is complete after tagc_ctx_sync, or on the
 * context stream after tagc_ctx_host_join. */
int tagc_reduce_shards_host(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                            const float* host_grad, float* acc, float* host_out,
                            tagc_peel_stats* stats);
/* Make the context stream wait for every copy tagc_reduce_shards_host has
 * enqueued (a CUDA event recorded on the context stream afterwards brackets
 * the host copies too). */
int tagc_ctx_host_join(tagc_ctx* ctx);
/* The exchange split around its collective, for a caller-provided transport
 * (the reference's in-process World, MPI, a test harness): _begin encodes
 * every shard into this rank's owner-major send blocks and returns them
 * (dev: world_size * block_f32 floats, world_size * block_u32 u32 words; the
 * layout of tagc_plan_exchange). The caller reduce-scatters them - owner o
 * receives the fp32 sum and the wrapping u32 sum of every rank's block o
 * (reference World::reduce / all_reduce_sum, collectives.cpp:143-166) - and
 * passes this rank's reduced blocks to _end, which decodes the owned shards
 * into `out` (given to _begin). Works for any world size without NCCL.
 * *send_f32 / *send_u32 non-NULL on input: encode straight into those
 * caller-owned buffers (sizes from tagc_plan_exchange), e.g. registered or
 * symmetric memory of the transport; NULL: engine workspace, returned. */
int tagc_reduce_shards_begin(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                             const float* grad, float* acc, float* out, float** send_f32,
                             uint32_t** send_u32, uint64_t* block_f32, uint64_t* block_u32);
/* 1-bit index only (index_lost / index_spurious, hook.cpp:176-188): after
 * _begin, this rank's index support as one byte (0/1) per position in
 * owner-major blocks of *block_bytes = 32 * block_u32 bytes (dev; into
 * *send_support when non-NULL on input, else engine workspace, returned).
 * The caller max-reduce-scatters them (max of 0/1 bytes = OR) and passes its
 * reduced block to _end_support. */
int tagc_reduce_shards_support(tagc_ctx* ctx, uint8_t** send_support, uint64_t* block_bytes);
int tagc_reduce_shards_end_support(tagc_ctx* ctx, const float* recv_f32, const uint32_t* recv_u32,
                                   const uint8_t* recv_support, tagc_peel_stats* stats);
/* tagc_reduce_shards with collect_audit = true: audit (dev, laid out like
 * out) = audit_exchanged_sum of the owned shards (hook.cpp:191-195), zeros
 * over raw segments. NCCL world or world_size 1 (a peer-exchange context
 * returns TAGC_INVALID). Diagnostic: one extra fp32 reduce-scatter of the
 * sparse vectors, and the call synchronises. */
int tagc_reduce_shards_audit(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards, const float* grad,
                             float* acc, float* out, tagc_peel_stats* stats, float* audit);
int tagc_reduce_shards_end(tagc_ctx* ctx, const float* recv_f32, const uint32_t* recv_u32,
                           tagc_peel_stats* stats);
/* Pull-mode exchange over peer memory (NVLink / NVSwitch) instead of NCCL.
 * Each rank encodes into its own owner-major send blocks inside a region its
 * peers map through CUDA IPC, raises a step flag in every peer, and reduces
 * its own block straight out of the W regions: fp32 sums in ascending rank
 * order (the reference World's fold, collectives.cpp:127-166, so the reduced
 * sketch and raw segments are bit-identical to it) and wrapping u32 sums of
 * the index words. Deterministic, no NCCL. Setup, after the shard layout is
 * known:
 *   tagc_ctx_peer_prepare  allocates this rank's region, returns its handle;
 *   (the caller all-gathers the world_size handles)
 *   tagc_ctx_peer_open     maps the peers' regions (handles: world_size x
 *                          TAGC_PEER_HANDLE_BYTES, rank order).
 * tagc_ctx_peer_attach_local does the same for contexts of one process (all
 * ranks on one GPU, tests). Afterwards tagc_reduce_shards(_host) uses the
 * peers; a rank that never signals makes the step fail with TAGC_RUNTIME
 * after TAGC_PEER_TIMEOUT_MS (default 20000) instead of hanging. */
#define TAGC_PEER_HANDLE_BYTES 64
int tagc_ctx_peer_prepare(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                          uint8_t handle[TAGC_PEER_HANDLE_BYTES]);
int tagc_ctx_peer_open(tagc_ctx* ctx, const uint8_t* handles);
int tagc_ctx_peer_attach_local(tagc_ctx* ctx, tagc_ctx* const* ranks, uint32_t n_ranks);
/* The owner-major exchange layout tagc_reduce_shards uses on `rank` (pure
 * host computation; exposed so a foreign transport can reproduce the
 * exchange). Owner o's f32 block is [o*block_f32, (o+1)*block_f32) of the
 * send buffer: compressed-segment sketches at sk_off, raw segments at raw_off;
 * its u32 block [o*block_u32, ...) holds index words at word_off. `out` may be
 * NULL to query *n_out (one entry per segment, shard order). */
typedef struct tagc_seg_plan {
  uint32_t shard, seg, compressed, buckets_per_row, n_words, owner;
  uint64_t lo, len, word_off, sk_off, raw_off, out_off;
} tagc_seg_plan;
int tagc_plan_exchange(const tagc_config* cfg, const tagc_shard* shards, uint32_t n_shards,
                       uint32_t world_size, uint32_t rank, tagc_seg_plan* out, uint32_t* n_out,
                       uint64_t* block_f32, uint64_t* block_u32);
/* Uncompressed comparator: ncclReduceScatter fp32 of the shards (requires
 * n_shards == world_size with shard i owned by rank i, as make_shards(W, W)
 * gives). out: dev, shard size floats. */
int tagc_baseline_reduce_shards(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                                const float* grad, float* out);

/* ------------------------------------- backward / exchange overlap (§8f)
 * tagc_reduce_shards split along the gradient's production (paper §3.3): the
 * exchange is opened before the gradient exists, every segment is sparsified
 * and encoded as soon as the flat range [begin, end) holding it is ready, and
 * the collective + decode run at finish. cuda_event (a cudaEvent_t recorded on
 * the producer's stream after it wrote the range, may be NULL) is waited on by
 * the context's stream, so encoding overlaps the rest of the backward pass.
 * A segment is encoded by the first ready call whose range contains it;
 * finish encodes whatever no call covered. grad must stay valid and unwritten
 * until finish has been enqueued (its reads end there). Results are those of
 * tagc_reduce_shards on the same inputs. */
int tagc_overlap_begin(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards, const float* grad, float* acc,
                       float* out);
int tagc_overlap_ready(tagc_ctx* ctx, uint64_t begin, uint64_t end, void* cuda_event);
int tagc_overlap_finish(tagc_ctx* ctx, tagc_peel_stats* stats);

/* ------------------------------------------- owner-side consumer (§8f)
 * The step after the exchange in the reference's training loop
 * (train.cpp:355-364): the owner takes the mean over ranks of its decoded
 * shard and updates its parameter slice, then every rank re-gathers the
 * padded flat parameter space.
 * tagc_apply_optimizer: decoded (dev, len, the summed shard; the mean
 * g = decoded * (1/world) of train.cpp:356-357 is formed on the fly and not
 * written back), params (dev, len, in/out), adam_v (dev, len,
 * in/out, zero before step 1; NULL for sgd). kind 0 = sgd (scale_sub_inplace,
 * kernels.cpp:32-41), 1 = adamw_nm (apply_optimizer, train.cpp:202-220; step
 * >= 1). Bit-identical to the reference's fp32 loop. */
int tagc_apply_optimizer(tagc_ctx* ctx, int32_t kind, double lr, double weight_decay, uint32_t world,
                         uint32_t step, float* params, const float* decoded, float* adam_v, uint64_t len);
/* tagc_reduce_shards followed by the owner's step, fused: the mean and the
 * optimizer update run inside the kernels that produce the decoded values
 * (the decode's dense emit and the owned raw segments' unpack), so the
 * decoded shard is not written and re-read. params / adam_v (dev) are laid
 * out like tagc_reduce_shards' out (the owned shards, concatenated); out may
 * be NULL (decoded values not stored) or a buffer that receives them too.
 * Bit-identical to tagc_reduce_shards + tagc_apply_optimizer(world = the
 * context's world size). */
int tagc_reduce_shards_step(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards, const float* grad,
                            float* acc, float* out, int32_t kind, double lr, double weight_decay, uint32_t step,
                            float* params, float* adam_v, tagc_peel_stats* stats);
/* World::all_gather of the owner slices (collectives.cpp:197-212, call site
 * train.cpp:364): params dev, padded = world * L floats; this rank's slice
 * [rank*L, (rank+1)*L) is gathered in place into every rank's buffer (NCCL). */
int tagc_allgather_params(tagc_ctx* ctx, float* params, uint64_t padded);

/* ------------------------------------------------- per-layer codec (device)
 * Each mirrors one reference function on one vector of n elements. */
/* apply_accumulator (sparsify.cpp:9-16): out = g + acc */
int tagc_apply_accumulator(tagc_ctx* ctx, const float* g, const float* acc, float* out,
                           uint64_t n);
/* sparsify (sparsify.cpp:18-49). sparse/residual dev (n each); tau and
 * zero_count host out-pointers (may be NULL). */
int tagc_sparsify(tagc_ctx* ctx, const float* g, uint32_t n, double theta, float* sparse,
                  float* residual, float* tau, uint64_t* zero_count);
/* Index::create (index.cpp:32-41): words dev, tagc_index_words(n,width) u32 */
int tagc_index_create(tagc_ctx* ctx, const float* values, uint32_t n, uint32_t width,
                      uint32_t* words);
/* merge_indices (index.cpp:80-93): wrapping u32 word sum of `world` inputs */
int tagc_merge_indices(tagc_ctx* ctx, const uint32_t* const* words, uint32_t world,
                       uint32_t n_words, uint32_t* out);
/* Index::presence (index.cpp:51-57): positions (dev, capacity n) ascending */
int tagc_index_presence(tagc_ctx* ctx, const uint32_t* words, uint32_t n, uint32_t width,
                        uint32_t* positions, uint32_t* count);
/* CountSketch::compress (sketch.cpp:37-67): sketch dev, rows*m floats */
int tagc_sketch_compress(tagc_ctx* ctx, const float* values, uint32_t n, uint32_t ratio,
                         uint32_t rows, uint64_t seed, float* sketch);
/* sketch_add (sketch.cpp:69-75): out = a + b */
int tagc_sketch_add(tagc_ctx* ctx, const float* a, const float* b, float* out, uint64_t len);
/* peeling_decompress (decode.cpp:53-140). presence dev (count entries),
 * sketch dev (rows*m, not modified), values dev (n). unresolved dev
 * (capacity count, ascending) may be NULL; n_unresolved / peeled_fraction
 * host out-pointers may be NULL. */
int tagc_peeling_decompress(tagc_ctx* ctx, const uint32_t* presence, uint32_t count, uint32_t n,
                            uint32_t ratio, uint32_t rows, uint64_t seed, const float* sketch,
                            float* values, uint32_t* unresolved, uint32_t* n_unresolved,
                            double* peeled_fraction);
/* estimation_decompress (decode.cpp:24-51): out dev, one value per target */
int tagc_estimation_decompress(tagc_ctx* ctx, const uint32_t* presence, uint32_t count,
                               uint32_t n, uint32_t ratio, uint32_t rows, uint64_t seed,
                               const float* sketch, const uint32_t* targets, uint32_t n_targets,
                               float* out);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* TAGC_B200_H */
