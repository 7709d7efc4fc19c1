// engine.hpp — the B200 exchange engine behind the C-ABI: plans device
// layouts for a shard list, owns workspaces, enqueues the sm_100a kernels and
// the NCCL exchange on one stream. C++ mirror of reference hook.cpp:98-200.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "host.hpp"
#include "kernels.hpp"

namespace tagc_b200 {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void cuda_check(cudaError_t e, const char* what);
void nccl_check(ncclResult_t r, const char* what);

// Device arena of named, grow-only buffers (memory laid out once per plan and
// reused across steps).
class Workspace {
 public:
  ~Workspace();
  void* get(const std::string& name, size_t bytes, bool zero_on_alloc = false,
            cudaStream_t s = nullptr);
  uint64_t bytes() const { return total_; }
  // bumped on every (re)allocation: captured graphs hold raw pointers
  uint64_t generation() const { return gen_; }
  // Regrowth keeps the old buffer until destruction instead of syncing and
  // freeing it: cudaFree synchronises the whole device, which must never
  // happen while a peer exchange may be spinning on this device.
  void set_defer_free(bool on) { defer_free_ = on; }

 private:
  uint64_t gen_ = 0;
  bool defer_free_ = false;
  std::vector<void*> graveyard_;
  struct Buf {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  std::map<std::string, Buf> bufs_;
  uint64_t total_ = 0;
};

struct SegPlan {
  uint32_t shard = 0;        // index into the shard list
  uint32_t seg = 0;          // index into shard.segments
  uint64_t lo = 0, len = 0;  // shard-relative offset, length
  bool compressed = false;
  uint32_t m = 0, n_words = 0;
  uint64_t word_off = 0, sk_off = 0, raw_off = 0;  // offsets inside an owner block
  std::string tag;
};

// Owner-major exchange layout for one rank (reference hook.cpp:117-166 per
// segment; the blocks are what one grouped reduce-scatter moves): owner o's
// float block [o*Bf, (o+1)*Bf) holds the sketches of its compressed segments
// followed by its raw segments, its u32 block [o*Bu, (o+1)*Bu) the index
// words.
struct ExchangePlan {
  std::vector<SegPlan> segs;
  std::vector<uint64_t> skc, rawc, wc;  // per-owner sketch / raw / word totals
  uint64_t Bf = 0, Bu = 0;
  std::vector<uint64_t> out_off;  // per shard: offset in the owner's output, ~0 if not owned
};
ExchangePlan plan_exchange(const std::vector<ShardSpec>& shards, const CompressionConfig& cfg,
                           uint32_t world, uint32_t rank);

struct PlanTotals {
  uint64_t enc_tiles = 0, enc_samples = 0, cand = 0;
  uint64_t dec_word_tiles = 0, dec_slots = 0, dec_bitmap_words = 0, dec_list = 0;
};

class Engine {
 public:
  Engine(const CompressionConfig& cfg, uint32_t world, uint32_t rank, int device, void* nccl_comm,
         void* stream);
  ~Engine();

  void set_config(const CompressionConfig& cfg);
  const CompressionConfig& config() const { return cfg_; }
  uint32_t world() const { return world_; }
  uint32_t rank() const { return rank_; }
  cudaStream_t stream() const { return stream_; }
  TrafficLedger& ledger() { return ledger_; }
  void download(const void* dev, uint64_t bytes, void* host);
  uint64_t workspace_bytes() const { return ws_.bytes(); }
  void init_nccl(const uint8_t id[128]);
  void set_timing(bool on) { timing_ = on; }
  // stage times (ms) of the last call: prep, select+fused pass, select finish, exchange, decode
  static constexpr int kStages = 5;
  void last_timing(float out[kStages]) const;
  uint64_t last_launches() const { return launches_; }
  // timing mode: device execution spans (ms) of the last call's sampled
  // select + fused pass (k_sample start .. k_fused end) and decode (k_build
  // start .. k_final end), from %globaltimer stamps written by the kernels
  void last_kernel_spans(float out_ms[2]);
  // peel rounds of the last decode that returned stats: {grid rounds, single-CTA tail rounds}
  void last_peel_rounds(uint32_t out[2]) const { out[0] = rounds_[0]; out[1] = rounds_[1]; }

  // hook.cpp:98-200 with `world` logical ranks on this GPU.
  // audit (optional, dev, shard.size() floats): audit_exchanged_sum
  // (hook.cpp:191-195), the rank-ordered sum of the sparse vectors exchanged
  // for compressed segments, zeros elsewhere.
  void reduce_shard_sim(const ShardSpec& shard, uint32_t world, const float* const* grads,
                        float* const* accs, float* out, PeelStats* stats, float* audit = nullptr);
  // hook.cpp:90-96
  void baseline_sim(const ShardSpec& shard, uint32_t world, const float* const* grads, float* out);
  // One process per GPU, NCCL exchange.
  void reduce_shards(const std::vector<ShardSpec>& shards, const float* grad, float* acc,
                     float* out, PeelStats* stats);
  void baseline_shards(const std::vector<ShardSpec>& shards, const float* grad, float* out);
  // CUDA-graph replay of reduce_shards: a call whose shard layout, config and
  // buffers repeat is captured once (on its second occurrence) and replayed
  // with one cudaGraphLaunch. TAGC_GRAPHS=0 disables.
  void set_graphs(bool on);
  // Host-buffer form of reduce_shards (the end-to-end call): the gradient is
  // copied H2D on a copy stream into one of two device buffers, the owner's
  // decoded shard D2H on a second copy stream from one of two device buffers,
  // so consecutive calls overlap D2H(k), H2D(k+1) and the exchange itself.
  // host_out is complete once host_join() (or sync_check) has run.
  void reduce_shards_host(const std::vector<ShardSpec>& shards, const float* host_grad, float* acc,
                          float* host_out, PeelStats* stats);
  // The context stream waits for every copy the host-buffer path enqueued.
  void host_join();
  // Pull-mode exchange over peer memory instead of NCCL (peer.cu). prepare
  // lays out and allocates this rank's exchange region for the shard layout
  // and returns its CUDA IPC handle; open maps every peer's region from the
  // gathered handles; attach_local takes the regions of contexts living in
  // this process (one GPU, tests). Afterwards reduce_shards uses the peers.
  static constexpr size_t kPeerHandleBytes = 64;
  void peer_prepare(const std::vector<ShardSpec>& shards, uint8_t handle[kPeerHandleBytes]);
  void peer_open(const uint8_t* handles);
  void peer_attach_local(const std::vector<Engine*>& ranks);
  // The exchange split around its collective, for a caller-provided
  // transport: exchange_begin encodes into the owner-major send blocks
  // (world * block_f32 floats, world * block_u32 words; layout of
  // plan_exchange), the caller reduce-scatters them (f32 sum, wrapping u32
  // sum), exchange_end decodes this rank's block.
  void exchange_begin(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                      float* user_send_f = nullptr, uint32_t* user_send_u = nullptr);
  // Overlapped exchange: open before the gradient exists, encode each range
  // as it becomes ready (ready: an event on the producer's stream, or null),
  // then the collective + decode. Same results as reduce_shards.
  void overlap_begin(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out);
  void overlap_ready(uint64_t lo, uint64_t hi, cudaEvent_t ready);
  void overlap_finish(PeelStats* stats);
  void open_exchange(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out);
  void finish_exchange(PeelStats* stats);
  // The pieces of exchange_begin: prologue (plan, send blocks), encode of the
  // segments inside a flat range, seal (the rest, end of gradient reads).
  void exchange_prologue(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                         float* user_send_f = nullptr, uint32_t* user_send_u = nullptr);
  void exchange_encode(uint64_t lo, uint64_t hi);
  void exchange_seal();
  void exchange_end(const float* recv_f, const uint32_t* recv_u, PeelStats* stats,
                    const std::function<void()>& pre_decode = nullptr);
  float* exchange_send_f() const { return xs_.send_f; }
  uint32_t* exchange_send_u() const { return xs_.send_u; }
  // Split API, 1-bit index: this rank's support (one byte per position,
  // owner-major blocks of block_bytes = 32 * block_u32) for the caller to
  // max-reduce-scatter; exchange_end then takes the reduced block as
  // xs_.support_recv (set_support_recv) and reports index_lost / _spurious.
  void exchange_support(uint8_t** send_support, uint64_t* block_bytes);
  void set_support_recv(const uint8_t* recv) { xs_.support_recv = recv; }
  // reduce_shards plus audit_exchanged_sum (hook.cpp:191-195) for the owned
  // shards (dev, laid out like out): the sum over ranks of the exchanged
  // sparse vectors of compressed segments, zeros elsewhere. NCCL world (or
  // W = 1); diagnostic: an extra uncompressed reduce-scatter.
  void reduce_shards_audit(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                           PeelStats* stats, float* audit);
  uint64_t exchange_block_f() const { return xs_.P.Bf; }
  uint64_t exchange_block_u() const { return xs_.P.Bu; }

  // Per-stage codec entry points (single vector).
  void sparsify(const float* g, uint32_t n, double theta, float* sparse, float* residual,
                float* tau, uint64_t* zero_count);
  void index_create(const float* v, uint32_t n, uint32_t width, uint32_t* words);
  void merge_indices(const uint32_t* const* words, uint32_t world, uint32_t n_words, uint32_t* out);
  void index_presence(const uint32_t* words, uint32_t n, uint32_t width, uint32_t* positions,
                      uint32_t* count);
  void sketch_compress(const float* v, uint32_t n, uint32_t ratio, uint32_t rows, uint64_t seed,
                       float* sketch);
  void add(const float* a, const float* b, float* out, uint64_t n);
  // Owner-side consumer: mean over ranks + optimizer step (train.cpp:202-220, 355-359)
  void apply_optimizer(int kind, double lr, double weight_decay, uint32_t world, uint32_t step, float* params,
                       const float* decoded, float* adam_v, uint64_t n);
  // reduce_shards followed by the owner-side optimizer step, fused into the
  // kernels that produce the decoded values. params / adam_v / out (optional)
  // are laid out like reduce_shards' out (the owned shards, concatenated).
  void reduce_shards_step(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                          int kind, double lr, double weight_decay, uint32_t step, float* params, float* adam_v,
                          PeelStats* stats);
  // Parameter all-gather after the owners' updates (train.cpp:364): params is
  // the padded flat space (padded = W * L, train.cpp:242); rank i's slice
  // [i*L, (i+1)*L) goes to every rank, in place.
  void allgather_params(float* params, uint64_t padded);
  void peeling_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                          uint32_t rows, uint64_t seed, const float* sketch, float* values,
                          uint32_t* unresolved, uint32_t* n_unresolved, double* pf);
  void estimation_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                             uint32_t rows, uint64_t seed, const float* sketch,
                             const uint32_t* targets, uint32_t n_targets, float* out);
  // Synchronise and surface deferred device errors (NaN input -> invalid).
  void sync_check();
  void clear_err_word(uint32_t seen);
  void trace(const char* phase) const;

 private:
  struct EncBatch;
  friend struct CallScope;
  void enqueue_reduce_shards(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                             PeelStats* stats);
  struct ExchangeState {  // between exchange_begin and exchange_end
    bool begun = false;   // prologue done, segments may still be encoded
    bool active = false;  // sealed: waiting for exchange_end
    bool side_used = false;
    const float* grad = nullptr;
    float* acc = nullptr;
    std::vector<uint8_t> encoded;  // per plan segment
    std::vector<ShardSpec> shards;
    ExchangePlan P;
    float* out = nullptr;
    float* send_f = nullptr;
    uint32_t* send_u = nullptr;
    cudaEvent_t zero_done = nullptr;
    // index_lost / index_spurious of a 1-bit index over several ranks: the
    // OR of the ranks' supports, as one byte per position of this rank's
    // owner block (NCCL / split), or the peer send set holding them
    const uint8_t* support_recv = nullptr;
    int peer_set = -1;
  };
  ExchangeState xs_;
  OptEpilogue* opt_dev_ = nullptr;  // device slot of the fused optimizer's scalars
  bool opt_on_ = false;             // set for the duration of reduce_shards_step
  OptEpilogue make_opt(int kind, double lr, double weight_decay, uint32_t world, uint32_t step, float* params,
                       float* adam_v, const float* out_base, bool write_out) const;
  struct PeerState {
    bool attached = false;
    char* region = nullptr;
    size_t bytes = 0;
    uint64_t Bf = 0, Bu = 0;
    size_t off_f[2] = {0, 0}, off_u[2] = {0, 0}, off_flags = 0, off_counter = 0;
    PeerView view{};
    int set = 0;
    std::vector<void*> opened;
  };
  PeerState peer_;
  void peer_release();
  void peer_fill(const std::vector<char*>& bases);
  struct LedgerEntry {
    CollectiveOp op;
    std::string tag;
    uint64_t bits, params;
  };
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    uint64_t gen = 0, launches = 0, wire = 0;
    std::vector<LedgerEntry> ledger;
    std::vector<char*> pinned;  // descriptor uploads frozen into the graph
    std::vector<void*> dev;     // graph-private descriptor buffers, filled once at capture
  };
  cudaStream_t desc_stream_ = nullptr;  // capture-time descriptor copies (never captured)
  // A descriptor buffer: the workspace's, or while capturing a graph-private
  // one that upload() fills once (no copy kernel in the replayed graph).
  void* desc_buffer(const char* name, size_t bytes);
  static void free_graph(GraphEntry& g);
  static constexpr size_t kMaxGraphs = 16;
  std::map<std::string, GraphEntry> graphs_;
  std::map<std::string, int> graph_seen_;
  bool graphs_on_ = true;
  GraphEntry* capturing_ = nullptr;  // upload() / ledger record target while capturing
  void drop_graphs();
  void record(CollectiveOp op, const std::string& tag, uint64_t bits, uint64_t params);
  // Descriptor uploads go through pinned staging (a pageable cudaMemcpyAsync
  // would synchronise the stream): two halves, one per public call, each
  // reused only after the call that last filled it has finished on the GPU.
  struct Staging {
    char* ptr = nullptr;  // mapped pinned host memory
    char* dev = nullptr;  // its device alias
    size_t cap = 0, off = 0;
    cudaEvent_t ev = nullptr;
  };
  std::vector<char*> stage_graveyard_;  // outgrown staging buffers (peer mode: freed at destruction)
  void stage_grow(Staging& s, size_t bytes);
  Staging stage_[2];
  int stage_cur_ = 0, call_depth_ = 0;
  void call_begin();
  void call_end();
  // host-buffer path (reduce_shards_host)
  cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
  cudaEvent_t hev_in_[2] = {}, hev_gfree_[2] = {}, hev_dec_[2] = {}, hev_out_[2] = {}, hev_join_ = nullptr;
  uint64_t host_calls_ = 0, host_grad_cap_ = 0, host_out_cap_ = 0;
  cudaEvent_t grad_read_ev_ = nullptr;  // recorded by reduce_shards once the gradient is consumed
  void run_select_encode(std::vector<EncItem>& items, bool w4, const HashParams& hp,
                         bool want_kept, const char* tag);
  // Decode into the items' outputs; the final emit waits on `zero_done` (if
  // set), the side stream's join event.
  // pre_launch (if set) is enqueued after the decode's allocations and
  // descriptor uploads, right before its kernels (the peer exchange goes
  // there: nothing that may synchronise the device follows its wait).
  void run_decode(std::vector<DecItem>& items, const HashParams& hp, bool want_unresolved,
                  bool ordered, cudaEvent_t zero_done = nullptr,
                  const std::function<void()>& pre_launch = nullptr, uint32_t stats_base = 0);
  void run_decode_grouped(std::vector<DecItem>& items, const HashParams& hp, bool ordered,
                          cudaEvent_t zero_done, const std::function<void()>& pre_launch);
  // Side stream for bandwidth work that overlaps the latency-bound peel
  // (W == 1 raw-segment copies); fork/join by events.
  cudaStream_t aux_ = nullptr;
  cudaEvent_t aux_fork_ = nullptr, aux_join_ = nullptr;
  void ensure_aux();
  // W == 1 exchange: the deferred sketch scatter runs on ds_stream_ while the
  // decode builds its presence list from the (already final) index; round 0
  // waits on ds_done_ (sketch_pending_) before it reads the sketch.
  cudaStream_t ds_stream_ = nullptr;
  cudaEvent_t ds_fork_ = nullptr, ds_done_ = nullptr;
  bool ds_side_ok_ = false;       // set by the W == 1 exchange encode
  bool sketch_pending_ = false;   // ds_done_ recorded, not yet waited on by stream_
  cudaEvent_t take_sketch_event();  // the event to wait on before reading sketches (or nullptr)
  void join_sketch();             // stream_ waits on a pending sketch scatter
  void upload(const void* host, size_t bytes, void* dev);
  // zero byte ranges with one kernel launch (no copy-engine memset)
  void zero(const std::vector<std::pair<void*, uint64_t>>& ranges);
  void ev_record(int i);
  void span_reset();
  unsigned long long* spans_ = nullptr;
  // sketches above this size are scattered by the region-ordered pass
  // (TAGC_DEFER_SCATTER_BYTES; 0 defers every compressed segment's)
  uint64_t defer_scatter_bytes_ = 32ull << 20;
  // sketches whose scatter is deferred to the region-ordered pass (> 32 MB)
  bool big_sketch(uint64_t floats) const { return floats * 4 > defer_scatter_bytes_; }
  // counter-mode decode with round 0 inside the dense emit (TAGC_FUSED_EMIT=1; off: 0.68 vs 0.50 ms on C4)
  bool fused_emit_ = false;
  // TAGC_FORCE_COLLECTIVE=1: a one-rank NCCL context runs the grouped
  // reduce-scatters anyway (exercises the NCCL data path on one GPU)
  bool force_collective_ = false;
  bool side_stream_ = true;  // W = 1 raw copies on the low-priority side stream (TAGC_SIDE_STREAM=0: in order)
  bool use_tma_ = true;  // TMA-staged fused pass (TAGC_FUSED_TMA=0 selects the register path)
  uint32_t* err_flag();

  CompressionConfig cfg_;
  uint32_t world_, rank_;
  int device_;
  DevInfo di_;
  cudaStream_t stream_ = nullptr;
  bool own_stream_ = false;
  ncclComm_t comm_ = nullptr;
  bool own_comm_ = false;
  Workspace ws_;
  TrafficLedger ledger_;
  bool timing_ = false;
  cudaEvent_t ev_[kStages + 1] = {};
  uint64_t launches_ = 0;
  // host mirrors of the last decode's per-item stats (device -> host)
  std::vector<DecStats> dec_stats_;
  uint32_t rounds_[2] = {0, 0};
  bool last_ordered_ = false;
  bool ord_epoch_set_ = false;  // TAGC_ORD_EPOCH_START applied
  uint64_t nvtx_range_ = 0;  // nvtxRangeId_t of the open stage range
  bool nvtx_open_ = false;
  void fetch_rounds();
};

}  // namespace tagc_b200
