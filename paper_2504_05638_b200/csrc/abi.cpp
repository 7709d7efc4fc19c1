// abi.cpp — extern "C" boundary (include/tagc_b200.h) over the C++ engine.
// Status mapping follows the reference CLI (cli.cpp:375-382): invalid argument
// -> 2, any other failure -> 1; the message is kept per thread.
#include "../../include/tagc_b200.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "engine.hpp"
#include "nccl_dl.hpp"

using namespace tagc_b200;

struct tagc_ctx {
  std::unique_ptr<Engine> engine;
};

struct tagc_shard_set {
  std::vector<ShardSpec> shards;
  std::vector<std::vector<tagc_segment>> segs;  // C views, names point into shards
};

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_error.clear();
    return TAGC_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return TAGC_INVALID;
  } catch (const std::exception& e) {
    g_error = e.what();
    return TAGC_RUNTIME;
  } catch (...) {
    g_error = "unknown error";
    return TAGC_RUNTIME;
  }
}

CompressionConfig to_cfg(const tagc_config* c) {
  if (!c) throw InvalidArgument("null config");
  CompressionConfig o;
  o.theta = c->theta;
  o.ratio = c->ratio;
  o.index_width = c->index_width;
  if (c->policy < 0 || c->policy > 2) throw InvalidArgument("unknown policy");
  o.policy = static_cast<Policy>(c->policy);
  o.include_out_proj = c->include_out_proj != 0;
  o.seed = c->seed;
  o.sketch_rows = c->sketch_rows;
  o.allow_low_theta = c->allow_low_theta != 0;
  o.min_compress_segment = c->min_compress_segment;
  return o;
}

LayerKind to_kind(int32_t k) {
  if (k < 0 || k > 8) throw InvalidArgument("unknown layer kind");
  return static_cast<LayerKind>(k);
}

ShardSpec to_shard(const tagc_shard* s) {
  if (!s) throw InvalidArgument("null shard");
  if (s->end < s->begin) throw InvalidArgument("shard end before begin");
  ShardSpec o;
  o.id = s->id;
  o.owner = s->owner;
  o.begin = s->begin;
  o.end = s->end;
  for (uint32_t i = 0; i < s->num_segments; ++i) {
    const tagc_segment& g = s->segments[i];
    o.segments.push_back({g.name ? g.name : "", to_kind(g.kind), g.begin, g.end});
  }
  return o;
}

Engine& eng(tagc_ctx* ctx) {
  if (!ctx || !ctx->engine) throw InvalidArgument("null context");
  return *ctx->engine;
}

}  // namespace

extern "C" {

const char* tagc_last_error(void) { return g_error.c_str(); }
int tagc_abi_version(void) { return TAGC_B200_ABI_VERSION; }

int tagc_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void tagc_config_default(tagc_config* out) {
  const CompressionConfig d;
  out->theta = d.theta;
  out->ratio = d.ratio;
  out->index_width = d.index_width;
  out->policy = static_cast<int32_t>(d.policy);
  out->include_out_proj = d.include_out_proj;
  out->seed = d.seed;
  out->sketch_rows = d.sketch_rows;
  out->allow_low_theta = d.allow_low_theta;
  out->min_compress_segment = d.min_compress_segment;
}

int tagc_config_validate(const tagc_config* cfg, uint32_t world_size) {
  return guarded([&] { to_cfg(cfg).validate_for_world(world_size); });
}

int tagc_theta_floor(uint32_t ratio, double* out) {
  return guarded([&] { *out = CompressionConfig::theta_floor(ratio); });
}

int tagc_kind_compressible(int32_t kind, int32_t policy, int32_t include_out_proj) {
  if (kind < 0 || kind > 8 || policy < 0 || policy > 2) return -1;
  return kind_compressible(static_cast<LayerKind>(kind), static_cast<Policy>(policy),
                           include_out_proj != 0)
             ? 1
             : 0;
}

int tagc_sketch_geometry(uint32_t n, uint32_t ratio, uint32_t rows, tagc_sketch_geom* out) {
  return guarded([&] {
    const SketchGeometry g = sketch_geometry(n, ratio, rows);
    *out = tagc_sketch_geom{g.n, g.ratio, g.rows, g.buckets_per_row};
  });
}

uint32_t tagc_index_words(uint32_t n, uint32_t width) { return words_needed(n, width); }

int tagc_comm_volume_model(const tagc_config* cfg, uint32_t world_size, uint64_t n,
                           tagc_comm_volume* out) {
  return guarded([&] {
    const CommVolume v = comm_volume_model(to_cfg(cfg), world_size,
                                           n ? std::optional<uint64_t>(n) : std::nullopt);
    *out = tagc_comm_volume{v.index_bits, v.sketch_bits, v.total_bits, v.factor};
  });
}

int tagc_lhc_comm_volume_model(const tagc_config* cfg, uint32_t world_size, uint64_t n,
                               tagc_comm_volume* out) {
  return guarded([&] {
    const CommVolume v = lhc_comm_volume_model(to_cfg(cfg), world_size,
                                               n ? std::optional<uint64_t>(n) : std::nullopt);
    *out = tagc_comm_volume{v.index_bits, v.sketch_bits, v.total_bits, v.factor};
  });
}

int tagc_make_shards(const tagc_layer_spec* layers, uint32_t n_layers, uint32_t shard_count,
                     uint32_t world_size, tagc_shard_set** out) {
  return guarded([&] {
    std::vector<LayerSpec> specs;
    for (uint32_t i = 0; i < n_layers; ++i)
      specs.push_back({layers[i].name ? layers[i].name : "", to_kind(layers[i].kind),
                       layers[i].param_count});
    auto set = std::make_unique<tagc_shard_set>();
    set->shards = make_shards(specs, shard_count, world_size);
    for (const ShardSpec& sh : set->shards) {
      std::vector<tagc_segment> v;
      for (const LayerSegment& s : sh.segments)
        v.push_back(tagc_segment{static_cast<int32_t>(s.kind), s.begin, s.end, s.name.c_str()});
      set->segs.push_back(std::move(v));
    }
    *out = set.release();
  });
}

uint32_t tagc_shard_set_count(const tagc_shard_set* set) {
  return set ? uint32_t(set->shards.size()) : 0;
}

int tagc_shard_set_get(const tagc_shard_set* set, uint32_t i, tagc_shard* out) {
  return guarded([&] {
    if (!set || i >= set->shards.size()) throw InvalidArgument("shard index out of range");
    const ShardSpec& s = set->shards[i];
    *out = tagc_shard{s.id, s.owner, s.begin, s.end, set->segs[i].data(),
                      uint32_t(set->segs[i].size())};
  });
}

void tagc_shard_set_destroy(tagc_shard_set* set) { delete set; }

int tagc_ctx_create(const tagc_config* cfg, uint32_t world_size, uint32_t rank, int device,
                    void* nccl_comm, void* cuda_stream, tagc_ctx** out) {
  return guarded([&] {
    auto c = std::make_unique<tagc_ctx>();
    c->engine = std::make_unique<Engine>(to_cfg(cfg), world_size, rank, device, nccl_comm, cuda_stream);
    *out = c.release();
  });
}

void tagc_ctx_destroy(tagc_ctx* ctx) { delete ctx; }

int tagc_ctx_set_config(tagc_ctx* ctx, const tagc_config* cfg) {
  return guarded([&] { eng(ctx).set_config(to_cfg(cfg)); });
}

void* tagc_ctx_stream(tagc_ctx* ctx) { return ctx && ctx->engine ? ctx->engine->stream() : nullptr; }

int tagc_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, 128);
  });
}

int tagc_ctx_init_nccl(tagc_ctx* ctx, const uint8_t unique_id[128]) {
  return guarded([&] { eng(ctx).init_nccl(unique_id); });
}

int tagc_ctx_ledger_csv(tagc_ctx* ctx, char* buf, size_t len, size_t* needed) {
  return guarded([&] {
    const std::string s = eng(ctx).ledger().to_csv();
    if (needed) *needed = s.size() + 1;
    if (buf && len) {
      const size_t k = std::min(len - 1, s.size());
      std::memcpy(buf, s.data(), k);
      buf[k] = 0;
    }
  });
}

}  // extern "C"

namespace {
int copy_out(const std::string& s, char* buf, size_t len, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && len) {
    const size_t k = std::min(len - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = 0;
  }
  return 0;
}
TrafficLedger& led(tagc_ledger* l) {
  if (!l) throw InvalidArgument("null ledger");
  return *reinterpret_cast<TrafficLedger*>(l);
}
}  // namespace

extern "C" {

tagc_ledger* tagc_ledger_create(void) {
  try {
    return reinterpret_cast<tagc_ledger*>(new TrafficLedger());
  } catch (...) {
    return nullptr;
  }
}

void tagc_ledger_destroy(tagc_ledger* l) { delete reinterpret_cast<TrafficLedger*>(l); }

int tagc_ledger_record(tagc_ledger* l, int32_t op, const char* tag, uint64_t payload_bits, uint64_t params) {
  return guarded([&] {
    if (op < 0 || op > 3) throw InvalidArgument("unknown collective op");
    led(l).record(static_cast<CollectiveOp>(op), tag ? tag : "", payload_bits, params);
  });
}

int tagc_ledger_csv(tagc_ledger* l, char* buf, size_t len, size_t* needed) {
  return guarded([&] { copy_out(led(l).to_csv(), buf, len, needed); });
}

int tagc_ledger_json(tagc_ledger* l, char* buf, size_t len, size_t* needed) {
  return guarded([&] { copy_out(led(l).to_json(), buf, len, needed); });
}

int tagc_ledger_bits_per_param(tagc_ledger* l, const char* prefix, double* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("null output");
    *out = led(l).bits_per_param_per_rank(prefix ? prefix : "");
  });
}

int tagc_ledger_row_count(tagc_ledger* l, uint32_t* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("null output");
    *out = uint32_t(led(l).rows().size());
  });
}

int tagc_ledger_row(tagc_ledger* l, uint32_t i, int32_t* op, char* tag, size_t tag_len, uint64_t* calls,
                    uint64_t* payload_bits, uint64_t* charged_bits, uint64_t* params) {
  return guarded([&] {
    const std::vector<LedgerRow> rows = led(l).rows();
    if (i >= rows.size()) throw InvalidArgument("ledger row out of range");
    const LedgerRow& r = rows[i];
    if (op) *op = int32_t(r.op);
    if (tag && tag_len) {
      const size_t k = std::min(tag_len - 1, r.tag.size());
      std::memcpy(tag, r.tag.data(), k);
      tag[k] = 0;
    }
    if (calls) *calls = r.calls;
    if (payload_bits) *payload_bits = r.payload_bits;
    if (charged_bits) *charged_bits = r.charged_bits;
    if (params) *params = r.params;
  });
}

int tagc_ledger_clear(tagc_ledger* l) {
  return guarded([&] { led(l).clear(); });
}

tagc_ledger* tagc_ctx_ledger(tagc_ctx* ctx) {
  if (!ctx || !ctx->engine) return nullptr;
  return reinterpret_cast<tagc_ledger*>(&ctx->engine->ledger());
}

int tagc_ctx_wire_bytes(tagc_ctx* ctx, uint64_t* out) {
  return guarded([&] {
    if (!out) throw InvalidArgument("null output");
    *out = eng(ctx).ledger().wire_bytes;
  });
}

int tagc_wire_bytes_from_device(tagc_ctx* ctx, const void* dev, uint64_t n_words, uint8_t* host_out) {
  return guarded([&] {
    static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "the wire format is the little-endian word layout");
    if (n_words && (!dev || !host_out)) throw InvalidArgument("null buffer");
    eng(ctx).download(dev, n_words * 4, host_out);
  });
}

int tagc_ctx_ledger_reset(tagc_ctx* ctx) {
  return guarded([&] { eng(ctx).ledger().clear(); });
}

uint64_t tagc_ctx_workspace_bytes(const tagc_ctx* ctx) {
  return ctx && ctx->engine ? ctx->engine->workspace_bytes() : 0;
}

int tagc_ctx_set_timing(tagc_ctx* ctx, int enabled) {
  return guarded([&] { eng(ctx).set_timing(enabled != 0); });
}

int tagc_ctx_last_timing(tagc_ctx* ctx, float out_ms[5]) {
  return guarded([&] {
    cuda_check(cudaStreamSynchronize(eng(ctx).stream()), "sync");
    eng(ctx).last_timing(out_ms);
  });
}

int tagc_ctx_set_graphs(tagc_ctx* ctx, int enabled) {
  return guarded([&] { eng(ctx).set_graphs(enabled != 0); });
}

int tagc_ctx_last_kernel_spans(tagc_ctx* ctx, float out_ms[2]) {
  return guarded([&] { eng(ctx).last_kernel_spans(out_ms); });
}

uint64_t tagc_ctx_last_launches(const tagc_ctx* ctx) {
  return ctx && ctx->engine ? ctx->engine->last_launches() : 0;
}

int tagc_ctx_last_peel_rounds(tagc_ctx* ctx, uint32_t out[2]) {
  return guarded([&] { eng(ctx).last_peel_rounds(out); });
}

int tagc_ctx_sync(tagc_ctx* ctx) {
  return guarded([&] { eng(ctx).sync_check(); });
}

int tagc_reduce_shard_sim(tagc_ctx* ctx, const tagc_shard* shard, uint32_t world,
                          const float* const* grads, float* const* accs, float* out,
                          tagc_peel_stats* stats) {
  return guarded([&] {
    PeelStats st;
    eng(ctx).reduce_shard_sim(to_shard(shard), world, grads, accs, out, stats ? &st : nullptr);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_reduce_shard_sim_audit(tagc_ctx* ctx, const tagc_shard* shard, uint32_t world,
                                const float* const* grads, float* const* accs, float* out,
                                tagc_peel_stats* stats, float* audit) {
  return guarded([&] {
    if (!audit) throw InvalidArgument("null audit buffer");
    PeelStats st;
    eng(ctx).reduce_shard_sim(to_shard(shard), world, grads, accs, out, stats ? &st : nullptr, audit);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_reduce_shards_support(tagc_ctx* ctx, uint8_t** send_support, uint64_t* block_bytes) {
  return guarded([&] { eng(ctx).exchange_support(send_support, block_bytes); });
}

int tagc_reduce_shards_end_support(tagc_ctx* ctx, const float* recv_f32, const uint32_t* recv_u32,
                                   const uint8_t* recv_support, tagc_peel_stats* stats) {
  return guarded([&] {
    PeelStats st;
    Engine& e = eng(ctx);
    e.set_support_recv(recv_support);
    e.exchange_end(recv_f32, recv_u32, stats ? &st : nullptr);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_reduce_shards_audit(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards, const float* grad,
                             float* acc, float* out, tagc_peel_stats* stats, float* audit) {
  return guarded([&] {
    if (!audit) throw InvalidArgument("null audit buffer");
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    PeelStats st;
    eng(ctx).reduce_shards_audit(v, grad, acc, out, stats ? &st : nullptr, audit);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_baseline_reduce_shard_sim(tagc_ctx* ctx, const tagc_shard* shard, uint32_t world,
                                   const float* const* grads, float* out) {
  return guarded([&] { eng(ctx).baseline_sim(to_shard(shard), world, grads, out); });
}

int tagc_reduce_shards(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                       const float* grad, float* acc, float* out, tagc_peel_stats* stats) {
  return guarded([&] {
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    PeelStats st;
    eng(ctx).reduce_shards(v, grad, acc, out, stats ? &st : nullptr);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_reduce_shard(tagc_ctx* ctx, const tagc_shard* shard, const float* grad, float* acc,
                      float* out, tagc_peel_stats* stats) {
  return tagc_reduce_shards(ctx, shard, 1, grad, acc, out, stats);
}

int tagc_reduce_shards_host(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                            const float* host_grad, float* acc, float* host_out,
                            tagc_peel_stats* stats) {
  return guarded([&] {
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    PeelStats st;
    eng(ctx).reduce_shards_host(v, host_grad, acc, host_out, stats ? &st : nullptr);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_reduce_shards_begin(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards, const float* grad,
                             float* acc, float* out, float** send_f32, uint32_t** send_u32, uint64_t* block_f32,
                             uint64_t* block_u32) {
  return guarded([&] {
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    Engine& e = eng(ctx);
    e.config().validate_for_world(e.world());
    e.exchange_begin(v, grad, acc, out, send_f32 ? *send_f32 : nullptr, send_u32 ? *send_u32 : nullptr);
    if (send_f32) *send_f32 = e.exchange_send_f();
    if (send_u32) *send_u32 = e.exchange_send_u();
    if (block_f32) *block_f32 = e.exchange_block_f();
    if (block_u32) *block_u32 = e.exchange_block_u();
  });
}

int tagc_overlap_begin(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards, const float* grad, float* acc,
                       float* out) {
  return guarded([&] {
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    eng(ctx).overlap_begin(v, grad, acc, out);
  });
}

int tagc_overlap_ready(tagc_ctx* ctx, uint64_t begin, uint64_t end, void* cuda_event) {
  return guarded([&] { eng(ctx).overlap_ready(begin, end, static_cast<cudaEvent_t>(cuda_event)); });
}

int tagc_overlap_finish(tagc_ctx* ctx, tagc_peel_stats* stats) {
  return guarded([&] {
    PeelStats st;
    eng(ctx).overlap_finish(stats ? &st : nullptr);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_reduce_shards_end(tagc_ctx* ctx, const float* recv_f32, const uint32_t* recv_u32,
                           tagc_peel_stats* stats) {
  return guarded([&] {
    PeelStats st;
    eng(ctx).exchange_end(recv_f32, recv_u32, stats ? &st : nullptr);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_ctx_peer_prepare(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                          uint8_t handle[TAGC_PEER_HANDLE_BYTES]) {
  return guarded([&] {
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    eng(ctx).peer_prepare(v, handle);
  });
}

int tagc_ctx_peer_open(tagc_ctx* ctx, const uint8_t* handles) {
  return guarded([&] {
    if (!handles) throw InvalidArgument("null handles");
    eng(ctx).peer_open(handles);
  });
}

int tagc_ctx_peer_attach_local(tagc_ctx* ctx, tagc_ctx* const* ranks, uint32_t n_ranks) {
  return guarded([&] {
    std::vector<Engine*> v;
    for (uint32_t i = 0; i < n_ranks; ++i) v.push_back(&eng(ranks[i]));
    eng(ctx).peer_attach_local(v);
  });
}

int tagc_ctx_host_join(tagc_ctx* ctx) {
  return guarded([&] { eng(ctx).host_join(); });
}

int tagc_plan_exchange(const tagc_config* cfg, const tagc_shard* shards, uint32_t n_shards,
                       uint32_t world_size, uint32_t rank, tagc_seg_plan* out, uint32_t* n_out,
                       uint64_t* block_f32, uint64_t* block_u32) {
  return guarded([&] {
    const CompressionConfig c = to_cfg(cfg);
    c.validate_for_world(world_size);
    if (rank >= world_size) throw InvalidArgument("rank must be below the world size");
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    const ExchangePlan P = plan_exchange(v, c, world_size, rank);
    if (n_out) *n_out = uint32_t(P.segs.size());
    if (block_f32) *block_f32 = P.Bf;
    if (block_u32) *block_u32 = P.Bu;
    if (out)
      for (size_t i = 0; i < P.segs.size(); ++i) {
        const SegPlan& p = P.segs[i];
        const uint64_t oo = P.out_off[p.shard];
        out[i] = tagc_seg_plan{p.shard, p.seg, p.compressed ? 1u : 0u, p.m, p.n_words,
                               v[p.shard].owner, p.lo, p.len, p.word_off, p.sk_off, p.raw_off,
                               oo == ~0ull ? ~0ull : oo + p.lo};
      }
  });
}

int tagc_baseline_reduce_shards(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards,
                                const float* grad, float* out) {
  return guarded([&] {
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    eng(ctx).baseline_shards(v, grad, out);
  });
}

int tagc_apply_accumulator(tagc_ctx* ctx, const float* g, const float* acc, float* out, uint64_t n) {
  return guarded([&] { eng(ctx).add(g, acc, out, n); });
}

int tagc_sparsify(tagc_ctx* ctx, const float* g, uint32_t n, double theta, float* sparse,
                  float* residual, float* tau, uint64_t* zero_count) {
  return guarded([&] { eng(ctx).sparsify(g, n, theta, sparse, residual, tau, zero_count); });
}

int tagc_index_create(tagc_ctx* ctx, const float* values, uint32_t n, uint32_t width,
                      uint32_t* words) {
  return guarded([&] { eng(ctx).index_create(values, n, width, words); });
}

int tagc_merge_indices(tagc_ctx* ctx, const uint32_t* const* words, uint32_t world,
                       uint32_t n_words, uint32_t* out) {
  return guarded([&] { eng(ctx).merge_indices(words, world, n_words, out); });
}

int tagc_index_presence(tagc_ctx* ctx, const uint32_t* words, uint32_t n, uint32_t width,
                        uint32_t* positions, uint32_t* count) {
  return guarded([&] { eng(ctx).index_presence(words, n, width, positions, count); });
}

int tagc_sketch_compress(tagc_ctx* ctx, const float* values, uint32_t n, uint32_t ratio,
                         uint32_t rows, uint64_t seed, float* sketch) {
  return guarded([&] { eng(ctx).sketch_compress(values, n, ratio, rows, seed, sketch); });
}

int tagc_sketch_add(tagc_ctx* ctx, const float* a, const float* b, float* out, uint64_t len) {
  return guarded([&] { eng(ctx).add(a, b, out, len); });
}

int tagc_apply_optimizer(tagc_ctx* ctx, int32_t kind, double lr, double weight_decay, uint32_t world,
                         uint32_t step, float* params, const float* decoded, float* adam_v, uint64_t len) {
  return guarded([&] { eng(ctx).apply_optimizer(kind, lr, weight_decay, world, step, params, decoded, adam_v, len); });
}

int tagc_reduce_shards_step(tagc_ctx* ctx, const tagc_shard* shards, uint32_t n_shards, const float* grad,
                            float* acc, float* out, int32_t kind, double lr, double weight_decay, uint32_t step,
                            float* params, float* adam_v, tagc_peel_stats* stats) {
  return guarded([&] {
    std::vector<ShardSpec> v;
    for (uint32_t i = 0; i < n_shards; ++i) v.push_back(to_shard(&shards[i]));
    PeelStats st;
    eng(ctx).reduce_shards_step(v, grad, acc, out, kind, lr, weight_decay, step, params, adam_v,
                                stats ? &st : nullptr);
    if (stats)
      *stats = tagc_peel_stats{st.presence, st.peeled, st.unresolved, st.index_lost,
                               st.index_spurious, st.compressed_segments, st.baseline_segments};
  });
}

int tagc_allgather_params(tagc_ctx* ctx, float* params, uint64_t padded) {
  return guarded([&] { eng(ctx).allgather_params(params, padded); });
}

int tagc_peeling_decompress(tagc_ctx* ctx, const uint32_t* presence, uint32_t count, uint32_t n,
                            uint32_t ratio, uint32_t rows, uint64_t seed, const float* sketch,
                            float* values, uint32_t* unresolved, uint32_t* n_unresolved,
                            double* peeled_fraction) {
  return guarded([&] {
    eng(ctx).peeling_decompress(presence, count, n, ratio, rows, seed, sketch, values, unresolved,
                                n_unresolved, peeled_fraction);
  });
}

int tagc_estimation_decompress(tagc_ctx* ctx, const uint32_t* presence, uint32_t count,
                               uint32_t n, uint32_t ratio, uint32_t rows, uint64_t seed,
                               const float* sketch, const uint32_t* targets, uint32_t n_targets,
                               float* out) {
  return guarded([&] {
    eng(ctx).estimation_decompress(presence, count, n, ratio, rows, seed, sketch, targets, n_targets,
                                   out);
  });
}

}  // extern "C"
