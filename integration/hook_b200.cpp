// hook_b200.cpp — the reference-side binding a maintainer adds to drop
// libtagc_b200 into the reference. It is a replacement
// translation unit for proj/src/hook.cpp: it defines every symbol hook.hpp
// declares (hook.hpp:42-104) with the same signatures, and routes the
// exchange itself through the C-ABI (include/tagc_b200.h) onto the B200:
//
//   tagc_reduce_shard      (hook.hpp:76-80, hook.cpp:98-200)  -> tagc_reduce_shard_sim[_audit]
//   baseline_reduce_shard  (hook.hpp:84-86, hook.cpp:90-96)   -> tagc_baseline_reduce_shard_sim
//   make_shards            (hook.hpp:42-43, hook.cpp:30-61)   -> tagc_make_shards
//   comm_volume_model / lhc_comm_volume_model (hook.cpp:202-236) -> tagc_(lhc_)comm_volume_model
//   PeelStats::operator+= / index_collision_rate (hook.cpp:13-28): plain struct arithmetic
//
// The reference's World keeps doing the bookkeeping its callers read: the
// library's ledger rows for the call (same tags, same charges) are replayed
// into world.ledger(). Status codes map back onto the reference's exceptions
// (TAGC_INVALID -> std::invalid_argument, anything else -> std::runtime_error).
//
// Linked together with the reference's other sources and its own test files
// (test_hook.cpp, acceptance.cpp) by integration/Makefile, so the reference's
// tests exercise the GPU path unmodified (tests/test_gpu_integration.py).
#include "tagc/hook.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "tagc_b200.h"

namespace tagc {
namespace {

void check(int st) {
  if (st == TAGC_OK) return;
  if (st == TAGC_INVALID) throw std::invalid_argument(tagc_last_error());
  throw std::runtime_error(tagc_last_error());
}

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

tagc_config to_c(const CompressionConfig& c) {
  tagc_config o;
  tagc_config_default(&o);
  o.theta = c.theta;
  o.ratio = c.ratio;
  o.index_width = c.index_width;
  o.policy = static_cast<int32_t>(c.policy);  // enum values identical (config.hpp:11)
  o.include_out_proj = c.include_out_proj ? 1 : 0;
  o.seed = c.seed;
  o.sketch_rows = c.sketch_rows;
  o.allow_low_theta = c.allow_low_theta ? 1 : 0;
  o.min_compress_segment = c.min_compress_segment;
  return o;
}

// One context per process (world_size 1: the simulated W comes with each
// call) and grow-only device staging for the host vectors the reference
// passes around.
struct Session {
  tagc_ctx* ctx = nullptr;
  void* buf = nullptr;
  size_t cap = 0;

  tagc_ctx* get(const tagc_config& cfg) {
    if (!ctx) {
      tagc_config base;
      tagc_config_default(&base);
      check(tagc_ctx_create(&base, 1, 0, 0, nullptr, nullptr, &ctx));
    }
    check(tagc_ctx_set_config(ctx, &cfg));
    return ctx;
  }
  float* floats(size_t n) {
    if (n * 4 > cap) {
      if (buf) cuda(cudaFree(buf), "cudaFree");
      cap = std::max<size_t>(n * 4, 1 << 20);
      cuda(cudaMalloc(&buf, cap), "cudaMalloc");
    }
    return static_cast<float*>(buf);
  }
  ~Session() {
    if (ctx) tagc_ctx_destroy(ctx);
    if (buf) cudaFree(buf);
  }
};

Session& session() {
  static Session s;
  return s;
}

void check_shard_inputs(const ShardSpec& shard, std::span<const std::vector<float>> grads, uint32_t w) {
  if (grads.size() != w) throw std::invalid_argument("need one gradient slice per rank");
  for (const auto& g : grads)
    if (g.size() != shard.size()) throw std::invalid_argument("gradient slice length does not match the shard");
  if (shard.owner >= w) throw std::invalid_argument("shard owner rank out of range");
}

struct CShard {
  std::vector<tagc_segment> segs;
  tagc_shard s{};
  explicit CShard(const ShardSpec& sh) {
    for (const LayerSegment& g : sh.segments)
      segs.push_back(tagc_segment{static_cast<int32_t>(g.kind), g.begin, g.end, g.name.c_str()});
    s = tagc_shard{sh.id, sh.owner, sh.begin, sh.end, segs.data(), uint32_t(segs.size())};
  }
};

// The call's rows of the library's ledger, recorded into the reference World.
void replay_ledger(tagc_ctx* ctx, World& world) {
  tagc_ledger* l = tagc_ctx_ledger(ctx);
  uint32_t n = 0;
  check(tagc_ledger_row_count(l, &n));
  for (uint32_t i = 0; i < n; ++i) {
    int32_t op = 0;
    char tag[512];
    uint64_t calls = 0, payload = 0, charged = 0, params = 0;
    check(tagc_ledger_row(l, i, &op, tag, sizeof(tag), &calls, &payload, &charged, &params));
    for (uint64_t c = 0; c < calls; ++c)  // per-call shares (one call per tag per exchange)
      world.ledger().record(static_cast<CollectiveOp>(op), tag, payload / calls, params / calls);
  }
  check(tagc_ctx_ledger_reset(ctx));
}

}  // namespace

PeelStats& PeelStats::operator+=(const PeelStats& o) {
  presence += o.presence;
  peeled += o.peeled;
  unresolved += o.unresolved;
  index_lost += o.index_lost;
  index_spurious += o.index_spurious;
  compressed_segments += o.compressed_segments;
  baseline_segments += o.baseline_segments;
  return *this;
}

double PeelStats::index_collision_rate() const {
  const std::uint64_t truth = presence + index_lost - index_spurious;
  return truth == 0 ? 0.0 : double(index_lost + index_spurious) / double(truth);
}

std::vector<ShardSpec> make_shards(const std::vector<LayerSpec>& layers, std::uint32_t shard_count,
                                   std::uint32_t world_size) {
  std::vector<tagc_layer_spec> c;
  for (const LayerSpec& l : layers)
    c.push_back(tagc_layer_spec{l.name.c_str(), static_cast<int32_t>(l.kind), l.param_count});
  tagc_shard_set* set = nullptr;
  check(tagc_make_shards(c.data(), uint32_t(c.size()), shard_count, world_size, &set));
  std::vector<ShardSpec> out;
  for (uint32_t i = 0; i < tagc_shard_set_count(set); ++i) {
    tagc_shard s;
    check(tagc_shard_set_get(set, i, &s));
    ShardSpec sh;
    sh.id = s.id;
    sh.owner = s.owner;
    sh.begin = s.begin;
    sh.end = s.end;
    for (uint32_t k = 0; k < s.num_segments; ++k) {
      const tagc_segment& g = s.segments[k];
      sh.segments.push_back(LayerSegment{g.name ? g.name : "", static_cast<LayerKind>(g.kind), g.begin, g.end});
    }
    out.push_back(std::move(sh));
  }
  tagc_shard_set_destroy(set);
  return out;
}

std::vector<float> baseline_reduce_shard(const ShardSpec& shard, std::span<const std::vector<float>> grads,
                                         World& world) {
  const uint32_t w = world.size();
  check_shard_inputs(shard, grads, w);
  const size_t n = shard.size();
  Session& S = session();
  tagc_config cfg;
  tagc_config_default(&cfg);
  tagc_ctx* ctx = S.get(cfg);
  float* d = S.floats((w + 1) * n + 1);
  std::vector<const float*> dg(w);
  for (uint32_t r = 0; r < w; ++r) {
    dg[r] = d + r * n;
    cuda(cudaMemcpy(d + r * n, grads[r].data(), n * 4, cudaMemcpyHostToDevice), "H2D");
  }
  CShard cs(shard);
  check(tagc_ctx_ledger_reset(ctx));
  check(tagc_baseline_reduce_shard_sim(ctx, &cs.s, w, dg.data(), d + w * n));
  // the context works on its own non-blocking stream and this call returns
  // no statistics (so it does not synchronise): wait before the legacy-stream
  // copy reads the result, and before the next call overwrites the inputs
  check(tagc_ctx_sync(ctx));
  std::vector<float> out(n);
  cuda(cudaMemcpy(out.data(), d + w * n, n * 4, cudaMemcpyDeviceToHost), "D2H");
  replay_ledger(ctx, world);
  return out;
}

ShardReduceResult tagc_reduce_shard(const ShardSpec& shard, std::span<const std::vector<float>> grads,
                                    std::span<ResidualAccumulator> accs, const CompressionConfig& config,
                                    World& world, bool collect_audit) {
  const uint32_t w = world.size();
  check_shard_inputs(shard, grads, w);
  const tagc_config cfg = to_c(config);
  check(tagc_config_validate(&cfg, w));
  if (accs.size() != w) throw std::invalid_argument("need one accumulator per rank");
  for (const auto& a : accs)
    if (a.values.size() != shard.size()) throw std::invalid_argument("accumulator length does not match the shard");
  const size_t n = shard.size();
  Session& S = session();
  tagc_ctx* ctx = S.get(cfg);
  // device layout: grads[W] | accs[W] | out | audit
  float* d = S.floats((2 * w + 2) * n + 1);
  std::vector<const float*> dg(w);
  std::vector<float*> da(w);
  for (uint32_t r = 0; r < w; ++r) {
    dg[r] = d + r * n;
    da[r] = d + (w + r) * n;
    cuda(cudaMemcpy(d + r * n, grads[r].data(), n * 4, cudaMemcpyHostToDevice), "H2D grad");
    cuda(cudaMemcpy(da[r], accs[r].values.data(), n * 4, cudaMemcpyHostToDevice), "H2D acc");
  }
  float* d_out = d + 2 * w * n;
  float* d_audit = d_out + n;
  CShard cs(shard);
  tagc_peel_stats st{};
  check(tagc_ctx_ledger_reset(ctx));
  if (collect_audit)
    check(tagc_reduce_shard_sim_audit(ctx, &cs.s, w, dg.data(), da.data(), d_out, &st, d_audit));
  else
    check(tagc_reduce_shard_sim(ctx, &cs.s, w, dg.data(), da.data(), d_out, &st));
  check(tagc_ctx_sync(ctx));  // (a call with statistics has synchronised already; kept explicit)
  ShardReduceResult res;
  res.decoded.emplace(n);
  cuda(cudaMemcpy(res.decoded->data(), d_out, n * 4, cudaMemcpyDeviceToHost), "D2H out");
  for (uint32_t r = 0; r < w; ++r)
    cuda(cudaMemcpy(accs[r].values.data(), da[r], n * 4, cudaMemcpyDeviceToHost), "D2H acc");
  if (collect_audit) {
    res.audit_exchanged_sum.emplace(n);
    cuda(cudaMemcpy(res.audit_exchanged_sum->data(), d_audit, n * 4, cudaMemcpyDeviceToHost), "D2H audit");
  }
  res.stats.presence = st.presence;
  res.stats.peeled = st.peeled;
  res.stats.unresolved = st.unresolved;
  res.stats.index_lost = st.index_lost;
  res.stats.index_spurious = st.index_spurious;
  res.stats.compressed_segments = st.compressed_segments;
  res.stats.baseline_segments = st.baseline_segments;
  replay_ledger(ctx, world);
  return res;
}

CommVolume comm_volume_model(const CompressionConfig& config, std::uint32_t world_size,
                             std::optional<std::uint64_t> n) {
  const tagc_config cfg = to_c(config);
  tagc_comm_volume v;
  check(tagc_comm_volume_model(&cfg, world_size, n.value_or(0), &v));
  return CommVolume{v.index_bits, v.sketch_bits, v.total_bits, v.factor};
}

CommVolume lhc_comm_volume_model(const CompressionConfig& config, std::uint32_t world_size,
                                 std::optional<std::uint64_t> n) {
  const tagc_config cfg = to_c(config);
  tagc_comm_volume v;
  check(tagc_lhc_comm_volume_model(&cfg, world_size, n.value_or(0), &v));
  return CommVolume{v.index_bits, v.sketch_bits, v.total_bits, v.factor};
}

}  // namespace tagc
