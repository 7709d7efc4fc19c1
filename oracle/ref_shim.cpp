// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libtagc_ref.so.
//
// TEST INFRASTRUCTURE ONLY: it exists so tests can pin the C restatement
// (oracle/tagc_oracle.c) against the reference's own outputs, and so
// bench.py --impl reference can time the reference's tagc_reduce_shard on the
// box's host cores. Struct types are borrowed from tagc_oracle.h (plain C).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "tagc/kernels.hpp"
#include "tagc/collectives.hpp"
#include "tagc/config.hpp"
#include "tagc/decode.hpp"
#include "tagc/hash.hpp"
#include "tagc/hook.hpp"
#include "tagc/index.hpp"
#include "tagc/layers.hpp"
#include "tagc/model.hpp"
#include "tagc/roundtrip.hpp"
#include "tagc/sketch.hpp"
#include "tagc/sparsify.hpp"
#include "tagc/train.hpp"
#include "tagc_oracle.h"

using namespace tagc;

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 2;
  } catch (const std::exception&) {
    return 1;
  }
}

CompressionConfig to_config(const or_config* c) {
  CompressionConfig out;
  out.theta = c->theta;
  out.ratio = c->ratio;
  out.index_width = c->index_width;
  out.policy = static_cast<Policy>(c->policy);
  out.include_out_proj = c->include_out_proj != 0;
  out.seed = c->seed;
  out.sketch_rows = c->sketch_rows;
  out.allow_low_theta = c->allow_low_theta != 0;
  out.min_compress_segment = c->min_compress_segment;
  return out;
}

ShardSpec to_shard(const or_shard* s) {
  ShardSpec out;
  out.id = s->id;
  out.owner = s->owner;
  out.begin = s->begin;
  out.end = s->end;
  for (uint32_t i = 0; i < s->num_segments; ++i) {
    const or_segment& g = s->segments[i];
    out.segments.push_back({"seg" + std::to_string(i), static_cast<LayerKind>(g.kind), g.begin, g.end});
  }
  return out;
}

CountSketch make_sketch(const float* v, uint32_t n, uint32_t ratio, uint32_t rows, uint64_t seed) {
  CountSketch s = CountSketch::zeros(sketch_geometry(n, ratio, rows), seed);
  std::memcpy(s.values.data(), v, s.values.size() * sizeof(float));
  return s;
}

void copy_str(const std::string& s, char* buf, size_t len) {
  if (!buf || len == 0) return;
  const size_t k = std::min(len - 1, s.size());
  std::memcpy(buf, s.data(), k);
  buf[k] = 0;
}

}  // namespace

extern "C" {

uint64_t ref_splitmix64(uint64_t x) { return splitmix64(x); }
uint32_t ref_bucket(uint64_t seed, uint32_t row, uint32_t p, uint32_t m) {
  return RowHash(seed, row).bucket(p, m);
}
float ref_sign(uint64_t seed, uint32_t row, uint32_t p) { return RowHash(seed, row).sign(p); }

int ref_stream(uint64_t n, double mu, double sigma, uint64_t seed, uint32_t count, float* out) {
  return guarded([&] {
    SyntheticStream s({static_cast<std::size_t>(n), mu, sigma, seed});
    for (uint32_t c = 0; c < count; ++c) {
      const std::vector<float> v = s.next();
      std::memcpy(out + static_cast<size_t>(c) * n, v.data(), n * sizeof(float));
    }
  });
}

int ref_sparsify(const float* g, size_t n, double theta, float* sparse, float* residual,
                 float* tau, uint64_t* zero_count) {
  return guarded([&] {
    SparsifyResult r = sparsify(std::span<const float>(g, n), theta);
    std::memcpy(sparse, r.sparse.data(), n * sizeof(float));
    std::memcpy(residual, r.residual.data(), n * sizeof(float));
    *tau = r.tau;
    *zero_count = r.zero_count;
  });
}

int ref_index_create(const float* v, uint32_t n, uint32_t w, uint32_t* words) {
  return guarded([&] {
    const Index idx = Index::create(std::span<const float>(v, n), w);
    std::memcpy(words, idx.words.data(), idx.words.size() * 4);
  });
}

int ref_merge_indices(const uint32_t* const* words, uint32_t world, uint32_t n, uint32_t w,
                      uint32_t* out) {
  return guarded([&] {
    std::vector<Index> locals;
    for (uint32_t r = 0; r < world; ++r) {
      Index idx = Index::zeros(n, w);
      std::memcpy(idx.words.data(), words[r], idx.words.size() * 4);
      locals.push_back(std::move(idx));
    }
    const Index merged = merge_indices(locals);
    std::memcpy(out, merged.words.data(), merged.words.size() * 4);
  });
}

int ref_index_presence(const uint32_t* words, uint32_t n, uint32_t w, uint32_t* out,
                       uint32_t* count) {
  return guarded([&] {
    Index idx = Index::zeros(n, w);
    std::memcpy(idx.words.data(), words, idx.words.size() * 4);
    const std::vector<uint32_t> p = idx.presence();
    std::memcpy(out, p.data(), p.size() * 4);
    *count = static_cast<uint32_t>(p.size());
  });
}

int ref_index_debug_json(const float* v, uint32_t n, uint32_t w, char* buf, size_t len) {
  return guarded([&] { copy_str(Index::create(std::span<const float>(v, n), w).debug_json().dump(), buf, len); });
}

int ref_sketch_compress(const float* v, uint32_t n, uint32_t ratio, uint32_t rows, uint64_t seed,
                        float* out) {
  return guarded([&] {
    const CountSketch s =
        CountSketch::compress(std::span<const float>(v, n), sketch_geometry(n, ratio, rows), seed);
    std::memcpy(out, s.values.data(), s.values.size() * sizeof(float));
  });
}

// TrafficLedger::to_csv / to_json().dump() (collectives.cpp:70-93) of a
// ledger fed the given records; also bits_per_param_per_rank(prefix).
int ref_ledger_dump(const int32_t* ops, const char* const* tags, const uint64_t* bits, const uint64_t* params,
                    uint32_t n, const char* prefix, char* csv, size_t csv_len, char* json, size_t json_len,
                    double* bpp) {
  return guarded([&] {
    TrafficLedger l;
    for (uint32_t i = 0; i < n; ++i) l.record(static_cast<CollectiveOp>(ops[i]), tags[i], bits[i], params[i]);
    std::ostringstream os;
    l.to_csv(os);
    copy_str(os.str(), csv, csv_len);
    copy_str(l.to_json().dump(), json, json_len);
    *bpp = l.bits_per_param_per_rank(prefix);
  });
}

// Index::to_bytes / CountSketch::to_bytes (index.cpp:59-69, sketch.cpp:77-89).
int ref_index_to_bytes(const float* v, uint32_t n, uint32_t w, uint8_t* out) {
  return guarded([&] {
    const std::vector<uint8_t> b = Index::create(std::span<const float>(v, n), w).to_bytes();
    std::memcpy(out, b.data(), b.size());
  });
}
int ref_sketch_to_bytes(const float* v, uint32_t n, uint32_t ratio, uint32_t rows, uint64_t seed, uint8_t* out) {
  return guarded([&] {
    const std::vector<uint8_t> b =
        CountSketch::compress(std::span<const float>(v, n), sketch_geometry(n, ratio, rows), seed).to_bytes();
    std::memcpy(out, b.data(), b.size());
  });
}

// The SGD step of the owner-side consumer (train.cpp:205-207).
int ref_scale_sub_inplace(float* dst, const float* src, size_t n, float scale) {
  return guarded([&] {
    tagc::kernels::scale_sub_inplace(std::span<float>(dst, n), std::span<const float>(src, n), scale,
                                     tagc::kernels::Exec::serial);
  });
}

int ref_sketch_debug_json(const float* v, uint32_t n, uint32_t ratio, uint32_t rows,
                          uint64_t seed, char* buf, size_t len) {
  return guarded([&] {
    const CountSketch s =
        CountSketch::compress(std::span<const float>(v, n), sketch_geometry(n, ratio, rows), seed);
    copy_str(s.debug_json().dump(), buf, len);
  });
}

int ref_peeling_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                           uint32_t rows, uint64_t seed, const float* sketch, float* values,
                           uint32_t* unresolved, uint32_t* n_unresolved, double* pf) {
  return guarded([&] {
    const CountSketch s = make_sketch(sketch, n, ratio, rows, seed);
    const DecodeResult r =
        peeling_decompress(std::span<const uint32_t>(presence, count), s);
    std::memcpy(values, r.values.data(), n * sizeof(float));
    std::memcpy(unresolved, r.unresolved.data(), r.unresolved.size() * 4);
    *n_unresolved = static_cast<uint32_t>(r.unresolved.size());
    *pf = r.peeled_fraction;
  });
}

int ref_estimation_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                              uint32_t rows, uint64_t seed, const float* sketch,
                              const uint32_t* targets, uint32_t nt, float* out) {
  return guarded([&] {
    const CountSketch s = make_sketch(sketch, n, ratio, rows, seed);
    const std::vector<float> e = estimation_decompress(std::span<const uint32_t>(presence, count), s,
                                                       std::span<const uint32_t>(targets, nt));
    std::memcpy(out, e.data(), nt * sizeof(float));
  });
}

// mode: 0 = sequential world, 1 = parallel world (collectives.hpp:171)
int ref_tagc_reduce_shard(const or_shard* shard, const float* const* grads, float* const* accs,
                          uint32_t world, const or_config* config, int mode, float* decoded,
                          or_peel_stats* stats, char* ledger_csv, size_t csv_len) {
  return guarded([&] {
    const ShardSpec sh = to_shard(shard);
    const uint64_t len = sh.size();
    std::vector<std::vector<float>> g(world);
    std::vector<ResidualAccumulator> acc(world, ResidualAccumulator(len));
    for (uint32_t r = 0; r < world; ++r) {
      g[r].assign(grads[r], grads[r] + len);
      std::memcpy(acc[r].values.data(), accs[r], len * sizeof(float));
    }
    World w(world, mode ? WorldMode::parallel : WorldMode::sequential);
    const ShardReduceResult res = tagc_reduce_shard(sh, g, acc, to_config(config), w);
    for (uint32_t r = 0; r < world; ++r) std::memcpy(accs[r], acc[r].values.data(), len * sizeof(float));
    std::memcpy(decoded, res.decoded->data(), len * sizeof(float));
    stats->presence = res.stats.presence;
    stats->peeled = res.stats.peeled;
    stats->unresolved = res.stats.unresolved;
    stats->index_lost = res.stats.index_lost;
    stats->index_spurious = res.stats.index_spurious;
    stats->compressed_segments = res.stats.compressed_segments;
    stats->baseline_segments = res.stats.baseline_segments;
    if (ledger_csv) {
      std::ostringstream os;
      w.ledger().to_csv(os);
      copy_str(os.str(), ledger_csv, csv_len);
    }
  });
}

// tagc_reduce_shard(..., collect_audit = true): the decoded shard and
// ShardReduceResult::audit_exchanged_sum (hook.cpp:191-195).
int ref_tagc_reduce_shard_audit(const or_shard* shard, const float* const* grads, float* const* accs,
                                uint32_t world, const or_config* config, float* decoded, float* audit) {
  return guarded([&] {
    const ShardSpec sh = to_shard(shard);
    const uint64_t len = sh.size();
    std::vector<std::vector<float>> g(world);
    std::vector<ResidualAccumulator> acc(world, ResidualAccumulator(len));
    for (uint32_t r = 0; r < world; ++r) {
      g[r].assign(grads[r], grads[r] + len);
      std::memcpy(acc[r].values.data(), accs[r], len * sizeof(float));
    }
    World w(world, WorldMode::sequential);
    const ShardReduceResult res = tagc_reduce_shard(sh, g, acc, to_config(config), w, true);
    for (uint32_t r = 0; r < world; ++r) std::memcpy(accs[r], acc[r].values.data(), len * sizeof(float));
    std::memcpy(decoded, res.decoded->data(), len * sizeof(float));
    std::memcpy(audit, res.audit_exchanged_sum->data(), len * sizeof(float));
  });
}

// Timing entry for bench.py --impl reference: the caller's buffers are
// converted to the reference's containers OUTSIDE the timed region, and only
// tagc_reduce_shard itself is timed (BASELINE.md §2 "What is timed").
int ref_time_reduce_shards(const or_shard* shards, uint32_t n_shards, const float* const* grads,
                           uint32_t world, const or_config* config, int reps, double* seconds) {
  return guarded([&] {
    std::vector<ShardSpec> specs;
    for (uint32_t s = 0; s < n_shards; ++s) specs.push_back(to_shard(&shards[s]));
    std::vector<std::vector<std::vector<float>>> g(n_shards);
    std::vector<std::vector<ResidualAccumulator>> acc(n_shards);
    for (uint32_t s = 0; s < n_shards; ++s) {
      const uint64_t len = specs[s].size();
      for (uint32_t r = 0; r < world; ++r)
        g[s].emplace_back(grads[r] + specs[s].begin, grads[r] + specs[s].begin + len);
      acc[s].assign(world, ResidualAccumulator(len));
    }
    const CompressionConfig cfg = to_config(config);
    double best = 1e300;
    for (int rep = 0; rep < reps; ++rep) {
      World w(world, WorldMode::parallel);
      const auto t0 = std::chrono::steady_clock::now();
      for (uint32_t s = 0; s < n_shards; ++s) tagc_reduce_shard(specs[s], g[s], acc[s], cfg, w);
      const double dt =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      seconds[rep] = dt;
      best = std::min(best, dt);
    }
  });
}

int ref_baseline_reduce_shard(const or_shard* shard, const float* const* grads, uint32_t world,
                              float* out) {
  return guarded([&] {
    const ShardSpec sh = to_shard(shard);
    std::vector<std::vector<float>> g(world);
    for (uint32_t r = 0; r < world; ++r) g[r].assign(grads[r], grads[r] + sh.size());
    World w(world, WorldMode::sequential);
    const std::vector<float> res = baseline_reduce_shard(sh, g, w);
    std::memcpy(out, res.data(), res.size() * sizeof(float));
  });
}

int ref_config_validate(const or_config* c, uint32_t world) {
  return guarded([&] { to_config(c).validate_for_world(world); });
}

int ref_comm_volume(const or_config* c, uint32_t world, uint64_t n, int lhc, double* out4) {
  return guarded([&] {
    const std::optional<std::uint64_t> nn = n ? std::optional<std::uint64_t>(n) : std::nullopt;
    const CommVolume v = lhc ? lhc_comm_volume_model(to_config(c), world, nn)
                             : comm_volume_model(to_config(c), world, nn);
    out4[0] = v.index_bits;
    out4[1] = v.sketch_bits;
    out4[2] = v.total_bits;
    out4[3] = v.factor;
  });
}

int ref_model_layer_specs(uint32_t layers, uint32_t d_model, uint32_t heads, uint32_t ffn_mult,
                          uint32_t vocab, uint32_t ctx, int untied, uint64_t* counts,
                          int32_t* kinds, uint32_t cap, uint32_t* n) {
  return guarded([&] {
    TinyModelConfig c;
    c.layers = layers;
    c.d_model = d_model;
    c.heads = heads;
    c.ffn_mult = ffn_mult;
    c.vocab = vocab;
    c.ctx = ctx;
    c.untied_head = untied != 0;
    const std::vector<LayerSpec> specs = model_layer_specs(c);
    *n = static_cast<uint32_t>(specs.size());
    for (uint32_t i = 0; i < specs.size() && i < cap; ++i) {
      counts[i] = specs[i].param_count;
      kinds[i] = static_cast<int32_t>(specs[i].kind);
    }
  });
}

int ref_make_shards(const uint64_t* counts, const int32_t* kinds, uint32_t n_layers,
                    uint32_t shard_count, uint32_t world, uint64_t* shard_len, or_segment* segs,
                    uint32_t* seg_shard, uint32_t cap, uint32_t* n_segments) {
  return guarded([&] {
    std::vector<LayerSpec> layers;
    for (uint32_t i = 0; i < n_layers; ++i)
      layers.push_back({"l" + std::to_string(i), static_cast<LayerKind>(kinds[i]), counts[i]});
    const std::vector<ShardSpec> shards = make_shards(layers, shard_count, world);
    *shard_len = shards[0].size();
    uint32_t k = 0;
    for (const ShardSpec& sh : shards) {
      for (const LayerSegment& s : sh.segments) {
        if (k < cap) {
          segs[k].kind = static_cast<int32_t>(s.kind);
          segs[k].begin = s.begin;
          segs[k].end = s.end;
          seg_shard[k] = sh.id;
        }
        ++k;
      }
    }
    *n_segments = k;
  });
}

// roundtrip.cpp:31-144 — out: mean_pf, min_pf, max_rel_resolved, max_rel_any;
// counts: trials_fully_peeled, presence_total, unresolved_total, index_lost,
// index_spurious, integer_exact, pass
// Trial t of roundtrip_experiment (roundtrip.cpp:65-95): the per-rank
// gradients and the trial's compression seed, drawn with the reference's own
// Rng / splitmix64 in the reference's draw order. sample_support
// (roundtrip.cpp:17-28) is file-static in the reference, so its partial
// Fisher-Yates is restated here; tests pin this generator by reproducing the
// reference's roundtrip reports from it (tests/test_oracle.py).
int ref_roundtrip_trial(uint32_t n, double theta, uint32_t world, uint64_t seed, uint32_t t, float* grads,
                        uint64_t* trial_seed) {
  return guarded([&] {
    const uint32_t zeros = static_cast<uint32_t>(std::ceil(theta * static_cast<double>(n) / 100.0));
    const uint32_t support = n - std::min(zeros, n);
    Rng rng(splitmix64(seed + 0x9E3779B97F4A7C15ULL * (t + 1)));
    const bool integer_trial = (t % 2 == 0);
    std::vector<uint32_t> all(n);
    for (uint32_t i = 0; i < n; ++i) all[i] = i;
    for (uint32_t i = 0; i < support; ++i) {
      const uint32_t j = i + static_cast<uint32_t>(rng.next_below(n - i));
      std::swap(all[i], all[j]);
    }
    all.resize(support);
    std::sort(all.begin(), all.end());
    std::memset(grads, 0, sizeof(float) * size_t(world) * n);
    for (uint32_t p : all) {
      const uint64_t mask = rng.next_below((1ull << world) - 1) + 1;
      for (uint32_t r = 0; r < world; ++r) {
        if (!(mask >> r & 1)) continue;
        float v;
        if (integer_trial) {
          v = static_cast<float>(1 + static_cast<int>(rng.next_below(16)));
          if (rng.next_u64() & 1) v = -v;
        } else {
          do {
            v = static_cast<float>(rng.next_double() * 2.0 - 1.0);
          } while (v == 0.0f);
        }
        grads[size_t(r) * n + p] = v;
      }
    }
    *trial_seed = rng.next_u64();
  });
}

int ref_roundtrip(uint32_t n, uint32_t trials, double theta, uint32_t ratio, uint32_t width,
                  uint32_t world, uint32_t rows, uint64_t seed, double* out4, uint64_t* counts7) {
  return guarded([&] {
    RoundtripParams p;
    p.n = n;
    p.trials = trials;
    p.theta = theta;
    p.ratio = ratio;
    p.index_width = width;
    p.world_size = world;
    p.sketch_rows = rows;
    p.seed = seed;
    const RoundtripReport r = roundtrip_experiment(p);
    out4[0] = r.mean_peeled_fraction;
    out4[1] = r.min_peeled_fraction;
    out4[2] = r.max_rel_error_resolved;
    out4[3] = r.max_rel_error_any;
    counts7[0] = r.trials_fully_peeled;
    counts7[1] = r.presence_total;
    counts7[2] = r.unresolved_total;
    counts7[3] = r.index_lost;
    counts7[4] = r.index_spurious;
    counts7[5] = r.integer_exact_when_resolved;
    counts7[6] = r.pass;
  });
}

}  // extern "C"
