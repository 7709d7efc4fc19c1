/*
 * tagc_oracle.h — CPU restatement of the TAGC compressed gradient-exchange
 * path (reference: /root/reference/proj, C++20).
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the
 * B200 CUDA path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. The product (paper_2504_05638_b200) never
 * links or calls it.
 *
 * Every function is a sequential restatement of the reference algorithm in
 * plain C and cites the reference file:line it follows. Sequential folds keep
 * the reference's float summation order (ascending position inside a sketch
 * row, ascending rank across ranks, FIFO peel order), so outputs are
 * bit-identical to the reference, which tests/test_oracle_vs_ref.py pins
 * against fixtures generated from the compiled reference (oracle/_ref).
 *
 * Status codes mirror the reference's error convention (cli.cpp:375-382):
 *   0 = ok, 2 = invalid argument (std::invalid_argument), 1 = runtime error.
 */
#ifndef TAGC_ORACLE_H
#define TAGC_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_RUNTIME = 1, OR_INVALID = 2 };

/* ---- hash family (hash.hpp) ---- */
uint64_t or_splitmix64(uint64_t x);
typedef struct or_rowhash {
  uint64_t pos_a, pos_b, sgn_a, sgn_b;
} or_rowhash;
void or_rowhash_init(or_rowhash* h, uint64_t seed, uint32_t row);
uint32_t or_bucket(const or_rowhash* h, uint32_t position, uint32_t m);
float or_sign(const or_rowhash* h, uint32_t position);

/* ---- deterministic RNG (hash.hpp:52-76) and SyntheticStream (train.cpp:445-459) ---- */
typedef struct or_rng {
  uint64_t state;
} or_rng;
uint64_t or_rng_next_u64(or_rng* r);
double or_rng_next_double(or_rng* r);
uint64_t or_rng_next_below(or_rng* r, uint64_t bound);
double or_rng_normal(or_rng* r);
typedef struct or_stream {
  uint64_t n;
  double mu, sigma;
  or_rng rng;
} or_stream;
int or_stream_init(or_stream* s, uint64_t n, double mu, double sigma, uint64_t seed);
void or_stream_next(or_stream* s, float* out);

/* ---- config / policy (config.cpp:27-59, layers.cpp:42-65) ---- */
enum { OR_POLICY_ALL_LAYERS = 0, OR_POLICY_NON_ATTENTION_LINEAR = 1, OR_POLICY_NONE = 2 };
enum {
  OR_KIND_EMBEDDING = 0,
  OR_KIND_POSITIONAL_EMBEDDING = 1,
  OR_KIND_ATTENTION_QKV = 2,
  OR_KIND_ATTENTION_OUT_PROJ = 3,
  OR_KIND_FEED_FORWARD = 4,
  OR_KIND_LM_HEAD = 5,
  OR_KIND_NORM = 6,
  OR_KIND_BIAS = 7,
  OR_KIND_OTHER = 8
};
typedef struct or_config {
  double theta;
  uint32_t ratio;
  uint32_t index_width;
  int32_t policy;
  int32_t include_out_proj;
  uint64_t seed;
  uint32_t sketch_rows;
  int32_t allow_low_theta;
  uint64_t min_compress_segment;
} or_config;
int or_config_validate(const or_config* c, uint32_t world_size);
int or_kind_compressible(int32_t kind, int32_t policy, int32_t include_out_proj);

/* ---- elementwise loops (kernels.cpp) ---- */
void or_add_inplace(float* dst, const float* src, size_t n);
void or_rank_sum(float* out, const float* const* inputs, uint32_t world, size_t n);
void or_rank_sum_words(uint32_t* out, const uint32_t* const* inputs, uint32_t world, size_t n);

/* ---- owner-side consumer (train.cpp:355-359, 202-220) ----
 * decoded *= 1/W, then SGD (kind 0: params -= lr * g) or the momentum-free
 * AdamW (kind 1: v = b2 v + (1-b2) g g; params -= lr (g / (sqrt(v / (1 - b2^step)) + eps) + wd params)).
 * decoded is scaled in place, as the reference does. */
void or_apply_optimizer(int32_t kind, float lr, float weight_decay, uint32_t world, uint32_t step, float* params,
                        float* decoded, float* adam_v, size_t n);
void or_threshold_split(const float* g, size_t n, float tau, float* sparse, float* residual);

/* ---- sparsify (sparsify.cpp:18-49) ---- */
int or_sparsify(const float* g, size_t n, double theta, float* sparse, float* residual,
                float* tau, uint64_t* zero_count);

/* ---- index (index.cpp) ---- */
uint32_t or_words_needed(uint32_t n, uint32_t width);
int or_index_create(const float* values, uint32_t n, uint32_t width, uint32_t* words);
uint32_t or_index_field(const uint32_t* words, uint32_t width, uint32_t p);
/* Writes the presence list (ascending) into out (capacity n); returns count. */
uint32_t or_index_presence(const uint32_t* words, uint32_t n, uint32_t width, uint32_t* out);

/* ---- count sketch (sketch.cpp) ---- */
int or_sketch_geometry(uint32_t n, uint32_t ratio, uint32_t rows, uint32_t* buckets_per_row);
/* out: rows*m floats, row-major, overwritten */
int or_sketch_compress(const float* values, uint32_t n, uint32_t ratio, uint32_t rows,
                       uint64_t seed, float* out);

/* ---- decode (decode.cpp) ---- */
/* values: n floats (overwritten); unresolved: capacity `count`; returns status */
int or_peeling_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                          uint32_t rows, uint64_t seed, const float* sketch, float* values,
                          uint32_t* unresolved, uint32_t* n_unresolved, double* peeled_fraction);
int or_estimation_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                             uint32_t rows, uint64_t seed, const float* sketch,
                             const uint32_t* targets, uint32_t n_targets, float* out);

/* ---- hook (hook.cpp) ---- */
typedef struct or_segment {
  int32_t kind;
  uint64_t begin, end; /* global flat coordinates */
} or_segment;
typedef struct or_shard {
  uint32_t id, owner;
  uint64_t begin, end;
  const or_segment* segments;
  uint32_t num_segments;
} or_shard;
typedef struct or_peel_stats {
  uint64_t presence, peeled, unresolved, index_lost, index_spurious, compressed_segments,
      baseline_segments;
} or_peel_stats;

/* tagc_reduce_shard (hook.cpp:98-200) over a simulated W-rank world.
 * grads[r], accs[r]: shard.size() floats; accs mutated; decoded: shard.size(). */
int or_tagc_reduce_shard(const or_shard* shard, const float* const* grads, float* const* accs,
                         uint32_t world, const or_config* config, float* decoded,
                         or_peel_stats* stats);
/* baseline_reduce_shard (hook.cpp:90-96) */
int or_baseline_reduce_shard(const or_shard* shard, const float* const* grads, uint32_t world,
                             float* out);

/* make_shards (hook.cpp:30-61). layer_counts: param counts in layer order.
 * Two-phase: returns the number of segments via *n_segments; segments may be
 * NULL to size. Each output segment carries its shard id in seg_shard[i] and
 * its layer index in seg_layer[i] (-1 for "pad"). */
int or_make_shards(const uint64_t* layer_counts, const int32_t* layer_kinds, uint32_t n_layers,
                   uint32_t shard_count, uint32_t world_size, uint64_t* shard_len,
                   or_segment* segments, uint32_t* seg_shard, int32_t* seg_layer,
                   uint32_t* n_segments);

#ifdef __cplusplus
}
#endif
#endif
