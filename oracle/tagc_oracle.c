/*
 * tagc_oracle.c — sequential CPU restatement of the TAGC exchange path.
 * TEST INFRASTRUCTURE ONLY (see tagc_oracle.h). Citations are file:line into
 * /root/reference/proj.
 */
#include "tagc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ hash */

/* hash.hpp:15-20 */
uint64_t or_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

/* hash.hpp:27-33 — coefficient chain seeded by (seed, row) */
void or_rowhash_init(or_rowhash* h, uint64_t seed, uint32_t row) {
  uint64_t s = or_splitmix64(seed ^ (0xA24BAED4963EE407ULL * (uint64_t)(row + 1u)));
  h->pos_a = or_splitmix64(s) | 1ULL;
  h->pos_b = or_splitmix64(h->pos_a);
  h->sgn_a = or_splitmix64(h->pos_b) | 1ULL;
  h->sgn_b = or_splitmix64(h->sgn_a);
}

/* hash.hpp:35-38 */
uint32_t or_bucket(const or_rowhash* h, uint32_t position, uint32_t m) {
  uint64_t x = h->pos_a * ((uint64_t)position + 0x9E3779B9ULL) + h->pos_b;
  return (uint32_t)((x >> 32) % m);
}

/* hash.hpp:40-43 */
float or_sign(const or_rowhash* h, uint32_t position) {
  uint64_t x = h->sgn_a * ((uint64_t)position + 0x85EBCA77ULL) + h->sgn_b;
  return (x >> 63) ? 1.0f : -1.0f;
}

/* ------------------------------------------------------------------- rng */

/* hash.hpp:56 */
uint64_t or_rng_next_u64(or_rng* r) { return or_splitmix64(r->state++); }
/* hash.hpp:61 */
double or_rng_next_double(or_rng* r) { return (double)(or_rng_next_u64(r) >> 11) * 0x1.0p-53; }
/* hash.hpp:64 */
uint64_t or_rng_next_below(or_rng* r, uint64_t bound) { return or_rng_next_u64(r) % bound; }
/* hash.hpp:71-76 (Box-Muller) */
double or_rng_normal(or_rng* r) {
  double u1 = or_rng_next_double(r);
  while (u1 <= 0.0) u1 = or_rng_next_double(r);
  const double u2 = or_rng_next_double(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* train.cpp:445-449 */
int or_stream_init(or_stream* s, uint64_t n, double mu, double sigma, uint64_t seed) {
  if (n == 0 || sigma < 0.0) return OR_INVALID;
  s->n = n;
  s->mu = mu;
  s->sigma = sigma;
  s->rng.state = or_splitmix64(seed ^ 0xD1B54A32D192ED03ULL);
  return OR_OK;
}

/* train.cpp:451-459 — log-normal magnitude, fair sign */
void or_stream_next(or_stream* s, float* out) {
  for (uint64_t i = 0; i < s->n; ++i) {
    const double mag = exp(s->mu + s->sigma * or_rng_normal(&s->rng));
    const int negative = (or_rng_next_u64(&s->rng) & 1) != 0;
    out[i] = (float)(negative ? -mag : mag);
  }
}

/* ---------------------------------------------------------------- config */

/* config.cpp:27-35 */
static int theta_floor(uint32_t ratio, double* floor_out) {
  switch (ratio) {
    case 1: *floor_out = 0.0; return OR_OK;
    case 2: *floor_out = 80.0; return OR_OK;
    case 4: *floor_out = 90.0; return OR_OK;
    case 10: *floor_out = 98.75; return OR_OK;
    default: return OR_INVALID;
  }
}

/* config.cpp:37-59 (validate + validate_for_world) */
int or_config_validate(const or_config* c, uint32_t world_size) {
  double floor;
  if (!(c->theta >= 0.0 && c->theta <= 100.0)) return OR_INVALID;
  if (c->index_width != 1 && c->index_width != 4) return OR_INVALID;
  if (c->sketch_rows == 0) return OR_INVALID;
  if (theta_floor(c->ratio, &floor) != OR_OK) return OR_INVALID;
  if (c->ratio > 1 && c->theta < floor && !c->allow_low_theta) return OR_INVALID;
  if (c->ratio > 1 && c->index_width == 4 && world_size > 15) return OR_INVALID;
  return OR_OK;
}

/* layers.cpp:42-65 */
int or_kind_compressible(int32_t kind, int32_t policy, int32_t include_out_proj) {
  switch (policy) {
    case OR_POLICY_NONE: return 0;
    case OR_POLICY_ALL_LAYERS: return 1;
    case OR_POLICY_NON_ATTENTION_LINEAR:
      switch (kind) {
        case OR_KIND_EMBEDDING:
        case OR_KIND_POSITIONAL_EMBEDDING:
        case OR_KIND_FEED_FORWARD:
        case OR_KIND_LM_HEAD: return 1;
        case OR_KIND_ATTENTION_OUT_PROJ: return include_out_proj != 0;
        default: return 0;
      }
    default: return 0;
  }
}

/* --------------------------------------------------------------- kernels */

/* kernels.cpp:21-30 */
void or_add_inplace(float* dst, const float* src, size_t n) {
  for (size_t i = 0; i < n; ++i) dst[i] += src[i];
}

/* kernels.cpp:43-63 — ascending-rank fold per element */
void or_rank_sum(float* out, const float* const* inputs, uint32_t world, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    float acc = 0.0f;
    for (uint32_t r = 0; r < world; ++r) acc += inputs[r][i];
    out[i] = acc;
  }
}

/* kernels.cpp:65-84 — wrapping u32 fold */
void or_rank_sum_words(uint32_t* out, const uint32_t* const* inputs, uint32_t world, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    uint32_t acc = 0;
    for (uint32_t r = 0; r < world; ++r) acc += inputs[r][i];
    out[i] = acc;
  }
}

/* kernels.cpp:86-107 — drop iff v<=tau && v>=-tau (kernels.cpp:95) */
void or_threshold_split(const float* g, size_t n, float tau, float* sparse, float* residual) {
  for (size_t i = 0; i < n; ++i) {
    const float v = g[i];
    const int drop = (v <= tau && v >= -tau);
    sparse[i] = drop ? 0.0f : v;
    residual[i] = drop ? v : 0.0f;
  }
}

/* -------------------------------------------------------------- sparsify */

/* Exact k-th smallest (0-based) of non-negative, non-NaN floats. The order of
 * such floats equals the order of their IEEE bit patterns, so an LSD-free MSD
 * radix select on the bits returns exactly the value nth_element returns at
 * sparsify.cpp:35-36. */
static float select_kth_nonneg(const float* mags, size_t n, size_t k) {
  uint32_t prefix = 0, mask = 0;
  size_t rank = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    size_t hist[256];
    memset(hist, 0, sizeof(hist));
    for (size_t i = 0; i < n; ++i) {
      uint32_t b;
      memcpy(&b, &mags[i], 4);
      if ((b & mask) == prefix) hist[(b >> shift) & 0xFFu]++;
    }
    uint32_t d = 0;
    while (rank >= hist[d]) {
      rank -= hist[d];
      ++d;
    }
    prefix |= d << shift;
    mask |= 0xFFu << shift;
  }
  float out;
  memcpy(&out, &prefix, 4);
  return out;
}

/* sparsify.cpp:18-49 */
int or_sparsify(const float* g, size_t n, double theta, float* sparse, float* residual,
                float* tau_out, uint64_t* zero_count) {
  if (!(theta >= 0.0 && theta <= 100.0)) return OR_INVALID; /* :19-20 */
  if (n == 0) return OR_INVALID;                              /* :21 */
  float* mags = (float*)malloc(n * sizeof(float));
  if (!mags) return OR_RUNTIME;
  for (size_t i = 0; i < n; ++i) { /* :24-28 */
    if (isnan(g[i])) {
      free(mags);
      return OR_INVALID;
    }
    mags[i] = fabsf(g[i]);
  }
  size_t c = (size_t)ceil(theta * (double)n / 100.0); /* :30 */
  if (c > n) c = n;                                   /* :31 */
  float tau = 0.0f;
  if (c > 0) tau = select_kth_nonneg(mags, n, c - 1); /* :33-37 */
  free(mags);
  or_threshold_split(g, n, tau, sparse, residual); /* :43 */
  uint64_t zc = 0;
  for (size_t i = 0; i < n; ++i)
    if (sparse[i] == 0.0f) ++zc; /* :44-47 */
  if (tau_out) *tau_out = tau;
  if (zero_count) *zero_count = zc;
  return OR_OK;
}

/* ----------------------------------------------------------------- index */

/* index.cpp:17-20 */
uint32_t or_words_needed(uint32_t n, uint32_t width) {
  const uint64_t bits = (uint64_t)n * width;
  return (uint32_t)((bits + 31) / 32);
}

/* index.cpp:32-41 — field set iff values[p] != 0 (-0 stays clear) */
int or_index_create(const float* values, uint32_t n, uint32_t width, uint32_t* words) {
  if (width != 1 && width != 4) return OR_INVALID;
  if (n == 0) return OR_INVALID;
  memset(words, 0, (size_t)or_words_needed(n, width) * 4);
  for (uint32_t p = 0; p < n; ++p) {
    if (values[p] != 0.0f) {
      const uint64_t bit = (uint64_t)p * width;
      words[bit >> 5] |= 1u << (bit & 31);
    }
  }
  return OR_OK;
}

/* index.cpp:43-49 */
uint32_t or_index_field(const uint32_t* words, uint32_t width, uint32_t p) {
  const uint64_t bit = (uint64_t)p * width;
  const uint32_t mask = (width == 1) ? 1u : 0xFu;
  return (words[bit >> 5] >> (bit & 31)) & mask;
}

/* index.cpp:51-57 */
uint32_t or_index_presence(const uint32_t* words, uint32_t n, uint32_t width, uint32_t* out) {
  uint32_t cnt = 0;
  for (uint32_t p = 0; p < n; ++p)
    if (or_index_field(words, width, p) != 0) out[cnt++] = p;
  return cnt;
}

/* ---------------------------------------------------------------- sketch */

/* sketch.cpp:11-27 */
int or_sketch_geometry(uint32_t n, uint32_t ratio, uint32_t rows, uint32_t* m) {
  if (ratio != 2 && ratio != 4 && ratio != 10) return OR_INVALID;
  if (rows == 0 || n == 0) return OR_INVALID;
  const uint32_t mm = n / (ratio * rows);
  if (mm == 0) return OR_INVALID;
  *m = mm;
  return OR_OK;
}

/* sketch.cpp:37-67 — per row, ascending position: row[h(p)] += s(p)*v */
int or_sketch_compress(const float* values, uint32_t n, uint32_t ratio, uint32_t rows,
                       uint64_t seed, float* out) {
  uint32_t m;
  int st = or_sketch_geometry(n, ratio, rows, &m);
  if (st != OR_OK) return st;
  memset(out, 0, (size_t)rows * m * sizeof(float));
  for (uint32_t r = 0; r < rows; ++r) {
    or_rowhash h;
    or_rowhash_init(&h, seed, r);
    float* row = out + (size_t)r * m;
    for (uint32_t p = 0; p < n; ++p) {
      const float v = values[p];
      if (v != 0.0f) row[or_bucket(&h, p, m)] += or_sign(&h, p) * v;
    }
  }
  return OR_OK;
}

/* ---------------------------------------------------------------- decode */

static void sort_floats_small(float* a, uint32_t k) {
  for (uint32_t i = 1; i < k; ++i) {
    float x = a[i];
    uint32_t j = i;
    while (j > 0 && x < a[j - 1]) {
      a[j] = a[j - 1];
      --j;
    }
    a[j] = x;
  }
}

/* decode.cpp:24-51 — median-of-rows estimator (middle order statistic) */
int or_estimation_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                             uint32_t rows, uint64_t seed, const float* sketch,
                             const uint32_t* targets, uint32_t n_targets, float* out) {
  uint32_t m;
  int st = or_sketch_geometry(n, ratio, rows, &m);
  if (st != OR_OK) return st;
  for (uint32_t i = 0; i < count; ++i)
    if (presence[i] >= n) return OR_INVALID; /* decode.cpp:15-20 */
  uint8_t* in_presence = (uint8_t*)calloc(n, 1);
  or_rowhash* hs = (or_rowhash*)malloc(rows * sizeof(or_rowhash));
  float* est = (float*)malloc(rows * sizeof(float));
  if (!in_presence || !hs || !est) {
    free(in_presence);
    free(hs);
    free(est);
    return OR_RUNTIME;
  }
  for (uint32_t i = 0; i < count; ++i) in_presence[presence[i]] = 1;
  st = OR_OK;
  for (uint32_t i = 0; i < n_targets; ++i) /* decode.cpp:30-33 */
    if (targets[i] >= n || !in_presence[targets[i]]) st = OR_INVALID;
  if (st == OR_OK) {
    for (uint32_t r = 0; r < rows; ++r) or_rowhash_init(&hs[r], seed, r);
    for (uint32_t i = 0; i < n_targets; ++i) {
      const uint32_t t = targets[i];
      for (uint32_t r = 0; r < rows; ++r)
        est[r] = or_sign(&hs[r], t) * sketch[(size_t)r * m + or_bucket(&hs[r], t, m)];
      sort_floats_small(est, rows);
      float e = est[rows / 2];
      if (e == 0.0f) e = 0.0f; /* decode.cpp:47 canonical zero */
      out[i] = e;
    }
  }
  free(in_presence);
  free(hs);
  free(est);
  return st;
}

/* decode.cpp:53-140 — FIFO peel over (count, key_sum) bucket state */
int or_peeling_decompress(const uint32_t* presence, uint32_t count, uint32_t n, uint32_t ratio,
                          uint32_t rows, uint64_t seed, const float* sketch, float* values,
                          uint32_t* unresolved, uint32_t* n_unresolved, double* peeled_fraction) {
  uint32_t m;
  int st = or_sketch_geometry(n, ratio, rows, &m);
  if (st != OR_OK) return st;
  for (uint32_t i = 0; i < count; ++i)
    if (presence[i] >= n) return OR_INVALID; /* :55 */
  memset(values, 0, (size_t)n * sizeof(float)); /* :60 */
  *n_unresolved = 0;
  if (count == 0) { /* :61-64 */
    *peeled_fraction = 1.0;
    return OR_OK;
  }
  const uint32_t k = rows;
  const size_t buckets = (size_t)k * m;
  or_rowhash* hs = (or_rowhash*)malloc(k * sizeof(or_rowhash));
  uint32_t* cnt = (uint32_t*)calloc(buckets, sizeof(uint32_t));
  uint64_t* key_sum = (uint64_t*)calloc(buckets, sizeof(uint64_t));
  float* residual = (float*)malloc(buckets * sizeof(float));
  uint32_t* slots = (uint32_t*)malloc((size_t)count * k * sizeof(uint32_t));
  uint32_t* pos_entry = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  uint8_t* recovered = (uint8_t*)calloc(count, 1);
  const size_t qcap = buckets + (size_t)count * k;
  uint32_t* queue = (uint32_t*)malloc(qcap * sizeof(uint32_t));
  if (!hs || !cnt || !key_sum || !residual || !slots || !pos_entry || !recovered || !queue) {
    st = OR_RUNTIME;
    goto done;
  }
  for (uint32_t r = 0; r < k; ++r) or_rowhash_init(&hs[r], seed, r);
  memcpy(residual, sketch, buckets * sizeof(float));
  for (uint32_t i = 0; i < count; ++i) { /* :79-88 */
    const uint32_t p = presence[i];
    for (uint32_t r = 0; r < k; ++r) {
      const uint32_t slot = r * m + or_bucket(&hs[r], p, m);
      slots[(size_t)i * k + r] = slot;
      cnt[slot] += 1;
      key_sum[slot] += p;
    }
  }
  for (uint32_t p = 0; p < n; ++p) pos_entry[p] = UINT32_MAX;
  for (uint32_t i = 0; i < count; ++i) { /* :89-94 duplicate check */
    if (pos_entry[presence[i]] != UINT32_MAX) {
      st = OR_INVALID;
      goto done;
    }
    pos_entry[presence[i]] = i;
  }
  size_t qh = 0, qt = 0;
  for (uint32_t slot = 0; slot < buckets; ++slot) /* :96-99 seed ascending */
    if (cnt[slot] == 1) queue[qt++] = slot;
  uint64_t peeled = 0;
  while (qh < qt) { /* :103-122 */
    const uint32_t slot = queue[qh++];
    if (cnt[slot] != 1) continue;
    const uint32_t p = (uint32_t)key_sum[slot];
    const uint32_t entry = pos_entry[p];
    const uint32_t row = slot / m;
    float value = or_sign(&hs[row], p) * residual[slot];
    if (value == 0.0f) value = 0.0f; /* :111 */
    values[p] = value;
    recovered[entry] = 1;
    ++peeled;
    for (uint32_t r = 0; r < k; ++r) {
      const uint32_t s = slots[(size_t)entry * k + r];
      residual[s] -= or_sign(&hs[r], p) * value;
      cnt[s] -= 1;
      key_sum[s] -= p;
      if (cnt[s] == 1) queue[qt++] = s;
    }
  }
  uint32_t nu = 0;
  for (uint32_t i = 0; i < count; ++i) /* :124-127 */
    if (!recovered[i]) unresolved[nu++] = presence[i];
  /* sort ascending (presence may be unsorted in the standalone API) */
  for (uint32_t i = 1; i < nu; ++i) {
    uint32_t x = unresolved[i], j = i;
    while (j > 0 && x < unresolved[j - 1]) {
      unresolved[j] = unresolved[j - 1];
      --j;
    }
    unresolved[j] = x;
  }
  *n_unresolved = nu;
  *peeled_fraction = (double)peeled / (double)count; /* :128 */
  if (nu > 0) {                                      /* :130-138 estimation on the residual */
    float* est = (float*)malloc((size_t)nu * sizeof(float));
    if (!est) {
      st = OR_RUNTIME;
      goto done;
    }
    st = or_estimation_decompress(presence, count, n, ratio, rows, seed, residual, unresolved, nu,
                                  est);
    if (st == OR_OK)
      for (uint32_t i = 0; i < nu; ++i) values[unresolved[i]] = est[i];
    free(est);
  }
done:
  free(hs);
  free(cnt);
  free(key_sum);
  free(residual);
  free(slots);
  free(pos_entry);
  free(recovered);
  free(queue);
  return st;
}

/* ------------------------------------------------------------------ hook */

/* hook.cpp:65-74 + :104-111 input checks are the caller's (pointers). */

/* hook.cpp:98-200 over a simulated world (sequential rank order). */
int or_tagc_reduce_shard(const or_shard* shard, const float* const* grads, float* const* accs,
                         uint32_t world, const or_config* config, float* decoded,
                         or_peel_stats* stats) {
  if (world == 0 || shard->owner >= world) return OR_INVALID;
  int st = or_config_validate(config, world); /* :105 */
  if (st != OR_OK) return st;
  memset(stats, 0, sizeof(*stats));
  const uint64_t shard_len = shard->end - shard->begin;
  memset(decoded, 0, shard_len * sizeof(float));
  for (uint32_t si = 0; si < shard->num_segments; ++si) { /* :117 */
    const or_segment* seg = &shard->segments[si];
    const uint64_t lo = seg->begin - shard->begin;
    const uint32_t len = (uint32_t)(seg->end - seg->begin);
    const int flagged = or_kind_compressible(seg->kind, config->policy, config->include_out_proj);
    const int compressed = flagged && config->ratio > 1 && len >= config->min_compress_segment;
    if (!compressed) { /* :125-135 raw path: rank-ordered sum */
      for (uint64_t i = 0; i < len; ++i) {
        float acc = 0.0f;
        for (uint32_t r = 0; r < world; ++r) acc += grads[r][lo + i];
        decoded[lo + i] = acc;
      }
      stats->baseline_segments += 1;
      continue;
    }
    uint32_t m;
    st = or_sketch_geometry(len, config->ratio, config->sketch_rows, &m); /* :138-139 */
    if (st != OR_OK) return st;
    const uint32_t rows = config->sketch_rows;
    const uint32_t w = config->index_width;
    const uint32_t nw = or_words_needed(len, w);
    float** sparse = (float**)calloc(world, sizeof(float*));
    uint32_t** words = (uint32_t**)calloc(world, sizeof(uint32_t*));
    float** sketches = (float**)calloc(world, sizeof(float*));
    float* combined = (float*)malloc((size_t)len * sizeof(float));
    float* residual = (float*)malloc((size_t)len * sizeof(float));
    uint32_t* merged = (uint32_t*)malloc((size_t)nw * 4);
    uint32_t* presence = (uint32_t*)malloc((size_t)len * 4);
    uint32_t* unresolved = (uint32_t*)malloc((size_t)len * 4);
    float* summed = (float*)malloc((size_t)rows * m * sizeof(float));
    float* dec = (float*)malloc((size_t)len * sizeof(float));
    st = OR_OK;
    if (!sparse || !words || !sketches || !combined || !residual || !merged || !presence ||
        !unresolved || !summed || !dec)
      st = OR_RUNTIME;
    for (uint32_t r = 0; r < world && st == OR_OK; ++r) { /* :143-152 */
      sparse[r] = (float*)malloc((size_t)len * sizeof(float));
      words[r] = (uint32_t*)malloc((size_t)nw * 4);
      sketches[r] = (float*)malloc((size_t)rows * m * sizeof(float));
      if (!sparse[r] || !words[r] || !sketches[r]) {
        st = OR_RUNTIME;
        break;
      }
      memcpy(combined, grads[r] + lo, (size_t)len * sizeof(float));
      or_add_inplace(combined, accs[r] + lo, len); /* :146-147 */
      st = or_sparsify(combined, len, config->theta, sparse[r], residual, NULL, NULL); /* :148 */
      if (st != OR_OK) break;
      memcpy(accs[r] + lo, residual, (size_t)len * sizeof(float)); /* :149 */
      or_index_create(sparse[r], len, w, words[r]);                 /* :151 */
    }
    if (st == OR_OK) {
      or_rank_sum_words(merged, (const uint32_t* const*)words, world, nw); /* :155-157 */
      const uint32_t np = or_index_presence(merged, len, w, presence);    /* :158 */
      for (uint32_t r = 0; r < world; ++r)                                 /* :160-163 */
        or_sketch_compress(sparse[r], len, config->ratio, rows, config->seed, sketches[r]);
      or_rank_sum(summed, (const float* const*)sketches, world, (size_t)rows * m); /* :164-166 */
      uint32_t nu = 0;
      double pf = 1.0;
      st = or_peeling_decompress(presence, np, len, config->ratio, rows, config->seed, summed,
                                 dec, unresolved, &nu, &pf); /* :168 */
      if (st == OR_OK) {
        memcpy(decoded + lo, dec, (size_t)len * sizeof(float));
        stats->presence += np; /* :171-189 */
        stats->unresolved += nu;
        stats->peeled += np - nu;
        stats->compressed_segments += 1;
        for (uint32_t i = 0; i < len; ++i) {
          int truth = 0;
          for (uint32_t r = 0; r < world; ++r)
            if (sparse[r][i] != 0.0f) truth = 1;
          const int present = or_index_field(merged, w, i) != 0;
          if (truth && !present) stats->index_lost += 1;
          if (present && !truth) stats->index_spurious += 1;
        }
      }
    }
    for (uint32_t r = 0; r < world; ++r) {
      if (sparse) free(sparse[r]);
      if (words) free(words[r]);
      if (sketches) free(sketches[r]);
    }
    free(sparse);
    free(words);
    free(sketches);
    free(combined);
    free(residual);
    free(merged);
    free(presence);
    free(unresolved);
    free(summed);
    free(dec);
    if (st != OR_OK) return st;
  }
  return OR_OK;
}

/* hook.cpp:90-96 → exchange_raw (hook.cpp:78-86) → rank_sum */
int or_baseline_reduce_shard(const or_shard* shard, const float* const* grads, uint32_t world,
                             float* out) {
  if (world == 0 || shard->owner >= world) return OR_INVALID;
  or_rank_sum(out, grads, world, shard->end - shard->begin);
  return OR_OK;
}

/* hook.cpp:30-61 */
int or_make_shards(const uint64_t* layer_counts, const int32_t* layer_kinds, uint32_t n_layers,
                   uint32_t shard_count, uint32_t world_size, uint64_t* shard_len_out,
                   or_segment* segments, uint32_t* seg_shard, int32_t* seg_layer,
                   uint32_t* n_segments) {
  if (shard_count == 0 || world_size == 0) return OR_INVALID;
  uint64_t total = 0;
  for (uint32_t i = 0; i < n_layers; ++i) total += layer_counts[i];
  if (total == 0) return OR_INVALID;
  const uint64_t shard_len = (total + shard_count - 1) / shard_count;
  if (shard_len_out) *shard_len_out = shard_len;
  uint32_t ns = 0;
  /* Segments are emitted shard-major (shards[s].segments in layer order), as
   * a caller iterating shards[s].segments would see them. */
  for (uint32_t s = 0; s < shard_count; ++s) {
    const uint64_t sb = (uint64_t)s * shard_len, se = sb + shard_len;
    uint64_t off = 0;
    for (uint32_t i = 0; i < n_layers; ++i) {
      const uint64_t lb = off, le = off + layer_counts[i];
      const uint64_t b = lb > sb ? lb : sb;
      const uint64_t e = le < se ? le : se;
      if (b < e) {
        if (segments) {
          segments[ns].kind = layer_kinds[i];
          segments[ns].begin = b;
          segments[ns].end = e;
          seg_shard[ns] = s;
          seg_layer[ns] = (int32_t)i;
        }
        ++ns;
      }
      off = le;
    }
    if (s == shard_count - 1 && total < se) { /* :57-59 pad */
      if (segments) {
        segments[ns].kind = OR_KIND_OTHER;
        segments[ns].begin = total;
        segments[ns].end = se;
        seg_shard[ns] = s;
        seg_layer[ns] = -1;
      }
      ++ns;
    }
  }
  *n_segments = ns;
  return OR_OK;
}

/* train.cpp:355-359 (mean over ranks) and apply_optimizer, train.cpp:202-220. */
void or_apply_optimizer(int32_t kind, float lr, float weight_decay, uint32_t world, uint32_t step, float* params,
                        float* decoded, float* adam_v, size_t n) {
  const float inv_w = 1.0f / (float)world;                    /* train.cpp:355 */
  for (size_t i = 0; i < n; ++i) decoded[i] *= inv_w;         /* train.cpp:356 */
  if (kind == 0) {                                            /* kernels.cpp:32-41 */
    for (size_t i = 0; i < n; ++i) params[i] -= lr * decoded[i];
    return;
  }
  const float b2 = 0.999f, eps = 1e-8f;                       /* train.cpp:209-210 */
  const float bias_fix = 1.0f - powf(b2, (float)step);        /* train.cpp:213 */
  for (size_t i = 0; i < n; ++i) {
    const float g = decoded[i];
    adam_v[i] = b2 * adam_v[i] + (1.0f - b2) * g * g;          /* train.cpp:216 */
    const float vhat = adam_v[i] / bias_fix;
    params[i] -= lr * (g / (sqrtf(vhat) + eps) + weight_decay * params[i]);
  }
}
