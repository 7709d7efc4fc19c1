// encode.cu — sm_100a kernels for the rank-local half of the exchange:
//   threshold selection   (reference sparsify.cpp:18-49: tau = c-th smallest |g+acc|)
//   split + encode        (kernels.cpp:86-107 split, index.cpp:32-41 Index::create,
//                          sketch.cpp:37-67 CountSketch::compress)
// plus the elementwise rank folds used by the simulated world and the raw path.
//
// Data layout: each work item is one (rank, segment) vector in HBM. Kernels are
// persistent (grid = SMs x resident CTAs) and walk 4096-element tiles; a tile
// maps to its item by binary search over the items' tile prefix. A thread owns
// 16 elements as four 16-byte quads, so every warp load/store is a contiguous
// 512-byte request.
//
// Selection is exact (bit-identical tau) and costs one HBM pass in the common
// case: a 1/32 sample pre-pass brackets the target order statistic into a key
// window, the main pass counts keys below the window and compacts the keys
// inside it, and a per-item CTA radix-selects tau from the compacted keys. If
// the bracket misses (or overflows), a 3-digit radix select over the full item
// runs instead (kernels launched unconditionally, early-exiting per item).
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <cstdlib>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace tagc_b200 {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t find_tile_item(const EncItem* items, uint32_t n_items,
                                                   uint64_t tile) {
  uint32_t lo = 0, hi = n_items - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (items[mid].tile_begin <= tile) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ uint32_t find_sample_item(const EncItem* items, uint32_t n_items,
                                                     uint64_t w) {
  uint32_t lo = 0, hi = n_items - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (items[mid].sample_begin <= w) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Loads 4 consecutive floats starting at element `pos` (< n); lanes past n read 0.
__device__ __forceinline__ void load_quad(const float* __restrict__ p, uint32_t pos, uint32_t n,
                                          bool vec, float (&o)[4]) {
  if (vec && pos + 4 <= n) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p + pos));
    o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = (pos + j < n) ? __ldg(p + pos + j) : 0.0f;
  }
}

__device__ __forceinline__ void load_quad_rw(const float* p, uint32_t pos, uint32_t n, bool vec,
                                             float (&o)[4]) {
  if (vec && pos + 4 <= n) {
    const float4 f = *reinterpret_cast<const float4*>(p + pos);
    o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = (pos + j < n) ? p[pos + j] : 0.0f;
  }
}

__device__ __forceinline__ void store_quad(float* p, uint32_t pos, uint32_t n, bool vec,
                                           const float (&o)[4]) {
  if (vec && pos + 4 <= n) {
    *reinterpret_cast<float4*>(p + pos) = make_float4(o[0], o[1], o[2], o[3]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (pos + j < n) p[pos + j] = o[j];
  }
}

// combined = g + acc (hook.cpp:146-147: one fp32 add, even when acc is zero).
__device__ __forceinline__ void load_combined(const EncItem& e, uint32_t pos, float (&v)[4]) {
  const bool vec = (e.flags & kAligned16) != 0;
  load_quad(e.g, pos, e.n, vec, v);
  if (e.flags & kHasAcc) {
    float a[4];
    load_quad_rw(e.acc, pos, e.n, vec, a);
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = v[j] + a[j];
  }
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

// Contiguous tile range of this CTA (persistent grid): consecutive tiles stay
// in the same item, so per-item staging is flushed rarely. 32-bit arithmetic:
// tile counts stay far below 2^32 and a 64-bit divide would pull a subroutine
// call into every persistent kernel.
__device__ __forceinline__ void cta_range(uint64_t total, uint64_t& t0, uint64_t& t1) {
  const uint32_t T = uint32_t(total), G = gridDim.x;
  const uint32_t chunk = T / G, extra = T % G, b = blockIdx.x;
  t0 = uint64_t(b) * chunk + min(b, extra);
  t1 = t0 + chunk + (b < extra ? 1u : 0u);
}

// --------------------------------------------------------------- sampling
__global__ void __launch_bounds__(kTileThreads) k_sample(const EncItem* __restrict__ items,
                                                         uint32_t n_items, uint64_t total,
                                                         uint32_t* __restrict__ sample_hist,
                                                         unsigned long long* span) {
  (void)span;
  __shared__ uint32_t hist[kSampleBins];
  for (uint32_t i = threadIdx.x; i < kSampleBins; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  int cur = -1;
  auto flush = [&](int item) {
    __syncthreads();
    uint32_t* dst = sample_hist + uint64_t(item) * kSampleStride;
    for (uint32_t i = threadIdx.x; i < kSampleBins; i += blockDim.x) {
      const uint32_t h = hist[i];
      if (h) atomicAdd(dst + i, h);
      hist[i] = 0;
    }
    __syncthreads();
  };
  // contiguous range of sample works per CTA: one histogram flush per item
  // touched instead of one per work
  uint64_t w0, w1;
  cta_range(total, w0, w1);
  uint32_t it = w0 < w1 ? find_sample_item(items, n_items, w0) : 0;
  constexpr int kU = 4;  // sample works in flight per thread
  for (uint64_t w = w0; w < w1; w += kU) {
    float v[kU][4];
    uint32_t wit[kU];
    bool ok[kU];
    uint64_t pos[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t wu = w + u;
      ok[u] = wu < w1;
      while (ok[u] && it + 1 < n_items && items[it + 1].sample_begin <= wu) ++it;
      wit[u] = it;
      const EncItem& e = items[it];
      pos[u] = ok[u] ? (wu - e.sample_begin) * uint64_t(e.sample_stride) * kTile + 4ull * threadIdx.x : 0;
      ok[u] = ok[u] && pos[u] < e.n;
      if (ok[u]) load_combined(e, uint32_t(pos[u]), v[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (int(wit[u]) != cur) {  // block-uniform (same work ids in every thread)
        if (cur >= 0) flush(cur);
        cur = int(wit[u]);
      }
      if (!ok[u]) continue;
      const uint32_t n = items[wit[u]].n;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (pos[u] + j < n) atomicAdd(&hist[mag_key(v[u][j]) >> kSampleShift], 1u);
    }
  }
  if (cur >= 0) flush(cur);
}

// --------------------------------------------------------------- window
// Two levels, so the window rests on sample order statistics rather than on
// an assumption about how keys spread inside a bin: k_window_coarse finds the
// 1/16-octave sample bins holding the bracketing ranks t -+ 6 sigma,
// k_sample_fine histograms the sample keys of those two bins at 128-ulp
// resolution, and k_window_fine sets the window to the outer edges of the
// fine bins holding the ranks. The only error left is the sample's own
// (covered by the 6 sigma margin) whatever the keys look like inside a bin.
// Interpolating inside a coarse bin instead assumed uniform keys there; error
// feedback leaves a cliff near tau (the previous step's threshold) where that
// fails, and the exact fallback then costs ~0.6 ms on GPT-2.

struct RankBinSmem {
  cub::BlockScan<uint32_t, 256>::TempStorage scan;
  uint32_t bin[2], below[2], total;
};

// Bins of a 256-thread CTA's histogram h[kSampleBins] holding the 0-based
// ranks r0, r1 (negative: none) into sm.bin / sm.below (bin 0xFFFFFFFF: no
// bin holds it), plus the total count, in one scan.
__device__ __forceinline__ void rank_bins_256(const uint32_t* h, double r0, double r1, RankBinSmem& sm) {
  constexpr int kPer = kSampleBins / 256;
  uint32_t loc[kPer];
  const uint4* h4 = reinterpret_cast<const uint4*>(h + threadIdx.x * kPer);
#pragma unroll
  for (int i = 0; i < kPer / 4; ++i) {
    const uint4 q = __ldcg(h4 + i);
    loc[4 * i] = q.x;
    loc[4 * i + 1] = q.y;
    loc[4 * i + 2] = q.z;
    loc[4 * i + 3] = q.w;
  }
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) sum += loc[i];
  uint32_t pre, total;
  cub::BlockScan<uint32_t, 256>(sm.scan).ExclusiveSum(sum, pre, total);
  if (threadIdx.x == 0) {
    sm.bin[0] = sm.bin[1] = 0xFFFFFFFFu;
    sm.below[0] = sm.below[1] = 0;
    sm.total = total;
  }
  __syncthreads();
  uint32_t cum = pre;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const double c0 = double(cum), c1 = double(cum + loc[i]);
    if (r0 >= 0.0 && c0 <= r0 && r0 < c1) {
      sm.bin[0] = threadIdx.x * kPer + i;
      sm.below[0] = cum;
    }
    if (r1 >= 0.0 && c0 <= r1 && r1 < c1) {
      sm.bin[1] = threadIdx.x * kPer + i;
      sm.below[1] = cum;
    }
    cum += loc[i];
  }
  __syncthreads();
}

// One CTA per item: coarse bins of the bracketing sample ranks, kept in the
// item's SelState until k_window_fine: prefix / kept = lo / hi coarse bin
// (0xFFFFFFFF: no bound), rank / n_sel = the ranks inside them.
__global__ void __launch_bounds__(256) k_window_coarse(const EncItem* __restrict__ items,
                                                       SelState* __restrict__ state,
                                                       const uint32_t* __restrict__ sample_hist,
                                                       unsigned long long* span) {
  PDL_WAIT();
  (void)span;
  __shared__ RankBinSmem sm;
  const uint32_t item = blockIdx.x;
  const EncItem e = items[item];
  SelState st{};
  st.prefix = st.kept = 0xFFFFFFFFu;
  if (e.sample_tiles > 0) {
    const uint32_t* h = sample_hist + uint64_t(item) * kSampleStride;
    rank_bins_256(h, -1.0, -1.0, sm);
    const double s = double(sm.total);
    const double p = double(e.c) / double(e.n);
    const double t = double(e.c > 0 ? e.c - 1 : 0) * s / double(e.n);
    const double delta = 6.0 * sqrt(fmax(s * p * (1.0 - p), 0.0)) + 16.0;
    const double lo = floor(t - delta), hi = ceil(t + delta);
    rank_bins_256(h, lo, hi < s ? hi : -1.0, sm);
    if (lo >= 0.0 && sm.bin[0] != 0xFFFFFFFFu) {
      st.prefix = sm.bin[0];
      st.rank = uint32_t(lo - double(sm.below[0]));
    }
    if (hi < s && sm.bin[1] != 0xFFFFFFFFu) {
      st.kept = sm.bin[1];
      st.n_sel = uint32_t(hi - double(sm.below[1]));
    }
  }
  if (threadIdx.x == 0) state[item] = st;
}

// Fine histograms (128-ulp bins) of the sample keys inside the two coarse
// bins, over the same sample works as k_sample.
__global__ void __launch_bounds__(kTileThreads) k_sample_fine(const EncItem* __restrict__ items,
                                                              const SelState* __restrict__ state,
                                                              uint32_t n_items, uint64_t total,
                                                              uint32_t* __restrict__ sample_hist) {
  PDL_WAIT();
  uint64_t w0, w1;
  cta_range(total, w0, w1);
  uint32_t it = w0 < w1 ? find_sample_item(items, n_items, w0) : 0;
  constexpr int kU = 4;
  for (uint64_t w = w0; w < w1; w += kU) {
    float v[kU][4];
    uint32_t wit[kU];
    bool ok[kU];
    uint64_t pos[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t wu = w + u;
      ok[u] = wu < w1;
      while (ok[u] && it + 1 < n_items && items[it + 1].sample_begin <= wu) ++it;
      wit[u] = it;
      const EncItem& e = items[it];
      pos[u] = ok[u] ? (wu - e.sample_begin) * uint64_t(e.sample_stride) * kTile + 4ull * threadIdx.x : 0;
      ok[u] = ok[u] && pos[u] < e.n;
      if (ok[u]) load_combined(e, uint32_t(pos[u]), v[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (!ok[u]) continue;
      const uint32_t n = items[wit[u]].n;
      const uint32_t blo = __ldg(&state[wit[u]].prefix), bhi = __ldg(&state[wit[u]].kept);
      uint32_t* h = sample_hist + uint64_t(wit[u]) * kSampleStride;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (pos[u] + j >= n) continue;
        const uint32_t key = mag_key(v[u][j]);
        const uint32_t cb = key >> kSampleShift, fb = (key >> kFineShift) & (kSampleBins - 1u);
        if (cb == blo) atomicAdd(h + kSampleBins + fb, 1u);
        if (cb == bhi) atomicAdd(h + 2 * kSampleBins + fb, 1u);
      }
    }
  }
}

// One CTA per item: the window from the fine bins (sampled items) or the
// default window, and the fused pass's fine-bin shift. Leaves the item's
// histograms zeroed for the next call.
__global__ void __launch_bounds__(256) k_window_fine(const EncItem* __restrict__ items,
                                                     SelState* __restrict__ state,
                                                     uint32_t* __restrict__ sample_hist) {
  PDL_WAIT();
  __shared__ RankBinSmem sm;
  const uint32_t item = blockIdx.x;
  const EncItem e = items[item];
  uint32_t klo = 1u, khi = 0x7F800000u;  // no sample: every nonzero key is a candidate
  if (e.sample_tiles > 0) {
    uint32_t* h = sample_hist + uint64_t(item) * kSampleStride;
    const SelState sc = state[item];
    if (sc.prefix != 0xFFFFFFFFu) {
      rank_bins_256(h + kSampleBins, double(sc.rank), -1.0, sm);
      if (sm.bin[0] != 0xFFFFFFFFu) klo = max(1u, (sc.prefix << kSampleShift) | (sm.bin[0] << kFineShift));
    }
    if (sc.kept != 0xFFFFFFFFu) {
      rank_bins_256(h + 2 * kSampleBins, double(sc.n_sel), -1.0, sm);
      if (sm.bin[0] != 0xFFFFFFFFu)
        khi = min(0x7F800000u, (sc.kept << kSampleShift) | (sm.bin[0] << kFineShift) | ((1u << kFineShift) - 1u));
    }
    uint4* h4 = reinterpret_cast<uint4*>(h);
    for (uint32_t i = threadIdx.x; i < kSampleStride / 4; i += blockDim.x) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (e.c == 0) {  // tau = 0 without selection: every nonzero key is kept
    klo = 1u;
    khi = 0u;
  }
  if (threadIdx.x == 0) {
    SelState st{};
    st.klo = klo;
    st.khi = khi;
    uint32_t fs = 0;
    while (khi >= klo && ((khi - klo) >> fs) >= kRadixBins) ++fs;
    st.fshift = fs;
    state[item] = st;
  }
}

// --------------------------------------------------------------- helpers
constexpr uint32_t kStatusReady = 0, kStatusFallback = 1, kStatusCollect = 3, kStatusFbReady = 4;

// Values a fallback pass reads: after k_restore an accumulator holds the
// combined value g + acc of every element, so it is read alone.
__device__ __forceinline__ void load_source(const EncItem& e, uint32_t pos, bool restored,
                                            float (&v)[4]) {
  if (restored && (e.flags & kHasAcc)) {
    load_quad_rw(e.acc, pos, e.n, (e.flags & kAligned16) != 0, v);
  } else {
    load_combined(e, pos, v);
  }
}

__device__ __forceinline__ void scatter_sketch(const EncItem& e, const HashParams& hp, uint32_t p,
                                               float v) {
  _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows)
    red_add_f32(e.sketch + uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m, e.mmul), dev_sign(hp.row[r], p) * v);
}

// --------------------------------------------------------------- fused pass
// ONE HBM pass per element does the selection bookkeeping AND a speculative
// encode (reference sparsify.cpp:18-49 + kernels.cpp:86-107 + index.cpp:32-41
// + sketch.cpp:37-67). The sampled key window [klo, khi] brackets tau:
//   key == 0 or key < klo : dropped (residual = v)
//   key >  khi            : kept   (residual 0, index bit, sketch scatter) and
//                           logged as (position, value) so a bracket miss can
//                           restore the accumulator
//   klo <= key <= khi     : undecided: written as dropped and logged as a
//                           candidate; k_fixup keeps those with key > tau.
// Candidates and kept elements are staged per warp in shared memory and
// appended to global pools with one atomic per 200+ entries.
constexpr uint32_t kWarpStage = 128;

// kHook: the exchange path (accumulator in/out, index + sketch). !kHook: the
// per-stage sparsify entry point (separate sparse/residual outputs). Separate
// template instances keep the hot kernel small enough for the instruction
// cache.
template <bool kW4, bool kHook>
__global__ void __launch_bounds__(kTileThreads, 4) k_fused(const EncItem* __restrict__ items,
                                                           SelState* __restrict__ state,
                                                           uint32_t n_items, uint64_t total_tiles,
                                                           const HashParams hp,
                                                           uint2* __restrict__ cand,
                                                           uint2* __restrict__ hi_pool,
                                                           uint32_t* __restrict__ fine_hist,
                                                           uint32_t* __restrict__ err,
                                                           unsigned long long* span) {
  span_begin(span);
  __shared__ uint2 s_cand[kTileThreads / 32][kWarpStage];
  __shared__ uint2 s_kept[kTileThreads / 32][kWarpStage];
  __shared__ float s_v[16][kTileThreads];  // a thread's 16 values, read back by bit index
  __shared__ uint32_t s_hist[kRadixBins];
  __shared__ uint32_t s_zero, s_lo;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t t0, t1;
  cta_range(total_tiles, t0, t1);
  if (t0 >= t1) return;
  bool nan = false;
  uint32_t it = find_tile_item(items, n_items, t0);
  for (uint64_t tile = t0; tile < t1;) {
    const EncItem e = items[it];
    const uint64_t item_end = e.tile_begin + (uint64_t(e.n) + kTile - 1) / kTile;
    const uint64_t tend = item_end < t1 ? item_end : t1;
    const uint32_t klo = state[it].klo, khi = state[it].khi, fshift = state[it].fshift;
    const bool vec = (e.flags & kAligned16) != 0;
    const uint32_t n_words = kW4 ? (e.n + 7u) / 8u : (e.n + 31u) / 32u;
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) s_hist[i] = 0;
    if (threadIdx.x == 0) s_zero = s_lo = 0;
    __syncthreads();
    uint32_t c_zero = 0, c_lo = 0, wc = 0, wk = 0;
    // warp-level flushes of the staged candidates / kept elements
    auto flush_cand = [&]() {
      __syncwarp();
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&state[it].cnt_in, wc);
      base = __shfl_sync(kFull, base, 0);
      for (uint32_t i = lane; i < wc; i += 32)
        if (base + i < e.cand_cap) cand[e.cand_off + base + i] = s_cand[warp][i];
      __syncwarp();
      wc = 0;
    };
    auto flush_kept = [&]() {
      __syncwarp();
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&state[it].cnt_hi, wk);
      base = __shfl_sync(kFull, base, 0);
      for (uint32_t i = lane; i < wk; i += 32) {
        const uint2 kv = s_kept[warp][i];
        const float v = __uint_as_float(kv.y);
        if (kHook && !(e.flags & kDeferScatter)) scatter_sketch(e, hp, kv.x, v);
        if (base + i < e.hi_cap) {
          hi_pool[e.hi_off + base + i] = kv;
        } else if (kHook) {  // pool full (bracket miss): keep v recoverable
          e.acc[kv.x] = v;
        }
      }
      __syncwarp();
      wk = 0;
    };
    for (; tile < tend; ++tile) {
      const uint32_t q0 = uint32_t(tile - e.tile_begin) * (kTile / 4);
      float v[4][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t pos = 4u * (q0 + k * kTileThreads + threadIdx.x);
        if (pos < e.n) {
          load_quad(e.g, pos, e.n, vec, v[k]);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) v[k][j] = 0.0f;
        }
      }
      if (kHook) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t pos = 4u * (q0 + k * kTileThreads + threadIdx.x);
          if (pos < e.n) {
            float a[4];
            load_quad_rw(e.acc, pos, e.n, vec, a);
#pragma unroll
            for (int j = 0; j < 4; ++j) v[k][j] = v[k][j] + a[j];
          }
        }
      }
      // classify the thread's 16 elements into bit masks (bit 4k+j)
      uint32_t in_m = 0, hi_m = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t pos = 4u * (q0 + k * kTileThreads + threadIdx.x);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const bool valid = pos + j < e.n;
          const uint32_t key = mag_key(v[k][j]);
          const uint32_t bit = 1u << (4 * k + j);
          hi_m |= (valid && key > khi) ? bit : 0u;
          in_m |= (valid && key >= klo && key <= khi && key != 0) ? bit : 0u;
          c_zero += valid && key == 0;
          c_lo += valid && key != 0 && key < klo;
          nan |= valid && key > 0x7F800000u;
        }
      }
      // element b = 4k + j sits at position 4*(q0 + k*256 + tid) + j
      const uint32_t pbase = 4u * (q0 + threadIdx.x);
      if (in_m | hi_m) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < 4; ++j) s_v[4 * k + j][threadIdx.x] = v[k][j];
      }
      // warp-level placement in the stages: one packed scan per tile
      const uint32_t cnt = uint32_t(__popc(in_m)) | (uint32_t(__popc(hi_m)) << 16);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= uint32_t(o)) incl += y;
      }
      const uint32_t tot = __shfl_sync(kFull, incl, 31);
      const uint32_t tot_c = tot & 0xFFFFu, tot_k = tot >> 16;
      if (tot_c) {
        if (wc + tot_c > kWarpStage) flush_cand();
        const bool direct = tot_c > kWarpStage;  // dense tile: straight to the pool
        uint32_t gbase = 0;
        if (direct) {
          if (lane == 0) gbase = atomicAdd(&state[it].cnt_in, tot_c);
          gbase = __shfl_sync(kFull, gbase, 0);
        }
        uint32_t o = (incl - cnt) & 0xFFFFu;
        for (uint32_t m = in_m; m; m &= m - 1) {
          const uint32_t b = __ffs(m) - 1;
          const float x = s_v[b][threadIdx.x];
          const uint2 kv = make_uint2(pbase + (b >> 2) * 4u * kTileThreads + (b & 3u), __float_as_uint(x));
          if (!direct) s_cand[warp][wc + o] = kv;
          else if (gbase + o < e.cand_cap) cand[e.cand_off + gbase + o] = kv;
          atomicAdd(&s_hist[(mag_key(x) - klo) >> fshift], 1u);
          ++o;
        }
        if (!direct) wc += tot_c;
      }
      if (tot_k) {
        if (wk + tot_k > kWarpStage) flush_kept();
        const bool direct = tot_k > kWarpStage;
        uint32_t gbase = 0;
        if (direct) {
          if (lane == 0) gbase = atomicAdd(&state[it].cnt_hi, tot_k);
          gbase = __shfl_sync(kFull, gbase, 0);
        }
        uint32_t o = (incl - cnt) >> 16;
        for (uint32_t m = hi_m; m; m &= m - 1) {
          const uint32_t b = __ffs(m) - 1;
          const float x = s_v[b][threadIdx.x];
          const uint2 kv = make_uint2(pbase + (b >> 2) * 4u * kTileThreads + (b & 3u), __float_as_uint(x));
          if (!direct) {
            s_kept[warp][wk + o] = kv;
          } else {
            if (kHook && !(e.flags & kDeferScatter)) scatter_sketch(e, hp, kv.x, x);
            if (gbase + o < e.hi_cap) hi_pool[e.hi_off + gbase + o] = kv;
            else hi_m &= ~(1u << b);  // pool full: the element keeps v in place
          }
          ++o;
        }
        if (!direct) wk += tot_k;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t q = q0 + k * kTileThreads + threadIdx.x;
        const uint32_t pos = 4u * q;
        const uint32_t nib = (hi_m >> (4 * k)) & 0xFu;
        if (pos < e.n) {
          float r[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) r[j] = (nib >> j & 1u) ? 0.0f : v[k][j];
          if (kHook) {
            store_quad(e.acc, pos, e.n, vec, r);
          } else {
            store_quad(e.residual, pos, e.n, false, r);
            float sp[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) sp[j] = (nib >> j & 1u) ? v[k][j] : 0.0f;
            store_quad(e.sparse, pos, e.n, false, sp);
          }
        }
        if (kHook) {
          if (kW4) {
            if (q < 2u * n_words) {
              const uint32_t hw = (nib & 1u) | (nib >> 1 & 1u) << 4 | (nib >> 2 & 1u) << 8 |
                                  (nib >> 3 & 1u) << 12;
              reinterpret_cast<uint16_t*>(e.index)[q] = uint16_t(hw);
            }
          } else {
            uint32_t x = nib << (4u * (lane & 7u));
            x |= __shfl_xor_sync(kFull, x, 1);
            x |= __shfl_xor_sync(kFull, x, 2);
            x |= __shfl_xor_sync(kFull, x, 4);
            if ((lane & 7u) == 0 && q / 8u < n_words) e.index[q / 8u] = x;
          }
        }
      }
    }
    // item done: drain the warp stages, then the CTA's counts and histogram
    __syncwarp();
    if (wc) flush_cand();
    if (wk) flush_kept();
    c_zero = warp_sum(c_zero);
    c_lo = warp_sum(c_lo);
    if (lane == 0) {
      if (c_zero) atomicAdd(&s_zero, c_zero);
      if (c_lo) atomicAdd(&s_lo, c_lo);
    }
    __syncthreads();
    uint32_t* fh = fine_hist + uint64_t(it) * kRadixBins;
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x)
      if (s_hist[i]) atomicAdd(fh + i, s_hist[i]);
    if (threadIdx.x == 0) {
      if (s_zero) atomicAdd(&state[it].cnt_zero, s_zero);
      if (s_lo) atomicAdd(&state[it].cnt_lo, s_lo);
    }
    __syncthreads();
    ++it;
  }
  if (nan) atomicOr(err, 1u);
  span_end(span);
}


// --------------------------------------------------------------- fused pass (TMA)
// The same single pass as k_fused for the exchange path (accumulator in/out),
// restructured around bulk async copies (cp.async.bulk, the 1-D TMA path):
// one persistent CTA per SM = one producer warp + kConsumerWarps consumer
// warps sharing a kFusedStages-deep ring of 32 KB stages (a 4096-element tile
// of g and of acc). The producer keeps the ring full (full/empty mbarriers,
// no CTA-wide barrier per tile), so HBM sees a steady stream of 16 KB
// requests while the consumers classify tiles out of shared memory. Items must
// be 16-byte aligned (the host checks); a tile's last <16 bytes are read
// directly from global memory.
constexpr int kFusedStages = 3;
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kFusedThreads = kConsumers + 32;
constexpr int kQuads = kTile / 4 / kConsumers;  // quads (4 elements) per consumer thread per tile
constexpr int kFusedCtasPerSm = 2;
constexpr uint32_t kWarpStageT = 64;
struct alignas(128) FusedStage {
  float g[kTile];
  float a[kTile];
  unsigned long long tile;  // which tile the stage holds (kNoTile: the producer is done)
};
constexpr unsigned long long kNoTile = ~0ull;
constexpr size_t kFusedSmem = size_t(kFusedStages) * sizeof(FusedStage) + 2 * kFusedStages * 8 + 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra.uni WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier; the streamed operands
// are marked evict-first in L2 so the sketch rows being scattered into stay hot
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         unsigned long long* b, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

template <bool kW4>
__global__ void __launch_bounds__(kFusedThreads, 2) k_fused_tma(const EncItem* __restrict__ items,
                                                                SelState* __restrict__ state,
                                                                uint32_t n_items, uint64_t total_tiles,
                                                                const HashParams hp,
                                                                uint2* __restrict__ cand,
                                                                uint2* __restrict__ hi_pool,
                                                                uint32_t* __restrict__ fine_hist,
                                                                uint32_t* __restrict__ err,
                                                                unsigned long long* span, uint32_t chunk) {
  PDL_WAIT();
  extern __shared__ __align__(128) unsigned char fsm[];
  FusedStage* stg = reinterpret_cast<FusedStage*>(fsm);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(fsm + size_t(kFusedStages) * sizeof(FusedStage));
  unsigned long long* empty = full + kFusedStages;
  __shared__ uint2 s_cand[kConsumerWarps][kWarpStageT];
  __shared__ uint2 s_kept[kConsumerWarps][kWarpStageT];
  __shared__ uint32_t s_hist[kRadixBins];
  __shared__ uint32_t s_zero, s_lo;
  span_begin(span);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // Tile order. chunk == 0: the contiguous balanced range of cta_range (every
  // sketch fits in L2 together). Otherwise the producer claims `chunk`-tile
  // chunks from a global counter (err[3]), so all CTAs advance through the
  // shard together inside a window of about G x chunk tiles and the sketch
  // rows being scattered into stay L2-resident even when the shard's
  // sketches total GBs (Llama-3-8B: 2.9 GB per rank). Consumers read each
  // stage's tile id from the stage itself.
  uint64_t t0 = 0, t1 = 0;
  if (chunk == 0) {
    cta_range(total_tiles, t0, t1);
    if (t0 >= t1) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFusedStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kConsumerWarps) {  // ------------------------------ producer warp
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      uint32_t pit = 0;
      uint32_t i = 0;
      auto push = [&](uint64_t tile) {
        const int s = int(i % kFusedStages);
        if (i >= uint32_t(kFusedStages)) mbar_wait(&empty[s], ((i / kFusedStages) - 1) & 1u);
        ++i;
        stg[s].tile = tile;
        if (tile == kNoTile) {
          mbar_arrive(&full[s]);
          return;
        }
        while (tile >= items[pit].tile_begin + (uint64_t(items[pit].n) + kTile - 1) / kTile) ++pit;
        const EncItem& pe = items[pit];
        const uint32_t start = uint32_t(tile - pe.tile_begin) * kTile;
        const uint32_t len = min(kTile, pe.n - start);
        const uint32_t bytes = (len * 4u) & ~15u;
        mbar_arrive_expect_tx(&full[s], 2u * bytes);
        if (bytes) {
          bulk_g2s(stg[s].g, pe.g + start, bytes, &full[s], policy);
          bulk_g2s(stg[s].a, pe.acc + start, bytes, &full[s], policy);
        }
      };
      if (chunk == 0) {
        pit = find_tile_item(items, n_items, t0);
        for (uint64_t tile = t0; tile < t1; ++tile) push(tile);
      } else {
        // the next claim is issued before the current chunk's tiles are
        // pushed, so its round trip overlaps the waits for free stages
        uint64_t c0 = uint64_t(atomicAdd(err + 3, 1u)) * chunk;
        while (c0 < total_tiles) {
          const uint64_t cn = uint64_t(atomicAdd(err + 3, 1u)) * chunk;
          const uint64_t c1 = min(total_tiles, c0 + chunk);
          for (uint64_t tile = c0; tile < c1; ++tile) push(tile);
          c0 = cn;
        }
      }
      push(kNoTile);
    }
    span_end(span);
    return;
  }

  // ------------------------------------------------------------ consumers
  const uint32_t ctid = threadIdx.x;
  bool nan = false;
  uint32_t iter = 0;
  // the first tile (tiles arrive in increasing order, items with it); the
  // contiguous order is known here, the claimed one is read from the stage
  uint64_t tile = t0;
  if (chunk != 0) {
    mbar_wait(&full[0], 0u);
    tile = *reinterpret_cast<volatile unsigned long long*>(&stg[0].tile);
  }
  uint32_t it = tile == kNoTile ? 0u : find_tile_item(items, n_items, tile);
  while (tile != kNoTile) {
    while (tile >= items[it].tile_begin + (uint64_t(items[it].n) + kTile - 1) / kTile) ++it;  // skip items with no tile here
    const EncItem e = items[it];
    const uint64_t item_end = e.tile_begin + (uint64_t(e.n) + kTile - 1) / kTile;
    const uint32_t klo = state[it].klo, khi = state[it].khi, fshift = state[it].fshift;
    const uint32_t n_words = kW4 ? (e.n + 7u) / 8u : (e.n + 31u) / 32u;
    for (uint32_t i = ctid; i < kRadixBins; i += kConsumers) s_hist[i] = 0;
    if (ctid == 0) s_zero = s_lo = 0;
    consumer_sync();
    uint32_t c_zero = 0, c_lo = 0, wc = 0, wk = 0;
    auto flush_cand = [&]() {
      __syncwarp();
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&state[it].cnt_in, wc);
      base = __shfl_sync(kFull, base, 0);
      for (uint32_t i = lane; i < wc; i += 32)
        if (base + i < e.cand_cap) cand[e.cand_off + base + i] = s_cand[warp][i];
      __syncwarp();
      wc = 0;
    };
    auto flush_kept = [&]() {
      __syncwarp();
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&state[it].cnt_hi, wk);
      base = __shfl_sync(kFull, base, 0);
      for (uint32_t i = lane; i < wk; i += 32) {
        const uint2 kv = s_kept[warp][i];
        const float v = __uint_as_float(kv.y);
        if (!(e.flags & kDeferScatter)) scatter_sketch(e, hp, kv.x, v);
        if (base + i < e.hi_cap) hi_pool[e.hi_off + base + i] = kv;
        else e.acc[kv.x] = v;  // pool full (bracket miss): keep v recoverable
      }
      __syncwarp();
      wk = 0;
    };
    for (;;) {  // stage `iter` holds `tile`
      const int s = int(iter % kFusedStages);
      const uint32_t start = uint32_t(tile - e.tile_begin) * kTile;
      const uint32_t len = min(kTile, e.n - start);
      mbar_wait(&full[s], (iter / kFusedStages) & 1u);  // returns at once after a peek
      float* sg = stg[s].g;
      const float* sa = stg[s].a;
      float v[kQuads][4];
      uint32_t hi_m = 0, lo_m = 0, z_m = 0, valid_m = (1u << (4 * kQuads)) - 1u;
#pragma unroll
      for (int k = 0; k < kQuads; ++k) {
        const uint32_t e0 = 4u * (k * kConsumers + ctid);
        if (e0 + 4 <= len) {
          const float4 x = *reinterpret_cast<const float4*>(sg + e0);
          const float4 y = *reinterpret_cast<const float4*>(sa + e0);
          v[k][0] = x.x + y.x; v[k][1] = x.y + y.y; v[k][2] = x.z + y.z; v[k][3] = x.w + y.w;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const bool in = e0 + j < len;
            v[k][j] = in ? __ldg(e.g + start + e0 + j) + e.acc[start + e0 + j] : 0.0f;
            if (!in) valid_m &= ~(1u << (4 * k + j));
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t key = mag_key(v[k][j]);
          const uint32_t bit = 1u << (4 * k + j);
          hi_m |= key > khi ? bit : 0u;
          lo_m |= key < klo ? bit : 0u;
          z_m |= key == 0u ? bit : 0u;
        }
      }
      hi_m &= valid_m;
      lo_m &= valid_m;
      z_m &= valid_m;
      const uint32_t in_m = valid_m & ~hi_m & ~lo_m;
      c_zero += __popc(z_m);
      c_lo += __popc(lo_m & ~z_m);
      // a thread with flagged elements parks its combined values in the stage
      // (its own slots only) for the compaction below
      if (in_m | hi_m) {
#pragma unroll
        for (int k = 0; k < kQuads; ++k)
          *reinterpret_cast<float4*>(sg + 4u * (k * kConsumers + ctid)) =
              make_float4(v[k][0], v[k][1], v[k][2], v[k][3]);
      }
      // warp placement of the flagged elements: counts are almost always 0 or
      // 1 per thread, so the exclusive prefix is a few ballots (one per count
      // level present in the warp) instead of a dependent shuffle scan
      const uint32_t n_c = __popc(in_m), n_k = __popc(hi_m);
      const uint32_t lt = (1u << lane) - 1u;
      uint32_t pre_c = 0, pre_k = 0, tot_c = 0, tot_k = 0;
      const uint32_t levels = __reduce_max_sync(kFull, max(n_c, n_k));
      for (uint32_t lv = 1; lv <= levels; ++lv) {
        const uint32_t mc = __ballot_sync(kFull, n_c >= lv), mk = __ballot_sync(kFull, n_k >= lv);
        pre_c += __popc(mc & lt);
        pre_k += __popc(mk & lt);
        tot_c += __popc(mc);
        tot_k += __popc(mk);
      }
      const uint32_t pbase = start + 4u * ctid;  // element b = 4k + j -> pbase + k*4*kConsumers + j
      if (tot_c) {
        if (wc + tot_c > kWarpStageT) flush_cand();
        const bool direct = tot_c > kWarpStageT;
        uint32_t gbase = 0;
        if (direct) {
          if (lane == 0) gbase = atomicAdd(&state[it].cnt_in, tot_c);
          gbase = __shfl_sync(kFull, gbase, 0);
        }
        uint32_t o = pre_c;
        for (uint32_t m = in_m; m; m &= m - 1) {
          const uint32_t b = __ffs(m) - 1;
          const uint32_t off = (b >> 2) * 4u * kConsumers + (b & 3u);
          const float x = sg[4u * ctid + off];
          const uint2 kv = make_uint2(pbase + off, __float_as_uint(x));
          if (!direct) s_cand[warp][wc + o] = kv;
          else if (gbase + o < e.cand_cap) cand[e.cand_off + gbase + o] = kv;
          atomicAdd(&s_hist[(mag_key(x) - klo) >> fshift], 1u);
          ++o;
        }
        if (!direct) wc += tot_c;
      }
      if (tot_k) {
        if (wk + tot_k > kWarpStageT) flush_kept();
        const bool direct = tot_k > kWarpStageT;
        uint32_t gbase = 0;
        if (direct) {
          if (lane == 0) gbase = atomicAdd(&state[it].cnt_hi, tot_k);
          gbase = __shfl_sync(kFull, gbase, 0);
        }
        uint32_t o = pre_k;
        for (uint32_t m = hi_m; m; m &= m - 1) {
          const uint32_t b = __ffs(m) - 1;
          const uint32_t off = (b >> 2) * 4u * kConsumers + (b & 3u);
          const float x = sg[4u * ctid + off];
          nan |= mag_key(x) > 0x7F800000u;
          const uint2 kv = make_uint2(pbase + off, __float_as_uint(x));
          if (!direct) {
            s_kept[warp][wk + o] = kv;
          } else {
            if (!(e.flags & kDeferScatter)) scatter_sketch(e, hp, kv.x, x);
            if (gbase + o < e.hi_cap) hi_pool[e.hi_off + gbase + o] = kv;
            else hi_m &= ~(1u << b);  // pool full: the element keeps v in place
          }
          ++o;
        }
        if (!direct) wk += tot_k;
      }
#pragma unroll
      for (int k = 0; k < kQuads; ++k) {
        const uint32_t qt = k * kConsumers + ctid;  // quad within the tile
        const uint32_t e0 = 4u * qt;
        const uint32_t nib = (hi_m >> (4 * k)) & 0xFu;
        float r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = (nib >> j & 1u) ? 0.0f : v[k][j];
        if (e0 + 4 <= len) {
          __stcs(reinterpret_cast<float4*>(e.acc + start + e0), make_float4(r[0], r[1], r[2], r[3]));
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (e0 + j < len) e.acc[start + e0 + j] = r[j];
        }
        const uint32_t q = start / 4u + qt;
        if (kW4) {
          if (q < 2u * n_words) {
            const uint32_t hw = (nib & 1u) | (nib >> 1 & 1u) << 4 | (nib >> 2 & 1u) << 8 | (nib >> 3 & 1u) << 12;
            reinterpret_cast<uint16_t*>(e.index)[q] = uint16_t(hw);
          }
        } else {
          uint32_t x = nib << (4u * (lane & 7u));
          x |= __shfl_xor_sync(kFull, x, 1);
          x |= __shfl_xor_sync(kFull, x, 2);
          x |= __shfl_xor_sync(kFull, x, 4);
          if ((lane & 7u) == 0 && q / 8u < n_words) e.index[q / 8u] = x;
        }
      }
      // parked values were generic-proxy writes into the stage: order them
      // before the bulk copy that refills it, then release the stage
      if (in_m | hi_m) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      // the next tile: same item, or the end of this item's run
      ++iter;
      if (chunk == 0) {
        tile = tile + 1 < t1 ? tile + 1 : kNoTile;
      } else {  // peek at the next stage
        const int ns = int(iter % kFusedStages);
        mbar_wait(&full[ns], (iter / kFusedStages) & 1u);
        tile = *reinterpret_cast<volatile unsigned long long*>(&stg[ns].tile);
      }
      if (tile >= item_end) break;  // kNoTile included
    }
    __syncwarp();
    if (wc) flush_cand();
    if (wk) flush_kept();
    c_zero = warp_sum(c_zero);
    c_lo = warp_sum(c_lo);
    if (lane == 0) {
      if (c_zero) atomicAdd(&s_zero, c_zero);
      if (c_lo) atomicAdd(&s_lo, c_lo);
    }
    consumer_sync();
    uint32_t* fh = fine_hist + uint64_t(it) * kRadixBins;
    for (uint32_t i = ctid; i < kRadixBins; i += kConsumers)
      if (s_hist[i]) atomicAdd(fh + i, s_hist[i]);
    if (ctid == 0) {
      if (s_zero) atomicAdd(&state[it].cnt_zero, s_zero);
      if (s_lo) atomicAdd(&state[it].cnt_lo, s_lo);
    }
    consumer_sync();
    ++it;
  }
  if (nan) atomicOr(err, 1u);
  span_end(span);
}

// Block-wide search over `kRadixBins` counters: finds the digit whose
// inclusive prefix first exceeds `rank`; returns the digit and the count of
// keys in lower digits.
template <int kThreads>
__device__ __forceinline__ void find_digit(const uint32_t* hist, uint32_t nbins, uint32_t rank,
                                           uint32_t* s_digit, uint32_t* s_below) {
  using Scan = cub::BlockScan<uint32_t, kThreads>;
  __shared__ typename Scan::TempStorage tmp;
  constexpr int kPer = kRadixBins / kThreads;
  uint32_t loc[kPer];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const uint32_t b = threadIdx.x * kPer + i;
    loc[i] = b < nbins ? hist[b] : 0u;
    sum += loc[i];
  }
  uint32_t pre;
  Scan(tmp).ExclusiveSum(sum, pre);
  uint32_t cum = pre;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    if (cum <= rank && rank < cum + loc[i]) {
      *s_digit = threadIdx.x * kPer + i;
      *s_below = cum;
    }
    cum += loc[i];
  }
  __syncthreads();
}

__host__ __device__ constexpr int digit_shift(int pass) { return pass == 0 ? 20 : (pass == 1 ? 10 : 0); }
__host__ __device__ constexpr int digit_bits(int pass) { return pass == 0 ? 11 : 10; }

constexpr uint32_t kFinalKeys = 8192;  // per-item capacity of the target sub-bin list

// --------------------------------------------------------------- finalize
// k_finish_select, a grid of kFinishCtas CTAs per item (blockIdx.y = item):
// (1) every CTA checks that tau (the c-th smallest key, sparsify.cpp:33-37)
//     falls inside the window, so every speculative decision outside it was
//     right, and names the fine sub-bin holding it (the same answer in every
//     CTA: the item's fine histogram is read-only here);
// (2) the CTAs gather that sub-bin's keys from their slice of the item's
//     candidates into the item's key list (sel_list, kFinalKeys per item);
// (3) the last CTA of the item to finish radix-selects tau exactly among
//     them (streaming all candidates again if the sub-bin overflowed the
//     list: massive ties) and leaves the fine histogram and the counters
//     zeroed for the next call.
// Bit-identical to nth_element (sparsify.cpp:35-36).
constexpr uint32_t kFinishCtas = 16;
constexpr uint32_t kFinishThreads = 256;

__global__ void __launch_bounds__(kFinishThreads) k_finish_select(const EncItem* __restrict__ items,
                                                                  SelState* __restrict__ state,
                                                                  uint32_t* __restrict__ fine_hist,
                                                                  const uint2* __restrict__ cand,
                                                                  uint32_t* __restrict__ sel_list,
                                                                  uint32_t* __restrict__ err) {
  __shared__ uint32_t keys[kFinalKeys];
  __shared__ uint32_t hist[kRadixBins];
  __shared__ uint32_t s_digit, s_below, s_last;
  const uint32_t item = blockIdx.y;
  const EncItem e = items[item];
  const SelState s = state[item];
  uint32_t* fh = fine_hist + uint64_t(item) * kRadixBins;
  uint32_t* list = sel_list + uint64_t(item) * kFinalKeys;
  const bool overflow = s.cnt_in > e.cand_cap || s.cnt_hi > e.hi_cap;
  const uint32_t Z = s.cnt_zero, L = s.cnt_lo, I = s.cnt_in;
  int action = 0;  // 0 none (NaN), 1 tau = 0, 2 select among candidates, 3 fallback
  if (!(*err & 1u)) {
    if (e.c <= Z) action = (L == 0 && !overflow) ? 1 : 3;  // tau = 0: every nonzero key is kept
    else if (!overflow && Z + L < e.c && e.c <= Z + L + I) action = 2;
    else action = 3;
  }
  uint32_t rank = 0, sub = 0;
  if (action == 2) {
    find_digit<kFinishThreads>(fh, kRadixBins, e.c - Z - L - 1, &s_digit, &s_below);
    sub = s_digit;  // target sub-bin
    rank = e.c - Z - L - 1 - s_below;
    // (2) this CTA's slice of the candidates
    const uint2* ck = cand + e.cand_off;
    const uint32_t nc = min(s.cnt_in, e.cand_cap);
    const uint32_t per = (nc + gridDim.x - 1) / gridDim.x;
    const uint32_t c0 = min(nc, blockIdx.x * per), c1 = min(nc, c0 + per);
    constexpr uint32_t kB = 4;  // candidate loads in flight per thread
    const uint32_t lane = threadIdx.x & 31;
    // warp-uniform trip count (the ballots below need every lane)
    for (uint32_t w0 = c0 + (threadIdx.x & ~31u); w0 < c1; w0 += kB * blockDim.x) {
      uint32_t kk[kB];
#pragma unroll
      for (uint32_t b = 0; b < kB; ++b) {
        const uint32_t i = w0 + lane + b * blockDim.x;
        kk[b] = i < c1 ? (__ldcs(&ck[i].y) & 0x7FFFFFFFu) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (uint32_t b = 0; b < kB; ++b) {
        const bool hit = kk[b] != 0xFFFFFFFFu && ((kk[b] - s.klo) >> s.fshift) == sub;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, hit);
        if (!m) continue;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&state[item].n_sel, uint32_t(__popc(m)));
        base = __shfl_sync(0xFFFFFFFFu, base, 0) + __popc(m & ((1u << lane) - 1u));
        if (hit && base < kFinalKeys) list[base] = kk[b];
      }
    }
  }
  // (3) the last CTA of the item finishes it
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&state[item].pad, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) fh[i] = 0;  // left zero for the next call
  if (action != 2) {
    if (threadIdx.x == 0) {
      if (action == 1) {
        state[item].tau_key = 0;
        state[item].status = kStatusReady;
      } else if (action == 3) {  // bracket missed: restore + full radix select
        state[item].status = kStatusFallback;
        state[item].prefix = 0;
        state[item].rank = e.c - 1;
        atomicOr(err + 1, 1u);
      }
      state[item].n_sel = 0;
      state[item].pad = 0;
    }
    return;
  }
  const uint32_t nk = __ldcg(&state[item].n_sel);
  const bool in_smem = nk <= kFinalKeys;
  if (in_smem)
    for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) keys[i] = __ldcg(list + i);
  const uint2* ck = cand + e.cand_off;
  const uint32_t nc = min(s.cnt_in, e.cand_cap);
  uint32_t prefix = 0;
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int shift = digit_shift(pass), bits = digit_bits(pass), hs = shift + bits;
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    if (in_smem) {
      for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) {
        const uint32_t key = keys[i];
        if ((key >> hs) == (prefix >> hs)) atomicAdd(&hist[(key >> shift) & ((1u << bits) - 1u)], 1u);
      }
    } else {  // massive ties inside one sub-bin: stream the candidates again
      for (uint32_t i = threadIdx.x; i < nc; i += blockDim.x) {
        const uint32_t key = ck[i].y & 0x7FFFFFFFu;
        if (((key - s.klo) >> s.fshift) == sub && (key >> hs) == (prefix >> hs))
          atomicAdd(&hist[(key >> shift) & ((1u << bits) - 1u)], 1u);
      }
    }
    __syncthreads();
    find_digit<kFinishThreads>(hist, 1u << bits, rank, &s_digit, &s_below);
    rank -= s_below;
    prefix |= s_digit << shift;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    state[item].tau_key = prefix;
    state[item].status = kStatusReady;
    state[item].n_sel = 0;
    state[item].pad = 0;
  }
}

// --------------------------------------------------------------- fixup
// Window candidates with key > tau were written as dropped: make them kept
// (residual 0, index field set, sketch scatter). Each CTA walks a contiguous
// range of the flattened candidates in 256-wide chunks; a chunk inside one
// item (the common case) takes its kept count and its deferred-scatter log
// slots with ONE atomic per chunk (block count / scan), a mixed chunk per
// warp and item - per-warp atomics on one item's counters serialised at a
// single L2 address once an item had 10^5 candidates.
template <bool kW4>
__global__ void __launch_bounds__(256) k_fixup(const EncItem* __restrict__ items,
                                               SelState* __restrict__ state, uint32_t n_items,
                                               const uint2* __restrict__ cand, const HashParams hp,
                                               const uint32_t* __restrict__ err, uint2* __restrict__ hi_pool) {
  using Scan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t pref[kMaxFlatItems + 1];
  __shared__ uint32_t s_tau[kMaxFlatItems];
  __shared__ uint32_t s_base;
  if (err[0]) return;
  for (uint32_t i = threadIdx.x; i < n_items; i += blockDim.x) s_tau[i] = state[i].tau_key;
  const uint32_t total = flat_prefix(n_items, [&](uint32_t i) {
    return state[i].status == kStatusReady ? min(state[i].cnt_in, items[i].cand_cap) : 0u;
  }, pref);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t per = ((total + gridDim.x - 1) / gridDim.x + 255u) & ~255u;
  const uint32_t j0 = min(total, blockIdx.x * per), j1 = min(total, j0 + per);
  for (uint32_t c = j0; c < j1; c += blockDim.x) {
    const uint32_t j = c + threadIdx.x;
    const bool valid = j < j1;
    uint32_t it = 0xFFFFFFFFu;
    bool keep = false;
    uint2 kv = make_uint2(0u, 0u);
    if (valid) {
      it = flat_item(pref, n_items, j);
      kv = cand[items[it].cand_off + (j - pref[it])];
      keep = (kv.y & 0x7FFFFFFFu) > s_tau[it];
    }
    const uint32_t it0 = flat_item(pref, n_items, c);
    const bool uni = __syncthreads_and(!valid || it == it0) != 0;  // block-uniform
    const EncItem& e0 = items[it0];
    const bool log0 = (e0.flags & kWriteSketch) && (e0.flags & kDeferScatter);
    uint32_t slot = 0;
    if (uni) {
      uint32_t off, nk;
      Scan(scan_tmp).ExclusiveSum(keep ? 1u : 0u, off, nk);
      if (threadIdx.x == 0) {
        if (nk) atomicAdd(&state[it0].kept, nk);
        s_base = (log0 && nk) ? atomicAdd(&state[it0].cnt_hi, nk) : 0u;
      }
      __syncthreads();
      slot = s_base + off;
      __syncthreads();  // s_base / scan storage reuse
    } else {
      // kept counts, aggregated over the lanes of the same item
      const uint32_t grp = __match_any_sync(kFull, it);
      const uint32_t km = __ballot_sync(kFull, keep) & grp;
      if (keep && lane == __ffs(km) - 1) atomicAdd(&state[it].kept, __popc(km));
      if (keep && (items[it].flags & kWriteSketch) && (items[it].flags & kDeferScatter)) {
        const uint32_t leader = __ffs(km) - 1;
        uint32_t b0 = 0;
        if (lane == leader) b0 = atomicAdd(&state[it].cnt_hi, __popc(km));
        b0 = __shfl_sync(km, b0, leader);
        slot = b0 + __popc(km & ((1u << lane) - 1u));
      }
    }
    if (!keep) continue;
    const EncItem& e = items[it];
    const uint32_t p = kv.x;
    const float v = __uint_as_float(kv.y);
    if (e.flags & kHasAcc) e.acc[p] = 0.0f;
    if (e.flags & kWriteResidual) e.residual[p] = 0.0f;
    if (e.flags & kWriteSparse) e.sparse[p] = v;
    if (e.flags & kWriteIndex) {
      if (kW4) red_or_u32(e.index + (p >> 3), 1u << (4u * (p & 7u)));
      else red_or_u32(e.index + (p >> 5), 1u << (p & 31u));
    }
    if ((e.flags & kWriteSketch) && !(e.flags & kDeferScatter)) {
      scatter_sketch(e, hp, p, v);
    } else if (e.flags & kWriteSketch) {  // log it with the speculatively kept: the deferred scatter takes both
      if (slot < e.hi_cap) hi_pool[e.hi_off + slot] = kv;  // kept <= n - c < hi_cap
    }
  }
}

// --------------------------------------------------------------- deferred scatter
// Items whose sketch is far bigger than L2 (kDeferScatter) skip the sketch
// REDs in the fused pass and in k_fixup: every kept entry (pos, v) is logged
// in the item's hi_pool instead. Once tau is final, the (entry, row) updates
// are binned by region of the sketch address space and applied region by
// region.
//  * k_ds_place: each CTA stages a batch of updates in shared memory, sorts
//    it by bin there (counting sort) and writes every bin's run contiguously
//    into that bin's fixed-capacity slice (bins are hash-uniform: capacity =
//    mean * 17/16 + 1024, the excess goes to an overflow list). No count
//    pass, no global scan, coalesced runs instead of 8-byte scatters.
//  * groups spanning up to 2^27 floats (512 MB; the engine splits larger
//    sets of deferred sketches into such groups): bins of 32K floats, and
//    k_ds_apply_smem sums each 16K-float region in shared memory (the two
//    CTAs of a bin read the bin's run, L2 resident, and keep their region's
//    updates) and stores it with plain
//    coalesced stores over the deferred sketches' part of the region — no
//    zeroing pass, no L2 atomics. Larger spans: zeroing pass + L2 REDs bin by
//    bin (k_ds_apply).
//  * k_ds_overflow adds the overflow list with REDs, after the apply.
// Same sums as the direct scatter; only the float summation order differs,
// as it does between any two runs of the direct scatter.
constexpr uint32_t kApplyShift = 14;  // 16K floats = 64 KB per shared-memory region (2 per 32K-float bin)
constexpr uint32_t kApplyRegion = 1u << kApplyShift;
constexpr uint32_t kDsBatch = 4096;   // staged updates per place batch
constexpr uint32_t kDsThreads = 512;  // place: 2 CTAs per SM
constexpr uint32_t kApplyThreads = 512;
using BlockScanDs = cub::BlockScan<uint32_t, kDsThreads>;

__device__ __forceinline__ bool ds_member(const EncItem& e, const SelState& st, uint32_t group) {
  return st.status == kStatusReady && (e.flags & kDeferScatter) && (e.flags & kWriteSketch) && e.ds_group == group;
}
__device__ __forceinline__ uint32_t ds_entries(const EncItem& e, const SelState& st, uint32_t group) {
  return ds_member(e, st, group) ? min(st.cnt_hi, e.hi_cap) : 0u;
}

__device__ __forceinline__ uint32_t ds_cap(uint32_t total_updates, uint32_t n_bins) {
  const uint64_t mean = (uint64_t(total_updates) + n_bins - 1) / n_bins;
  return uint32_t(mean + mean / 16 + 1024);
}

// fill[n_bins] (zero on entry) counts each bin's updates; records hold bin b
// at [b * cap, b * cap + min(fill[b], cap)); ctl[0] = overflow count,
// ctl[1] = cap.
__global__ void __launch_bounds__(kDsThreads, 2) k_ds_place(const EncItem* __restrict__ items,
                                                         const SelState* __restrict__ state, uint32_t n_items,
                                                         const uint2* __restrict__ hi_pool, const HashParams hp,
                                                         const float* base, uint32_t group, uint32_t shift,
                                                         uint32_t n_bins, uint32_t tight, uint32_t* __restrict__ fill,
                                                         uint32_t* __restrict__ ctl,
                                                         uint2* __restrict__ records, uint2* __restrict__ ovf) {
  __shared__ uint32_t pref[kMaxFlatItems + 1];
  __shared__ typename BlockScanDs::TempStorage s_scan;
  extern __shared__ uint2 s_dyn[];
  uint2* s_u = s_dyn;               // unsorted batch
  uint2* s_s = s_dyn + kDsBatch;    // sorted batch
  uint32_t* s_hist = reinterpret_cast<uint32_t*>(s_dyn + 2 * kDsBatch);  // [n_bins]: count, then cursor
  uint32_t* s_loff = s_hist + n_bins;                                     // [n_bins]: local offset
  uint32_t* s_gb = s_loff + n_bins;                                       // [n_bins]: global base
  const uint32_t rows = hp.rows;
  const uint32_t total =
      flat_prefix(n_items, [&](uint32_t i) { return ds_entries(items[i], state[i], group); }, pref);
  // tight (test hook TAGC_DS_TIGHT): a quarter of the mean per bin, so most
  // updates take the overflow path
  const uint32_t cap = tight ? max(1u, (total * rows / n_bins) / 4u) : ds_cap(total * rows, n_bins);
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl[1] = cap;
  const uint32_t per_batch = kDsBatch / rows;
  const uint32_t per_cta = (total + gridDim.x - 1) / gridDim.x;
  const uint32_t j0 = min(total, blockIdx.x * per_cta), j1 = min(total, j0 + per_cta);
  for (uint32_t b0 = j0; b0 < j1; b0 += per_batch) {
    const uint32_t b1 = min(j1, b0 + per_batch);
    const uint32_t nrec = (b1 - b0) * rows;
    for (uint32_t i = threadIdx.x; i < n_bins; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    // kPer entries per thread loaded before any is hashed (memory-level parallelism)
    constexpr uint32_t kPer = 4;
    for (uint32_t q0 = b0; q0 < b1; q0 += kPer * blockDim.x) {
    uint2 kv[kPer];
    uint32_t kit[kPer];
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      const uint32_t j = q0 + q * blockDim.x + threadIdx.x;
      kit[q] = 0;
      kv[q] = make_uint2(0, 0);
      if (j < b1) {
        kit[q] = flat_item(pref, n_items, j);
        kv[q] = __ldcs(hi_pool + items[kit[q]].hi_off + (j - pref[kit[q]]));
      }
    }
#pragma unroll
    for (uint32_t q = 0; q < kPer; ++q) {
      const uint32_t j = q0 + q * blockDim.x + threadIdx.x;
      if (j >= b1) continue;
      const EncItem& e = items[kit[q]];
      const uint64_t sk = uint64_t(e.sketch - base);
      _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < rows) {
        const uint32_t off = uint32_t(sk + uint64_t(r) * e.m + dev_bucket(hp.row[r], kv[q].x, e.m, e.mmul));
        s_u[(j - b0) * rows + r] =
            make_uint2(off, __float_as_uint(dev_sign(hp.row[r], kv[q].x) * __uint_as_float(kv[q].y)));
        atomicAdd(&s_hist[off >> shift], 1u);
      }
    }
    }
    __syncthreads();
    {  // exclusive scan of the bin counts (each thread a run of bins); global slices reserved in parallel
      const uint32_t per = (n_bins + blockDim.x - 1) / blockDim.x;
      const uint32_t c0 = min(n_bins, threadIdx.x * per), c1 = min(n_bins, c0 + per);
      uint32_t sum = 0;
      for (uint32_t b = c0; b < c1; ++b) sum += s_hist[b];
      uint32_t off;
      BlockScanDs(s_scan).ExclusiveSum(sum, off);
      for (uint32_t b = c0; b < c1; ++b) {
        const uint32_t h = s_hist[b];
        s_gb[b] = h ? atomicAdd(fill + b, h) : 0u;
        s_loff[b] = off;
        s_hist[b] = off;  // becomes the placement cursor
        off += h;
      }
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nrec; k += blockDim.x) {
      const uint2 rec = s_u[k];
      s_s[atomicAdd(&s_hist[rec.x >> shift], 1u)] = rec;
    }
    __syncthreads();
    for (uint32_t k = threadIdx.x; k < nrec; k += blockDim.x) {
      const uint2 rec = s_s[k];
      const uint32_t b = rec.x >> shift;
      const uint32_t g = s_gb[b] + (k - s_loff[b]);
      if (g < cap) records[uint64_t(b) * cap + g] = rec;
      else ovf[atomicAdd(ctl, 1u)] = rec;
    }
    __syncthreads();
  }
}

// One CTA per 16K-float region (2^(shift - kApplyShift) CTAs per bin): the bin's run
// is read by each of its CTAs (L2 resident), each keeps its region's updates
// in shared memory, then stores the region over the part that belongs to
// deferred, finally-selected sketches (gaps and fallen-back items are left
// alone).
__global__ void __launch_bounds__(kApplyThreads) k_ds_apply_smem(const EncItem* __restrict__ items,
                                                              const SelState* __restrict__ state, uint32_t n_items,
                                                              uint32_t group, uint32_t rows, uint32_t shift,
                                                              const uint2* __restrict__ records,
                                                              const uint32_t* __restrict__ fill,
                                                              const uint32_t* __restrict__ ctl, float* base) {
  extern __shared__ float4 s_acc4[];
  float* s_acc = reinterpret_cast<float*>(s_acc4);
  const uint32_t reg = blockIdx.x;
  const uint32_t b = reg >> (shift - kApplyShift);
  for (uint32_t i = threadIdx.x; i < kApplyRegion / 4; i += blockDim.x) s_acc4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  const uint32_t cap = ctl[1];
  const uint32_t n = min(fill[b], cap);
  const uint2* run = records + uint64_t(b) * cap;
  constexpr uint32_t kDepth = 8;  // loads in flight per thread
  for (uint32_t i0 = 0; i0 < n; i0 += blockDim.x * kDepth) {
    uint2 r[kDepth];
#pragma unroll
    for (uint32_t q = 0; q < kDepth; ++q) {
      const uint32_t i = i0 + q * blockDim.x + threadIdx.x;
      r[q] = i < n ? __ldcg(run + i) : make_uint2(0xFFFFFFFFu, 0u);
    }
#pragma unroll
    for (uint32_t q = 0; q < kDepth; ++q)
      if ((r[q].x >> kApplyShift) == reg) atomicAdd(s_acc + (r[q].x & (kApplyRegion - 1u)), __uint_as_float(r[q].y));
  }
  __syncthreads();
  const uint64_t g0 = uint64_t(reg) << kApplyShift, g1 = g0 + kApplyRegion;
  for (uint32_t it = 0; it < n_items; ++it) {
    const EncItem& e = items[it];
    if (!ds_member(e, state[it], group)) continue;
    const uint64_t a = uint64_t(e.sketch - base), z = a + uint64_t(rows) * e.m;
    const uint64_t lo = a > g0 ? a : g0, hi = z < g1 ? z : g1;
    for (uint64_t x = lo + threadIdx.x; x < hi; x += blockDim.x) base[x] = s_acc[x - g0];
  }
}

// The RED path's sketches start at zero: written right before the apply
// (full-sector stores allocate their lines in L2 without a DRAM read), for
// the items whose select is final (a fallen-back item was re-encoded exactly
// and scattered directly into its freshly cleared sketch).
__global__ void __launch_bounds__(256) k_ds_zero(const EncItem* __restrict__ items,
                                                 const SelState* __restrict__ state, uint32_t n_items,
                                                 uint32_t group, uint32_t rows) {
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint32_t it = 0; it < n_items; ++it) {
    const EncItem& e = items[it];
    if (!ds_member(e, state[it], group)) continue;
    const uint64_t n = uint64_t(rows) * e.m;
    float* p = e.sketch;
    const uint64_t mis = ((16u - (reinterpret_cast<uintptr_t>(p) & 15u)) & 15u) / 4u;
    const uint64_t head = n < mis ? n : mis;
    for (uint64_t i = tid; i < head; i += stride) p[i] = 0.0f;
    float4* p4 = reinterpret_cast<float4*>(p + head);
    const uint64_t n4 = (n - head) / 4;
    for (uint64_t i = tid; i < n4; i += stride) p4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint64_t i = head + 4 * n4 + tid; i < n; i += stride) p[i] = 0.0f;
  }
}

// RED path: bins in order (CTA-strided over bins, grid-stride inside), so all
// CTAs sweep the address space together and the REDs hit L2.
__global__ void __launch_bounds__(256) k_ds_apply(const uint2* __restrict__ records, const uint32_t* __restrict__ fill,
                                                  const uint32_t* __restrict__ ctl, uint32_t n_bins, float* base) {
  const uint32_t cap = ctl[1];
  for (uint32_t b = 0; b < n_bins; ++b) {
    const uint32_t n = min(fill[b], cap);
    const uint2* run = records + uint64_t(b) * cap;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const uint2 r = __ldcs(run + i);
      red_add_f32(base + r.x, __uint_as_float(r.y));
    }
  }
}

// Updates beyond their bin's capacity (never, for hash-uniform bins), after
// the apply.
__global__ void __launch_bounds__(256) k_ds_overflow(const uint2* __restrict__ ovf, const uint32_t* __restrict__ ctl,
                                                     float* base) {
  const uint32_t n = ctl[0];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint2 r = ovf[i];
    red_add_f32(base + r.x, __uint_as_float(r.y));
  }
}

// --------------------------------------------------------------- fallback
// Bracket missed: put the combined value back into the accumulator of every
// speculatively kept element, clear the sketch, and rerun an exact radix
// select + encode for that item only.
__device__ __forceinline__ void restore_body(const EncItem* __restrict__ items, SelState* __restrict__ state,
                                             uint32_t n_items, const uint2* __restrict__ hi_pool, uint32_t rows) {
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gstride = uint64_t(gridDim.x) * blockDim.x;
  for (uint32_t it = 0; it < n_items; ++it) {
    if (state[it].status != kStatusFallback) continue;
    const EncItem e = items[it];
    if (e.flags & kHasAcc) {
      const uint32_t cnt = min(state[it].cnt_hi, e.hi_cap);
      for (uint64_t i = gtid; i < cnt; i += gstride) {
        const uint2 kv = hi_pool[e.hi_off + i];
        e.acc[kv.x] = __uint_as_float(kv.y);
      }
    }
    if (e.flags & kWriteSketch)
      for (uint64_t i = gtid; i < uint64_t(rows) * e.m; i += gstride) e.sketch[i] = 0.0f;
  }
}

__device__ __forceinline__ void fb_hist_body(const EncItem* __restrict__ items,
                                             const SelState* __restrict__ state, uint32_t n_items,
                                             uint64_t total_tiles, uint32_t* __restrict__ fb_hist, int pass,
                                             uint32_t* hist) {
  const int shift = digit_shift(pass), bits = digit_bits(pass), hs = shift + bits;
  for (uint64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const uint32_t it = find_tile_item(items, n_items, tile);
    if (state[it].status != kStatusFallback) continue;  // block-uniform
    const EncItem e = items[it];
    const uint32_t prefix = state[it].prefix;
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t q0 = uint32_t(tile - e.tile_begin) * (kTile / 4);
    for (int k = 0; k < 4; ++k) {
      const uint32_t pos = 4u * (q0 + k * kTileThreads + threadIdx.x);
      if (pos >= e.n) continue;
      float v[4];
      load_source(e, pos, true, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = mag_key(v[j]);
        if (pos + j < e.n && (key >> hs) == (prefix >> hs))
          atomicAdd(&hist[(key >> shift) & ((1u << bits) - 1u)], 1u);
      }
    }
    __syncthreads();
    uint32_t* dst = fb_hist + uint64_t(it) * kRadixBins;
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x)
      if (hist[i]) atomicAdd(dst + i, hist[i]);
    __syncthreads();
  }
}

__device__ __forceinline__ void fb_scan_body(SelState* __restrict__ state, uint32_t n_items,
                                             uint32_t* __restrict__ fb_hist, int pass, uint32_t* s_digit,
                                             uint32_t* s_below) {
  for (uint32_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    if (state[item].status != kStatusFallback) continue;  // block-uniform
    uint32_t* h = fb_hist + uint64_t(item) * kRadixBins;
    const uint32_t rank = state[item].rank;
    find_digit<kTileThreads>(h, 1u << digit_bits(pass), rank, s_digit, s_below);
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) h[i] = 0;
    if (threadIdx.x == 0) {
      const uint32_t prefix = state[item].prefix | (*s_digit << digit_shift(pass));
      state[item].prefix = prefix;
      state[item].rank = rank - *s_below;
      if (pass == 2) {
        state[item].tau_key = prefix;
        state[item].status = kStatusFbReady;
        state[item].kept = 0;
      }
    }
    __syncthreads();
  }
}

// --------------------------------------------------------------- exact encode
// Split + index + sketch for a known tau. mode 0: every item, tau = 0
// (CountSketch::compress / Index::create entry points); mode 1: only items
// whose selection fell back (status 4), reading the restored values.
constexpr uint32_t kKeptStage = 1024;  // kept elements staged per tile (overflow: direct)

template <bool kW4>
__device__ __forceinline__ void encode_body(const EncItem* __restrict__ items, SelState* __restrict__ state,
                                            uint32_t n_items, uint64_t total_tiles, const HashParams& hp,
                                            int mode, uint32_t* s_pos, float* s_val, uint32_t& s_n) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t t0, t1;
  cta_range(total_tiles, t0, t1);
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  uint32_t it = t0 < t1 ? find_tile_item(items, n_items, t0) : 0;
  for (uint64_t tile = t0; tile < t1; ++tile) {
    while (it + 1 < n_items && items[it + 1].tile_begin <= tile) ++it;
    if (mode == 1 && state[it].status != kStatusFbReady) continue;  // block-uniform
    const EncItem e = items[it];
    const uint32_t tau = mode == 1 ? state[it].tau_key : 0u;
    const bool vec = (e.flags & kAligned16) != 0;
    const uint32_t n_words = kW4 ? (e.n + 7u) / 8u : (e.n + 31u) / 32u;
    const uint32_t q0 = uint32_t(tile - e.tile_begin) * (kTile / 4);
    float v[4][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t pos = 4u * (q0 + k * kTileThreads + threadIdx.x);
      if (pos < e.n) {
        load_source(e, pos, mode == 1, v[k]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) v[k][j] = 0.0f;
      }
    }
    uint32_t kept = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t q = q0 + k * kTileThreads + threadIdx.x;
      const uint32_t pos = 4u * q;
      uint32_t nib = 0;
      if (pos < e.n) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (pos + j < e.n && mag_key(v[k][j]) > tau) nib |= 1u << j;
        if (e.flags & kHasAcc) {
          float r[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) r[j] = (nib >> j & 1u) ? 0.0f : v[k][j];
          store_quad(e.acc, pos, e.n, vec, r);
        }
        if (e.flags & kWriteResidual) {
          float r[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) r[j] = (nib >> j & 1u) ? 0.0f : v[k][j];
          store_quad(e.residual, pos, e.n, false, r);
        }
        if (e.flags & kWriteSparse) {
          float sp[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) sp[j] = (nib >> j & 1u) ? v[k][j] : 0.0f;
          store_quad(e.sparse, pos, e.n, false, sp);
        }
        if ((e.flags & kWriteSketch) && nib) {
          const uint32_t base = atomicAdd(&s_n, uint32_t(__popc(nib)));
          uint32_t o = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (nib >> j & 1u) {
              if (base + o < kKeptStage) {
                s_pos[base + o] = pos + j;
                s_val[base + o] = v[k][j];
              } else {  // dense tile: scatter directly
                scatter_sketch(e, hp, pos + j, v[k][j]);
              }
              ++o;
            }
        }
        kept += __popc(nib);
      }
      if (e.flags & kWriteIndex) {
        if (kW4) {
          if (q < 2u * n_words) {
            const uint32_t hw = (nib & 1u) | (nib >> 1 & 1u) << 4 | (nib >> 2 & 1u) << 8 |
                                (nib >> 3 & 1u) << 12;
            reinterpret_cast<uint16_t*>(e.index)[q] = uint16_t(hw);
          }
        } else {
          uint32_t x = nib << (4u * (lane & 7u));
          x |= __shfl_xor_sync(kFull, x, 1);
          x |= __shfl_xor_sync(kFull, x, 2);
          x |= __shfl_xor_sync(kFull, x, 4);
          if ((lane & 7u) == 0 && q / 8u < n_words) e.index[q / 8u] = x;
        }
      }
    }
    kept = warp_sum(kept);
    if (lane == 0 && kept) atomicAdd(&state[it].kept, kept);
    if (e.flags & kWriteSketch) {
      __syncthreads();
      const uint32_t nk = min(s_n, kKeptStage);
      for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) scatter_sketch(e, hp, s_pos[i], s_val[i]);
      __syncthreads();
      if (threadIdx.x == 0) s_n = 0;
      __syncthreads();
    }
  }
}

template <bool kW4>
__global__ void __launch_bounds__(kTileThreads, 5) k_encode(const EncItem* __restrict__ items,
                                                            SelState* __restrict__ state,
                                                            uint32_t n_items, uint64_t total_tiles,
                                                            const HashParams hp,
                                                            const uint32_t* __restrict__ err) {
  __shared__ uint32_t s_pos[kKeptStage];
  __shared__ float s_val[kKeptStage];
  __shared__ uint32_t s_n;
  if (err && err[0]) return;  // NaN anywhere: nothing more is written
  encode_body<kW4>(items, state, n_items, total_tiles, hp, 0, s_pos, s_val, s_n);
}

// The whole bracket-miss repair in one cooperative launch: restore, three
// radix-select digit passes, exact re-encode of the fallen-back items. In the
// normal case (no item fell back, or NaN) every CTA returns at once.
template <bool kW4>
__global__ void __launch_bounds__(kTileThreads) k_fallback(const EncItem* __restrict__ items,
                                                           SelState* __restrict__ state, uint32_t n_items,
                                                           uint64_t total_tiles, const HashParams hp,
                                                           const uint2* __restrict__ hi_pool,
                                                           uint32_t* __restrict__ fb_hist,
                                                           const uint32_t* __restrict__ err) {
  __shared__ uint32_t s_hist[kRadixBins];
  __shared__ uint32_t s_pos[kKeptStage];
  __shared__ float s_val[kKeptStage];
  __shared__ uint32_t s_n, s_digit, s_below;
  if (err[0] || !err[1]) return;  // grid-uniform
  cg::grid_group grid = cg::this_grid();
  restore_body(items, state, n_items, hi_pool, hp.rows);
  for (int pass = 0; pass < 3; ++pass) {
    grid.sync();
    fb_hist_body(items, state, n_items, total_tiles, fb_hist, pass, s_hist);
    grid.sync();
    fb_scan_body(state, n_items, fb_hist, pass, &s_digit, &s_below);
  }
  grid.sync();
  encode_body<kW4>(items, state, n_items, total_tiles, hp, 1, s_pos, s_val, s_n);
}

// --------------------------------------------------------------- folds
__global__ void k_rank_sum_f32(const float* const* __restrict__ in, uint32_t world,
                               float* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    float acc = 0.0f;
    for (uint32_t r = 0; r < world; ++r) acc += in[r][i];
    out[i] = acc;
  }
}

__global__ void k_rank_sum_u32(const uint32_t* const* __restrict__ in, uint32_t world,
                               uint32_t* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t acc = 0;
    for (uint32_t r = 0; r < world; ++r) acc += in[r][i];
    out[i] = acc;
  }
}

__global__ void k_add(const float* __restrict__ a, const float* __restrict__ b,
                      float* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = a[i] + b[i];
}

// Owner-side consumer of the decoded shard as a standalone pass (the fused
// form is the OptEpilogue of k_emit / k_copy_items): params / adam_v updated
// from decoded (read only).
template <bool kAdam>
__global__ void __launch_bounds__(256) k_apply_optimizer(OptEpilogue o, uint64_t n) {
  constexpr uint64_t kChunk = 256 * 8;
  for (uint64_t c0 = uint64_t(blockIdx.x) * kChunk; c0 < n; c0 += uint64_t(gridDim.x) * kChunk)
    opt_range<kAdam, true>(o, const_cast<float*>(o.out_base) + c0, o.out_base + c0,
                           uint32_t(n - c0 < kChunk ? n - c0 : kChunk));
}

// Raw-segment pack/unpack: flat 4096-element tiles over all items, 16-byte
// accesses when source and destination are both aligned.
template <bool kOpt>
__global__ void __launch_bounds__(256) k_copy_items(const CopyItem* __restrict__ items,
                                                    uint32_t n_items, uint64_t total_tiles,
                                                    const OptEpilogue* __restrict__ opt) {
  for (uint64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    uint32_t lo = 0, hi = n_items - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (items[mid].tile_begin <= tile) lo = mid;
      else hi = mid - 1;
    }
    const CopyItem it = items[lo];
    const uint64_t b = (tile - it.tile_begin) * kCopyTile;
    const uint64_t e = min(it.n, b + kCopyTile);
    if (!it.src) {  // zero-fill item
      if ((reinterpret_cast<uintptr_t>(it.dst) & 15u) == 0) {
        for (uint64_t i = b + 4ull * threadIdx.x; i < e; i += 4ull * blockDim.x) {
          if (i + 4 <= e) __stcs(reinterpret_cast<float4*>(it.dst + i), make_float4(0.f, 0.f, 0.f, 0.f));
          else for (uint64_t j = i; j < e; ++j) it.dst[j] = 0.0f;
        }
      } else {
        for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) it.dst[i] = 0.0f;
      }
      continue;
    }
    if (kOpt) {  // owner's raw segment: the optimizer step on the summed value
      const OptEpilogue o = *opt;
      if (o.kind == 1) opt_range<true, true>(o, it.dst + b, it.src + b, uint32_t(e - b));
      else opt_range<false, true>(o, it.dst + b, it.src + b, uint32_t(e - b));
      continue;
    }
    const bool vec = ((reinterpret_cast<uintptr_t>(it.src) | reinterpret_cast<uintptr_t>(it.dst)) & 15u) == 0;
    if (vec) {
      for (uint64_t i = b + 4ull * threadIdx.x; i < e; i += 4ull * blockDim.x) {
        if (i + 4 <= e) {
          *reinterpret_cast<float4*>(it.dst + i) = __ldg(reinterpret_cast<const float4*>(it.src + i));
        } else {
          for (uint64_t j = i; j < e; ++j) it.dst[j] = it.src[j];
        }
      }
    } else {
      for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) it.dst[i] = it.src[i];
    }
  }
}

__global__ void k_raw_sum(const RawItem* __restrict__ items, const float* const* __restrict__ bases,
                          uint32_t world) {
  const RawItem it = items[blockIdx.y];
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < it.n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    float acc = 0.0f;
    for (uint32_t r = 0; r < world; ++r) acc += bases[r][it.src_off + i];
    it.dst[i] = acc;
  }
}

__global__ void k_index_diag(const DiagItem* __restrict__ items,
                             const uint32_t* const* __restrict__ rank_words, uint32_t world,
                             unsigned long long* __restrict__ out) {
  const DiagItem it = items[blockIdx.y];
  uint32_t lost = 0, spur = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < it.n_words;
       w += gridDim.x * blockDim.x) {
    uint32_t truth = 0;
    for (uint32_t r = 0; r < world; ++r) truth |= rank_words[r][it.word_off + w];
    const uint32_t x = it.merged[w];
    uint32_t present, valid;
    const uint64_t first = uint64_t(w) * (it.width == 4 ? 8u : 32u);
    const uint64_t left = it.n > first ? it.n - first : 0;
    if (it.width == 4) {
      present = (x | x >> 1 | x >> 2 | x >> 3) & 0x11111111u;
      truth &= 0x11111111u;
      valid = left >= 8 ? 0x11111111u : (0x11111111u & ((1u << (4 * left)) - 1u));
    } else {
      present = x;
      valid = left >= 32 ? 0xFFFFFFFFu : ((1u << left) - 1u);
    }
    present &= valid;
    truth &= valid;
    lost += __popc(truth & ~present);
    spur += __popc(present & ~truth);
  }
  lost = warp_sum(lost);
  spur = warp_sum(spur);
  if ((threadIdx.x & 31) == 0) {
    if (lost) atomicAdd(&out[2 * blockIdx.y], (unsigned long long)lost);
    if (spur) atomicAdd(&out[2 * blockIdx.y + 1], (unsigned long long)spur);
  }
}

__global__ void __launch_bounds__(256) k_zero(const ZeroRanges r) {
  for (int k = 0; k < r.n; ++k) {
    char* p = static_cast<char*>(r.ptr[k]);
    const uint64_t n = r.bytes[k];
    const uint64_t mis = (16u - (reinterpret_cast<uintptr_t>(p) & 15u)) & 15u;
    const uint64_t head = mis < n ? mis : n;
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < head; i += stride) p[i] = 0;
    const uint64_t nv = (n - head) / 16;
    uint4* v = reinterpret_cast<uint4*>(p + head);
    for (uint64_t i = tid; i < nv; i += stride) v[i] = make_uint4(0u, 0u, 0u, 0u);
    for (uint64_t i = head + nv * 16 + tid; i < n; i += stride) p[i] = 0;
  }
}

__global__ void __launch_bounds__(256) k_stage_copy(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                                    uint64_t n16) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += uint64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

int persistent_grid(const void* fn, int threads, const DevInfo& di, uint64_t work) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
  if (per_sm < 1) per_sm = 1;
  const uint64_t g = uint64_t(per_sm) * di.sms;
  return int(work < g ? (work ? work : 1) : g);
}

int flat_grid(uint64_t n, int threads) {
  const uint64_t b = (n + threads - 1) / threads;
  return int(b < 4096 ? (b ? b : 1) : 4096);
}

}  // namespace

int launch_select_fused(const DevInfo& di, const EncItem* items, SelState* state, uint32_t n_items,
                        uint64_t total_tiles, uint64_t total_samples, const HashParams& hp, bool w4,
                        int per_stage, uint32_t* sample_hist, uint32_t* fine_hist, uint2* cand,
                        uint2* hi_pool, uint32_t* err, cudaStream_t stream, unsigned long long* span,
                        bool tma, uint64_t sketch_bytes) {
  if (n_items == 0) return 0;
  int launches = 0;
  if (total_samples) {
    k_sample<<<persistent_grid((const void*)k_sample, kTileThreads, di, total_samples), kTileThreads,
               0, stream>>>(items, n_items, total_samples, sample_hist, span);
    ++launches;
  }
  if (total_samples) {
    launch_pdl(k_window_coarse, dim3(n_items), dim3(256), 0, stream, items, state, sample_hist, span);
    launch_pdl(k_sample_fine, dim3(persistent_grid((const void*)k_sample_fine, kTileThreads, di, total_samples)),
               dim3(kTileThreads), 0, stream, items, state, n_items, total_samples, sample_hist);
    launches += 2;
  }
  launch_pdl(k_window_fine, dim3(n_items), dim3(256), 0, stream, items, state, sample_hist);
  // every item of a batch shares the path: hook (accumulator) or per-stage outputs
  const bool hook = per_stage == 0;
  auto launch = [&](auto kern) {
    kern<<<persistent_grid((const void*)kern, kTileThreads, di, total_tiles), kTileThreads, 0, stream>>>(
        items, state, n_items, total_tiles, hp, cand, hi_pool, fine_hist, err, span);
  };
  if (tma && hook) {
    auto launch_tma = [&](auto kern) {
      // opt-in to > 48 KB of dynamic shared memory (cheap; per launch keeps it per device)
      cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kFusedSmem));
      // A batch that scatters into no sketch (every sketch deferred: C4) is a
      // pure stream: non-persistent, ceil(tiles / 10) CTAs of 10 contiguous
      // tiles each, a retiring CTA's slot refilled, so no SM waits on the
      // slowest share (C4: 0.580 -> 0.522 ms; K = 4 / 6 / 8 / 12 / 16:
      // 0.581 / 0.535 / 0.525 / 0.525 / 0.530; the bare ring of
      // tools/micro/tma_ring.cu: 6.2 -> 6.6 TB/s). Batches with direct
      // scatters stay persistent (GPT-2 0.25 -> 0.30 ms, Llama-3-8B 18.4 ->
      // 23.2 ms non-persistent). TAGC_FUSED_TILES_PER_CTA overrides (0:
      // persistent).
      static const char* per_env = std::getenv("TAGC_FUSED_TILES_PER_CTA");
      const uint64_t per_cta = per_env ? std::strtoull(per_env, nullptr, 10) : (sketch_bytes == 0 ? 10 : 0);
      const uint64_t g = per_cta ? (total_tiles + per_cta - 1) / per_cta
                                 : std::min<uint64_t>(uint64_t(di.sms) * kFusedCtasPerSm, total_tiles);
      // one contiguous range per CTA while every sketch fits in L2 together;
      // beyond that, small chunks claimed from a counter keep every CTA in
      // one narrow window of the shard, whose sketch rows stay L2-resident
      // (Llama-3-8B fused pass: 64-tile chunks 19.1 ms, 8: 18.6, 2: 18.35,
      // 1: 18.9 — the counter atomics start to cost; TAGC_FUSED_CHUNK)
      const uint64_t contiguous = (total_tiles + (g ? g : 1) - 1) / (g ? g : 1);
      static const uint64_t chunk_tiles = std::getenv("TAGC_FUSED_CHUNK") ? std::strtoull(std::getenv("TAGC_FUSED_CHUNK"), nullptr, 10) : 2;
      static const uint64_t chunk_above = (std::getenv("TAGC_FUSED_CHUNK_ABOVE_MB") ? std::strtoull(std::getenv("TAGC_FUSED_CHUNK_ABOVE_MB"), nullptr, 10) : 48ull) << 20;
      const uint32_t chunk = uint32_t(per_cta || sketch_bytes <= chunk_above ? 0 : std::min<uint64_t>(chunk_tiles, contiguous));
      launch_pdl(kern, dim3(unsigned(g ? g : 1)), dim3(kFusedThreads), kFusedSmem, stream, items, state, n_items,
                 total_tiles, hp, cand, hi_pool, fine_hist, err, span, chunk);
    };
    if (w4) launch_tma(k_fused_tma<true>);
    else launch_tma(k_fused_tma<false>);
  } else if (w4 && hook) launch(k_fused<true, true>);
  else if (w4) launch(k_fused<true, false>);
  else if (hook) launch(k_fused<false, true>);
  else launch(k_fused<false, false>);
  return launches + 2;
}

int launch_select_finish(const DevInfo& di, const EncItem* items, SelState* state, uint32_t n_items,
                         uint64_t total_tiles, const HashParams& hp, bool w4, uint32_t* fine_hist,
                         uint32_t* fb_hist, uint2* cand, uint2* hi_pool, uint32_t* sel_list,
                         uint32_t* err, cudaStream_t stream) {
  if (n_items == 0) return 0;
  k_finish_select<<<dim3(kFinishCtas, n_items), kFinishThreads, 0, stream>>>(items, state, fine_hist, cand,
                                                                           sel_list, err);
  if (w4) k_fixup<true><<<di.sms * 4, 256, 0, stream>>>(items, state, n_items, cand, hp, err, hi_pool);
  else k_fixup<false><<<di.sms * 4, 256, 0, stream>>>(items, state, n_items, cand, hp, err, hi_pool);
  // bracket-miss repair: one cooperative launch that exits at once unless some item fell back
  auto launch_fb = [&](auto kern) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kern, kTileThreads, 0);
    const uint64_t g = std::min<uint64_t>(uint64_t(coop_grid(di, std::max(per_sm, 1))), std::max<uint64_t>(total_tiles, 1));
    const EncItem* a0 = items;
    SelState* a1 = state;
    uint32_t a2 = n_items;
    uint64_t a3 = total_tiles;
    HashParams a4 = hp;
    const uint2* a5 = hi_pool;
    uint32_t* a6 = fb_hist;
    const uint32_t* a7 = err;
    void* args[] = {&a0, &a1, &a2, &a3, &a4, &a5, &a6, &a7};
    cudaLaunchCooperativeKernel((const void*)kern, dim3(unsigned(g)), dim3(kTileThreads), args, 0, stream);
  };
  if (w4) launch_fb(k_fallback<true>);
  else launch_fb(k_fallback<false>);
  return 3;
}

int launch_encode_exact(const DevInfo& di, const EncItem* items, SelState* state, uint32_t n_items,
                        uint64_t total_tiles, const HashParams& hp, const uint32_t* err, bool w4,
                        cudaStream_t stream) {
  if (n_items == 0) return 0;
  if (w4) {
    const int g = persistent_grid((const void*)k_encode<true>, kTileThreads, di, total_tiles);
    k_encode<true><<<g, kTileThreads, 0, stream>>>(items, state, n_items, total_tiles, hp, err);
  } else {
    const int g = persistent_grid((const void*)k_encode<false>, kTileThreads, di, total_tiles);
    k_encode<false><<<g, kTileThreads, 0, stream>>>(items, state, n_items, total_tiles, hp, err);
  }
  return 1;
}

int launch_zero(const ZeroRanges& r, cudaStream_t stream) {
  uint64_t mx = 0;
  for (int k = 0; k < r.n; ++k) mx = std::max<uint64_t>(mx, r.bytes[k]);
  if (!mx) return 0;
  const uint64_t blocks = std::min<uint64_t>((mx / 16 + 255) / 256 + 1, 148ull * 8);
  k_zero<<<int(blocks), 256, 0, stream>>>(r);
  return 1;
}

// dst and mapped_src 16-byte aligned, bytes a multiple of 16 (the staging
// arena rounds every upload up).
int launch_stage_copy(void* dst, const void* mapped_src, uint64_t bytes, cudaStream_t stream) {
  const uint64_t n16 = bytes / 16;
  if (!n16) return 0;
  const uint64_t blocks = std::min<uint64_t>((n16 + 255) / 256, 64);
  k_stage_copy<<<int(blocks), 256, 0, stream>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(mapped_src),
                                                n16);
  return 1;
}

int launch_rank_sum_f32(const float* const* in_ptrs, uint32_t world, float* out, uint64_t n,
                        cudaStream_t stream) {
  if (!n) return 0;
  k_rank_sum_f32<<<flat_grid(n, 256), 256, 0, stream>>>(in_ptrs, world, out, n);
  return 1;
}

int launch_rank_sum_u32(const uint32_t* const* in_ptrs, uint32_t world, uint32_t* out, uint64_t n,
                        cudaStream_t stream) {
  if (!n) return 0;
  k_rank_sum_u32<<<flat_grid(n, 256), 256, 0, stream>>>(in_ptrs, world, out, n);
  return 1;
}

__global__ void k_set_opt(OptEpilogue* dst, OptEpilogue o) { *dst = o; }

__global__ void k_set_u32(uint32_t* dst, uint32_t v) { *dst = v; }

int launch_set_u32(uint32_t* dst, uint32_t v, cudaStream_t stream) {
  k_set_u32<<<1, 1, 0, stream>>>(dst, v);
  return 1;
}

int launch_set_opt(OptEpilogue* dev_opt, const OptEpilogue& o, cudaStream_t stream) {
  k_set_opt<<<1, 1, 0, stream>>>(dev_opt, o);
  return 1;
}

int launch_deferred_scatter(const DevInfo& di, const EncItem* items, const SelState* state, uint32_t n_items,
                            uint32_t group, const uint2* hi_pool, const HashParams& hp, float* base,
                            uint64_t span_floats, uint32_t* fill, uint32_t* ctl, uint2* records, uint2* ovf,
                            cudaStream_t stream) {
  if (!n_items) return 0;
  if (span_floats > 0xFFFFFFFFull || span_floats == 0) return -1;  // caller scatters directly
  uint32_t lg = 0;
  while ((1ull << lg) < span_floats) ++lg;
  const bool smem = lg <= 27;  // bins of 2 shared-memory regions, <= 4096 bins
  static const uint32_t extra = std::getenv("TAGC_DS_BIN_SHIFT") ? uint32_t(std::atoi(std::getenv("TAGC_DS_BIN_SHIFT"))) : 1u;
  const uint32_t shift = smem ? std::max<uint32_t>(kApplyShift + extra, lg > 12 ? lg - 12 : 0)
                              : std::max<uint32_t>(22, lg - 12);
  const uint32_t n_bins = uint32_t((span_floats + (1ull << shift) - 1) >> shift);
  const int smem_place = int(2 * kDsBatch * sizeof(uint2) + 3 * n_bins * sizeof(uint32_t));
  const uint32_t tight = std::getenv("TAGC_DS_TIGHT") && std::atoi(std::getenv("TAGC_DS_TIGHT")) != 0 ? 1u : 0u;
  cudaFuncSetAttribute((const void*)k_ds_place, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_place);
  static const int place_per_sm = std::getenv("TAGC_DS_PLACE_PER_SM") ? std::max(1, std::atoi(std::getenv("TAGC_DS_PLACE_PER_SM"))) : 2;
  k_ds_place<<<di.sms * place_per_sm, kDsThreads, smem_place, stream>>>(items, state, n_items, hi_pool, hp, base, group, shift,
                                                         n_bins, tight, fill, ctl, records, ovf);
  int l = 1;
  if (smem) {
    const uint32_t regions = uint32_t((span_floats + kApplyRegion - 1) >> kApplyShift);
    cudaFuncSetAttribute((const void*)k_ds_apply_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kApplyRegion * 4));
    k_ds_apply_smem<<<regions, kApplyThreads, kApplyRegion * 4, stream>>>(items, state, n_items, group, hp.rows,
                                                                           shift, records, fill, ctl, base);
    ++l;
  } else {
    k_ds_zero<<<di.sms * 4, 256, 0, stream>>>(items, state, n_items, group, hp.rows);
    k_ds_apply<<<di.sms * 8, 256, 0, stream>>>(records, fill, ctl, n_bins, base);
    l += 2;
  }
  k_ds_overflow<<<di.sms, 256, 0, stream>>>(ovf, ctl, base);
  return l + 1;
}

int launch_apply_optimizer(const OptEpilogue& o, uint64_t n, cudaStream_t stream) {
  if (!n) return 0;
  const int g = int(std::min<uint64_t>((n + 2047) / 2048, 148ull * 16));
  if (o.kind == 0) k_apply_optimizer<false><<<g, 256, 0, stream>>>(o, n);
  else k_apply_optimizer<true><<<g, 256, 0, stream>>>(o, n);
  return 1;
}

int launch_add(const float* a, const float* b, float* out, uint64_t n, cudaStream_t stream) {
  if (!n) return 0;
  k_add<<<flat_grid(n, 256), 256, 0, stream>>>(a, b, out, n);
  return 1;
}

uint64_t copy_tiles(CopyItem* items, uint32_t n_items) {
  uint64_t t = 0;
  for (uint32_t i = 0; i < n_items; ++i) {
    items[i].tile_begin = t;
    t += (items[i].n + kCopyTile - 1) / kCopyTile;
  }
  return t;
}

int launch_copy_items(const DevInfo& di, const CopyItem* items, uint32_t n_items, uint64_t total_tiles,
                      cudaStream_t stream, bool one_tile_per_cta, const OptEpilogue* dev_opt) {
  if (!n_items || !total_tiles) return 0;
  // one tile per CTA: short CTAs that a higher-priority stream's kernels can
  // interleave with as SMs free up (side-stream copies)
  const uint64_t g = one_tile_per_cta ? std::min<uint64_t>(total_tiles, 0x7FFFFFFFull)
                                      : std::min<uint64_t>(total_tiles, uint64_t(di.sms) * 8);
  if (dev_opt) k_copy_items<true><<<int(g), 256, 0, stream>>>(items, n_items, total_tiles, dev_opt);
  else k_copy_items<false><<<int(g), 256, 0, stream>>>(items, n_items, total_tiles, nullptr);
  return 1;
}

int launch_raw_sum(const RawItem* items, uint32_t n_items, uint64_t max_n,
                   const float* const* rank_bases, uint32_t world, cudaStream_t stream) {
  if (!n_items || !max_n) return 0;
  dim3 grid(std::min<uint64_t>((max_n + 255) / 256, 1024), n_items);
  k_raw_sum<<<grid, 256, 0, stream>>>(items, rank_bases, world);
  return 1;
}

int launch_index_diag(const DiagItem* items, uint32_t n_items, uint32_t max_words,
                      const uint32_t* const* rank_words, uint32_t world,
                      unsigned long long* lost_spurious, cudaStream_t stream) {
  if (!n_items) return 0;
  dim3 grid(std::min<uint32_t>((max_words + 255) / 256, 512), n_items);
  k_index_diag<<<grid, 256, 0, stream>>>(items, rank_words, world, lost_spurious);
  return 1;
}

// Loads every kernel of this file now (see preload_all_kernels).
void preload_encode_kernels() {
  const void* fns[] = {(const void*)k_add, (const void*)k_apply_optimizer<false>, (const void*)k_apply_optimizer<true>, (const void*)k_copy_items<false>, (const void*)k_copy_items<true>, (const void*)k_ds_apply, (const void*)k_ds_apply_smem, (const void*)k_ds_zero, (const void*)k_ds_overflow, (const void*)k_ds_place, (const void*)k_encode<false>, (const void*)k_encode<true>, (const void*)k_fallback<false>, (const void*)k_fallback<true>, (const void*)k_finish_select, (const void*)k_fixup<false>, (const void*)k_fixup<true>, (const void*)k_fused<false, false>, (const void*)k_fused<false, true>, (const void*)k_fused<true, false>, (const void*)k_fused<true, true>, (const void*)k_fused_tma<false>, (const void*)k_fused_tma<true>, (const void*)k_index_diag, (const void*)k_rank_sum_f32, (const void*)k_rank_sum_u32, (const void*)k_raw_sum, (const void*)k_sample, (const void*)k_sample_fine, (const void*)k_set_opt, (const void*)k_set_u32, (const void*)k_stage_copy, (const void*)k_window_coarse, (const void*)k_window_fine, (const void*)k_zero};
  cudaFuncAttributes a;
  for (const void* f : fns) cudaFuncGetAttributes(&a, f);
  cudaGetLastError();
}

}  // namespace tagc_b200
