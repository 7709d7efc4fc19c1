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
#include <cub/block/block_scan.cuh>

#include "kernels.hpp"

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

// --------------------------------------------------------------- sampling
__global__ void __launch_bounds__(kTileThreads) k_sample(const EncItem* __restrict__ items,
                                                         uint32_t n_items, uint64_t total,
                                                         uint32_t* __restrict__ sample_hist) {
  __shared__ uint32_t hist[kSampleBins];
  for (uint32_t i = threadIdx.x; i < kSampleBins; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  int cur = -1;
  auto flush = [&](int item) {
    __syncthreads();
    uint32_t* dst = sample_hist + uint64_t(item) * kSampleBins;
    for (uint32_t i = threadIdx.x; i < kSampleBins; i += blockDim.x) {
      const uint32_t h = hist[i];
      if (h) atomicAdd(dst + i, h);
      hist[i] = 0;
    }
    __syncthreads();
  };
  for (uint64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const uint32_t it = find_sample_item(items, n_items, w);
    if (int(it) != cur) {
      if (cur >= 0) flush(cur);
      cur = int(it);
    }
    const EncItem e = items[it];
    const uint64_t start = (w - e.sample_begin) * uint64_t(e.sample_stride) * kTile;
    const uint64_t pos = start + 4ull * threadIdx.x;
    if (pos < e.n) {
      float v[4];
      load_combined(e, uint32_t(pos), v);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (pos + j < e.n) atomicAdd(&hist[mag_key(v[j]) >> kSampleShift], 1u);
    }
  }
  if (cur >= 0) flush(cur);
}

// --------------------------------------------------------------- window
// One CTA per item: bracket the target rank of the sample into a key window.
__global__ void __launch_bounds__(256) k_window(const EncItem* __restrict__ items,
                                                SelState* __restrict__ state,
                                                uint32_t* __restrict__ sample_hist) {
  using Scan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ uint32_t s_lo, s_hi;
  const uint32_t item = blockIdx.x;
  const EncItem e = items[item];
  uint32_t klo = 1u, khi = 0x7F800000u;
  if (e.sample_tiles > 0) {
    uint32_t* h = sample_hist + uint64_t(item) * kSampleBins;
    constexpr int kPer = kSampleBins / 256;
    uint32_t loc[kPer];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      loc[i] = h[threadIdx.x * kPer + i];
      sum += loc[i];
    }
    uint32_t pre, total;
    Scan(tmp).ExclusiveSum(sum, pre, total);
    if (threadIdx.x == 0) {
      s_lo = 0xFFFFFFFFu;  // "below every bin"
      s_hi = 0xFFFFFFFFu;  // "above every bin"
    }
    __syncthreads();
    const double s = double(total);
    const double p = double(e.c) / double(e.n);
    const double t = double(e.c > 0 ? e.c - 1 : 0) * s / double(e.n);
    const double delta = 6.0 * sqrt(fmax(s * p * (1.0 - p), 0.0)) + 16.0;
    const double lo = floor(t - delta), hi = ceil(t + delta);
    uint32_t cum = pre;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const uint32_t b = threadIdx.x * kPer + i;
      const double c0 = double(cum), c1 = double(cum + loc[i]);
      if (lo >= 0.0 && c0 <= lo && lo < c1) s_lo = b;
      if (hi < s && c0 <= hi && hi < c1) s_hi = b;
      cum += loc[i];
    }
    __syncthreads();
    if (s_lo != 0xFFFFFFFFu) klo = max(1u, s_lo << kSampleShift);
    if (s_hi != 0xFFFFFFFFu) khi = min(0x7F800000u, ((s_hi + 1u) << kSampleShift) - 1u);
    // leave the histogram zeroed for the next call
#pragma unroll
    for (int i = 0; i < kPer; ++i) h[threadIdx.x * kPer + i] = 0;
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

// --------------------------------------------------------------- count
// Contiguous tile range of this CTA (persistent grid): consecutive tiles stay
// in the same item, so per-item shared-memory staging is flushed rarely.
// (32-bit arithmetic: tile counts stay far below 2^32, and a 64-bit divide
// would pull a subroutine call into every persistent kernel.)
__device__ __forceinline__ void cta_range(uint64_t total, uint64_t& t0, uint64_t& t1) {
  const uint32_t T = uint32_t(total), G = gridDim.x;
  const uint32_t chunk = T / G, extra = T % G, b = blockIdx.x;
  t0 = uint64_t(b) * chunk + min(b, extra);
  t1 = t0 + chunk + (b < extra ? 1u : 0u);
}

constexpr uint32_t kStageKeys = 8192;  // per-CTA candidate staging (flushed at >= 4096)

// One HBM pass: NaN check (sparsify.cpp:24-28), counts of zero keys and keys
// below the window, compaction of in-window keys (staged in shared memory and
// appended with one global atomic per flush) and a 2048-bin histogram of the
// in-window keys that lets the finalize kernel jump to the right sub-bin.
__global__ void __launch_bounds__(kTileThreads) k_count(const EncItem* __restrict__ items,
                                                        SelState* __restrict__ state,
                                                        uint32_t n_items, uint64_t total_tiles,
                                                        uint32_t* __restrict__ cand,
                                                        uint32_t* __restrict__ fine_hist,
                                                        uint32_t* __restrict__ err) {
  __shared__ uint32_t s_keys[kStageKeys];
  __shared__ uint32_t s_hist[kRadixBins];
  __shared__ uint32_t s_n, s_base, s_zero, s_lo;
  const uint32_t lane = threadIdx.x & 31;
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
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) s_hist[i] = 0;
    if (threadIdx.x == 0) s_n = s_zero = s_lo = 0;
    __syncthreads();
    uint32_t c_zero = 0, c_lo = 0;
    auto flush_keys = [&]() {
      __syncthreads();
      if (threadIdx.x == 0) s_base = s_n ? atomicAdd(&state[it].cnt_in, s_n) : 0u;
      __syncthreads();
      const uint32_t nk = s_n, base = s_base, cap = e.cand_cap;
      uint32_t* cb = cand + e.cand_off;
      for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x)
        if (base + i < cap) cb[base + i] = s_keys[i];
      __syncthreads();
      if (threadIdx.x == 0) s_n = 0;
      __syncthreads();
    };
    for (; tile < tend; ++tile) {
      const uint32_t q0 = uint32_t(tile - e.tile_begin) * (kTile / 4);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t pos = 4u * (q0 + k * kTileThreads + threadIdx.x);
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (pos < e.n) load_combined(e, pos, v);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t key = mag_key(v[j]);
          const bool valid = pos + j < e.n;
          c_zero += valid && key == 0;
          c_lo += valid && key != 0 && key < klo;
          nan |= valid && key > 0x7F800000u;
          const bool in = valid && key >= klo && key <= khi;
          const uint32_t m = __ballot_sync(kFull, in);
          if (m) {  // warp-aggregated append into the CTA stage
            const uint32_t leader = __ffs(m) - 1;
            uint32_t base = 0;
            if (lane == leader) base = atomicAdd(&s_n, __popc(m));
            base = __shfl_sync(kFull, base, leader);
            if (in) {
              s_keys[base + __popc(m & ((1u << lane) - 1u))] = key;
              atomicAdd(&s_hist[(key - klo) >> fshift], 1u);
            }
          }
        }
      }
      __syncthreads();
      if (s_n >= kStageKeys - kTile) flush_keys();
    }
    flush_keys();
    // counts and fine histogram of this item
    c_zero = warp_sum(c_zero);
    c_lo = warp_sum(c_lo);
    if ((threadIdx.x & 31) == 0) {
      if (c_zero) atomicAdd(&s_zero, c_zero);
      if (c_lo) atomicAdd(&s_lo, c_lo);
    }
    uint32_t* fh = fine_hist + uint64_t(it) * kRadixBins;
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x)
      if (s_hist[i]) atomicAdd(fh + i, s_hist[i]);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_zero) atomicAdd(&state[it].cnt_zero, s_zero);
      if (s_lo) atomicAdd(&state[it].cnt_lo, s_lo);
    }
    __syncthreads();
    ++it;
  }
  if (nan) atomicOr(err, 1u);
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
// (1) k_pick, one CTA per item: the fine histogram names the sub-bin holding
//     the target rank; (2) k_collect, all SMs: the keys of that sub-bin
//     (typically tens) are gathered from the candidate pool; (3) k_select,
//     one CTA per item: exact radix select of the remaining rank in shared
//     memory. Bit-identical to nth_element (sparsify.cpp:35-36): tau is the
//     c-th smallest key.
constexpr uint32_t kStatusCollect = 3;

__global__ void __launch_bounds__(1024) k_pick(const EncItem* __restrict__ items,
                                               SelState* __restrict__ state,
                                               uint32_t* __restrict__ fine_hist,
                                               uint32_t* __restrict__ err) {
  __shared__ uint32_t s_digit, s_below;
  const uint32_t item = blockIdx.x;
  const EncItem e = items[item];
  const SelState s = state[item];
  uint32_t* fh = fine_hist + uint64_t(item) * kRadixBins;
  const bool nan = (*err & 1u) != 0;
  bool done = nan;
  if (!done && (e.c == 0 || e.c <= s.cnt_zero)) {  // tau = 0 (c == 0, or the rank falls on zeros)
    if (threadIdx.x == 0) {
      state[item].tau_key = 0;
      state[item].status = 0;
    }
    done = true;
  }
  const uint32_t r = e.c - s.cnt_zero;  // 1-based rank among nonzero keys
  if (!done && !(s.cnt_lo < r && r <= s.cnt_lo + s.cnt_in && s.cnt_in <= e.cand_cap)) {
    if (threadIdx.x == 0) {  // bracket missed: full radix select fallback
      state[item].status = 1;
      state[item].prefix = 0;
      state[item].rank = e.c - 1;
      atomicOr(err + 1, 1u);
    }
    done = true;
  }
  if (!done) {
    find_digit<1024>(fh, kRadixBins, r - s.cnt_lo - 1, &s_digit, &s_below);
    if (threadIdx.x == 0) {
      state[item].status = kStatusCollect;
      state[item].prefix = s_digit;  // target sub-bin
      state[item].rank = r - s.cnt_lo - 1 - s_below;
      state[item].pad1 = 0;          // collected keys
    }
  }
  for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) fh[i] = 0;
}

__global__ void __launch_bounds__(256) k_collect(const EncItem* __restrict__ items,
                                                 SelState* __restrict__ state, uint32_t n_items,
                                                 const uint32_t* __restrict__ cand,
                                                 uint32_t* __restrict__ sel_list) {
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gstride = uint64_t(gridDim.x) * blockDim.x;
  for (uint32_t it = 0; it < n_items; ++it) {
    const SelState s = state[it];
    if (s.status != kStatusCollect) continue;
    const uint32_t* ck = cand + items[it].cand_off;
    uint32_t* out = sel_list + uint64_t(it) * kFinalKeys;
    for (uint64_t i = gtid; i < s.cnt_in; i += gstride) {
      const uint32_t key = ck[i];
      if (((key - s.klo) >> s.fshift) == s.prefix) {
        const uint32_t idx = atomicAdd(&state[it].pad1, 1u);
        if (idx < kFinalKeys) out[idx] = key;
      }
    }
  }
}

__global__ void __launch_bounds__(1024) k_select(const EncItem* __restrict__ items,
                                                 SelState* __restrict__ state,
                                                 const uint32_t* __restrict__ cand,
                                                 const uint32_t* __restrict__ sel_list) {
  __shared__ uint32_t keys[kFinalKeys];
  __shared__ uint32_t hist[kRadixBins];
  __shared__ uint32_t s_digit, s_below;
  const uint32_t item = blockIdx.x;
  const SelState s = state[item];
  if (s.status != kStatusCollect) return;
  const uint32_t nk = s.pad1;
  const bool in_smem = nk <= kFinalKeys;
  const uint32_t* ck = cand + items[item].cand_off;
  if (in_smem)
    for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) keys[i] = sel_list[uint64_t(item) * kFinalKeys + i];
  uint32_t rank = s.rank, prefix = 0;
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
      for (uint32_t i = threadIdx.x; i < s.cnt_in; i += blockDim.x) {
        const uint32_t key = ck[i];
        if (((key - s.klo) >> s.fshift) == s.prefix && (key >> hs) == (prefix >> hs))
          atomicAdd(&hist[(key >> shift) & ((1u << bits) - 1u)], 1u);
      }
    }
    __syncthreads();
    find_digit<1024>(hist, 1u << bits, rank, &s_digit, &s_below);
    rank -= s_below;
    prefix |= s_digit << shift;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    state[item].tau_key = prefix;
    state[item].status = 0;
  }
}

// --------------------------------------------------------------- fallback
__global__ void __launch_bounds__(kTileThreads) k_fb_hist(const EncItem* __restrict__ items,
                                                          const SelState* __restrict__ state,
                                                          uint32_t n_items, uint64_t total_tiles,
                                                          uint32_t* __restrict__ fb_hist, int pass,
                                                          const uint32_t* __restrict__ err) {
  if (err[0] || !err[1]) return;  // NaN, or no item needs the fallback
  __shared__ uint32_t hist[kRadixBins];
  const int shift = digit_shift(pass), bits = digit_bits(pass), hs = shift + bits;
  for (uint64_t tile = blockIdx.x; tile < total_tiles; tile += gridDim.x) {
    const uint32_t it = find_tile_item(items, n_items, tile);
    if (state[it].status != 1) continue;  // block-uniform
    const EncItem e = items[it];
    const uint32_t prefix = state[it].prefix;
    for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t q0 = uint32_t(tile - e.tile_begin) * (kTile / 4);
    for (int k = 0; k < 4; ++k) {
      const uint32_t pos = 4u * (q0 + k * kTileThreads + threadIdx.x);
      if (pos >= e.n) continue;
      float v[4];
      load_combined(e, pos, v);
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

__global__ void __launch_bounds__(512) k_fb_scan(SelState* __restrict__ state,
                                                 uint32_t* __restrict__ fb_hist, int pass,
                                                 const uint32_t* __restrict__ err) {
  __shared__ uint32_t s_digit, s_below;
  if (err[0] || !err[1]) return;
  const uint32_t item = blockIdx.x;
  if (state[item].status != 1) return;
  uint32_t* h = fb_hist + uint64_t(item) * kRadixBins;
  const uint32_t rank = state[item].rank;
  find_digit<512>(h, 1u << digit_bits(pass), rank, &s_digit, &s_below);
  for (uint32_t i = threadIdx.x; i < kRadixBins; i += blockDim.x) h[i] = 0;
  if (threadIdx.x == 0) {
    const uint32_t prefix = state[item].prefix | (s_digit << digit_shift(pass));
    state[item].prefix = prefix;
    state[item].rank = rank - s_below;
    if (pass == 2) {
      state[item].tau_key = prefix;
      state[item].status = 0;
    }
  }
}

// --------------------------------------------------------------- encode
// Split (drop iff |v| <= tau: kernels.cpp:95, on the 31-bit key), residual
// write-back, packed index (field set iff the kept value is nonzero,
// index.cpp:35) and count-sketch scatter row[h_r(p)] += s_r(p)*v
// (sketch.cpp:52-53) with fp32 reductions at L2. All 16 elements of a thread
// are loaded before any is consumed (8 x 16-byte requests in flight per
// thread); kept elements are staged in shared memory and scattered by the
// whole CTA, so the rare hash work does not serialise the streaming loop.
constexpr uint32_t kKeptStage = 1024;  // kept elements staged per tile (overflow: direct)

template <bool kW4>
__global__ void __launch_bounds__(kTileThreads, 5) k_encode(const EncItem* __restrict__ items,
                                                         const SelState* __restrict__ state,
                                                         uint32_t n_items, uint64_t total_tiles,
                                                         const HashParams hp,
                                                         const uint32_t* __restrict__ err,
                                                         SelState* __restrict__ kept_state) {
  __shared__ uint32_t s_pos[kKeptStage];
  __shared__ float s_val[kKeptStage];
  __shared__ uint32_t s_n;
  if (err && *err) return;  // NaN anywhere: no accumulator is touched
  const uint32_t lane = threadIdx.x & 31;
  uint64_t t0, t1;
  cta_range(total_tiles, t0, t1);
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  uint32_t it = t0 < t1 ? find_tile_item(items, n_items, t0) : 0;
  for (uint64_t tile = t0; tile < t1; ++tile) {
    while (it + 1 < n_items && items[it + 1].tile_begin <= tile) ++it;
    const EncItem e = items[it];
    const uint32_t tau = (e.flags & kSelect) ? state[it].tau_key : 0u;
    const bool vec = (e.flags & kAligned16) != 0;
    const uint32_t n_words = kW4 ? (e.n + 7u) / 8u : (e.n + 31u) / 32u;
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
    if (e.flags & kHasAcc) {
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
                _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows)
                  atomicAdd(e.sketch + uint64_t(r) * e.m + dev_bucket(hp.row[r], pos + j, e.m),
                            dev_sign(hp.row[r], pos + j) * v[k][j]);
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
    if (kept_state && (e.flags & kWriteSparse)) {
      kept = warp_sum(kept);
      if (lane == 0 && kept) atomicAdd(&kept_state[it].kept, kept);
    }
    if (e.flags & kWriteSketch) {
      __syncthreads();
      const uint32_t nk = min(s_n, kKeptStage);
      float* sk = e.sketch;
      const uint32_t m = e.m;
      for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) {
        const uint32_t p = s_pos[i];
        const float x = s_val[i];
        _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows)
          atomicAdd(sk + uint64_t(r) * m + dev_bucket(hp.row[r], p, m), dev_sign(hp.row[r], p) * x);
      }
      __syncthreads();
      if (threadIdx.x == 0) s_n = 0;
      __syncthreads();
    }
  }
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

// Raw-segment pack/unpack: flat 4096-element tiles over all items, 16-byte
// accesses when source and destination are both aligned.
__global__ void __launch_bounds__(256) k_copy_items(const CopyItem* __restrict__ items,
                                                    uint32_t n_items, uint64_t total_tiles) {
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

int launch_select(const DevInfo& di, const EncItem* items, SelState* state, uint32_t n_items,
                  uint64_t total_tiles, uint64_t total_samples, uint32_t* sample_hist,
                  uint32_t* fb_hist, uint32_t* fine_hist, uint32_t* cand, uint32_t* sel_list,
                  uint32_t* err, cudaStream_t stream) {
  if (n_items == 0) return 0;
  int launches = 0;
  if (total_samples) {
    k_sample<<<persistent_grid((const void*)k_sample, kTileThreads, di, total_samples), kTileThreads,
               0, stream>>>(items, n_items, total_samples, sample_hist);
    ++launches;
  }
  k_window<<<n_items, 256, 0, stream>>>(items, state, sample_hist);
  k_count<<<persistent_grid((const void*)k_count, kTileThreads, di, total_tiles), kTileThreads, 0,
            stream>>>(items, state, n_items, total_tiles, cand, fine_hist, err);
  k_pick<<<n_items, 1024, 0, stream>>>(items, state, fine_hist, err);
  k_collect<<<di.sms * 2, 256, 0, stream>>>(items, state, n_items, cand, sel_list);
  k_select<<<n_items, 1024, 0, stream>>>(items, state, cand, sel_list);
  launches += 5;
  const int fg = persistent_grid((const void*)k_fb_hist, kTileThreads, di, total_tiles);
  for (int pass = 0; pass < 3; ++pass) {
    k_fb_hist<<<fg, kTileThreads, 0, stream>>>(items, state, n_items, total_tiles, fb_hist, pass, err);
    k_fb_scan<<<n_items, 512, 0, stream>>>(state, fb_hist, pass, err);
    launches += 2;
  }
  return launches;
}

int launch_encode(const DevInfo& di, const EncItem* items, const SelState* state, uint32_t n_items,
                    uint64_t total_tiles, const HashParams& hp, const uint32_t* err,
                    SelState* kept_state, bool w4, cudaStream_t stream) {
  if (n_items == 0) return 0;
  if (w4) {
    const int g = persistent_grid((const void*)k_encode<true>, kTileThreads, di, total_tiles);
    k_encode<true><<<g, kTileThreads, 0, stream>>>(items, state, n_items, total_tiles, hp, err,
                                                   kept_state);
  } else {
    const int g = persistent_grid((const void*)k_encode<false>, kTileThreads, di, total_tiles);
    k_encode<false><<<g, kTileThreads, 0, stream>>>(items, state, n_items, total_tiles, hp, err,
                                                    kept_state);
  }
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
                      cudaStream_t stream) {
  if (!n_items || !total_tiles) return 0;
  const uint64_t g = std::min<uint64_t>(total_tiles, uint64_t(di.sms) * 8);
  k_copy_items<<<int(g), 256, 0, stream>>>(items, n_items, total_tiles);
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

}  // namespace tagc_b200
