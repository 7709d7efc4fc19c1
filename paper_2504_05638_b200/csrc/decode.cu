// decode.cu — sm_100a owner-side decode (reference decode.cpp:24-140):
//   build      : walk the merged index words and list the present positions
//                in ascending order per word tile (plist / pitem, one block
//                scan per tile); remember each tile's list offset;
//   accumulate : per listed entry i, add (i, 1) into its k buckets' state;
//   round 0    : every listed position inspects its k buckets and peels from
//                its lowest singleton row (the reference's ascending seed
//                order, decode.cpp:96-99), then leaves the buckets it shares;
//   peel       : frontier rounds in ONE cooperative persistent kernel, a
//                single CTA finishing once the frontier is small;
//   estimate   : median-of-rows on the residual sketch for every listed
//                position the peel could not resolve (decode.cpp:130-138);
//   emit       : the dense shard chunk by chunk: a zeroed shared-memory
//                chunk takes the chunk's listed values and leaves by TMA
//                bulk store.
//
// Everything between build and emit is keyed by the presence-list index i,
// not the position: a bucket's state is (count, sum of list indices) in one
// u64, decoded values go to val[i] and the recovered flags to bit i. The
// randomly accessed working set is then the bucket state plus the residual
// sketch; the dense output is written once, at the end.
//
// Bucket state: (sum of list indices mod 2^40) << 24 | count (24 bits), so
// building and peeling cost one 64-bit L2 atomic per (entry, row). count == 1
// makes the low 32 bits of the sum the single remaining entry exactly
// (decode.cpp:104-106 keeps a u64 key_sum for the same reason).
//
// Parity: the recovered/unresolved position sets are those of the reference's
// FIFO peel (the peelable set is the complement of the 2-core, independent of
// order); values match within fp32 reassociation tolerance and bit-exactly on
// integer-valued inputs.
#include <cooperative_groups.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace tagc_b200 {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
constexpr unsigned long long kCountMask = (1ull << 24) - 1ull;
__device__ __forceinline__ unsigned long long st_add(uint32_t i) { return (uint64_t(i) << 24) | 1ull; }
__device__ __forceinline__ unsigned long long st_sub(uint32_t i) { return ~st_add(i) + 1ull; }
__device__ __forceinline__ uint32_t st_count(unsigned long long s) { return uint32_t(s & kCountMask); }
__device__ __forceinline__ uint32_t st_entry(unsigned long long s) { return uint32_t(s >> 24); }
constexpr uint32_t kWordTile = kDecWordTile;
constexpr uint32_t kTail = 512;  // frontier size at which one CTA finishes (<= kLocalQ, kPeelHandoff)

__device__ __forceinline__ uint32_t ldcg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ unsigned long long ldcg(const unsigned long long* p) { return __ldcg(p); }
__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }

__device__ __forceinline__ uint32_t find_word_item(const DecItem* items, uint32_t n, uint64_t t) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (items[mid].word_tile_begin <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Presence bits of one merged word: field != 0 (index.cpp:43-57). Width 4:
// bit 4j set iff nibble j nonzero; width 1: the word itself. Bits past the
// item's last position are cleared.
__device__ __forceinline__ uint32_t present_bits(uint32_t x, bool w4, uint32_t wi, uint32_t n) {
  x = w4 ? ((x | x >> 1 | x >> 2 | x >> 3) & 0x11111111u) : x;
  const uint64_t first = uint64_t(wi) * (w4 ? 8u : 32u);
  const uint64_t left = n > first ? n - first : 0;
  if (w4) {
    if (left < 8) x &= left ? (1u << (4 * left)) - 1u : 0u;
  } else if (left < 32) {
    x &= left ? (1u << left) - 1u : 0u;
  }
  return x;
}

// Same without the item-end mask: for words wholly inside the item.
__device__ __forceinline__ uint32_t present_bits_full(uint32_t x, bool w4) {
  return w4 ? ((x | x >> 1 | x >> 2 | x >> 3) & 0x11111111u) : x;
}
// Thread-owned words [w0, w0 + kPerThreadWords) all inside the item's n positions.
__device__ __forceinline__ bool words_full(uint32_t w0, uint32_t nwords, bool w4, uint32_t n) {
  return uint64_t(w0 + nwords) * (w4 ? 8u : 32u) <= uint64_t(n);
}

__device__ __forceinline__ float canonical(float v) { return v == 0.0f ? 0.0f : v; }

// Item of presence-list entry i: a one-item decode (one huge segment) keeps
// no per-entry item array (pitem is neither written nor read).
__device__ __forceinline__ uint32_t item_of(const DecodeWork& w, uint64_t i) {
  return w.n_items == 1 ? 0u : __ldcs(w.pitem + i);
}

// Counter mode: one counter of 2^cnt_shift bits (8 or 4) per bucket, packed
// into u32 words (w.cnt8).
__device__ __forceinline__ void cnt_add(const DecodeWork& w, uint64_t slot) {
  const uint32_t cs = w.cnt_shift, per = 5u - cs;
  red_add_u32(w.cnt8 + (slot >> per), 1u << (uint32_t(slot & ((1u << per) - 1u)) << cs));
}
__device__ __forceinline__ uint32_t cnt_get(const DecodeWork& w, uint64_t slot) {
  const uint32_t cs = w.cnt_shift, per = 5u - cs;
  return (ldcg(w.cnt8 + (slot >> per)) >> (uint32_t(slot & ((1u << per) - 1u)) << cs)) & ((1u << (1u << cs)) - 1u);
}

__device__ __forceinline__ uint32_t warp_sum32(uint32_t x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  return x;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PEEL_MARK(k)                                                         \
  do {                                                                       \
    const int mk_ = (k);                                                     \
    if (w.dbg && blockIdx.x == 0 && threadIdx.x == 0 && mk_ < 64) w.dbg[mk_] = gtimer(); \
  } while (0)

// Middle order statistic of k row estimates (decode.cpp:45: nth_element k/2).
__device__ __forceinline__ float median_rows(float (&e)[kMaxRows], uint32_t k) {
  if (k == 3) {
    const float a = e[0], b = e[1], c = e[2];
    return fmaxf(fminf(a, b), fminf(fmaxf(a, b), c));
  }
#pragma unroll
  for (uint32_t i = 1; i < kMaxRows; ++i) {
    if (i >= k) break;
    const float x = e[i];
    uint32_t j = i;
    while (j > 0 && x < e[j - 1]) {
      e[j] = e[j - 1];
      --j;
    }
    e[j] = x;
  }
  return e[k / 2];
}

// ------------------------------------------------------------------ build
// Word tiles of kWordTile merged-index words (16 per thread of a 256-thread
// CTA). One pass, k_list: each tile's present positions are counted, its
// list offset found by decoupled look-back (tile_base[wt]; the presence list
// is ordered by tile, ascending position inside a tile), the list entries
// (plist / pitem) written at their final index and (entry, 1) added into each
// entry's k buckets with fire-and-forget 64-bit reductions (the bucket state).
constexpr uint32_t kPerThreadWords = kWordTile / 256;

__device__ __forceinline__ void cta_tiles(uint64_t total, uint32_t& t0, uint32_t& t1) {
  const uint32_t T = uint32_t(total), G = gridDim.x, b = blockIdx.x;
  const uint32_t chunk = T / G, extra = T % G;
  t0 = b * chunk + min(b, extra);
  t1 = t0 + chunk + (b < extra ? 1u : 0u);
}

// Thread t of a tile owns words [wbase + 16 t, wbase + 16 t + 16): the block
// scan over threads then lists positions in ascending order (k_emit relies on
// it). 16-byte loads when the words are aligned.
__device__ __forceinline__ uint32_t tile_word(uint32_t wbase, uint32_t k) {
  return wbase + threadIdx.x * kPerThreadWords + k;
}
__device__ __forceinline__ void load_tile_bits(const DecItem& e, uint32_t wbase, bool w4,
                                               uint32_t (&bits)[kPerThreadWords], uint32_t& cnt) {
  uint32_t raw[kPerThreadWords];
  const uint32_t w0 = tile_word(wbase, 0);
  if (w0 + kPerThreadWords <= e.n_words && (reinterpret_cast<uintptr_t>(e.words + w0) & 15u) == 0) {
#pragma unroll
    for (uint32_t k = 0; k < kPerThreadWords; k += 4) {  // streamed: keep the bucket state in L2
      const uint4 x = __ldcs(reinterpret_cast<const uint4*>(e.words + w0 + k));
      raw[k] = x.x; raw[k + 1] = x.y; raw[k + 2] = x.z; raw[k + 3] = x.w;
    }
  } else {
#pragma unroll
    for (uint32_t k = 0; k < kPerThreadWords; ++k) raw[k] = w0 + k < e.n_words ? __ldcs(e.words + w0 + k) : 0u;
  }
  cnt = 0;
#pragma unroll
  for (uint32_t k = 0; k < kPerThreadWords; ++k) {
    bits[k] = present_bits(raw[k], w4, w0 + k, e.n);
    cnt += __popc(bits[k]);
  }
}

// List build in ONE pass over the merged index: word tiles are claimed in
// order from a counter (qcount[12]); each CTA publishes its tile's count and
// finds its list offset by a warp-wide decoupled look-back over the preceding
// tiles' published counts / inclusive prefixes (tile_state), then writes its
// list entries and inserts them into the bucket state. In-order claiming keeps
// the look-back deadlock-free (predecessors belong to running CTAs that
// publish their counts without waiting) and the REDs inside an L2-resident
// window of the state.
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__global__ void __launch_bounds__(256) k_list(DecodeWork w, const HashParams hp) {
  using Scan = cub::BlockScan<uint32_t, 256>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t s_wt, s_base;
  span_begin(w.span);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cap = uint32_t(w.list_cap < 0xFFFFFFFFull ? w.list_cap : 0xFFFFFFFFull);
  const uint32_t T = uint32_t(w.total_word_tiles);
  for (;;) {
    if (threadIdx.x == 0) s_wt = atomicAdd(&w.qcount[12], 1u);
    __syncthreads();
    const uint32_t wt = s_wt;
    if (wt >= T) break;
    const uint32_t it = find_word_item(w.items, w.n_items, wt);
    const DecItem& e = w.items[it];
    const bool w4 = (e.flags & kWidth4) != 0;
    const uint32_t P = w4 ? 8u : 32u;
    const uint32_t wbase = uint32_t(wt - e.word_tile_begin) * kWordTile;
    uint32_t bits[kPerThreadWords], cnt;
    load_tile_bits(e, wbase, w4, bits, cnt);
    uint32_t off, total;
    Scan(scan_tmp).ExclusiveSum(cnt, off, total);
    if (threadIdx.x < 32) {  // warp 0: publish, look back, publish
      unsigned long long* ts = w.tile_state;
      uint64_t prefix = 0;
      if (wt > 0) {
        if (lane == 0) atomicExch(ts + wt, (1ull << 32) | total);  // aggregate
        for (int k0 = int(wt) - 1;; k0 -= 32) {
          const int k = k0 - int(lane);
          unsigned long long v = 2ull << 32;  // before tile 0: an inclusive zero
          if (k >= 0) {
            do { v = ld_volatile_u64(ts + k); } while ((v >> 32) == 0);
          }
          const uint32_t incl = __ballot_sync(kFull, (v >> 32) == 2);
          const uint32_t stop = incl ? uint32_t(__ffs(incl) - 1) : 31u;  // nearest inclusive prefix
          prefix += warp_sum32(lane <= stop ? uint32_t(v) : 0u);
          if (incl) break;
        }
      }
      if (lane == 0) {
        atomicExch(ts + wt, (2ull << 32) | uint32_t(prefix + total));  // inclusive prefix
        s_base = uint32_t(prefix);
        w.tile_base[wt] = uint32_t(prefix);
        if (total) atomicAdd(&w.stats[it].presence, total);
        // a corrupt index (NaN input aborted the encode) may list more than the
        // capacity: then nothing is decoded (the call reports the NaN)
        if (wt == T - 1) w.qcount[5] = prefix + total <= cap ? uint32_t(prefix + total) : 0u;
      }
    }
    __syncthreads();
    const uint32_t base = s_base;
    const uint32_t n_in = base + total <= cap ? total : (base < cap ? cap - base : 0u);
    uint32_t j = base + off;
#pragma unroll
    for (uint32_t k = 0; k < kPerThreadWords; ++k) {  // list entries: cheap, divergent
      const uint32_t wi = tile_word(wbase, k);
      for (uint32_t x = bits[k]; x; x &= x - 1) {
        const uint32_t bb = __ffs(x) - 1;
        if (j < cap) {
          w.plist[j] = wi * P + (w4 ? bb / 4 : bb);
          if (w.n_items > 1) w.pitem[j] = it;
        }
        ++j;
      }
    }
    __syncthreads();  // the tile's entries are visible to the whole CTA
    // bucket counts, one entry per thread (hashing and reductions stay
    // converged): byte counters packed four to a word when the batch has
    // them (cnt8, L2-resident), else the full (count, index sum) state
    for (uint32_t q = threadIdx.x; q < n_in; q += blockDim.x) {
      const uint32_t i = base + q;
      const uint32_t p = w.plist[i];
      _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
        const uint64_t slot = e.slot_base + uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m, e.mmul);
        if (w.cnt8) cnt_add(w, slot);
        else atomicAdd(w.slot_state + slot, st_add(i));  // result unused: RED.ADD.64
      }
    }
    __syncthreads();  // scan storage reuse
  }
}

// Counter mode (bucket counters, no list indices in the bucket state): the
// bucket counts do not depend on the list order, so the build splits into
// two passes over the same per-CTA tile ranges, with no look-back chain
// between word tiles:
//   k_list_count : per word tile its present count (into the tile_state
//                  words, free in counter mode) and per CTA their sum, the
//                  next tile's words already in flight;
//   k_list_write : the CTA's list offset from the per-CTA sums, its tiles'
//                  offsets (tile_base) by a block scan, then per word tile the
//                  list entries at their final index and the counter REDs.
// The merged index is read twice (streamed), against a per-tile look-back
// whose latency chain grew with the number of CTAs in flight.
__device__ __forceinline__ void load_tile_raw(const DecItem& e, uint32_t wbase, uint32_t (&raw)[kPerThreadWords]) {
  const uint32_t w0 = tile_word(wbase, 0);
  if (w0 + kPerThreadWords <= e.n_words && (reinterpret_cast<uintptr_t>(e.words + w0) & 15u) == 0) {
#pragma unroll
    for (uint32_t k = 0; k < kPerThreadWords; k += 4) {
      const uint4 x = __ldcs(reinterpret_cast<const uint4*>(e.words + w0 + k));
      raw[k] = x.x; raw[k + 1] = x.y; raw[k + 2] = x.z; raw[k + 3] = x.w;
    }
  } else {
#pragma unroll
    for (uint32_t k = 0; k < kPerThreadWords; ++k) raw[k] = w0 + k < e.n_words ? __ldcs(e.words + w0 + k) : 0u;
  }
}

__global__ void __launch_bounds__(256) k_list_count(DecodeWork w) {
  using Reduce = cub::BlockReduce<uint32_t, 256>;
  __shared__ typename Reduce::TempStorage red_tmp[2];  // double-buffered: no barrier per tile
  span_begin(w.span);
  // two count CTAs per write CTA (k_list_write runs gridDim.x / 2 CTAs):
  // CTA c counts one half of write CTA c / 2's tile range
  uint32_t t0, t1;
  {
    const uint32_t sp = w.list_split;  // count CTAs per write CTA: 1 or 2
    const uint32_t T = uint32_t(w.total_word_tiles), G = gridDim.x / sp, b = blockIdx.x / sp;
    const uint32_t chunk = T / G, extra = T % G;
    const uint32_t b0 = b * chunk + min(b, extra), b1 = b0 + chunk + (b < extra ? 1u : 0u);
    const uint32_t mid = b0 + (b1 - b0) / 2;
    t0 = sp == 1 ? b0 : ((blockIdx.x & 1) ? mid : b0);
    t1 = sp == 1 ? b1 : ((blockIdx.x & 1) ? b1 : mid);
  }
  uint32_t* tile_cnt = reinterpret_cast<uint32_t*>(w.tile_state);  // counter mode: tile_state is free
  uint32_t cta_sum = 0, item_sum = 0;  // item_sum: presence of item `it` so far (one stats atomic per item run)
  if (t0 >= t1) {
    if (threadIdx.x == 0) w.cta_cnt[blockIdx.x] = 0;
    return;
  }
  uint32_t it = find_word_item(w.items, w.n_items, t0);
  uint32_t raw[kPerThreadWords];
  {
    const DecItem& e = w.items[it];
    load_tile_raw(e, uint32_t(t0 - e.word_tile_begin) * kWordTile, raw);
  }
  for (uint32_t wt = t0, buf = 0; wt < t1; ++wt, buf ^= 1u) {
    const DecItem& e = w.items[it];
    const bool w4 = (e.flags & kWidth4) != 0;
    const uint32_t wbase = uint32_t(wt - e.word_tile_begin) * kWordTile;
    uint32_t cnt = 0;
    if (words_full(tile_word(wbase, 0), kPerThreadWords, w4, e.n)) {
#pragma unroll
      for (uint32_t k = 0; k < kPerThreadWords; ++k) cnt += __popc(present_bits_full(raw[k], w4));
    } else {
#pragma unroll
      for (uint32_t k = 0; k < kPerThreadWords; ++k) cnt += __popc(present_bits(raw[k], w4, tile_word(wbase, k), e.n));
    }
    uint32_t nit = it;  // the next tile's words in flight during the reduction
    if (wt + 1 < t1) {
      while (nit + 1 < w.n_items && w.items[nit + 1].word_tile_begin <= wt + 1) ++nit;
      const DecItem& ne = w.items[nit];
      load_tile_raw(ne, uint32_t(wt + 1 - ne.word_tile_begin) * kWordTile, raw);
    }
    const uint32_t total = Reduce(red_tmp[buf]).Sum(cnt);
    if (threadIdx.x == 0) {
      tile_cnt[wt] = total;
      cta_sum += total;
      item_sum += total;
      if (nit != it || wt + 1 == t1) {
        if (item_sum) atomicAdd(&w.stats[it].presence, item_sum);
        item_sum = 0;
      }
    }
    it = nit;
  }
  if (threadIdx.x == 0) w.cta_cnt[blockIdx.x] = cta_sum;
}

constexpr uint32_t kListStage = 2048;  // staged positions per word tile (beyond: read back)

__global__ void __launch_bounds__(256, 4) k_list_write(DecodeWork w, const HashParams hp) {
  PDL_WAIT();
  using Scan = cub::BlockScan<uint32_t, 256>;
  // double-buffered per tile (scan storage, staged positions), so a tile
  // needs no trailing barrier: tile i + 2 reuses tile i's buffers only after
  // every thread has passed tile i + 1's scan
  __shared__ typename Scan::TempStorage scan_tmp[2];
  __shared__ uint32_t s_pos[2][kListStage];
  // this CTA's list offset and the list length from the per-CTA counts of
  // k_list_count (same grid, same tile ranges): no separate scan kernel
  __shared__ uint32_t s_pre[8], s_all[8];
  uint32_t pre = 0, all = 0;
  for (uint32_t b = threadIdx.x; b < w.list_split * gridDim.x; b += blockDim.x) {  // count CTAs of this pass
    const uint32_t c = ldcg(w.cta_cnt + b);
    all += c;
    pre += b < w.list_split * blockIdx.x ? c : 0u;
  }
  pre = warp_sum32(pre);
  all = warp_sum32(all);
  if ((threadIdx.x & 31) == 0) {
    s_pre[threadIdx.x >> 5] = pre;
    s_all[threadIdx.x >> 5] = all;
  }
  __syncthreads();
  uint64_t run = 0, tot = 0;
  for (uint32_t i = 0; i < blockDim.x / 32; ++i) {
    run += s_pre[i];
    tot += s_all[i];
  }
  // the list length, or 0 when it exceeds the capacity (a corrupt index
  // after a NaN-aborted encode lists nothing)
  const uint32_t total_list = tot <= w.list_cap ? uint32_t(tot) : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) w.qcount[5] = total_list;
  const uint32_t* tile_cnt = reinterpret_cast<const uint32_t*>(w.tile_state);
  uint32_t t0, t1;
  cta_tiles(w.total_word_tiles, t0, t1);
  uint64_t tile_base = run;  // list offset of the current tile (the tiles' counts run on from here)
  // list offset of every tile of this CTA (k_emit, this pass): a block scan
  // of the tiles' counts, 256 tiles at a time
  for (uint32_t b0 = t0; b0 < t1; b0 += blockDim.x) {
    const uint32_t wt = b0 + threadIdx.x;
    const uint32_t c = wt < t1 ? ldcg(tile_cnt + wt) : 0u;
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, d);
      if ((threadIdx.x & 31) >= uint32_t(d)) incl += y;
    }
    __syncthreads();  // s_pre reuse
    if ((threadIdx.x & 31) == 31) s_pre[threadIdx.x >> 5] = incl;
    __syncthreads();
    uint64_t wbase = 0, btot = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) {
      wbase += i < (threadIdx.x >> 5) ? s_pre[i] : 0u;
      btot += s_pre[i];
    }
    const uint64_t off = run + wbase + incl - c;
    if (wt < t1) w.tile_base[wt] = uint32_t(off < 0xFFFFFFFFull ? off : 0xFFFFFFFFull);
    run += btot;
  }
  if (t0 >= t1 || total_list == 0) return;
  __syncthreads();
  uint32_t it = find_word_item(w.items, w.n_items, t0);
  uint32_t raw[kPerThreadWords];
  {
    const DecItem& e = w.items[it];
    load_tile_raw(e, uint32_t(t0 - e.word_tile_begin) * kWordTile, raw);
  }
  for (uint32_t wt = t0, buf = 0; wt < t1; ++wt, buf ^= 1u) {
    const DecItem& e = w.items[it];
    const bool w4 = (e.flags & kWidth4) != 0;
    const uint32_t P = w4 ? 8u : 32u;
    const uint32_t wbase = uint32_t(wt - e.word_tile_begin) * kWordTile;
    uint32_t bits[kPerThreadWords], cnt = 0;
    const bool full = words_full(tile_word(wbase, 0), kPerThreadWords, w4, e.n);
#pragma unroll
    for (uint32_t k = 0; k < kPerThreadWords; ++k) {
      bits[k] = full ? present_bits_full(raw[k], w4) : present_bits(raw[k], w4, tile_word(wbase, k), e.n);
      cnt += __popc(bits[k]);
    }
    uint32_t nit = it;
    if (wt + 1 < t1) {
      while (nit + 1 < w.n_items && w.items[nit + 1].word_tile_begin <= wt + 1) ++nit;
      const DecItem& ne = w.items[nit];
      load_tile_raw(ne, uint32_t(wt + 1 - ne.word_tile_begin) * kWordTile, raw);
    }
    uint32_t off, tile_n;
    Scan(scan_tmp[buf]).ExclusiveSum(cnt, off, tile_n);
    // = tile_base[wt] (same counts as k_list_count), no load
    const uint32_t base = uint32_t(tile_base < 0xFFFFFFFFull ? tile_base : 0xFFFFFFFFull);
    tile_base += tile_n;
    const bool staged = tile_n <= kListStage;
    uint32_t j = base + off;
    // a thread's words cover consecutive positions: pack their presence into
    // 32-position masks (w = 4: four words of 8 positions per mask, the
    // nibble-any bits compressed to one bit each), so position = pos0 + 32 g
    // + bit and the extraction loop runs over 4 masks instead of 16 words
    uint32_t msk[kPerThreadWords];
    if (w4) {
#pragma unroll
      for (uint32_t g = 0; g < kPerThreadWords / 4; ++g) {
        uint32_t c = 0;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
          uint32_t x = bits[4 * g + q];  // bits 0, 4, ..., 28
          x = (x | x >> 3) & 0x03030303u;
          x = (x | x >> 6) & 0x000F000Fu;
          x = (x | x >> 12) & 0xFFu;
          c |= x << (8 * q);
        }
        msk[g] = c;
      }
    } else {
#pragma unroll
      for (uint32_t k = 0; k < kPerThreadWords; ++k) msk[k] = bits[k];
    }
    const uint32_t groups = w4 ? kPerThreadWords / 4 : kPerThreadWords;
    const uint32_t pos0 = tile_word(wbase, 0) * P;
#pragma unroll
    for (uint32_t g = 0; g < kPerThreadWords; ++g) {
      if (g >= groups) break;
      for (uint32_t x = msk[g]; x; x &= x - 1) {
        const uint32_t p = pos0 + 32u * g + uint32_t(__ffs(x) - 1);
        if (j < total_list) {
          w.plist[j] = p;
          if (w.n_items > 1) w.pitem[j] = it;
        }
        if (staged) s_pos[buf][j - base] = p;
        ++j;
      }
    }
    __syncthreads();  // the tile's positions are visible to the whole CTA
    // bucket byte counters, one entry per thread (hashing and REDs converged)
    const uint32_t n_in = base + tile_n <= total_list ? tile_n : (base < total_list ? total_list - base : 0u);
    for (uint32_t q = threadIdx.x; q < n_in; q += blockDim.x) {
      const uint32_t p = staged ? s_pos[buf][q] : __ldcg(w.plist + base + q);
      _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
        const uint64_t slot = e.slot_base + uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m, e.mmul);
        cnt_add(w, slot);
      }
    }
    it = nit;
  }
}

// ------------------------------------------------------------------ staging
// Warp-aggregated appends into a per-CTA shared-memory stage, flushed with one
// global atomic per CTA; a single list counter hit by every warp serialises at
// one L2 slice otherwise. s_n[0] = reserved entries, s_n[1] = end of the
// contiguous written prefix (an overflowing warp goes straight to the list).
// Returns (warp-uniform) whether the stage now holds more than flush_at
// entries: a caller whose loop is CTA-uniform flushes mid-loop when any warp
// saw that (__syncthreads_or), so the direct path stays a rare fallback.
template <typename T, uint32_t kCap>
__device__ __forceinline__ bool stage_push(bool push, T val, T* s_buf, uint32_t* s_n, T* g_buf,
                                           uint32_t* g_count, uint32_t lane, uint32_t flush_at = kCap) {
  const uint32_t mask = __ballot_sync(kFull, push);
  if (!mask) return false;
  const uint32_t leader = __ffs(mask) - 1, cnt = __popc(mask);
  uint32_t b = 0, direct = 0;
  if (lane == leader) {
    b = atomicAdd(s_n, cnt);
    if (b + cnt > kCap) {
      if (b < kCap) atomicMin(s_n + 1, b);  // [b, cap) stays unwritten
      direct = 1;
      b = atomicAdd(g_count, cnt);
    }
  }
  b = __shfl_sync(kFull, b, leader);
  direct = __shfl_sync(kFull, direct, leader);
  if (push) {
    const uint32_t idx = b + __popc(mask & ((1u << lane) - 1u));
    if (direct) g_buf[idx] = val;
    else s_buf[idx] = val;
  }
  return direct || b + cnt > flush_at;
}

template <typename T, uint32_t kCap>
__device__ __forceinline__ void stage_flush(T* s_buf, uint32_t* s_n, uint32_t* s_base, T* g_buf,
                                            uint32_t* g_count) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t n = min(min(s_n[0], kCap), s_n[1]);
    *s_base = n ? atomicAdd(g_count, n) : 0u;
    s_n[0] = n;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < s_n[0]; i += blockDim.x) g_buf[*s_base + i] = s_buf[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    s_n[0] = 0;
    s_n[1] = kCap;
  }
  __syncthreads();
}

constexpr uint32_t kPushStage = 8192;  // next-frontier slots per CTA
constexpr uint32_t kR0Stage = 2048;    // round-0 subtraction entries per phase-1 CTA

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Item of a global slot id: the items' slot bases are cached in shared
// memory when they fit (binary search in L1/L2 otherwise).
constexpr uint32_t kPeelItemsSmem = 512;
struct SlotItems {
  const unsigned long long* sbase;  // shared copy, or nullptr
  const DecItem* items;
  uint32_t n;
  __device__ __forceinline__ uint32_t find(uint64_t s) const {
    uint32_t lo = 0, hi = n - 1;
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      const uint64_t b = sbase ? sbase[mid] : items[mid].slot_base;
      if (b <= s) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  }
};

__device__ __forceinline__ uint32_t slot_row(uint64_t local, uint32_t m) {
  uint32_t row = 0;
  while (local >= m) {
    local -= m;
    ++row;
  }
  return row;
}

// ------------------------------------------------------------------ round 0
// Every listed entry i (position p) inspects its k buckets at round start
// and peels from its lowest singleton row (lowest slot id: the reference's
// ascending seed order, decode.cpp:96-99), writing value = sign * residual
// (decode.cpp:110-111) to val[i]; pinfo[i] keeps (value, rows shared with
// other positions, peel row) for the subtraction pass. Recovered flags of a
// warp's 32 consecutive entries are written as one word (no atomics).
__device__ __forceinline__ void round0_phase1(const DecodeWork& w, const HashParams& hp,
                                              uint64_t start, uint64_t stride, uint32_t* s_q = nullptr,
                                              uint32_t* s_n = nullptr, uint32_t* s_u = nullptr,
                                              uint32_t* s_un = nullptr) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t won = 0;
  const uint32_t total = ldcg(&w.qcount[5]);
  for (uint64_t base = start - lane; base < total; base += stride) {
    const uint64_t i = base + lane;
    bool peeled = false, sub = false;  // sub: peeled with a shared bucket (k_r0_subtract's work)
    if (i < total) {
      const uint32_t p = __ldcs(w.plist + i);
      const DecItem& e = w.items[item_of(w, i)];
      uint64_t ls[kMaxRows];
      unsigned long long st[kMaxRows];
#pragma unroll
      for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) {
        if (r < hp.rows) {  // issue every row's load before inspecting any
          ls[r] = uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m, e.mmul);
          if (w.cnt8) {
            const uint64_t sl = e.slot_base + ls[r];
            st[r] = cnt_get(w, sl);
          } else {
            st[r] = ldcg(w.slot_state + e.slot_base + ls[r]);
          }
        }
      }
      int best = -1;
      uint64_t local = 0;
      float sg = 0.0f;
      uint32_t shared = 0;  // rows whose bucket holds other positions too
#pragma unroll
      for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) {
        if (r >= hp.rows) continue;
        const uint32_t c = st_count(st[r]);
        shared |= uint32_t(c >= 2u) << r;
        if (best < 0 && c == 1u) {
          best = int(r);
          local = ls[r];
          sg = dev_sign(hp.row[r], p);
        }
      }
      uint2 info = make_uint2(0u, 0u);
      if (best < 0 && w.slot_mark) {  // unresolved after round 0: its buckets still matter
#pragma unroll
        for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r)
          if (r < hp.rows) {
            const uint64_t sl = e.slot_base + ls[r];
            red_or_u32(w.slot_mark + (sl >> 5), 1u << (sl & 31));
            // counter mode: only these buckets get a (count, index sum)
            // state, built by k_r0_subtract from the unresolved entries
            if (w.cnt8 && !w.state_zeroed) w.slot_state[sl] = 0ull;
          }
      }
      if (best >= 0) {
        const float v = canonical(sg * ldcg(e.sketch + local));
        w.val[i] = v;
        info = make_uint2(__float_as_uint(v), shared | 0x100u | (uint32_t(best) << 12));
        if (w.wmask && shared) {  // ordered peel: winner slot of an entry that pushes
          const uint64_t ws = e.slot_base + local;
          red_or_u32(w.wmask + (ws >> 5), 1u << (ws & 31));
        }
        peeled = true;
        sub = shared != 0u;
        ++won;
      }
      w.pinfo[i] = info;
    }
    const uint32_t m = __ballot_sync(kFull, peeled);
    if (lane == 0 && base < total) w.bitmap[base >> 5] = m;  // base is a multiple of 32
    if (s_q) stage_push<uint32_t, kR0Stage>(sub, uint32_t(i), s_q, s_n, w.r0_list, &w.qcount[13], lane);
    if (s_u) stage_push<uint32_t, kR0Stage>(i < total && !peeled, uint32_t(i), s_u, s_un, w.ulist,
                                            &w.qcount[14], lane);
  }
  won = warp_sum32(won);
  if (lane == 0 && won) atomicAdd(&w.qcount[kPeeledWord], won);
}

__global__ void __launch_bounds__(256) k_r0_phase1(DecodeWork w, const HashParams hp) {
  __shared__ uint32_t s_q[kR0Stage], s_u[kR0Stage];
  __shared__ uint32_t s_n[2], s_un[2], s_base;
  const bool compact = w.r0_list != nullptr;
  const bool ulist = w.cnt8 != nullptr;
  if (threadIdx.x == 0) {
    s_n[0] = s_un[0] = 0;
    s_n[1] = s_un[1] = kR0Stage;
  }
  __syncthreads();
  round0_phase1(w, hp, uint64_t(blockIdx.x) * blockDim.x + threadIdx.x, uint64_t(gridDim.x) * blockDim.x,
                compact ? s_q : nullptr, s_n, ulist ? s_u : nullptr, s_un);
  if (compact) stage_flush<uint32_t, kR0Stage>(s_q, s_n, &s_base, w.r0_list, &w.qcount[13]);
  if (ulist) stage_flush<uint32_t, kR0Stage>(s_u, s_un, &s_base, w.ulist, &w.qcount[14]);
}

// Round 0 with the row count fixed at compile time (k = R, the common k = 3)
// and PER list entries per thread: every entry's bucket probes, then every
// peeled entry's residual load, are issued before any of them is consumed,
// so PER x R probes and PER sketch gathers are in flight per thread (the
// generic kernel has R and 1). Same outputs as round0_phase1; pinfo only
// where a later pass reads it (compact list: entries with a shared bucket).
template <int R, int PER>
__global__ void __launch_bounds__(256) k_r0_phase1_k(DecodeWork w, const HashParams hp) {
  __shared__ uint32_t s_q[kR0Stage], s_u[kR0Stage];
  __shared__ uint32_t s_n[2], s_un[2], s_base, s_won;
  const bool compact = w.r0_list != nullptr;
  const bool ulist = w.cnt8 != nullptr;
  if (threadIdx.x == 0) {
    s_won = 0;
    s_n[0] = s_un[0] = 0;
    s_n[1] = s_un[1] = kR0Stage;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t won = 0;
  const uint32_t total = ldcg(&w.qcount[5]);
  const uint64_t step = uint64_t(gridDim.x) * blockDim.x * PER;
  // a warp covers PER consecutive groups of 32 entries (one bitmap word each);
  // the loop bound is CTA-uniform (stage flushes need every thread)
  for (uint64_t cb = uint64_t(blockIdx.x) * blockDim.x * PER; cb < total; cb += step) {
    const uint64_t wb = cb + uint64_t(threadIdx.x & ~31u) * PER;
    bool full = false;
    uint32_t p[PER], it[PER];
    bool act[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint64_t i = wb + 32u * k + lane;
      act[k] = i < total;
      p[k] = act[k] ? __ldcs(w.plist + i) : 0u;
      it[k] = act[k] ? item_of(w, i) : 0u;
    }
    uint64_t ls[PER][R];
    uint32_t c[PER][R];
    const float* sk[PER];
    uint64_t sb[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const DecItem& e = w.items[it[k]];
      const uint32_t m = e.m;
      const uint64_t mm = e.mmul;
      sk[k] = e.sketch;
      sb[k] = e.slot_base;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ls[k][r] = uint64_t(r) * m + dev_bucket(hp.row[r], p[k], m, mm);
        const uint64_t sl = sb[k] + ls[k][r];
        if (!act[k]) c[k][r] = 0u;
        else if (w.cnt8) c[k][r] = cnt_get(w, sl);
        else c[k][r] = st_count(ldcg(w.slot_state + sl));
      }
    }
    int best[PER];
    uint32_t shared[PER];
    float resid[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      best[k] = -1;
      shared[k] = 0u;
      uint64_t local = 0;
#pragma unroll
      for (int r = R - 1; r >= 0; --r) {  // lowest singleton row wins
        shared[k] |= uint32_t(c[k][r] >= 2u) << r;
        if (c[k][r] == 1u) {
          best[k] = r;
          local = ls[k][r];
        }
      }
      resid[k] = best[k] >= 0 ? ldcg(sk[k] + local) : 0.0f;  // every gather in flight together
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint64_t i = wb + 32u * k + lane;
      const bool peeled = act[k] && best[k] >= 0;
      const bool sub = peeled && shared[k] != 0u;
      if (act[k]) {
        uint2 info = make_uint2(0u, 0u);
        if (peeled) {
          float sg = 0.0f;
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (r == best[k]) sg = dev_sign(hp.row[r], p[k]);
          const float v = canonical(sg * resid[k]);
          w.val[i] = v;
          info = make_uint2(__float_as_uint(v), shared[k] | 0x100u | (uint32_t(best[k]) << 12));
          ++won;
          if (w.wmask && shared[k]) {  // ordered peel: winner slot of an entry that pushes
            uint64_t lb = 0;
#pragma unroll
            for (int r = 0; r < R; ++r)
              if (r == best[k]) lb = ls[k][r];
            const uint64_t ws = sb[k] + lb;
            red_or_u32(w.wmask + (ws >> 5), 1u << (ws & 31));
          }
        } else if (w.slot_mark) {  // unresolved after round 0: its buckets still matter
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint64_t sl = sb[k] + ls[k][r];
            red_or_u32(w.slot_mark + (sl >> 5), 1u << (sl & 31));
            if (w.cnt8 && !w.state_zeroed) w.slot_state[sl] = 0ull;  // built by k_r0_subtract_cnt
          }
        }
        if (!compact || sub) w.pinfo[i] = info;
      }
      const uint32_t bm = __ballot_sync(kFull, peeled);
      if (lane == 0 && wb + 32u * k < total) w.bitmap[(wb >> 5) + k] = bm;
      // flush once a stage could not take another iteration's entries
      constexpr uint32_t kAt = kR0Stage - 256u * PER;
      if (compact) full |= stage_push<uint32_t, kR0Stage>(sub, uint32_t(i), s_q, s_n, w.r0_list, &w.qcount[13], lane, kAt);
      if (ulist) full |= stage_push<uint32_t, kR0Stage>(act[k] && !peeled, uint32_t(i), s_u, s_un, w.ulist,
                                                        &w.qcount[14], lane, kAt);
    }
    // a single list counter hit by every overflowing warp serialised round 0
    // at high load (theta = 90: ~2M same-address atomics)
    if (__syncthreads_or(full)) {
      if (compact) stage_flush<uint32_t, kR0Stage>(s_q, s_n, &s_base, w.r0_list, &w.qcount[13]);
      if (ulist) stage_flush<uint32_t, kR0Stage>(s_u, s_un, &s_base, w.ulist, &w.qcount[14]);
    }
  }
  won = warp_sum32(won);
  if (lane == 0 && won) atomicAdd(&s_won, won);
  if (compact) stage_flush<uint32_t, kR0Stage>(s_q, s_n, &s_base, w.r0_list, &w.qcount[13]);
  if (ulist) stage_flush<uint32_t, kR0Stage>(s_u, s_un, &s_base, w.ulist, &w.qcount[14]);
  __syncthreads();
  if (threadIdx.x == 0 && s_won) atomicAdd(&w.qcount[kPeeledWord], s_won);  // one RED per CTA
}

// Every entry peeled in round 0 leaves the buckets it shares with other
// positions (decode.cpp:115-121); buckets whose count drops to one seed round
// 1 (queue 1, frontier counter qcount[9]). Only buckets that also hold an
// entry round 0 left unresolved (slot_mark, set by round0_phase1) are
// touched: every other bucket would only empty out, and nothing reads an
// empty bucket again (neither the frontier nor the median estimate).
// Counter mode (w.cnt8): round 0 kept no index sums, so the state of every
// bucket holding a round-0 unresolved entry (slot_mark; cleared by
// k_r0_phase1) is built here from those entries alone - exactly what the
// full state holds there once the round-0 peeled entries have left - while
// the peeled entries only take their values out of the marked buckets'
// residuals. k_peel seeds round 1 from the unresolved entries' buckets.
__global__ void __launch_bounds__(256) k_r0_subtract_cnt(DecodeWork w, const HashParams hp) {
  PDL_WAIT();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint32_t total = ldcg(&w.qcount[13]);
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < total; base += stride) {
    const uint64_t j = base + lane;
    if (j >= total) continue;
    const uint64_t i = ldcg(w.r0_list + j);
    const uint2 info = __ldcs(w.pinfo + i);
    const uint32_t rows = info.y & 0xFFu;
    const float v = __uint_as_float(info.x);
    const uint32_t p = __ldcs(w.plist + i);
    const DecItem* e = w.items + item_of(w, i);
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows && ((rows >> r) & 1u)) {
      const uint64_t loc = uint64_t(r) * e->m + dev_bucket(hp.row[r], p, e->m, e->mmul);
      const uint64_t sl = e->slot_base + loc;
      if ((__ldg(w.slot_mark + (sl >> 5)) >> (sl & 31)) & 1u) red_add_f32(e->sketch + loc, -(dev_sign(hp.row[r], p) * v));
    }
  }
  const uint32_t nu = ldcg(&w.qcount[14]);
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < nu; j += stride) {
    const uint32_t i = ldcg(w.ulist + j);
    const uint32_t p = __ldcs(w.plist + i);
    const DecItem* e = w.items + item_of(w, i);
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
      const uint64_t sl = e->slot_base + uint64_t(r) * e->m + dev_bucket(hp.row[r], p, e->m, e->mmul);
      atomicAdd(w.slot_state + sl, st_add(i));  // result unused: RED.ADD.64
    }
  }
}

__global__ void __launch_bounds__(256) k_r0_subtract(DecodeWork w, const HashParams hp) {
  __shared__ uint32_t s_q[kPushStage];
  __shared__ uint32_t s_n[2], s_base;
  if (threadIdx.x == 0) {
    s_n[0] = 0;
    s_n[1] = kPushStage;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  // only the round-0 peeled entries that share a bucket (compacted by
  // k_r0_phase1); the whole list when no compact list was built
  const bool compact = w.r0_list != nullptr;
  const uint32_t total = compact ? ldcg(&w.qcount[13]) : ldcg(&w.qcount[5]);
  uint32_t* nq = w.queue[1];
  uint32_t* ncount = &w.qcount[9];
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < total; base += stride) {
    const uint64_t j = base + lane;
    const uint64_t i = compact && j < total ? uint64_t(ldcg(w.r0_list + j)) : j;
    uint32_t p = 0, rows = 0;
    float v = 0.0f;
    const DecItem* e = w.items;
    if (j < total) {
      const uint2 info = __ldcs(w.pinfo + i);
      if (info.y & 0x100u) {
        rows = info.y & 0xFFu;
        v = __uint_as_float(info.x);
        p = __ldcs(w.plist + i);
        e = w.items + item_of(w, i);
      }
    }
    unsigned long long old[kMaxRows];
    uint64_t loc[kMaxRows];
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
      bool sh = (rows >> r) & 1u;
      loc[r] = sh ? uint64_t(r) * e->m + dev_bucket(hp.row[r], p, e->m, e->mmul) : 0;
      if (sh) {
        const uint64_t sl = e->slot_base + loc[r];
        sh = (__ldg(w.slot_mark + (sl >> 5)) >> (sl & 31)) & 1u;
      }
      old[r] = sh ? atomicAdd(w.slot_state + e->slot_base + loc[r], st_sub(uint32_t(i))) : 0ull;
      if (sh) red_add_f32(e->sketch + loc[r], -(dev_sign(hp.row[r], p) * v));
    }
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows)
      stage_push<uint32_t, kPushStage>(st_count(old[r]) == 2u, uint32_t(e->slot_base + loc[r]), s_q, s_n, nq,
                                       ncount, lane);
  }
  stage_flush<uint32_t, kPushStage>(s_q, s_n, &s_base, nq, ncount);
}

// ------------------------------------------------------------------ frontier
// Rounds >= 1 in ONE cooperative persistent kernel. A slot holding exactly
// one entry i (decode.cpp:104-106) claims i (an entry reachable through
// several singleton slots is claimed once: atomicOr on its recovered bit),
// reads value = sign * residual into val[i] and removes i from its other
// buckets; a bucket whose count drops to one is pushed for the next round
// together with its remaining entry, which the decrement's returned state
// names exactly (count 1: the low bits of the index sum).
//
// Per round the dependent chain is two L2 round trips: {claim, position,
// residual} then {residual REDs, count decrements}. No state re-read: a
// pushed (slot, entry) pair is stale only if entry was peeled elsewhere,
// which the claim detects. No fence between a removal's residual update and
// its count decrement: within a round a claimed slot's residual can only be
// changed by the removal of its own single entry, and rounds are separated
// by a barrier. The next frontier stays in the pushing CTA's shared memory
// (global overflow beyond kLocalQ); the grid barrier is one atomic per CTA
// that also sums the CTAs' push counts, so no CTA reads a global counter.
// Once a round's frontier is small, CTA 0 finishes alone with block
// barriers. The peeled set is the complement of the 2-core either way
// (order-independent); values match the reference's FIFO peel within fp32
// reassociation.
constexpr uint32_t kLocalQ = 2048;   // (slot, entry) pairs per CTA and round
constexpr uint32_t kOvfStage = 2048; // overflow slots staged per CTA before one global append

// Overflow beyond the local queue: the slot alone (its state names the entry
// next round), staged in shared memory and appended to the round's global
// queue with one atomic per flush (stage_push / stage_flush). A per-warp
// append on the one queue counter serialised millions of pushes at high load
// (theta = 90: 6 ms of k_peel).
struct PeelOvf {
  uint32_t* s_buf;   // kOvfStage slots
  uint32_t* s_n;     // stage_push's two words
  uint32_t* s_base;
  uint32_t* gq;      // the next round's global queue and its counter
  uint32_t* gcount;
};

// Returns (warp-uniform) whether the overflow stage should be flushed.
template <uint32_t kFlushAt>
__device__ __forceinline__ bool local_push(bool push, uint32_t slot, uint32_t entry, uint2* s_next,
                                           uint32_t* s_nn, const PeelOvf& ov, uint32_t lane) {
  const uint32_t mask = __ballot_sync(kFull, push);
  if (!mask) return false;
  const uint32_t leader = __ffs(mask) - 1;
  uint32_t b = 0;
  if (lane == leader) b = atomicAdd(s_nn, uint32_t(__popc(mask)));
  b = __shfl_sync(kFull, b, leader);
  const uint32_t idx = b + __popc(mask & ((1u << lane) - 1u));
  if (push && idx < kLocalQ) s_next[idx] = make_uint2(slot, entry);
  if (b + __popc(mask) <= kLocalQ) return false;
  return stage_push<uint32_t, kOvfStage>(push && idx >= kLocalQ, slot, ov.s_buf, ov.s_n, ov.gq, ov.gcount, lane,
                                         kFlushAt);
}

// kN frontier elements per lane, processed together (their L2 trips
// overlap). kPair: (slot, entry) from a local queue; otherwise a slot from a
// global queue (its state names the entry).
template <bool kPair, int kN, int R>
__device__ __forceinline__ uint32_t peel_n(const DecodeWork& w, const HashParams& hp, const SlotItems& si,
                                           const bool (&have_in)[kN], const uint32_t (&slot)[kN],
                                           const uint32_t (&i_in)[kN], uint2* s_next, uint32_t* s_nn,
                                           const PeelOvf& ov, bool& full, uint32_t lane) {
  bool have[kN];
  uint32_t i[kN];
#pragma unroll
  for (int k = 0; k < kN; ++k) {
    have[k] = have_in[k];
    i[k] = i_in[k];
  }
  if (!kPair) {
    unsigned long long st[kN];
#pragma unroll
    for (int k = 0; k < kN; ++k) st[k] = have[k] ? ldcg(w.slot_state + slot[k]) : 0ull;
#pragma unroll
    for (int k = 0; k < kN; ++k) {
      have[k] = have[k] && st_count(st[k]) == 1u;
      i[k] = st_entry(st[k]);
    }
  }
  bool win[kN];
  uint32_t p[kN], row[kN], pp[kN], old_bits[kN];
  float v[kN], resid[kN];
  const DecItem* e[kN];
  uint64_t local[kN];
#pragma unroll
  for (int k = 0; k < kN; ++k) {  // claims, positions and residuals of every element in flight together
    e[k] = w.items;
    local[k] = 0;
    pp[k] = 0;
    resid[k] = 0.0f;
    old_bits[k] = ~0u;
    if (have[k]) {
      e[k] = w.items + si.find(slot[k]);
      local[k] = slot[k] - e[k]->slot_base;
      pp[k] = __ldg(w.plist + i[k]);
      resid[k] = ldcg(e[k]->sketch + local[k]);
      old_bits[k] = atomicOr(w.bitmap + (i[k] >> 5), 1u << (i[k] & 31));
    }
  }
#pragma unroll
  for (int k = 0; k < kN; ++k) {
    win[k] = have[k] && !((old_bits[k] >> (i[k] & 31)) & 1u);
    p[k] = 0;
    row[k] = 0;
    v[k] = 0.0f;
    if (win[k]) {
      p[k] = pp[k];
      row[k] = slot_row(local[k], e[k]->m);
      float sg = 0.0f;
      _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(R); ++r) if (r == row[k]) sg = dev_sign(hp.row[r], p[k]);
      v[k] = canonical(sg * resid[k]);
      w.val[i[k]] = v[k];
    }
  }
  unsigned long long old[kN][R];
  uint32_t sl[kN][R];
#pragma unroll
  for (int k = 0; k < kN; ++k) {
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(R); ++r) if (r < hp.rows) {
      old[k][r] = 0ull;
      sl[k][r] = 0u;
      if (win[k] && r != row[k]) {
        const uint64_t loc = uint64_t(r) * e[k]->m + dev_bucket(hp.row[r], p[k], e[k]->m, e[k]->mmul);
        sl[k][r] = uint32_t(e[k]->slot_base + loc);
        red_add_f32(e[k]->sketch + loc, -(dev_sign(hp.row[r], p[k]) * v[k]));
        old[k][r] = atomicAdd(w.slot_state + e[k]->slot_base + loc, st_sub(i[k]));
      }
    }
  }
  uint32_t won = 0;
  // an iteration pushes at most blockDim * kN * (R - 1) slots
  constexpr uint32_t kAt = kOvfStage > 256u * kN * (R - 1) ? kOvfStage - 256u * kN * (R - 1) : 0u;
#pragma unroll
  for (int k = 0; k < kN; ++k) {
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(R); ++r) if (r < hp.rows) {
      const bool push = win[k] && r != row[k] && st_count(old[k][r]) == 2u;
      full |= local_push<kAt>(push, sl[k][r], st_entry(old[k][r] + st_sub(i[k])), s_next, s_nn, ov, lane);
    }
    won += win[k] ? 1u : 0u;
  }
  return won;
}

__device__ __forceinline__ void ovf_flush(const PeelOvf& ov) {
  stage_flush<uint32_t, kOvfStage>(ov.s_buf, ov.s_n, ov.s_base, ov.gq, ov.gcount);
}
// end of a loop: flush only a non-empty stage (no pushes until the next
// round's barrier, so every thread reads the same count)
__device__ __forceinline__ void ovf_flush_end(const PeelOvf& ov) {
  __syncthreads();
  if (ov.s_n[0] != 0u) ovf_flush(ov);
}

// One round's share of a CTA: the local pairs [0, nl) and the global slots
// [0, ng) strided by gstride from cta0 (CTA-uniform loop bounds: the
// overflow stage is flushed mid-round when a warp finds it nearly full),
// kPeelN per lane. The stage is flushed at the end.
constexpr int kPeelN = 2;
template <int R>
__device__ __forceinline__ uint32_t peel_round(const DecodeWork& w, const HashParams& hp, const SlotItems& si,
                                               const uint2* cur, uint32_t nl, const uint32_t* gsrc, uint32_t ng,
                                               uint64_t cta0, uint64_t gstride, uint2* s_next, uint32_t* s_nn,
                                               const PeelOvf& ov, uint32_t lane) {
  uint32_t won = 0;
  for (uint32_t b = 0; b < nl; b += blockDim.x * kPeelN) {
    bool have[kPeelN];
    uint32_t sl[kPeelN], en[kPeelN];
#pragma unroll
    for (int k = 0; k < kPeelN; ++k) {
      const uint32_t j = b + k * blockDim.x + threadIdx.x;
      have[k] = j < nl;
      const uint2 x = have[k] ? cur[j] : make_uint2(0, 0);
      sl[k] = x.x;
      en[k] = x.y;
    }
    bool full = false;
    won += peel_n<true, kPeelN, R>(w, hp, si, have, sl, en, s_next, s_nn, ov, full, lane);
    if (b + blockDim.x * kPeelN < nl && __syncthreads_or(full)) ovf_flush(ov);  // (CTA-uniform)
  }
  for (uint64_t b = cta0; b < ng; b += gstride * kPeelN) {
    bool have[kPeelN];
    uint32_t sl[kPeelN], en[kPeelN];
#pragma unroll
    for (int k = 0; k < kPeelN; ++k) {
      const uint64_t j = b + k * gstride + threadIdx.x;
      have[k] = j < ng;
      sl[k] = have[k] ? ldcg(gsrc + j) : 0u;
      en[k] = 0u;
    }
    bool full = false;
    won += peel_n<false, kPeelN, R>(w, hp, si, have, sl, en, s_next, s_nn, ov, full, lane);
    if (b + gstride * kPeelN < ng && __syncthreads_or(full)) ovf_flush(ov);
  }
  ovf_flush_end(ov);
  return won;
}

// Grid barrier that also sums a per-CTA value: barrier k adds
// (1 << 40 | add) into word k % 3 and waits for every CTA's arrival; the
// word of barrier k - 1 is free again once barrier k has passed (each CTA
// read it before arriving at k), so CTA 0 clears it for barrier k + 2.
constexpr unsigned kBarSleepNs = 64;  // poll back-off (0..300 ns measured alike; no back-off: ~7 % slower)
__device__ __forceinline__ uint32_t grid_barrier_sum(unsigned long long* bar, uint32_t k, uint32_t add,
                                                     uint32_t* s_out) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* word = bar + k % 3;
    __threadfence();
    atomicAdd(word, (1ull << 40) | uint64_t(add));
    const unsigned long long target = uint64_t(gridDim.x) << 40;
    unsigned long long v;
    while ((v = ld_acquire(word)) < target) __nanosleep(kBarSleepNs);  // 296 pollers on one line
    __threadfence();
    *s_out = uint32_t(v & ((1ull << 40) - 1ull));
    if (blockIdx.x == 0) bar[(k + 2) % 3] = 0ull;
  }
  __syncthreads();
  return *s_out;
}

// R: rows compiled in (3, the common k, or kMaxRows for any k <= 8).
template <int R>
__global__ void __launch_bounds__(256, 2) k_peel(DecodeWork w, const HashParams hp) {
  __shared__ uint2 s_lq[2][kLocalQ];
  __shared__ unsigned long long s_sbase[kPeelItemsSmem];
  __shared__ uint32_t s_ovf[kOvfStage];
  __shared__ uint32_t s_ln[2], s_on[2], s_obase, s_base, s_total, s_won;
  if (threadIdx.x == 0) {
    s_won = 0;
    s_ln[0] = s_ln[1] = 0;
    s_on[0] = 0;
    s_on[1] = kOvfStage;
  }
  const bool cache = w.n_items <= kPeelItemsSmem;
  if (cache)
    for (uint32_t i = threadIdx.x; i < w.n_items; i += blockDim.x) s_sbase[i] = w.items[i].slot_base;
  __syncthreads();
  const SlotItems si{cache ? s_sbase : nullptr, w.items, w.n_items};
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gstride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t* cnt = w.qcount + 8;
  uint32_t* const qbuf0 = w.queue[0];  // selected by value: a runtime index into the parameter
  uint32_t* const qbuf1 = w.queue[1];  // struct would copy it to local memory
  auto qbuf = [&](uint32_t k) { return (k & 1) ? qbuf1 : qbuf0; };
  int mk = 0;
  PEEL_MARK(mk++);
  if (gtid == 0) w.qcount[2] = 1;
  // round k reads the local queue s_lq[k & 1] and the global overflow
  // qbuf(k) / cnt[k % 3]; it pushes into s_lq[(k + 1) & 1] / qbuf(k + 1).
  // Grid barriers are numbered 0 (round 1's frontier), 1, 2, ...
  uint32_t total;
  if (w.cnt8) {
    // counter mode: round 1's frontier = the unresolved entries' single-
    // entry buckets, each pushed by its only entry as a local (slot, entry)
    // pair; two entries per lane in flight
    const uint32_t nu = ldcg(&w.qcount[14]);
    const PeelOvf ov{s_ovf, s_on, &s_obase, qbuf1, &cnt[1]};
    constexpr uint32_t kAt = kOvfStage > 256u * 2u * R ? kOvfStage - 256u * 2u * R : 0u;
    for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x; base < nu; base += 2 * gstride) {  // CTA-uniform
      uint32_t ii[2], p[2];
      const DecItem* e[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t j = base + h * gstride + threadIdx.x;
        ii[h] = j < nu ? ldcg(w.ulist + j) : 0u;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool ok = base + h * gstride + threadIdx.x < nu;
        p[h] = ok ? __ldcs(w.plist + ii[h]) : 0u;
        e[h] = w.items + (ok ? item_of(w, ii[h]) : 0u);
      }
      uint32_t sl[2][R];
      uint32_t one[2] = {0u, 0u};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool ok = base + h * gstride + threadIdx.x < nu;
        _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(R); ++r) if (r < hp.rows) {
          sl[h][r] = uint32_t(e[h]->slot_base + uint64_t(r) * e[h]->m + dev_bucket(hp.row[r], p[h], e[h]->m, e[h]->mmul));
          if (ok && st_count(ldcg(w.slot_state + sl[h][r])) == 1u) one[h] |= 1u << r;
        }
      }
      bool full = false;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(R); ++r) if (r < hp.rows)
          full |= local_push<kAt>((one[h] >> r) & 1u, sl[h][r], ii[h], s_lq[1], &s_ln[1], ov, lane);
      }
      if (base + 2 * gstride < nu && __syncthreads_or(full)) ovf_flush(ov);
    }
    ovf_flush_end(ov);
    total = grid_barrier_sum(w.bar, 0, s_ln[1], &s_total);
  } else {
    total = ldcg(&cnt[1]);  // k_r0_subtract's global pushes
  }
  // Grid rounds, then (once a round's frontier is <= kTail) the tail: CTA 0
  // alone with block barriers. ONE loop and one peel_round call site for
  // both, so the tail runs the grid rounds' instructions (a separate inlined
  // copy started with a cold instruction cache: its first round took 10 us
  // against 3.4 for the next ones at W = 8).
  uint32_t won = 0, k = 1;
  bool tail = false;
  for (;; ++k) {
    if (!tail) {
      if (total == 0) break;
      if (total <= kTail) {  // hand the local pairs to CTA 0 (w.handoff, count qcount[15])
        const uint32_t n = min(s_ln[k & 1], kLocalQ);
        if (threadIdx.x == 0) s_base = n ? atomicAdd(&w.qcount[15], n) : 0u;
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) w.handoff[s_base + j] = s_lq[k & 1][j];
        if (threadIdx.x == 0) s_ln[k & 1] = 0;
        grid_barrier_sum(w.bar, k, 0, &s_total);
        if (blockIdx.x != 0) break;
        const uint32_t nh = ldcg(&w.qcount[15]);  // <= total <= kTail <= kLocalQ
        for (uint32_t j = threadIdx.x; j < nh; j += blockDim.x) s_lq[k & 1][j] = __ldcg(w.handoff + j);
        if (threadIdx.x == 0) s_ln[k & 1] = nh;
        __syncthreads();
        tail = true;  // round k's global part is qbuf(k) / cnt[k % 3], later rounds local
      }
    }
    if (tail) {
      if (threadIdx.x == 0) cnt[(k + 2) % 3] = 0;
    } else if (gtid == 0) {
      cnt[(k + 2) % 3] = 0;
      w.qcount[2] += 1;
    }
    const uint32_t nl = min(s_ln[k & 1], kLocalQ);
    const uint32_t ng = ldcg(&cnt[k % 3]);
    if (tail && nl == 0 && ng == 0) break;
    uint2* nxt = s_lq[(k + 1) & 1];
    uint32_t* nn = &s_ln[(k + 1) & 1];
    const PeelOvf ov{s_ovf, s_on, &s_obase, qbuf(k + 1), &cnt[(k + 1) % 3]};
    won += peel_round<R>(w, hp, si, s_lq[k & 1], nl, qbuf(k), ng, tail ? 0ull : uint64_t(blockIdx.x) * blockDim.x,
                         tail ? uint64_t(blockDim.x) : gstride, nxt, nn, ov, lane);
    __syncthreads();
    if (!tail) total = grid_barrier_sum(w.bar, k, *nn, &s_total);
    if (threadIdx.x == 0) {
      s_ln[k & 1] = 0;  // read by every thread before the barrier
      if (tail) w.qcount[3] += 1;
    }
    PEEL_MARK(mk++);
    __syncthreads();
  }
  // one RED per CTA (per-warp REDs shared a line with the queue counters)
  won = warp_sum32(won);
  if (lane == 0 && won) atomicAdd(&s_won, won);
  __syncthreads();
  if (threadIdx.x == 0 && s_won) atomicAdd(&w.qcount[kPeeledWord], s_won);
}

// ------------------------------------------------------------------ ordered peel
// FIFO-order emulation for indices that can hide mass (1-bit merge carries
// drop positions whose contributions stay in the sketch, so the reference's
// values depend on its peel order, decode.cpp:96-122). Generation 0 is the
// entry-centric round above: every entry peels from its lowest singleton
// slot, exactly the reference's ascending seed order. Generation g+1 is the
// queue of slots whose count dropped to one while generation g was processed,
// ordered as the reference's deque orders it: by the FIFO position j of the
// peeled entry, then by row. A slot is queued when the LAST subtraction of
// the generation (in FIFO order) leaves one entry, so every subtraction
// atomicMax-es its key j * rows + r into the slot; keys are unique per slot
// and dense in [0, qlen * rows), so the order is a placement into a dense
// key array plus an order-preserving compaction — no sort. An entry that is a
// singleton in several queued slots is peeled from the first of them
// (epoch-tagged atomicMax claims on ~j).
//
// Everything runs in ONE cooperative kernel (k_ord_loop): generation 0's
// subtraction, then per generation place | count | write + claim | peel,
// separated by grid barriers; once a generation holds <= kOrdTail slots, CTA
// 0 finishes alone with block barriers. No host round trip, so the call is
// graph-capturable like the unordered decode.
constexpr uint32_t kOrdTail = 2048;
constexpr uint32_t kOrdWrap = 0xF0000000u;

__device__ __forceinline__ unsigned long long ord_tag(uint32_t ep, uint64_t key) {
  return (uint64_t(ep) << 32) | key;
}

template <int R, typename Sync>
__device__ __forceinline__ uint32_t ord_generation(const DecodeWork& w, const HashParams& hp, const OrdState& o,
                                                   uint32_t g, uint32_t n, uint64_t dom, uint32_t ep, uint32_t part,
                                                   uint32_t nparts, uint32_t* cnt, uint32_t* s_q, uint32_t* s_nq,
                                                   uint32_t* s_base, uint32_t* s_warp, Sync sync, int& mk) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t rows = hp.rows;
  const uint32_t* u = (g & 1) ? o.u1 : o.u0;
  // A: place every pushed slot at its FIFO key
  for (uint32_t t0 = part * blockDim.x + tid; t0 < n; t0 += 4 * nparts * blockDim.x) {
    uint32_t sl[4], key[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // four slots' key loads in flight per thread
      const uint32_t t = t0 + q * nparts * blockDim.x;
      sl[q] = t < n ? ldcg(u + t) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) key[q] = sl[q] != 0xFFFFFFFFu ? uint32_t(ldcg(o.slot_key + sl[q])) : 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (sl[q] != 0xFFFFFFFFu) o.dense[key[q]] = sl[q] + 1u;
  }
  sync();
  PEEL_MARK(mk++);
  // B: non-empty keys per part (contiguous chunks of 1024-key tiles)
  const uint64_t tiles = (dom + 1023) / 1024;
  const uint64_t per = (tiles + nparts - 1) / nparts;
  const uint64_t lo = min(dom, uint64_t(part) * per * 1024), hi = min(dom, lo + per * 1024);
  uint32_t c = 0;
  for (uint64_t k = lo + tid * 4; k < hi; k += blockDim.x * 4) {
    if (k + 4 <= hi) {
      const uint4 v = __ldcg(reinterpret_cast<const uint4*>(o.dense + k));
      c += (v.x != 0) + (v.y != 0) + (v.z != 0) + (v.w != 0);
    } else {
      for (uint64_t x = k; x < hi; ++x) c += ldcg(o.dense + x) != 0;
    }
  }
  c = warp_sum32(c);
  if (lane == 0) s_warp[wid] = c;
  __syncthreads();
  if (tid == 0) {
    uint32_t t = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) t += s_warp[i];
    o.cta[part] = t;
  }
  sync();
  PEEL_MARK(mk++);
  // C: ordered write of the queue (+ reset of the dense keys, + claims)
  uint32_t off = 0;
  for (uint32_t i = tid; i < part; i += blockDim.x) off += ldcg(o.cta + i);
  off = warp_sum32(off);
  __syncthreads();
  if (lane == 0) s_warp[wid] = off;
  __syncthreads();
  off = 0;
  for (uint32_t i = 0; i < blockDim.x / 32; ++i) off += s_warp[i];
  __syncthreads();
  for (uint64_t base = lo; base < hi; base += blockDim.x * 4) {
    const uint64_t k = base + tid * 4;
    uint32_t v[4] = {0, 0, 0, 0};
    if (k + 4 <= hi) {
      const uint4 x = __ldcg(reinterpret_cast<const uint4*>(o.dense + k));
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
      for (uint32_t x = 0; x < 4; ++x) if (k + x < hi) v[x] = ldcg(o.dense + k + x);
    }
    const uint32_t mine = (v[0] != 0) + (v[1] != 0) + (v[2] != 0) + (v[3] != 0);
    // block exclusive scan of mine (thread order = key order)
    uint32_t incl = mine;
    _Pragma("unroll") for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, d);
      if (lane >= uint32_t(d)) incl += y;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    uint32_t wbase = 0, total = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) {
      const uint32_t x = s_warp[i];
      wbase += i < wid ? x : 0u;
      total += x;
    }
    uint32_t pos = off + wbase + incl - mine;
    if (mine) {
      if (k + 4 <= hi) *reinterpret_cast<uint4*>(o.dense + k) = make_uint4(0, 0, 0, 0);
      else for (uint32_t x = 0; x < 4; ++x) if (k + x < hi) o.dense[k + x] = 0;
      unsigned long long st[4];
#pragma unroll
      for (uint32_t x = 0; x < 4; ++x) st[x] = v[x] ? ldcg(w.slot_state + (v[x] - 1u)) : 0ull;  // in flight together
#pragma unroll
      for (uint32_t x = 0; x < 4; ++x) if (v[x]) {
        o.q[pos] = v[x] - 1u;
        if (st_count(st[x]) == 1u) atomicMax(o.claim + st_entry(st[x]), ord_tag(ep, ~pos));
        ++pos;
      }
    }
    off += total;
    __syncthreads();
  }
  sync();
  PEEL_MARK(mk++);
  // D: peel the queue; subtractions are tagged with the next epoch
  uint32_t won = 0;
  uint32_t* un = (g & 1) ? o.u0 : o.u1;
  uint32_t* cn = cnt + (g + 1) % 3;
  // two queue entries per thread in flight; an entry's position, item and
  // residual are read together with its claim (one dependent trip less)
  constexpr int kD = 2;
  for (uint32_t base = part * blockDim.x * kD; base < n; base += nparts * blockDim.x * kD) {
    uint32_t jj[kD], slot[kD], i[kD], pp[kD], p[kD];
    bool live[kD], win[kD];
    unsigned long long st[kD], cl[kD];
    const DecItem* e[kD];
    float resid[kD], v[kD];
#pragma unroll
    for (int h = 0; h < kD; ++h) {
      jj[h] = base + h * blockDim.x + tid;
      live[h] = jj[h] < n;
      slot[h] = live[h] ? ldcg(o.q + jj[h]) : 0u;
    }
#pragma unroll
    for (int h = 0; h < kD; ++h) st[h] = live[h] ? ldcg(w.slot_state + slot[h]) : 0ull;
#pragma unroll
    for (int h = 0; h < kD; ++h) {
      live[h] = live[h] && st_count(st[h]) == 1u;
      i[h] = st_entry(st[h]);
      e[h] = w.items;
      cl[h] = 0ull;
      pp[h] = 0u;
      resid[h] = 0.0f;
      if (live[h]) {
        cl[h] = ldcg(o.claim + i[h]);
        pp[h] = w.plist[i[h]];
        e[h] = w.items + item_of(w, i[h]);
        resid[h] = ldcg(e[h]->sketch + (slot[h] - e[h]->slot_base));
      }
    }
#pragma unroll
    for (int h = 0; h < kD; ++h) {
      win[h] = live[h] && cl[h] == ord_tag(ep, ~jj[h]);
      p[h] = 0u;
      v[h] = 0.0f;
      if (win[h]) {
        p[h] = pp[h];
        const uint32_t row = uint32_t((slot[h] - e[h]->slot_base) / e[h]->m);
        v[h] = canonical(dev_sign(row_coef(hp, row), p[h]) * resid[h]);  // decode.cpp:110-111
        w.val[i[h]] = v[h];
        red_or_u32(w.bitmap + (i[h] >> 5), 1u << (i[h] & 31));
        ++won;
      }
    }
    unsigned long long old[kD][R];
    uint32_t ss[kD][R], sub[kD];
#pragma unroll
    for (int h = 0; h < kD; ++h) {
      sub[h] = 0u;
      _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(R); ++r) if (r < rows) {
        old[h][r] = 0ull;
        ss[h][r] = 0u;
        if (win[h]) {
          const uint64_t local = uint64_t(r) * e[h]->m + dev_bucket(hp.row[r], p[h], e[h]->m, e[h]->mmul);
          const uint64_t sl = e[h]->slot_base + local;
          if (sl != slot[h]) {
            sub[h] |= 1u << r;
            ss[h][r] = uint32_t(sl);
            red_add_f32(e[h]->sketch + local, -(dev_sign(hp.row[r], p[h]) * v[h]));
            atomicMax(o.slot_key + sl, ord_tag(ep + 1, uint64_t(jj[h]) * rows + r));
            old[h][r] = atomicAdd(w.slot_state + sl, st_sub(i[h]));
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < kD; ++h) {
      _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(R); ++r) if (r < rows) {
        const bool push = ((sub[h] >> r) & 1u) && st_count(old[h][r]) == 2u;
        stage_push<uint32_t, kPushStage>(push, ss[h][r], s_q, s_nq, un, cn, lane);
      }
    }
  }
  stage_flush<uint32_t, kPushStage>(s_q, s_nq, s_base, un, cn);
  return won;
}

// R: rows compiled in (3, or kMaxRows for any k <= 8).
template <int R>
__global__ void __launch_bounds__(256) k_ord_loop(DecodeWork w, const HashParams hp, OrdState o) {
  __shared__ uint32_t s_q[kPushStage];
  __shared__ uint32_t s_nq[2], s_base, s_warp[8];
  if (threadIdx.x == 0) {
    s_nq[0] = 0;
    s_nq[1] = kPushStage;
  }
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gstride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t* cnt = w.qcount + 8;
  int mk = 0;
  PEEL_MARK(mk++);
  uint32_t ep = ldcg(o.epoch);
  if (ep >= kOrdWrap) {  // once per 2^32 generations: restart the tags from zero
    for (uint64_t x = gtid; x < o.slot_key_cap; x += gstride) o.slot_key[x] = 0ull;
    for (uint64_t x = gtid; x < o.claim_cap; x += gstride) o.claim[x] = 0ull;
    ep = 0;
    grid.sync();
  }
  ++ep;  // generation 0's subtractions
  // Generation 0's FIFO keys are (winner slot, row); only winners of entries
  // with a shared bucket push, so the keys are made dense over those: rank of
  // the winner slot among them (popcount prefix of wmask), times rows.
  const uint64_t nwords = o.wwords;
  uint32_t n_win;
  {
    const uint64_t per = (nwords + gridDim.x - 1) / gridDim.x;
    const uint64_t w0 = min(nwords, uint64_t(blockIdx.x) * per), w1 = min(nwords, w0 + per);
    uint32_t c = 0;
    for (uint64_t x = w0 + threadIdx.x; x < w1; x += blockDim.x) c += __popc(ldcg(o.wmask + x));
    c = warp_sum32(c);
    if (lane == 0) s_warp[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (uint32_t i = 0; i < blockDim.x / 32; ++i) t += s_warp[i];
      o.cta[blockIdx.x] = t;
    }
    grid.sync();
    uint32_t off = 0, all = 0;
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      const uint32_t x = ldcg(o.cta + i);
      all += x;
      off += i < blockIdx.x ? x : 0u;
    }
    off = warp_sum32(off);
    all = warp_sum32(all);
    __syncthreads();
    if (lane == 0) s_warp[threadIdx.x >> 5] = off;
    __syncthreads();
    off = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) off += s_warp[i];
    __syncthreads();
    if (lane == 0) s_warp[threadIdx.x >> 5] = all;
    __syncthreads();
    n_win = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) n_win += s_warp[i];
    __syncthreads();
    // exclusive prefix per word of this CTA's range, 256 words at a time
    for (uint64_t b = w0; b < w1; b += blockDim.x) {
      const uint64_t x = b + threadIdx.x;
      const uint32_t pc = x < w1 ? __popc(ldcg(o.wmask + x)) : 0u;
      uint32_t incl = pc;
      _Pragma("unroll") for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, d);
        if (lane >= uint32_t(d)) incl += y;
      }
      if (lane == 31) s_warp[threadIdx.x >> 5] = incl;
      __syncthreads();
      uint32_t wbase = 0, tot = 0;
      for (uint32_t i = 0; i < blockDim.x / 32; ++i) {
        wbase += i < (threadIdx.x >> 5) ? s_warp[i] : 0u;
        tot += s_warp[i];
      }
      if (x < w1) o.wrank[x] = off + wbase + incl - pc;
      off += tot;
      __syncthreads();
    }
    grid.sync();
  }
  // ---- generation 0: round-0 peeled entries leave every bucket they share;
  // pushes keyed (winner slot, row) — the reference's ascending seed order
  // only round 0's compact list (entries peeled with a shared bucket) pushes
  const uint32_t total = ldcg(&w.qcount[13]);
  for (uint64_t base = gtid - lane; base < total; base += gstride) {
    const uint64_t j = base + lane;
    uint64_t i = 0;
    uint32_t p = 0, rows = 0;
    float v = 0.0f;
    uint64_t wkey = 0;
    const DecItem* e = w.items;
    if (j < total) {
      i = ldcg(w.r0_list + j);
      const uint2 info = w.pinfo[i];
      if (info.y & 0x100u) {
        rows = info.y & 0xFFu;
        v = __uint_as_float(info.x);
        p = w.plist[i];
        e = w.items + item_of(w, i);
        const uint32_t best = (info.y >> 12) & 0xFu;
        const uint64_t ws = e->slot_base + uint64_t(best) * e->m + dev_bucket(row_coef(hp, best), p, e->m, e->mmul);
        if (rows) {  // rank of the winner slot among the pushing entries' winners
          const uint32_t wm = ldcg(o.wmask + (ws >> 5));
          wkey = uint64_t(ldcg(o.wrank + (ws >> 5)) + __popc(wm & ((1u << (ws & 31)) - 1u))) * hp.rows;
        }
      }
    }
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
      bool push = false;
      uint64_t s = 0;
      if (rows >> r & 1u) {
        const uint64_t local = uint64_t(r) * e->m + dev_bucket(hp.row[r], p, e->m, e->mmul);
        s = e->slot_base + local;
        red_add_f32(e->sketch + local, -(dev_sign(hp.row[r], p) * v));
        atomicMax(o.slot_key + s, ord_tag(ep, wkey + r));
        const unsigned long long old = atomicAdd(w.slot_state + s, st_sub(uint32_t(i)));
        push = st_count(old) == 2u;
      }
      stage_push<uint32_t, kPushStage>(push, uint32_t(s), s_q, s_nq, o.u0, cnt, lane);
    }
  }
  stage_flush<uint32_t, kPushStage>(s_q, s_nq, &s_base, o.u0, cnt);
  PEEL_MARK(mk++);
  // ---- generations >= 1
  uint64_t dom = uint64_t(n_win) * hp.rows;
  // grid generations, then (at <= kOrdTail slots) CTA 0 alone with block
  // barriers: one loop and one ord_generation instance for both, so the
  // tail runs warm code (cf. k_peel)
  uint32_t won = 0, g = 0;
  bool tail = false;
  for (;; ++g) {
    if (tail) __syncthreads();
    else grid.sync();
    const uint32_t n = ldcg(cnt + g % 3);
    if (n == 0) break;
    if (!tail && n <= kOrdTail) {  // every CTA sees the same n
      if (blockIdx.x != 0) break;
      tail = true;
    }
    if (tail) {
      if (threadIdx.x == 0) {
        cnt[(g + 2) % 3] = 0;
        w.qcount[3] += 1;
      }
    } else if (gtid == 0) {
      cnt[(g + 2) % 3] = 0;
      w.qcount[2] += 1;
    }
    won += ord_generation<R>(w, hp, o, g, n, dom, ep, tail ? 0u : blockIdx.x, tail ? 1u : gridDim.x, cnt, s_q,
                             s_nq, &s_base, s_warp, [&] {
                               if (tail) __syncthreads();
                               else grid.sync();
                             }, mk);
    dom = uint64_t(n) * hp.rows;
    ++ep;
  }
  won = warp_sum32(won);
  if (lane == 0 && won) atomicAdd(&w.qcount[kPeeledWord], won);
  if (blockIdx.x != 0) return;
  if (threadIdx.x == 0) *o.epoch = ep;
}

// ------------------------------------------------------------------ estimate
// Median-of-rows estimate (decode.cpp:130-138 / :43-47) into val[i] for every
// listed entry the peel left unresolved.
__global__ void __launch_bounds__(256) k_final(DecodeWork w, const HashParams hp) {
  PDL_WAIT();
  const uint32_t total = w.qcount[5];
  if (total == w.qcount[kPeeledWord]) return;  // every listed entry peeled: nothing to estimate
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < total; base += stride) {
    const uint32_t i = uint32_t(base) + lane;
    // a warp's 32 entries share one recovered-bit word (base is a multiple of 32)
    const uint32_t word = ldcg(w.bitmap + (base >> 5));
    const bool todo = i < total && !(word >> lane & 1u);
    uint32_t it = 0xFFFFFFFFu, p = 0;
    if (todo) {
      p = w.plist[i];
      it = item_of(w, i);
      const DecItem& e = w.items[it];
      float est[kMaxRows];
#pragma unroll
      for (uint32_t r = 0; r < kMaxRows; ++r) {
        if (r >= hp.rows) break;
        est[r] = dev_sign(hp.row[r], p) * e.sketch[uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m, e.mmul)];
      }
      w.val[i] = canonical(median_rows(est, hp.rows));
    }
    // unresolved counts, one atomic per item group of the warp (a stalled
    // item's counter would otherwise take one atomic per entry)
    const uint32_t grp = __match_any_sync(kFull, it);
    if (todo) {
      const uint32_t leader = __ffs(grp) - 1;
      uint32_t b0 = 0;
      if (lane == leader) b0 = atomicAdd(&w.stats[it].unresolved, uint32_t(__popc(grp)));
      b0 = __shfl_sync(grp, b0, leader);
      if (w.unresolved) w.unresolved[w.items[it].list_off + b0 + __popc(grp & ((1u << lane) - 1u))] = p;
    }
  }
}

// ------------------------------------------------------------------ emit
// The dense shard, chunk by chunk (8192 positions): a shared-memory chunk is
// zeroed (decode.cpp:61-64 zero-initialises the output), the chunk's listed
// entries - a contiguous list range, ascending positions - drop their values
// into it, and one bulk async copy (1-D TMA store) writes it out. Two chunk
// buffers alternate, so a chunk is assembled while the previous one streams.
constexpr uint32_t kEmitChunk = 8192;
constexpr size_t kEmitSmem = 2 * kEmitChunk * sizeof(float);

__device__ __forceinline__ uint32_t emit_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// kOpt (the owner's optimizer step instead of the bulk store): one buffer,
// 4 CTAs per SM, so more parameter / state loads are in flight.
// Word tiles are claimed one at a time from a counter (qcount[6]) instead
// of a static per-CTA range: a persistent store stream with a fixed share per
// CTA ends with the slowest SM (1 GB: 6.3 TB/s static vs 7.4 TB/s claimed,
// tools/micro/write_pattern.cu). The next tile is claimed while the current
// one is stored, and its bounds and first two entry windows are loaded one
// chunk later, so a tile switch exposes no load latency.
template <bool kOpt>
__global__ void __launch_bounds__(256, kOpt ? 4 : 1) k_emit(DecodeWork w, const OptEpilogue* __restrict__ opt) {
  extern __shared__ __align__(128) float ebuf[];  // [2][kEmitChunk] ([1] with kOpt)
  __shared__ uint32_t s_claim;
  const uint32_t T = uint32_t(w.total_word_tiles);
  const uint32_t total = w.qcount[5];
  uint32_t n_chunks = 0;  // chunks stored by this CTA (ring position)
  auto tile_end = [&](uint32_t t) {
    uint32_t le = t + 1 < T ? __ldg(w.tile_base + t + 1) : total;
    return le < total ? le : total;
  };
  // entry window at list index base (thread t: entry base + t), bounded by lend
  auto load_win = [&](uint32_t base, uint32_t lend, uint32_t& p, float& v) {
    const uint32_t i = base + threadIdx.x;
    p = 0xFFFFFFFFu;
    v = 0.0f;
    if (i < lend) {
      p = __ldcs(w.plist + i);
      v = __ldcs(w.val + i);
    }
  };
  if (threadIdx.x == 0) s_claim = atomicAdd(&w.qcount[6], 1u);
  __syncthreads();
  uint32_t wt = s_claim;
  uint32_t lbeg = 0, le = 0, wp = 0, np = 0;
  float wv = 0.0f, nv = 0.0f;
  if (wt < T) {
    lbeg = __ldg(w.tile_base + wt);
    le = tile_end(wt);
    load_win(lbeg, le, wp, wv);
    load_win(lbeg + blockDim.x, le, np, nv);
  }
  while (wt < T) {
    __syncthreads();  // every thread has read s_claim
    if (threadIdx.x == 0) s_claim = atomicAdd(&w.qcount[6], 1u);  // the next tile, read after the first chunk's barrier
    const DecItem& e = w.items[find_word_item(w.items, w.n_items, wt)];
    const uint64_t P = (e.flags & kWidth4) ? 8u : 32u;
    const uint64_t wbase = uint64_t(wt - e.word_tile_begin) * kWordTile;
    const uint64_t p0 = wbase * P;
    const uint64_t p1 = min(uint64_t(e.n), (wbase + kWordTile) * P);
    uint32_t wb = lbeg;  // first entry of the current window
    uint32_t cons = 0;   // entries of the current window already placed
    uint32_t nt = T, nlb = 0, nle = 0;  // the next tile and its list range
    uint32_t fp = 0xFFFFFFFFu, gp = 0xFFFFFFFFu;  // its first two windows
    float fv = 0.0f, gv = 0.0f;
    bool next_loaded = false;
    uint32_t k = 0;  // chunk of this tile
    for (uint64_t c0 = p0; c0 < p1; c0 += kEmitChunk, ++n_chunks, ++k) {
      const uint32_t clen = uint32_t(p1 - c0 < kEmitChunk ? p1 - c0 : kEmitChunk);
      float* buf = kOpt ? ebuf : ebuf + (n_chunks & 1u) * kEmitChunk;
      if (kOpt && n_chunks) __syncthreads();  // every thread is done reading the previous chunk
      if (!kOpt && n_chunks >= 2) {  // the store issued from this buffer two chunks ago has read it
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
      }
      float4* b4 = reinterpret_cast<float4*>(buf);
      for (uint32_t q = threadIdx.x; q < kEmitChunk / 4; q += blockDim.x) b4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncthreads();
      if (k == 0) {  // the claim is visible: its list range in flight during this chunk
        nt = s_claim;
        if (nt < T) {
          nlb = __ldg(w.tile_base + nt);
          nle = tile_end(nt);
        }
      } else if (!next_loaded && nt < T) {  // bounds arrived: the next tile's first windows
        load_win(nlb, nle, fp, fv);
        load_win(nlb + blockDim.x, nle, gp, gv);
        next_loaded = true;
      }
      // this chunk's entries: the window's unplaced entries below c0 + clen
      // (list index < le: the tile's own entries)
      for (;;) {
        const uint32_t i = wb + threadIdx.x;
        const bool in = threadIdx.x >= cons && i < le && uint64_t(wp) < c0 + clen;
        if (in) buf[wp - c0] = wv;
        cons += __syncthreads_count(in);
        const uint32_t rest = min(wb + blockDim.x, le);
        if (wb + cons < rest) break;          // stopped inside the window: chunk done
        if (wb + blockDim.x > le) break;      // the tile's entries end inside the window
        wb += blockDim.x;                      // window used up: advance, prefetch the next
        cons = 0;
        wp = np;
        wv = nv;
        load_win(wb + blockDim.x, le, np, nv);
      }
      float* dst = e.out + c0;
      const uint32_t bytes = (clen * 4u) & ~15u;
      if (kOpt) {  // owner-side optimizer step on the chunk (no bulk store)
        const OptEpilogue o = *opt;
        if (o.kind == 1) opt_range<true, false>(o, dst, buf, clen);
        else opt_range<false, false>(o, dst, buf, clen);
      } else if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && bytes) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                       "r"(emit_smem_u32(buf)), "r"(bytes)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        for (uint32_t q = bytes / 4u + threadIdx.x; q < clen; q += blockDim.x) dst[q] = buf[q];
      } else {  // unaligned output: plain coalesced stores
        for (uint32_t q = threadIdx.x; q < clen; q += blockDim.x) dst[q] = buf[q];
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // keep the ring count
      }
    }
    if (k == 0) {  // no chunk (cannot happen for a listed tile): take the claim anyway
      __syncthreads();
      nt = s_claim;
      if (nt < T) {
        nlb = __ldg(w.tile_base + nt);
        nle = tile_end(nt);
      }
    }
    if (nt < T && !next_loaded) {  // a one-chunk tile: load now
      load_win(nlb, nle, fp, fv);
      load_win(nlb + blockDim.x, nle, gp, gv);
    }
    wt = nt;
    lbeg = nlb;
    le = nle;
    wp = fp;
    wv = fv;
    np = gp;
    nv = gv;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  span_end(w.span);
}

// ------------------------------------------------------------------ round 0 + emit
// Counter mode without an owner step: round 0 and the dense emit in ONE pass
// over the word tiles, so round 0's random probes hide under the emit's
// 4 B/position store stream instead of running as their own latency-bound
// kernel. Per word tile (all of one item):
//   (A) every listed entry probes its k byte counters and peels from its
//       lowest singleton row (the reference's ascending seed order,
//       decode.cpp:96-99) - value = sign * residual (decode.cpp:110-111),
//       staged in shared memory; entries sharing a bucket join the compact
//       subtraction list (pinfo), unresolved ones the ulist (their buckets
//       marked and their state cleared for k_r0_subtract_cnt);
//   (B) the tile's chunks are zero-filled (decode.cpp:61-64), take the staged
//       values and leave by TMA bulk store (the k_emit ring).
// Entries round 0 leaves unresolved stay zero here: k_final_fix writes them
// after the frontier rounds and the median estimate.
constexpr uint32_t kR0EmitCap = 1024;  // staged values per tile (beyond: through val[])
constexpr uint32_t kR0EStage = 512;    // subtraction / unresolved list staging per CTA (3 CTAs per SM)
constexpr size_t kR0EmitSmem = 2 * kEmitChunk * sizeof(float) + kR0EmitCap * sizeof(float);

__global__ void __launch_bounds__(256, 3) k_r0_emit(DecodeWork w, const HashParams hp) {
  extern __shared__ __align__(128) float ebuf[];  // [2][kEmitChunk] ring, then [kR0EmitCap] staged values
  float* s_val = ebuf + 2 * kEmitChunk;
  __shared__ uint32_t s_q[kR0EStage], s_u[kR0EStage];
  __shared__ uint32_t s_n[2], s_un[2], s_base;
  if (threadIdx.x == 0) {
    s_n[0] = s_un[0] = 0;
    s_n[1] = s_un[1] = kR0EStage;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t total = ldcg(&w.qcount[5]);
  const uint32_t T = uint32_t(w.total_word_tiles);
  uint32_t t0, t1;
  cta_tiles(w.total_word_tiles, t0, t1);
  uint32_t n_chunks = 0, won = 0;
  uint32_t it = t0 < t1 ? find_word_item(w.items, w.n_items, t0) : 0u;
  for (uint32_t wt = t0; wt < t1; ++wt) {
    while (it + 1 < w.n_items && w.items[it + 1].word_tile_begin <= wt) ++it;
    const DecItem& e = w.items[it];
    const uint32_t L0 = min(__ldg(w.tile_base + wt), total);
    const uint32_t L1 = wt + 1 < T ? min(__ldg(w.tile_base + wt + 1), total) : total;
    // (A) round 0 over the tile's entries, warps on 32-aligned groups (one
    // recovered-bit word each; words at tile edges are shared: red.or)
    for (uint32_t g0 = (L0 & ~31u) + (threadIdx.x & ~31u); g0 < L1; g0 += blockDim.x) {
      const uint32_t i = g0 + lane;
      const bool act = i >= L0 && i < L1;
      bool peeled = false, sub = false, unres = false;
      if (act) {
        const uint32_t p = __ldcs(w.plist + i);
        uint64_t ls[kMaxRows];
        uint32_t c[kMaxRows];
#pragma unroll
        for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r)
          if (r < hp.rows) {  // every row's probe in flight before any is inspected
            ls[r] = uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m, e.mmul);
            const uint64_t sl = e.slot_base + ls[r];
            c[r] = cnt_get(w, sl);
          }
        int best = -1;
        uint32_t shared = 0;
#pragma unroll
        for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) {
          if (r >= hp.rows) continue;
          shared |= uint32_t(c[r] >= 2u) << r;
          if (best < 0 && c[r] == 1u) best = int(r);
        }
        float v = 0.0f;
        if (best >= 0) {
          uint64_t local = 0;
          float sg = 0.0f;
#pragma unroll
          for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r)
            if (int(r) == best) {
              local = ls[r];
              sg = dev_sign(hp.row[r], p);
            }
          v = canonical(sg * ldcg(e.sketch + local));
          peeled = true;
          sub = shared != 0u;
          if (sub) w.pinfo[i] = make_uint2(__float_as_uint(v), shared | 0x100u | (uint32_t(best) << 12));
          ++won;
        } else {  // unresolved after round 0: its buckets get a (count, index sum) state
          unres = true;
#pragma unroll
          for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r)
            if (r < hp.rows) {
              const uint64_t sl = e.slot_base + ls[r];
              red_or_u32(w.slot_mark + (sl >> 5), 1u << (sl & 31));
              w.slot_state[sl] = 0ull;
            }
        }
        if (i - L0 < kR0EmitCap) s_val[i - L0] = v;
        else if (peeled) w.val[i] = v;
      }
      const uint32_t m = __ballot_sync(kFull, peeled);
      if (lane == 0 && m) red_or_u32(w.bitmap + (g0 >> 5), m);
      stage_push<uint32_t, kR0EStage>(sub, i, s_q, s_n, w.r0_list, &w.qcount[13], lane);
      stage_push<uint32_t, kR0EStage>(unres, i, s_u, s_un, w.ulist, &w.qcount[14], lane);
    }
    __syncthreads();  // staged values visible to the whole CTA
    // (B) the tile's chunks
    const uint64_t P = (e.flags & kWidth4) ? 8u : 32u;
    const uint64_t wbase = uint64_t(wt - e.word_tile_begin) * kWordTile;
    const uint64_t p0 = wbase * P;
    const uint64_t p1 = min(uint64_t(e.n), (wbase + kWordTile) * P);
    uint32_t cur = L0;
    for (uint64_t c0 = p0; c0 < p1; c0 += kEmitChunk, ++n_chunks) {
      const uint32_t clen = uint32_t(p1 - c0 < kEmitChunk ? p1 - c0 : kEmitChunk);
      float* buf = ebuf + (n_chunks & 1u) * kEmitChunk;
      if (n_chunks >= 2) {  // the store issued from this buffer two chunks ago has read it
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
      }
      float4* b4 = reinterpret_cast<float4*>(buf);
      for (uint32_t q = threadIdx.x; q < kEmitChunk / 4; q += blockDim.x) b4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      __syncthreads();
      for (;;) {
        const uint32_t i = cur + threadIdx.x;
        uint32_t p = 0xFFFFFFFFu;
        if (i < L1) p = __ldcg(w.plist + i);  // just read by (A): an L2 hit
        const bool in = uint64_t(p) < c0 + clen;
        if (in) buf[p - c0] = i - L0 < kR0EmitCap ? s_val[i - L0] : __ldcg(w.val + i);
        const uint32_t cnt = __syncthreads_count(in);
        cur += cnt;
        if (cnt < blockDim.x) break;
      }
      float* dst = e.out + c0;
      const uint32_t bytes = (clen * 4u) & ~15u;
      if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && bytes) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                       "r"(emit_smem_u32(buf)), "r"(bytes)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        for (uint32_t q = bytes / 4u + threadIdx.x; q < clen; q += blockDim.x) dst[q] = buf[q];
      } else {  // unaligned output: plain coalesced stores
        for (uint32_t q = threadIdx.x; q < clen; q += blockDim.x) dst[q] = buf[q];
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // keep the ring count
      }
    }
    __syncthreads();  // (B) is done reading s_val before the next tile's (A)
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  won = warp_sum32(won);
  if (lane == 0 && won) atomicAdd(&w.qcount[kPeeledWord], won);
  stage_flush<uint32_t, kR0EStage>(s_q, s_n, &s_base, w.r0_list, &w.qcount[13]);
  stage_flush<uint32_t, kR0EStage>(s_u, s_un, &s_base, w.ulist, &w.qcount[14]);
}

// Counter mode's last step after k_r0_emit: each entry round 0 left
// unresolved gets its final value into the dense output - the frontier
// rounds' value, or the median-of-rows estimate (decode.cpp:130-138, :43-47)
// where the peel stalled.
__global__ void __launch_bounds__(256) k_final_fix(DecodeWork w, const HashParams hp) {
  const uint32_t nu = ldcg(&w.qcount[14]);
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x - lane; base < nu; base += stride) {
    const uint64_t j = base + lane;
    uint32_t it = 0xFFFFFFFFu, p = 0;
    bool todo = false;
    if (j < nu) {
      const uint32_t i = ldcg(w.ulist + j);
      p = __ldg(w.plist + i);
      it = item_of(w, i);
      const DecItem& e = w.items[it];
      float v;
      if ((ldcg(w.bitmap + (i >> 5)) >> (i & 31)) & 1u) {
        v = ldcg(w.val + i);
      } else {
        todo = true;
        float est[kMaxRows];
#pragma unroll
        for (uint32_t r = 0; r < kMaxRows; ++r) {
          if (r >= hp.rows) break;
          est[r] = dev_sign(hp.row[r], p) * ldcg(e.sketch + uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m, e.mmul));
        }
        v = canonical(median_rows(est, hp.rows));
      }
      e.out[p] = v;
    }
    const uint32_t grp = __match_any_sync(kFull, todo ? it : 0xFFFFFFFFu);
    if (todo) {
      const uint32_t leader = __ffs(grp) - 1;
      uint32_t b0 = 0;
      if (lane == leader) b0 = atomicAdd(&w.stats[it].unresolved, uint32_t(__popc(grp)));
      b0 = __shfl_sync(grp, b0, leader);
      if (w.unresolved) w.unresolved[w.items[it].list_off + b0 + __popc(grp & ((1u << lane) - 1u))] = p;
    }
  }
  span_end(w.span);
}

// ------------------------------------------------------------------ helpers
__global__ void k_presence_to_bitmap(const uint32_t* __restrict__ presence, uint32_t count,
                                     uint32_t n, uint32_t* bitmap, uint32_t* err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const uint32_t p = presence[i];
    if (p >= n) {
      atomicOr(err, 1u);
      continue;
    }
    const uint32_t bit = 1u << (p & 31);
    if (atomicOr(bitmap + (p >> 5), bit) & bit) atomicOr(err, 2u);
  }
}

__global__ void k_estimate_targets(const uint32_t* __restrict__ targets, uint32_t nt,
                                   const uint32_t* __restrict__ bitmap, uint32_t n, uint32_t m,
                                   const float* __restrict__ sketch, const HashParams hp,
                                   float* __restrict__ out, uint32_t* err) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nt; i += gridDim.x * blockDim.x) {
    const uint32_t t = targets[i];
    if (t >= n || !(bitmap[t >> 5] >> (t & 31) & 1u)) {
      atomicOr(err, 4u);
      continue;
    }
    float est[kMaxRows];
#pragma unroll
    for (uint32_t r = 0; r < kMaxRows; ++r) {
      if (r >= hp.rows) break;
      est[r] = dev_sign(hp.row[r], t) * sketch[uint64_t(r) * m + dev_bucket(hp.row[r], t, m)];
    }
    out[i] = canonical(median_rows(est, hp.rows));
  }
}

__global__ void k_word_counts(const uint32_t* __restrict__ words, uint32_t n, uint32_t n_words,
                              bool w4, uint32_t* __restrict__ counts) {
  for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < n_words; wi += gridDim.x * blockDim.x) {
    counts[wi] = __popc(present_bits(words[wi], w4, wi, n));
  }
}

__global__ void k_word_positions(const uint32_t* __restrict__ words, uint32_t n, uint32_t n_words,
                                 bool w4, const uint32_t* __restrict__ offsets,
                                 uint32_t* __restrict__ out, uint32_t* count_dev) {
  for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < n_words; wi += gridDim.x * blockDim.x) {
    uint32_t bits = present_bits(words[wi], w4, wi, n);
    const uint32_t P = w4 ? 8u : 32u;
    uint32_t o = offsets[wi];
    const uint32_t c = __popc(bits);
    while (bits) {
      const uint32_t b = __ffs(bits) - 1;
      bits &= bits - 1;
      out[o++] = wi * P + (w4 ? b / 4 : b);
    }
    if (wi == n_words - 1) *count_dev = offsets[wi] + c;
  }
}

int grid_for(uint64_t n, int threads) {
  const uint64_t b = (n + threads - 1) / threads;
  return int(b < 2048 ? (b ? b : 1) : 2048);
}

// count -> scan -> list + bucket state (bucket state zeroed in between: it is
// first touched by k_list). Returns the grid used for the word-tile passes.
int build_passes(const DevInfo& di, const DecodeWork& w, const HashParams& hp, cudaStream_t stream) {
  if (w.cnt8) {  // counter mode: count, scan, write (no look-back)
    // count and write on the same grid (the same tile range per CTA): the
    // write pass turns the per-CTA counts into list offsets itself
    static const uint64_t list_ctas = std::getenv("TAGC_LIST_CTAS") ? std::strtoull(std::getenv("TAGC_LIST_CTAS"), nullptr, 10) : 0;
    const uint64_t gc = std::min<uint64_t>(std::max<uint64_t>(w.total_word_tiles, 1),
                                           std::min<uint64_t>(list_ctas ? list_ctas : uint64_t(di.sms) * 4, kListMaxCtas));
    k_list_count<<<int(w.list_split * gc), 256, 0, stream>>>(w);
    launch_pdl(k_list_write, dim3(unsigned(gc)), dim3(256), 0, stream, w, hp);  // counters were zeroed by the caller
    return int(gc);
  }
  const uint64_t g64 = std::min<uint64_t>(std::max<uint64_t>(w.total_word_tiles, 1), uint64_t(di.sms) * 4);
  const int g = int(g64);
  k_list<<<g, 256, 0, stream>>>(w, hp);  // bucket and tile state were zeroed by the caller
  return g;
}

}  // namespace

int launch_decode(const DevInfo& di, const DecodeWork& w, const HashParams& hp,
                  cudaStream_t stream, bool fused_emit, cudaEvent_t sketch_ready) {
  if (w.n_items == 0) {
    if (sketch_ready) cudaStreamWaitEvent(stream, sketch_ready, 0);
    return 0;
  }
  int per_sm = 0;
  build_passes(di, w, hp, stream);
  if (sketch_ready) cudaStreamWaitEvent(stream, sketch_ready, 0);
  const int list_launches = w.cnt8 ? 2 : 1;
  if (fused_emit) {
    const uint64_t ge = std::min<uint64_t>(std::max<uint64_t>(w.total_word_tiles, 1), uint64_t(di.sms) * 3);
    cudaFuncSetAttribute((const void*)k_r0_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kR0EmitSmem));
    k_r0_emit<<<int(ge), 256, kR0EmitSmem, stream>>>(w, hp);
  } else if (hp.rows == 3) {
    // TAGC_R0_GRID=0: one pass (ceil(list bound / 512) CTAs), else CTAs per SM
    static const int r0_grid = std::getenv("TAGC_R0_GRID") ? std::atoi(std::getenv("TAGC_R0_GRID")) : 8;
    const uint64_t g0 = r0_grid > 0 ? uint64_t(di.sms) * r0_grid
                                    : std::max<uint64_t>(1, (w.list_cap + 511) / 512);
    k_r0_phase1_k<3, 2><<<int(std::min<uint64_t>(g0, 1u << 20)), 256, 0, stream>>>(w, hp);
  } else {
    k_r0_phase1<<<di.sms * 8, 256, 0, stream>>>(w, hp);
  }
  if (w.cnt8) launch_pdl(k_r0_subtract_cnt, dim3(di.sms * 8), dim3(256), 0, stream, w, hp);
  else k_r0_subtract<<<di.sms * 8, 256, 0, stream>>>(w, hp);

  const void* peel = hp.rows == 3 ? (const void*)k_peel<3> : (const void*)k_peel<kMaxRows>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, peel, 256, 0);
  const int pg = coop_grid(di, std::max(per_sm, 1));
  DecodeWork wc = w;
  HashParams hc = hp;
  void* args[] = {&wc, &hc};
  cudaLaunchCooperativeKernel(peel, dim3(pg), dim3(256), args, 0, stream);

  if (fused_emit) {  // the dense output is complete after this one
    k_final_fix<<<di.sms * 4, 256, 0, stream>>>(w, hp);
    return list_launches + 4;  // list, round 0 + emit, subtraction, peel, final
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_final, 256, 0);
  launch_pdl(k_final, dim3(std::max(per_sm, 1) * di.sms), dim3(256), 0, stream, w, hp);
  return list_launches + 4;  // list, round 0 (2), peel, final
}

int ordered_loop_grid(const DevInfo& di) {  // the larger of the two instantiations' grids (per-CTA scratch)
  int a = 0, b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, (const void*)k_ord_loop<3>, 256, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, (const void*)k_ord_loop<kMaxRows>, 256, 0);
  return std::max(std::max(a, b), 1) * di.sms;
}

int launch_decode_ordered(const DevInfo& di, const DecodeWork& w, const HashParams& hp, const OrdState& o,
                          cudaStream_t stream, cudaEvent_t sketch_ready) {
  if (w.n_items == 0) {
    if (sketch_ready) cudaStreamWaitEvent(stream, sketch_ready, 0);
    return 0;
  }
  build_passes(di, w, hp, stream);
  if (sketch_ready) cudaStreamWaitEvent(stream, sketch_ready, 0);
  const int grid = di.sms * 4;
  if (hp.rows == 3) k_r0_phase1_k<3, 2><<<grid, 256, 0, stream>>>(w, hp);
  else k_r0_phase1<<<grid, 256, 0, stream>>>(w, hp);
  DecodeWork wa = w;
  HashParams ha = hp;
  OrdState oa = o;
  void* args[] = {&wa, &ha, &oa};
  const void* loop = hp.rows == 3 ? (const void*)k_ord_loop<3> : (const void*)k_ord_loop<kMaxRows>;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, loop, 256, 0);
  cudaLaunchCooperativeKernel(loop, dim3(std::max(per_sm, 1) * di.sms), dim3(256), args, 0, stream);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_final, 256, 0);
  launch_pdl(k_final, dim3(std::max(per_sm, 1) * di.sms), dim3(256), 0, stream, w, hp);
  return (w.cnt8 ? 2 : 1) + 3;  // build, round 0, loop, estimate
}

int launch_decode_emit(const DevInfo& di, const DecodeWork& w, cudaStream_t stream, const OptEpilogue* dev_opt) {
  if (w.n_items == 0) return 0;
  const uint64_t g = std::min<uint64_t>(std::max<uint64_t>(w.total_word_tiles, 1), uint64_t(di.sms) * 3);
  if (dev_opt) {
    const uint64_t go = std::min<uint64_t>(std::max<uint64_t>(w.total_word_tiles, 1), uint64_t(di.sms) * 4);
    k_emit<true><<<int(go), 256, kEmitSmem / 2, stream>>>(w, dev_opt);
  } else {
    cudaFuncSetAttribute((const void*)k_emit<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kEmitSmem));
    k_emit<false><<<int(g), 256, kEmitSmem, stream>>>(w, nullptr);
  }
  return 1;
}

int launch_presence_to_bitmap(const uint32_t* presence, uint32_t count, uint32_t n,
                              uint32_t* bitmap, uint32_t* err, cudaStream_t stream) {
  if (!count) return 0;
  k_presence_to_bitmap<<<grid_for(count, 256), 256, 0, stream>>>(presence, count, n, bitmap, err);
  return 1;
}

int launch_estimate_targets(const uint32_t* targets, uint32_t n_targets, const uint32_t* bitmap,
                            uint32_t n, uint32_t m, const float* sketch, const HashParams& hp,
                            float* out, uint32_t* err, cudaStream_t stream) {
  if (!n_targets) return 0;
  k_estimate_targets<<<grid_for(n_targets, 256), 256, 0, stream>>>(targets, n_targets, bitmap, n, m,
                                                                   sketch, hp, out, err);
  return 1;
}

size_t index_presence_scratch_bytes(uint32_t n, uint32_t width) {
  const uint32_t nw = uint32_t((uint64_t(n) * width + 31) / 32);
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, (uint32_t*)nullptr, (uint32_t*)nullptr, int(nw));
  return 2 * size_t(nw) * 4 + temp + 256;
}

int launch_index_presence(const uint32_t* words, uint32_t n, uint32_t width, uint32_t* positions,
                          uint32_t* count_dev, void* scratch, size_t scratch_bytes,
                          cudaStream_t stream) {
  const uint32_t nw = uint32_t((uint64_t(n) * width + 31) / 32);
  uint32_t* counts = static_cast<uint32_t*>(scratch);
  uint32_t* offsets = counts + nw;
  void* temp = reinterpret_cast<char*>(scratch) + ((2 * size_t(nw) * 4 + 255) / 256) * 256;
  size_t temp_bytes = scratch_bytes - ((2 * size_t(nw) * 4 + 255) / 256) * 256;
  const bool w4 = width == 4;
  k_word_counts<<<grid_for(nw, 256), 256, 0, stream>>>(words, n, nw, w4, counts);
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offsets, int(nw), stream);
  k_word_positions<<<grid_for(nw, 256), 256, 0, stream>>>(words, n, nw, w4, offsets, positions,
                                                          count_dev);
  return 3;
}

size_t sort_scratch_bytes(uint32_t count) {
  size_t temp = 0;
  cub::DoubleBuffer<uint32_t> db(nullptr, nullptr);
  cub::DeviceRadixSort::SortKeys(nullptr, temp, db, int(count));
  return temp;
}

int launch_sort_u32(uint32_t* keys, uint32_t* keys_alt, uint32_t count, void* scratch,
                    size_t scratch_bytes, cudaStream_t stream) {
  if (count < 2) return 0;
  cub::DoubleBuffer<uint32_t> db(keys, keys_alt);
  cub::DeviceRadixSort::SortKeys(scratch, scratch_bytes, db, int(count), 0, 32, stream);
  if (db.Current() != keys)
    cudaMemcpyAsync(keys, db.Current(), size_t(count) * 4, cudaMemcpyDeviceToDevice, stream);
  return 1;
}

// Loads every kernel of this file now (see preload_all_kernels).
void preload_decode_kernels() {
  const void* fns[] = {(const void*)k_r0_emit, (const void*)k_final_fix, (const void*)k_emit<false>, (const void*)k_emit<true>, (const void*)k_estimate_targets, (const void*)k_final, (const void*)k_list, (const void*)k_list_count, (const void*)k_list_write, (const void*)k_ord_loop<3>, (const void*)k_ord_loop<kMaxRows>, (const void*)k_peel<3>, (const void*)k_peel<kMaxRows>, (const void*)k_presence_to_bitmap, (const void*)k_r0_phase1, (const void*)k_r0_phase1_k<3, 2>, (const void*)k_r0_subtract, (const void*)k_r0_subtract_cnt, (const void*)k_word_counts, (const void*)k_word_positions};
  cudaFuncAttributes a;
  for (const void* f : fns) cudaFuncGetAttributes(&a, f);
  cudaGetLastError();
}

}  // namespace tagc_b200
