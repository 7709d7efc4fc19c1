// decode.cu — sm_100a owner-side decode (reference decode.cpp:24-140):
//   build    : zero-fill the dense shard, walk the merged index words and
//              accumulate per-bucket (count, key_sum) state in one 64-bit word
//              per bucket, collecting the presence list and first-touch
//              singleton candidates;
//   peel     : synchronous peeling rounds in ONE cooperative persistent kernel
//              (phase 1 claims singleton buckets, phase 2 subtracts the peeled
//              contributions from all k rows); when the frontier is small a
//              single CTA finishes the remaining rounds with block barriers;
//   estimate : median-of-rows on the residual sketch for every present
//              position the peel could not resolve.
//
// Bucket state: (count << 40) | sum(position) in one u64, so building and
// peeling cost one 64-bit L2 atomic per (position, row). count == 1 makes the
// low 40 bits equal to the single remaining position (decode.cpp:104-106 uses
// a u64 key_sum for the same reason). The sum field cannot carry for any
// bucket holding fewer than 2^40 / n positions; the build kernel flags that
// overflow (never reached at ratio <= 10) and the engine reports it.
//
// Parity: the recovered/unresolved position sets are those of the reference's
// FIFO peel (the peelable set is the complement of the 2-core, independent of
// order); values match within fp32 reassociation tolerance and bit-exactly on
// integer-valued inputs.
#include <cooperative_groups.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "kernels.hpp"

namespace cg = cooperative_groups;

namespace tagc_b200 {
namespace {

constexpr uint32_t kFull = 0xFFFFFFFFu;
// Bucket state word: (sum of positions mod 2^40) << 24 | count (24 bits).
// Adding (p << 24) | 1 never carries out of the count field unless one bucket
// holds 2^24 positions; the sum wraps harmlessly at the top, and when
// count == 1 its low 32 bits are the remaining position exactly.
constexpr unsigned long long kCountMask = (1ull << 24) - 1ull;
__device__ __forceinline__ unsigned long long st_add(uint32_t p) { return (uint64_t(p) << 24) | 1ull; }
__device__ __forceinline__ unsigned long long st_sub(uint32_t p) { return ~st_add(p) + 1ull; }
__device__ __forceinline__ uint32_t st_count(unsigned long long s) { return uint32_t(s & kCountMask); }
__device__ __forceinline__ uint32_t st_pos(unsigned long long s) { return uint32_t(s >> 24); }
constexpr uint32_t kWinner = 0x80000000u;
constexpr uint32_t kWordTile = kDecWordTile;
constexpr uint32_t kStage = 4096;
constexpr uint32_t kTail = 512;  // frontier size at which one CTA finishes

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

__device__ __forceinline__ uint32_t find_slot_item(const DecItem* items, uint32_t n, uint64_t s) {
  uint32_t lo = 0, hi = n - 1;
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (items[mid].slot_base <= s) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Presence bits of one merged word: field != 0 (index.cpp:43-57). Width 4:
// bit 4j set iff nibble j nonzero; width 1: the word itself.
__device__ __forceinline__ uint32_t present_bits(uint32_t x, bool w4) {
  return w4 ? ((x | x >> 1 | x >> 2 | x >> 3) & 0x11111111u) : x;
}

__device__ __forceinline__ float canonical(float v) { return v == 0.0f ? 0.0f : v; }

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
// Contiguous range of word tiles per CTA (kWordTile words per tile, 4 words
// per thread), bucket state updated with fire-and-forget 64-bit reductions.
__global__ void __launch_bounds__(256) k_build(DecodeWork w, const HashParams hp) {
  span_begin(w.span);
  __shared__ uint32_t s_list[kStage];
  __shared__ uint32_t s_nl, s_bl;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t T = uint32_t(w.total_word_tiles), G = gridDim.x, b = blockIdx.x;
  const uint32_t chunk = T / G, extra = T % G;
  const uint32_t t0 = b * chunk + min(b, extra), t1 = t0 + chunk + (b < extra ? 1u : 0u);
  if (t0 >= t1) return;
  if (threadIdx.x == 0) s_nl = 0;
  __syncthreads();
  uint32_t it = find_word_item(w.items, w.n_items, t0);
  for (uint32_t wt = t0; wt < t1; ++wt) {
    while (it + 1 < w.n_items && w.items[it + 1].word_tile_begin <= wt) ++it;
    const DecItem e = w.items[it];
    const bool w4 = (e.flags & kWidth4) != 0;
    const uint32_t P = w4 ? 8u : 32u;
    const uint32_t wbase = uint32_t(wt - e.word_tile_begin) * kWordTile;
    // zero-fill the tile's positions (coalesced 4-byte stores)
    {
      const uint64_t p0 = uint64_t(wbase) * P;
      const uint64_t p1 = min(uint64_t(e.n), p0 + uint64_t(kWordTile) * P);
      for (uint64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) e.out[p] = 0.0f;
    }
    uint32_t bits[kWordTile / 256];
#pragma unroll
    for (uint32_t k = 0; k < kWordTile / 256; ++k) {
      const uint32_t wi = wbase + k * 256 + threadIdx.x;
      uint32_t x = 0;
      if (wi < e.n_words) {
        x = present_bits(__ldg(e.words + wi), w4);
        const uint64_t first = uint64_t(wi) * P;
        const uint64_t left = e.n > first ? e.n - first : 0;
        if (w4) {
          if (left < 8) x &= (1u << (4 * left)) - 1u;
        } else if (left < 32) {
          x &= (1u << left) - 1u;
        }
      }
      bits[k] = x;
    }
#pragma unroll
    for (uint32_t k = 0; k < kWordTile / 256; ++k) {
      const uint32_t wi = wbase + k * 256 + threadIdx.x;
      uint32_t x = bits[k];
      while (x) {
        const uint32_t bb = __ffs(x) - 1;
        x &= x - 1;
        const uint32_t p = wi * P + (w4 ? bb / 4 : bb);
        const uint32_t li = atomicAdd(&s_nl, 1u);
        if (li < kStage) {
          s_list[li] = p;
        } else {
          atomicAdd(&w.stats[it].presence, 1u);
          const uint32_t gi = atomicAdd(&w.qcount[5], 1u);
          w.plist[gi] = p;
          w.pitem[gi] = it;
        }
        _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
          const uint64_t slot = e.slot_base + uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m);
          atomicAdd(w.slot_state + slot, st_add(p));  // result unused: RED.ADD.64
        }
      }
    }
    __syncthreads();
    const bool item_ends = wt + 1 == t1 || (it + 1 < w.n_items && w.items[it + 1].word_tile_begin <= wt + 1);
    if (item_ends || s_nl >= kStage / 2) {  // flush the staged presence list
      if (threadIdx.x == 0) {
        const uint32_t nl = min(s_nl, kStage);
        if (nl) atomicAdd(&w.stats[it].presence, nl);
        s_bl = nl ? atomicAdd(&w.qcount[5], nl) : 0;
        s_nl = nl;
      }
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < s_nl; i += blockDim.x) {
        w.plist[s_bl + i] = s_list[i];
        w.pitem[s_bl + i] = it;
      }
      __syncthreads();
      if (threadIdx.x == 0) s_nl = 0;
      __syncthreads();
    }
  }
  (void)lane;
}

// ------------------------------------------------------------------ peel
// Next-frontier pushes are staged in shared memory per CTA (warp-aggregated)
// and flushed with one global atomic per CTA per phase; a single queue
// counter hit by every warp serialises at one L2 slice otherwise.
constexpr uint32_t kPushStage = 8192;

__device__ __forceinline__ void push_slot(bool push, uint32_t s, uint32_t* s_q, uint32_t* s_nq,
                                          uint32_t* nq, uint32_t* ncount, uint32_t lane) {
  const uint32_t mask = __ballot_sync(kFull, push);
  if (!mask) return;
  const uint32_t leader = __ffs(mask) - 1, cnt = __popc(mask);
  uint32_t b = 0, direct = 0;
  if (lane == leader) {
    b = atomicAdd(s_nq, cnt);
    if (b + cnt > kPushStage) {  // stage full: straight to the global frontier
      if (b < kPushStage) atomicMin(s_nq + 1, b);  // [b, stage) stays unwritten
      direct = 1;
      b = atomicAdd(ncount, cnt);
    }
  }
  b = __shfl_sync(kFull, b, leader);
  direct = __shfl_sync(kFull, direct, leader);
  if (push) {
    const uint32_t idx = b + __popc(mask & ((1u << lane) - 1u));
    if (direct) nq[idx] = s;
    else s_q[idx] = s;
  }
}

__device__ __forceinline__ void flush_pushes(uint32_t* s_q, uint32_t* s_nq, uint32_t* s_base,
                                             uint32_t* nq, uint32_t* ncount) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t n = min(min(s_nq[0], kPushStage), s_nq[1]);
    *s_base = n ? atomicAdd(ncount, n) : 0u;
    s_nq[0] = n;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < s_nq[0]; i += blockDim.x) nq[*s_base + i] = s_q[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    s_nq[0] = 0;
    s_nq[1] = kPushStage;
  }
  __syncthreads();
}

// Phase 1: claim singleton buckets of the current frontier.
__device__ __forceinline__ void peel_phase1(const DecodeWork& w, const HashParams& hp,
                                            uint32_t cur, uint32_t qlen, uint64_t start,
                                            uint64_t stride) {
  uint32_t* q = w.queue[cur];
  for (uint64_t i = start; i < qlen; i += stride) {
    const uint32_t slot = ldcg(q + i);
    const unsigned long long st = ldcg(w.slot_state + slot);
    if (st_count(st) != 1u) continue;  // stale (decode.cpp:106)
    const uint32_t p = st_pos(st);
    const uint32_t it = find_slot_item(w.items, w.n_items, slot);
    const DecItem e = w.items[it];
    const uint64_t local = slot - e.slot_base;
    const uint32_t row = uint32_t(local / e.m);
    const float v = canonical(dev_sign(row_coef(hp, row), p) * ldcg(e.sketch + local));  // :110-111
    uint32_t* word = w.bitmap + e.bitmap_off + (p >> 5);
    const uint32_t bit = 1u << (p & 31);
    if (atomicOr(word, bit) & bit) continue;  // p already claimed via another row
    __stcg(e.out + p, v);
    q[i] = slot | kWinner;
    atomicAdd(&w.qcount[4], 1u);
  }
}

// Phase 2: subtract each claimed position from all k rows (decode.cpp:115-121),
// pushing buckets whose count drops to one onto the next frontier.
__device__ __forceinline__ void peel_phase2(const DecodeWork& w, const HashParams& hp,
                                            uint32_t cur, uint32_t qlen, uint64_t start,
                                            uint64_t stride, uint32_t* s_q, uint32_t* s_nq,
                                            uint32_t* s_base) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* q = w.queue[cur];
  uint32_t* nq = w.queue[cur ^ 1];
  uint32_t* ncount = &w.qcount[cur ^ 1];
  // warp-uniform trip count so pushes can be warp-aggregated
  const uint64_t wstart = start - lane;
  for (uint64_t base = wstart; base < qlen; base += stride) {
    const uint64_t i = base + lane;
    uint32_t slot = 0, p = 0;
    float v = 0.0f;
    DecItem e{};
    bool win = false;
    if (i < qlen) {
      const uint32_t x = ldcg(q + i);
      if (x & kWinner) {
        win = true;
        slot = x & ~kWinner;
        p = st_pos(ldcg(w.slot_state + slot));
        const uint32_t it = find_slot_item(w.items, w.n_items, slot);
        e = w.items[it];
        v = ldcg(e.out + p);
      }
    }
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
      bool push = false;
      uint64_t s = 0;
      if (win) {
        const uint64_t local = uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m);
        s = e.slot_base + local;
        if (s != slot) {  // the winner's own bucket held only p: leave it
          atomicAdd(e.sketch + local, -(dev_sign(hp.row[r], p) * v));
          const unsigned long long old = atomicAdd(w.slot_state + s, st_sub(p));
          push = st_count(old) == 2u;
        }
      }
      push_slot(push, uint32_t(s), s_q, s_nq, nq, ncount, lane);
    }
  }
  flush_pushes(s_q, s_nq, s_base, nq, ncount);
}

// Round 0, position-centric: every present position inspects its k buckets
// at round start and peels from its first singleton row (lowest slot id, the
// reference's ascending seed order, decode.cpp:96-99).
__device__ __forceinline__ void round0_phase1(const DecodeWork& w, const HashParams& hp,
                                              uint64_t start, uint64_t stride) {
  uint32_t won = 0;
  const uint32_t total = ldcg(&w.qcount[5]);  // flat presence list (all items)
  for (uint64_t i = start; i < total; i += stride) {
    const uint32_t p = w.plist[i];
    const DecItem e = w.items[w.pitem[i]];
    uint64_t ls[kMaxRows];
    unsigned long long st[kMaxRows];
#pragma unroll
    for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) {
      if (r < hp.rows) {  // issue every row's load before inspecting any
        ls[r] = uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m);
        st[r] = ldcg(w.slot_state + e.slot_base + ls[r]);
      }
    }
    int best = -1;
    uint64_t local = 0;
    float sg = 0.0f;
    uint32_t shared = 0;  // rows whose bucket holds other positions too
#pragma unroll
    for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) {
      if (r >= hp.rows) continue;
      const uint32_t cnt = st_count(st[r]);
      shared |= uint32_t(cnt >= 2u) << r;
      if (best < 0 && cnt == 1u) {
        best = int(r);
        local = ls[r];
        sg = dev_sign(hp.row[r], p);
      }
    }
    if (best < 0) {
      w.pinfo[i] = make_uint2(0u, 0u);
      continue;
    }
    const float v = canonical(sg * ldcg(e.sketch + local));
    __stcg(e.out + p, v);
    atomicOr(w.bitmap + e.bitmap_off + (p >> 5), 1u << (p & 31));
    // phase 2 needs the value and only the rows shared with other positions
    w.pinfo[i] = make_uint2(__float_as_uint(v), shared | 0x100u | (uint32_t(best) << 12));
    ++won;
  }
  won = warp_sum32(won);
  if ((threadIdx.x & 31) == 0 && won) atomicAdd(&w.qcount[4], won);
}

// Round 0 subtraction for every position peeled in round0_phase1. Buckets
// that held only the peeled position are left alone: nothing else reads them
// (their count drops 1 -> 0 in the reference, decode.cpp:115-121).
__device__ __forceinline__ void round0_phase2(const DecodeWork& w, const HashParams& hp,
                                              uint64_t start, uint64_t stride, uint32_t* s_q,
                                              uint32_t* s_nq, uint32_t* s_base) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t* nq = w.queue[1];
  uint32_t* ncount = &w.qcount[1];
  const uint32_t total = ldcg(&w.qcount[5]);
  for (uint64_t base = start - lane; base < total; base += stride) {
    const uint64_t i = base + lane;
    uint32_t p = 0, rows = 0;
    float v = 0.0f;
    DecItem e{};
    if (i < total) {
      const uint2 info = w.pinfo[i];
      if (info.y & 0x100u) {
        rows = info.y & 0xFFu;
        v = __uint_as_float(info.x);
        p = w.plist[i];
        e = w.items[w.pitem[i]];
      }
    }
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
      bool push = false;
      uint64_t s = 0;
      if (rows >> r & 1u) {
        const uint64_t local = uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m);
        s = e.slot_base + local;
        atomicAdd(e.sketch + local, -(dev_sign(hp.row[r], p) * v));
        const unsigned long long old = atomicAdd(w.slot_state + s, st_sub(p));
        push = st_count(old) == 2u;
      }
      push_slot(push, uint32_t(s), s_q, s_nq, nq, ncount, lane);
    }
  }
  flush_pushes(s_q, s_nq, s_base, nq, ncount);
}

__global__ void __launch_bounds__(256) k_peel(DecodeWork w, const HashParams hp) {
  __shared__ uint32_t s_q[kPushStage];
  __shared__ uint32_t s_nq[2], s_base;  // [0] reserved, [1] end of the contiguous written prefix
  if (threadIdx.x == 0) {
    s_nq[0] = 0;
    s_nq[1] = kPushStage;
  }
  __syncthreads();
  cg::grid_group grid = cg::this_grid();
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gstride = uint64_t(gridDim.x) * blockDim.x;
  int mk = 0;
  PEEL_MARK(mk++);
  round0_phase1(w, hp, gtid, gstride);
  PEEL_MARK(mk++);
  grid.sync();
  PEEL_MARK(mk++);
  round0_phase2(w, hp, gtid, gstride, s_q, s_nq, &s_base);
  PEEL_MARK(mk++);
  if (gtid == 0) w.qcount[2] = 1;
  uint32_t cur = 1;
  for (;;) {
    grid.sync();
    PEEL_MARK(mk++);
    const uint32_t qlen = ldcg(&w.qcount[cur]);
    if (qlen == 0) return;
    if (qlen <= kTail) break;  // every CTA sees the same qlen
    peel_phase1(w, hp, cur, qlen, gtid, gstride);
    PEEL_MARK(mk++);
    if (gtid == 0) {
      w.qcount[cur ^ 1] = 0;
      w.qcount[2] += 1;
    }
    grid.sync();
    PEEL_MARK(mk++);
    peel_phase2(w, hp, cur, qlen, gtid, gstride, s_q, s_nq, &s_base);
    PEEL_MARK(mk++);
    cur ^= 1;
  }
  // tail: one CTA finishes with block barriers
  if (blockIdx.x != 0) return;
  for (;;) {
    __syncthreads();
    const uint32_t qlen = ldcg(&w.qcount[cur]);
    if (qlen == 0) return;
    peel_phase1(w, hp, cur, qlen, threadIdx.x, blockDim.x);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      w.qcount[cur ^ 1] = 0;
      w.qcount[3] += 1;
    }
    __threadfence();
    __syncthreads();
    peel_phase2(w, hp, cur, qlen, threadIdx.x, blockDim.x, s_q, s_nq, &s_base);
    __threadfence();
    PEEL_MARK(mk++);
    cur ^= 1;
  }
}

// ------------------------------------------------------------------ ordered peel
// FIFO-order emulation for indices that can hide mass (1-bit merge carries
// drop positions whose contributions stay in the sketch, so the reference's
// values depend on its peel order, decode.cpp:96-122). Generation 0 is the
// position-centric round above: every position peels from its lowest
// singleton slot, exactly the reference's ascending seed order. Generation
// g+1 is the queue of slots whose count dropped to one while generation g was
// processed, ordered as the reference's deque orders it: by the processing
// order of the peeled position, then by row. Pushes carry that key, the host
// sorts each generation (cub radix sort), and a position that is a singleton
// in several queued slots is peeled from the first of them (epoch-tagged
// atomicMax claims).
struct OrdPush {
  unsigned long long* keys;
  uint32_t* slots;
  uint32_t* count;
  unsigned long long* slot_key;  // per slot: (epoch << 36) | max FIFO key of this generation
  unsigned long long tag;        // epoch << 36 of the generation doing the subtractions
};
constexpr unsigned long long kKeyMask = (1ull << 36) - 1ull;

constexpr uint32_t kOrdStage = 2048;

__device__ __forceinline__ void ord_push(bool push, unsigned long long key, uint32_t slot,
                                         unsigned long long* s_k, uint32_t* s_s, uint32_t* s_n,
                                         const OrdPush& o) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t mask = __ballot_sync(kFull, push);
  if (!mask) return;
  const uint32_t leader = __ffs(mask) - 1, cnt = __popc(mask);
  uint32_t b = 0, direct = 0;
  if (lane == leader) {
    b = atomicAdd(s_n, cnt);
    if (b + cnt > kOrdStage) {
      if (b < kOrdStage) atomicMin(s_n + 1, b);  // [b, stage) stays unwritten
      direct = 1;
      b = atomicAdd(o.count, cnt);
    }
  }
  b = __shfl_sync(kFull, b, leader);
  direct = __shfl_sync(kFull, direct, leader);
  if (push) {
    const uint32_t idx = b + __popc(mask & ((1u << lane) - 1u));
    if (direct) {
      o.keys[idx] = key;
      o.slots[idx] = slot;
    } else {
      s_k[idx] = key;
      s_s[idx] = slot;
    }
  }
}

__device__ __forceinline__ void ord_flush(unsigned long long* s_k, uint32_t* s_s, uint32_t* s_n,
                                          uint32_t* s_b, const OrdPush& o) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t n = min(min(s_n[0], kOrdStage), s_n[1]);
    *s_b = n ? atomicAdd(o.count, n) : 0u;
    s_n[0] = n;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < *s_n; i += blockDim.x) {
    o.keys[*s_b + i] = s_k[i];
    o.slots[*s_b + i] = s_s[i];
  }
}

__global__ void __launch_bounds__(256) k_r0_phase1(DecodeWork w, const HashParams hp) {
  round0_phase1(w, hp, uint64_t(blockIdx.x) * blockDim.x + threadIdx.x,
                uint64_t(gridDim.x) * blockDim.x);
}

// Generation-0 subtraction; pushes are keyed (winner slot, row).
__global__ void __launch_bounds__(256) k_r0_push(DecodeWork w, const HashParams hp, OrdPush o) {
  __shared__ unsigned long long s_k[kOrdStage];
  __shared__ uint32_t s_s[kOrdStage];
  __shared__ uint32_t s_n[2], s_b;  // [0] reserved, [1] end of the contiguous written prefix
  if (threadIdx.x == 0) {
    s_n[0] = 0;
    s_n[1] = kOrdStage;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t start = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint32_t total = w.qcount[5];
  for (uint64_t base = start - lane; base < total; base += stride) {
    const uint64_t i = base + lane;
    uint32_t p = 0, rows = 0;
    float v = 0.0f;
    unsigned long long wkey = 0;
    DecItem e{};
    if (i < total) {
      const uint2 info = w.pinfo[i];
      if (info.y & 0x100u) {
        rows = info.y & 0xFFu;
        v = __uint_as_float(info.x);
        p = w.plist[i];
        e = w.items[w.pitem[i]];
        const uint32_t best = (info.y >> 12) & 0xFu;
        const uint64_t ws = e.slot_base + uint64_t(best) * e.m + dev_bucket(row_coef(hp, best), p, e.m);
        wkey = ws * hp.rows;
      }
    }
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
      bool push = false;
      uint64_t s = 0;
      if (rows >> r & 1u) {
        const uint64_t local = uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m);
        s = e.slot_base + local;
        atomicAdd(e.sketch + local, -(dev_sign(hp.row[r], p) * v));
        // the reference queues a slot when its LAST subtraction of the
        // generation (in FIFO order) leaves one position: keep the max key
        atomicMax(o.slot_key + s, o.tag | (wkey + r));
        const unsigned long long old = atomicAdd(w.slot_state + s, st_sub(p));
        push = st_count(old) == 2u;
      }
      ord_push(push, 0ull, uint32_t(s), s_k, s_s, s_n, o);
    }
  }
  ord_flush(s_k, s_s, s_n, &s_b, o);
}

__global__ void __launch_bounds__(256) k_ord_keys(unsigned long long* keys, const uint32_t* slots,
                                                  uint32_t n, const unsigned long long* slot_key) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
    keys[j] = slot_key[slots[j]] & kKeyMask;
}

__global__ void __launch_bounds__(256) k_ord_claim(DecodeWork w, const uint32_t* __restrict__ q,
                                                   uint32_t qlen, unsigned long long* claim,
                                                   uint32_t epoch) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < qlen; i += gridDim.x * blockDim.x) {
    const uint32_t slot = q[i];
    const unsigned long long st = w.slot_state[slot];
    if (st_count(st) != 1u) continue;
    const uint32_t it = find_slot_item(w.items, w.n_items, slot);
    const uint64_t pos = w.items[it].bitmap_off * 32ull + st_pos(st);
    atomicMax(claim + pos, (uint64_t(epoch) << 32) | uint64_t(~i));
  }
}

__global__ void __launch_bounds__(256) k_ord_peel(DecodeWork w, const HashParams hp,
                                                  const uint32_t* __restrict__ q, uint32_t qlen,
                                                  const unsigned long long* __restrict__ claim,
                                                  uint32_t epoch, OrdPush o) {
  __shared__ unsigned long long s_k[kOrdStage];
  __shared__ uint32_t s_s[kOrdStage];
  __shared__ uint32_t s_n[2], s_b;  // [0] reserved, [1] end of the contiguous written prefix
  if (threadIdx.x == 0) {
    s_n[0] = 0;
    s_n[1] = kOrdStage;
  }
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * blockDim.x;
  uint32_t won = 0;
  for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x - lane; base < qlen; base += stride) {
    const uint32_t i = base + lane;
    bool win = false;
    uint32_t slot = 0, p = 0;
    DecItem e{};
    float v = 0.0f;
    if (i < qlen) {
      slot = q[i];
      const unsigned long long st = w.slot_state[slot];
      if (st_count(st) == 1u) {
        p = st_pos(st);
        const uint32_t it = find_slot_item(w.items, w.n_items, slot);
        e = w.items[it];
        win = claim[e.bitmap_off * 32ull + p] == ((uint64_t(epoch) << 32) | uint64_t(~i));
        if (win) {
          const uint64_t local = slot - e.slot_base;
          const uint32_t row = uint32_t(local / e.m);
          v = canonical(dev_sign(row_coef(hp, row), p) * e.sketch[local]);  // decode.cpp:110-111
          e.out[p] = v;
          atomicOr(w.bitmap + e.bitmap_off + (p >> 5), 1u << (p & 31));
          ++won;
        }
      }
    }
    _Pragma("unroll") for (uint32_t r = 0; r < uint32_t(kMaxRows); ++r) if (r < hp.rows) {
      bool push = false;
      uint64_t s = 0;
      if (win) {
        const uint64_t local = uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m);
        s = e.slot_base + local;
        if (s != slot) {
          atomicAdd(e.sketch + local, -(dev_sign(hp.row[r], p) * v));
          atomicMax(o.slot_key + s, o.tag | (uint64_t(i) * hp.rows + r));
          const unsigned long long old = atomicAdd(w.slot_state + s, st_sub(p));
          push = st_count(old) == 2u;
        }
      }
      ord_push(push, 0ull, uint32_t(s), s_k, s_s, s_n, o);
    }
  }
  won = warp_sum32(won);
  if (lane == 0 && won) atomicAdd(&w.qcount[4], won);
  ord_flush(s_k, s_s, s_n, &s_b, o);
}

// ------------------------------------------------------------------ estimate
__global__ void __launch_bounds__(256) k_final(DecodeWork w, const HashParams hp) {
  const uint32_t total = w.qcount[5];
  if (total == w.qcount[4]) {  // every present position peeled: nothing to estimate
    span_end(w.span);
    return;
  }
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gtid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gstride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t base = gtid - lane; base < total; base += gstride) {
    const uint64_t i = base + lane;
    bool unres = false;
    uint32_t p = 0, it = 0;
    DecItem e{};
    if (i < total) {
      p = w.plist[i];
      it = w.pitem[i];
      e = w.items[it];
      unres = !(w.bitmap[e.bitmap_off + (p >> 5)] >> (p & 31) & 1u);
      if (unres) {  // decode.cpp:130-138 / :43-47
        float est[kMaxRows];
#pragma unroll
        for (uint32_t r = 0; r < kMaxRows; ++r) {
          if (r >= hp.rows) break;
          est[r] = dev_sign(hp.row[r], p) * e.sketch[uint64_t(r) * e.m + dev_bucket(hp.row[r], p, e.m)];
        }
        e.out[p] = canonical(median_rows(est, hp.rows));
        const uint32_t b = atomicAdd(&w.stats[it].unresolved, 1u);
        if (w.unresolved) w.unresolved[e.list_off + b] = p;
      }
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
    uint32_t bits = present_bits(words[wi], w4);
    const uint32_t P = w4 ? 8u : 32u;
    const uint64_t first = uint64_t(wi) * P, left = n > first ? n - first : 0;
    if (w4) {
      if (left < 8) bits &= (1u << (4 * left)) - 1u;
    } else if (left < 32) {
      bits &= (1u << left) - 1u;
    }
    counts[wi] = __popc(bits);
  }
}

__global__ void k_word_positions(const uint32_t* __restrict__ words, uint32_t n, uint32_t n_words,
                                 bool w4, const uint32_t* __restrict__ offsets,
                                 uint32_t* __restrict__ out, uint32_t* count_dev) {
  for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < n_words; wi += gridDim.x * blockDim.x) {
    uint32_t bits = present_bits(words[wi], w4);
    const uint32_t P = w4 ? 8u : 32u;
    const uint64_t first = uint64_t(wi) * P, left = n > first ? n - first : 0;
    if (w4) {
      if (left < 8) bits &= (1u << (4 * left)) - 1u;
    } else if (left < 32) {
      bits &= (1u << left) - 1u;
    }
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

}  // namespace

int launch_decode(const DevInfo& di, const DecodeWork& w, const HashParams& hp,
                  cudaStream_t stream) {
  if (w.n_items == 0) return 0;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_build, 256, 0);
  uint64_t g = uint64_t(std::max(per_sm, 1)) * di.sms;
  if (w.total_word_tiles < g) g = w.total_word_tiles;
  k_build<<<int(g ? g : 1), 256, 0, stream>>>(w, hp);

  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_peel, 256, 0);
  const int pg = std::max(per_sm, 1) * di.sms;
  DecodeWork wc = w;
  HashParams hc = hp;
  void* args[] = {&wc, &hc};
  cudaLaunchCooperativeKernel((const void*)k_peel, dim3(pg), dim3(256), args, 0, stream);

  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_final, 256, 0);
  k_final<<<std::max(per_sm, 1) * di.sms, 256, 0, stream>>>(w, hp);
  return 3;
}

int launch_decode_ordered(const DevInfo& di, const DecodeWork& w, const HashParams& hp,
                          const OrderedBuffers& ob, cudaStream_t stream, uint32_t& epoch,
                          uint32_t* rounds) {
  if (w.n_items == 0) return 0;
  int launches = 0;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_build, 256, 0);
  uint64_t g = uint64_t(std::max(per_sm, 1)) * di.sms;
  if (w.total_word_tiles < g) g = w.total_word_tiles;
  k_build<<<int(g ? g : 1), 256, 0, stream>>>(w, hp);
  const int grid = di.sms * 4;
  k_r0_phase1<<<grid, 256, 0, stream>>>(w, hp);
  ++epoch;
  OrdPush o{ob.keys[0], ob.slots[0], ob.count, ob.slot_key, uint64_t(epoch) << 36};
  cudaMemsetAsync(ob.count, 0, 4, stream);
  k_r0_push<<<grid, 256, 0, stream>>>(w, hp, o);
  launches += 3;
  uint32_t gen = 1;
  unsigned long long* cur_keys = ob.keys[0];
  uint32_t* cur_slots = ob.slots[0];
  for (;;) {
    uint32_t cnt = 0;
    cudaMemcpyAsync(&cnt, ob.count, 4, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    if (cnt == 0) break;
    k_ord_keys<<<grid, 256, 0, stream>>>(cur_keys, cur_slots, cnt, ob.slot_key);
    cub::DoubleBuffer<unsigned long long> dk(cur_keys, cur_keys == ob.keys[0] ? ob.keys[1] : ob.keys[0]);
    cub::DoubleBuffer<uint32_t> dv(cur_slots, cur_slots == ob.slots[0] ? ob.slots[1] : ob.slots[0]);
    size_t tb = ob.scratch_bytes;
    cub::DeviceRadixSort::SortPairs(ob.scratch, tb, dk, dv, int(cnt), 0, 36, stream);
    const uint32_t* q = dv.Current();
    // the next generation's pushes go to the buffers the sort left free
    ++epoch;
    OrdPush no{dk.Alternate(), dv.Alternate(), ob.count, ob.slot_key, uint64_t(epoch) << 36};
    k_ord_claim<<<grid, 256, 0, stream>>>(w, q, cnt, ob.claim, epoch);
    cudaMemsetAsync(ob.count, 0, 4, stream);
    k_ord_peel<<<grid, 256, 0, stream>>>(w, hp, q, cnt, ob.claim, epoch, no);
    cur_keys = dk.Alternate();
    cur_slots = dv.Alternate();
    launches += 4;
    ++gen;
  }
  if (rounds) *rounds = gen;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)k_final, 256, 0);
  k_final<<<std::max(per_sm, 1) * di.sms, 256, 0, stream>>>(w, hp);
  return launches + 1;
}

size_t ordered_sort_scratch_bytes(uint32_t count) {
  size_t temp = 0;
  cub::DoubleBuffer<unsigned long long> dk(nullptr, nullptr);
  cub::DoubleBuffer<uint32_t> dv(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, temp, dk, dv, int(count), 0, 64);
  return temp;
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

}  // namespace tagc_b200
