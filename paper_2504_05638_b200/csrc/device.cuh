// device.cuh — descriptors shared by the host engine and the sm_100a kernels,
// plus the device forms of the wire-format hash (reference hash.hpp:25-47).
#pragma once

#include <cstdint>

namespace tagc_b200 {

constexpr int kMaxRows = 8;
// Elements per tile: 256 threads x 16 elements. Tiles are word-aligned for
// both index widths (multiple of 32 positions).
constexpr uint32_t kTile = 4096;
constexpr uint32_t kTileThreads = 256;
// Segments at or below this length skip the sampling pre-pass: every nonzero
// key is a threshold candidate.
constexpr uint32_t kSmallSegment = 65536;
// Sample geometry: first kSampleChunk elements of every `sample_stride`-th tile.
constexpr uint32_t kSampleChunk = 1024;
constexpr uint32_t kSampleBins = 4096;  // top 12 bits of the 31-bit magnitude key
constexpr uint32_t kSampleShift = 19;
constexpr uint32_t kFineShift = kSampleShift - 12;   // 4096 fine bins inside a sample bin
constexpr uint32_t kSampleStride = 3 * kSampleBins;  // per item: coarse, fine (lo), fine (hi)
// Large segments sample 1024 elements of every kSampleMaxStride-th tile
// (1/32 of the data); the window's rank margin scales with 1/sqrt(sample).
constexpr uint64_t kSampleMaxStride = 8;
// ... and at most kSampleMaxTiles chunks (2M samples) per segment: past that
// the stride grows (a 2^28-element bucket samples every 32nd tile, 1/128).
// sigma of the sampled rank then is ~140 at theta = 99, a window of ~0.1 %
// of the segment, still tiny against the fused pass's streaming.
constexpr uint64_t kSampleMaxTiles = 2048;
constexpr uint32_t kRadixBins = 2048;   // 11/10/10-bit digits of the key
constexpr uint32_t kDecWordTile = 4096; // merged-index words per decode word tile (16 per thread)
constexpr uint32_t kMaxFlatItems = 4096; // items per call (flattened iteration bound)

// Per-row hash coefficients (reference hash.hpp:27-33), derived on the host.
struct RowCoef {
  uint64_t pos_a, pos_b, sgn_a, sgn_b;
};
struct HashParams {
  RowCoef row[kMaxRows];
  uint32_t rows;
};

// Item flags
enum : uint32_t {
  kWidth4 = 1u << 0,     // index width 4 (else 1)
  kAligned16 = 1u << 1,  // g and acc (when present) are 16-byte aligned
  kHasAcc = 1u << 2,     // combined = g + acc, residual written back to acc
  kWriteIndex = 1u << 3,
  kWriteSketch = 1u << 4,
  kSelect = 1u << 5,      // tau from the select pipeline; else tau = 0
  kWriteSparse = 1u << 6, // per-stage sparsify outputs
  kWriteResidual = 1u << 7,
  kDeferScatter = 1u << 8,  // sketch bigger than L2: kept entries are logged, scattered region by region later
};

// One (rank, segment) unit of sparsify + encode work.
struct EncItem {
  const float* g;
  float* acc;
  float* sparse;    // optional (kWriteSparse)
  float* residual;  // optional (kWriteResidual)
  uint32_t* index;  // segment index words
  float* sketch;    // rows*m floats
  uint64_t tile_begin;
  uint64_t sample_begin;  // first sample-work id (sample kernel)
  uint64_t cand_off;      // offset into the candidate pool (uint2: position, value bits)
  uint64_t hi_off;        // offset into the speculatively-kept pool (uint2)
  uint32_t n, m, c, flags;
  uint32_t cand_cap, sample_stride, sample_tiles, hi_cap;
  uint64_t mmul;  // fastmod multiplier for m (fastmod_magic), set by the engine
  uint32_t ds_group;  // deferred-scatter group (kDeferScatter items; groups span <= 2^27 floats)
  uint32_t ds_pad;
};

// Select state per item (device; reset by the window kernel every call).
// status: 0 tau ready, 1 fallback, 3 collect sub-bin, 4 fallback tau ready.
struct SelState {
  uint32_t klo, khi;          // candidate window on the 31-bit key
  uint32_t cnt_zero, cnt_lo;  // keys == 0, 0 < key < klo
  uint32_t cnt_in, cnt_hi;    // window candidates, keys above the window (kept speculatively)
  uint32_t status, tau_key;
  uint32_t prefix, rank;      // collect: target sub-bin / rank; fallback: radix prefix / rank
  uint32_t kept, fshift;      // kept elements (zero_count); fine-bin shift of the window
  uint32_t n_sel, pad;        // keys gathered from the target sub-bin
};

// One owner-side decode unit (one compressed segment).
struct DecItem {
  const uint32_t* words;  // merged index (or presence bitmap, width 1)
  float* sketch;          // summed sketch rows*m (mutated into the residual)
  float* out;             // dense output for the segment (n floats)
  uint64_t slot_base;     // first global slot id (rows*m per item)
  uint64_t word_tile_begin;
  uint64_t list_off;      // presence list offset
  uint32_t n, m, flags, n_words;
  uint32_t list_cap, pad;  // bound on this item's presence (host-side sizing)
  uint64_t mmul;          // fastmod multiplier for m (fastmod_magic), set by the engine
};

struct DecStats {  // per decode item, device
  uint32_t presence, unresolved, overflow, pad;
};

// Owner-side optimizer epilogue parameters (see opt_update below).
struct OptEpilogue {
  int32_t kind;       // -1: none, 0: sgd, 1: adamw_nm
  int32_t write_out;  // also store the decoded value (else out_base aliases params, never written)
  // params, adam_v and out_base must be 16-byte aligned (the engine checks)
  const float* out_base;
  float* params;
  float* adam_v;
  float inv_w, lr, wd, bias_fix;
};

#ifdef __CUDACC__
// -------------------------------------------------------------- device hash
__device__ __forceinline__ uint32_t dev_bucket(const RowCoef& c, uint32_t p, uint32_t m) {
  const uint64_t h = c.pos_a * (uint64_t(p) + 0x9E3779B9ull) + c.pos_b;  // hash.hpp:36
  return uint32_t(h >> 32) % m;                                            // hash.hpp:37
}
// x % m without a divide: Lemire's fastmod, exact for every 32-bit x and
// m >= 1 with mmul = fastmod_magic(m) = floor((2^64 - 1) / m) + 1 (mod 2^64).
__device__ __forceinline__ uint32_t fastmod(uint32_t x, uint64_t mmul, uint32_t m) {
  return uint32_t(__umul64hi(mmul * uint64_t(x), uint64_t(m)));
}
__device__ __forceinline__ uint32_t dev_bucket(const RowCoef& c, uint32_t p, uint32_t m, uint64_t mmul) {
  const uint64_t h = c.pos_a * (uint64_t(p) + 0x9E3779B9ull) + c.pos_b;  // hash.hpp:36
  return fastmod(uint32_t(h >> 32), mmul, m);                              // hash.hpp:37
}
__device__ __forceinline__ float dev_sign(const RowCoef& c, uint32_t p) {
  const uint64_t h = c.sgn_a * (uint64_t(p) + 0x85EBCA77ull) + c.sgn_b;  // hash.hpp:41
  return (h >> 63) ? 1.0f : -1.0f;                                         // hash.hpp:42
}
__device__ __forceinline__ uint32_t mag_key(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }
// Fire-and-forget global reductions. A plain atomicAdd(float*) through a
// generic pointer compiles to a returning ATOM plus a shared-memory CAS
// fallback; these name the global state space and return nothing (RED).
// Like every GPU float atomic, red.add.f32 flushes subnormals.
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("{\n.reg .u64 ga;\ncvta.to.global.u64 ga, %0;\nred.global.add.f32 [ga], %1;\n}" ::"l"(p), "f"(v)
               : "memory");
}
__device__ __forceinline__ void red_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("{\n.reg .u64 ga;\ncvta.to.global.u64 ga, %0;\nred.global.add.u32 [ga], %1;\n}" ::"l"(p), "r"(v)
               : "memory");
}
__device__ __forceinline__ void red_or_u32(uint32_t* p, uint32_t v) {
  asm volatile("{\n.reg .u64 ga;\ncvta.to.global.u64 ga, %0;\nred.global.or.b32 [ga], %1;\n}" ::"l"(p), "r"(v)
               : "memory");
}
// Owner-side optimizer step (reference train.cpp:355-359, apply_optimizer
// :202-220) as an epilogue of whatever kernel produces a decoded value:
// g = decoded * (1/W), then SGD or momentum-free AdamW on params[i], with
// explicitly rounded operations in the reference's order (no FMA contraction)
// so the update is bit-identical to its fp32 loop. Element i of the owner's
// decoded output `out_base` maps to params[i] / adam_v[i].
template <bool kAdam>
__device__ __forceinline__ void opt_update(const OptEpilogue& o, float decoded, float& p, float& v) {
  constexpr float kB2 = 0.999f, kOneMinusB2 = 1.0f - 0.999f, kEps = 1e-8f;
  const float g = __fmul_rn(decoded, o.inv_w);
  if (!kAdam) {
    p = __fsub_rn(p, __fmul_rn(o.lr, g));
  } else {
    v = __fadd_rn(__fmul_rn(kB2, v), __fmul_rn(__fmul_rn(kOneMinusB2, g), g));
    // g / (sqrt(v / bias_fix) + eps) is exactly g (a signed zero) when g is
    // a zero and v >= 0: the denominator is then >= eps > 0 or +inf. Most of
    // a sparse decoded shard takes this branch and skips two IEEE divisions
    // and a square root; the result is bit-identical either way.
    float ratio = g;
    if (!(g == 0.0f && v >= 0.0f)) {
      const float vhat = __fdiv_rn(v, o.bias_fix);
      ratio = __fdiv_rn(g, __fadd_rn(__fsqrt_rn(vhat), kEps));
    }
    const float upd = __fadd_rn(ratio, __fmul_rn(o.wd, p));
    p = __fsub_rn(p, __fmul_rn(o.lr, upd));
  }
}
// The epilogue over a contiguous run of decoded values vals[0, len) (shared
// or global memory) landing at dst[0, len). The body moves params / adam_v
// (and the decoded values where their alignment allows) as float4: 4-byte
// accesses cap this HBM-bound update near 3.8 TB/s on B200, float4 reaches
// ~6.9 TB/s (tools/micro/opt_variants.cu). Each thread handles two float4
// groups per pass with both groups' loads issued before any store.
template <bool kAdam>
__device__ __forceinline__ void opt_one(const OptEpilogue& o, float* dst, uint64_t i, float d) {
  float p = o.params[i], v = kAdam ? o.adam_v[i] : 0.0f;
  if (o.write_out) *dst = d;
  opt_update<kAdam>(o, d, p, v);
  o.params[i] = p;
  if (kAdam) o.adam_v[i] = v;
}
template <bool kAdam>
__device__ __forceinline__ void opt_four(const OptEpilogue& o, float4 d, float4& p, float4& v) {
  opt_update<kAdam>(o, d.x, p.x, v.x);
  opt_update<kAdam>(o, d.y, p.y, v.y);
  opt_update<kAdam>(o, d.z, p.z, v.z);
  opt_update<kAdam>(o, d.w, p.w, v.w);
}
template <bool kAdam, bool kStreamVals>
__device__ __forceinline__ void opt_range(const OptEpilogue& o, float* dst, const float* vals, uint32_t len) {
  const uint64_t base = uint64_t(dst - o.out_base);
  // params, adam_v and out_base are 16-byte aligned (checked on the host), so
  // element base + head starts a float4 of each
  const uint32_t head = min(len, uint32_t((4u - (base & 3u)) & 3u));
  for (uint32_t q = threadIdx.x; q < head; q += blockDim.x)
    opt_one<kAdam>(o, dst + q, base + q, kStreamVals ? __ldcs(vals + q) : vals[q]);
  const uint32_t groups = (len - head) >> 2;
  const uint32_t tail0 = head + (groups << 2);
  for (uint32_t q = tail0 + threadIdx.x; q < len; q += blockDim.x)
    opt_one<kAdam>(o, dst + q, base + q, kStreamVals ? __ldcs(vals + q) : vals[q]);
  if (!groups) return;
  float4* __restrict__ P4 = reinterpret_cast<float4*>(o.params + base + head);
  float4* __restrict__ V4 = kAdam ? reinterpret_cast<float4*>(o.adam_v + base + head) : nullptr;
  float4* __restrict__ D4 = reinterpret_cast<float4*>(dst + head);
  const float* vh = vals + head;
  const bool vals4 = (reinterpret_cast<uintptr_t>(vh) & 15u) == 0;
  auto load_vals = [&](uint32_t g) {
    if (vals4) return kStreamVals ? __ldcs(reinterpret_cast<const float4*>(vh) + g)
                                  : reinterpret_cast<const float4*>(vh)[g];
    const float* x = vh + 4u * g;
    return kStreamVals ? make_float4(__ldcs(x), __ldcs(x + 1), __ldcs(x + 2), __ldcs(x + 3))
                       : make_float4(x[0], x[1], x[2], x[3]);
  };
  for (uint32_t g0 = threadIdx.x; g0 < groups; g0 += 2u * blockDim.x) {
    const uint32_t g1 = g0 + blockDim.x;
    const bool has1 = g1 < groups;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 d0 = load_vals(g0), p0 = P4[g0], v0 = kAdam ? V4[g0] : z;
    float4 d1 = z, p1 = z, v1 = z;
    if (has1) {
      d1 = load_vals(g1);
      p1 = P4[g1];
      if (kAdam) v1 = V4[g1];
    }
    if (o.write_out) {
      D4[g0] = d0;
      if (has1) D4[g1] = d1;
    }
    opt_four<kAdam>(o, d0, p0, v0);
    P4[g0] = p0;
    if (kAdam) V4[g0] = v0;
    if (has1) {
      opt_four<kAdam>(o, d1, p1, v1);
      P4[g1] = p1;
      if (kAdam) V4[g1] = v1;
    }
  }
}

// Device-side execution spans (timing mode): span[0] = earliest CTA start,
// span[1] = latest CTA end of a kernel chain, in %globaltimer ns. Independent
// of where the driver stamps stream events.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void span_begin(unsigned long long* span) {
  if (span && threadIdx.x == 0) atomicMin(span, globaltimer_ns());
}
// CTA-uniform call site (contains a barrier)
__device__ __forceinline__ void span_end(unsigned long long* span) {
  if (span) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(span + 1, globaltimer_ns());
  }
}
// Flattened iteration over per-item counts that live in device memory: one
// warp builds the exclusive prefix in shared memory (pref[0..n]), then every
// thread maps a flat index to (item, offset) by binary search. Keeps all SMs
// busy when items (segments) are many and uneven instead of walking them one
// after another.
template <typename CountFn>
__device__ __forceinline__ uint32_t flat_prefix(uint32_t n_items, CountFn count, uint32_t* pref) {
  if (threadIdx.x < 32) {
    uint32_t carry = 0;
    for (uint32_t base = 0; base < n_items; base += 32) {
      const uint32_t i = base + threadIdx.x;
      uint32_t c = i < n_items ? count(i) : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, c, o);
        if (threadIdx.x >= uint32_t(o)) c += y;
      }
      if (i < n_items) pref[i + 1] = carry + c;
      carry += __shfl_sync(0xFFFFFFFFu, c, 31);
    }
    if (threadIdx.x == 0) pref[0] = 0;
  }
  __syncthreads();
  return pref[n_items];
}
__device__ __forceinline__ uint32_t flat_item(const uint32_t* pref, uint32_t n_items, uint32_t j) {
  uint32_t lo = 0, hi = n_items - 1;  // largest i with pref[i] <= j
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= j) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Row coefficients with a runtime row index, without dynamic indexing into
// the kernel-parameter struct (which would spill it to local memory).
__device__ __forceinline__ RowCoef row_coef(const HashParams& hp, uint32_t row) {
  RowCoef c = hp.row[0];
#pragma unroll
  for (uint32_t r = 1; r < uint32_t(kMaxRows); ++r)
    if (row == r) c = hp.row[r];
  return c;
}
#endif

inline uint64_t fastmod_magic(uint32_t m) { return ~0ull / uint64_t(m ? m : 1) + 1ull; }

// Host: coefficient derivation (hash.hpp:15-33).
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
inline RowCoef make_row_coef(uint64_t seed, uint32_t row) {
  RowCoef c;
  const uint64_t s = splitmix64(seed ^ (0xA24BAED4963EE407ULL * (uint64_t)(row + 1u)));
  c.pos_a = splitmix64(s) | 1ULL;
  c.pos_b = splitmix64(c.pos_a);
  c.sgn_a = splitmix64(c.pos_b) | 1ULL;
  c.sgn_b = splitmix64(c.sgn_a);
  return c;
}
inline HashParams make_hash_params(uint64_t seed, uint32_t rows) {
  HashParams h{};
  h.rows = rows;
  for (uint32_t r = 0; r < rows && r < (uint32_t)kMaxRows; ++r) h.row[r] = make_row_coef(seed, r);
  return h;
}

}  // namespace tagc_b200

// ---------------------------------------------------------- dependent launch
// Programmatic dependent launch between consecutive kernels of a step: a
// kernel launched with launch_pdl may be scheduled while its predecessor
// drains, and waits (griddepcontrol.wait, its first statement) until the
// predecessor has completed and its writes are visible. Only kernels that
// open with PDL_WAIT() may be launched this way. TAGC_PDL=0 disables.
#if defined(__CUDACC__)
#include <cstdlib>
#include <utility>
#define PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
namespace tagc_b200 {
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TAGC_PDL");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
  if (!pdl_enabled()) {
    kern<<<grid, block, smem, stream>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace tagc_b200
#endif
