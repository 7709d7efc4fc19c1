// kernels.hpp — host launchers for the sm_100a kernels (encode.cu, decode.cu).
// All launchers enqueue on `stream` and return the number of kernel launches
// they issued (the engine reports the total as gpu_launches).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include <cstdint>

#include "device.cuh"

namespace tagc_b200 {

struct DevInfo {
  int sms = 148;
  int dev = 0;
  // CTAs per SM a cooperative launch leaves free: 1 while a peer exchange is
  // attached, so a peer's 1-CTA flag wait on the same GPU (all ranks in one
  // process) can never hold back the full-occupancy grid it waits for
  int coop_headroom = 0;
};
// cooperative grid: (blocks per SM - headroom) x SMs, at least one per SM
inline int coop_grid(const DevInfo& di, int per_sm) {
  const int b = per_sm - di.coop_headroom;
  return (b > 0 ? b : 1) * di.sms;
}

// ---------------------------------------------------------------- select + encode
// Speculative single-pass sparsify + encode for `n_items` items (all with
// kSelect): sample -> window -> fused pass. Device scratch: sample_hist
// [n_items * kSampleBins] and fine_hist [n_items * kRadixBins] (zero on entry,
// left zero), cand / hi_pool (uint2 pools at each item's cand_off / hi_off),
// err[4] (err[0] NaN, err[1] fallback needed).
int launch_select_fused(const DevInfo& di, const EncItem* items, SelState* state, uint32_t n_items,
                        uint64_t total_tiles, uint64_t total_samples, const HashParams& hp, bool w4,
                        int per_stage, uint32_t* sample_hist, uint32_t* fine_hist, uint2* cand,
                        uint2* hi_pool, uint32_t* err, cudaStream_t stream,
                        unsigned long long* span = nullptr, bool tma = false, uint64_t sketch_bytes = 0);
// Exact tau from the window candidates, fix-up of the candidates, and the
// (normally idle) restore + radix-select + re-encode fallback chain.
int launch_select_finish(const DevInfo& di, const EncItem* items, SelState* state, uint32_t n_items,
                         uint64_t total_tiles, const HashParams& hp, bool w4, uint32_t* fine_hist,
                         uint32_t* fb_hist, uint2* cand, uint2* hi_pool, uint32_t* sel_list,
                         uint32_t* err, cudaStream_t stream);
// tau = 0 encode (CountSketch::compress / Index::create entry points).
int launch_encode_exact(const DevInfo& di, const EncItem* items, SelState* state, uint32_t n_items,
                        uint64_t total_tiles, const HashParams& hp, const uint32_t* err, bool w4,
                        cudaStream_t stream);

// ------------------------------------------------------- plumbing kernels
// Zero up to kZeroRanges byte ranges in one launch, and copy bytes from mapped
// pinned host memory. Both run on the SMs, so the context stream never queues
// behind a bulk transfer on a copy engine (the host-buffer path keeps the
// copy engines busy with gradient / result transfers).
constexpr int kZeroRanges = 8;
struct ZeroRanges {
  void* ptr[kZeroRanges];
  uint64_t bytes[kZeroRanges];
  int n;
};
int launch_zero(const ZeroRanges& r, cudaStream_t stream);
int launch_stage_copy(void* dst, const void* mapped_src, uint64_t bytes, cudaStream_t stream);

// ------------------------------------------------------- elementwise / sums
// out[i] = sum_{r<world} in[r][i], ascending rank order (reference rank_sum,
// kernels.cpp:43-63). in_ptrs: device array of `world` pointers.
int launch_rank_sum_f32(const float* const* in_ptrs, uint32_t world, float* out, uint64_t n,
                        cudaStream_t stream);
// Wrapping u32 word sum (kernels.cpp:65-84).
int launch_rank_sum_u32(const uint32_t* const* in_ptrs, uint32_t world, uint32_t* out, uint64_t n,
                        cudaStream_t stream);
// Sketch scatter of the kDeferScatter items' logged kept entries, binned by
// region of [base, base + span_floats) (after launch_select_finish).
// fill: kDsMaxBins u32 and ctl: 4 u32, both zero on entry (the caller zeroes
// them per batch); records: rows x (sum of the items' hi_cap) x 17/16 +
// kDsMaxBins x 1024 uint2; ovf: rows x (sum of hi_cap) uint2. Returns -1
// when the span exceeds 2^32 floats (nothing launched). Spans up to 2^26
// floats are summed per region in shared memory and stored over the
// deferred sketches of items whose select did not fall back (the exact
// re-encode scatters directly), so callers leave those sketches unzeroed;
// larger spans are zeroed here and applied with L2 REDs bin by bin.
constexpr uint32_t kDsMaxBins = 4096;
// One call per deferred-scatter group: the items with ds_group == group,
// whose sketches lie in [base, base + span_floats).
int launch_deferred_scatter(const DevInfo& di, const EncItem* items, const SelState* state, uint32_t n_items,
                            uint32_t group, const uint2* hi_pool, const HashParams& hp, float* base,
                            uint64_t span_floats, uint32_t* fill, uint32_t* ctl, uint2* records, uint2* ovf,
                            cudaStream_t stream);
// Owner-side optimizer step on the decoded shard (train.cpp:202-220, 355-359):
// kind 0 SGD, 1 momentum-free AdamW (adam_v in/out).
int launch_apply_optimizer(const OptEpilogue& o, uint64_t n, cudaStream_t stream);
// out = a + b (sketch_add / apply_accumulator).
int launch_add(const float* a, const float* b, float* out, uint64_t n, cudaStream_t stream);

// Strided segment copies: dst[i] = src[i] for each item (pack/unpack raw
// segments around the reduce-scatter); src == nullptr zero-fills dst.
struct CopyItem {
  const float* src;
  float* dst;
  uint64_t n;
  uint64_t tile_begin;  // filled by launch_copy_items' caller via copy_tiles()
};
constexpr uint32_t kCopyTile = 4096;
// Assigns tile_begin; returns the total tile count.
uint64_t copy_tiles(CopyItem* items, uint32_t n_items);
int launch_copy_items(const DevInfo& di, const CopyItem* items, uint32_t n_items, uint64_t total_tiles,
                      cudaStream_t stream, bool one_tile_per_cta = false,
                      const OptEpilogue* dev_opt = nullptr);

// Raw (uncompressed) segments in a simulated world: dst[i] = sum_r src_r[i]
// in ascending rank order. srcs: device array [n_items * world].
struct RawItem {
  float* dst;
  uint64_t n;
  uint64_t src_off;  // offset added to every rank's base pointer
};
int launch_raw_sum(const RawItem* items, uint32_t n_items, uint64_t max_n,
                   const float* const* rank_bases, uint32_t world, cudaStream_t stream);

// Index diagnostics (hook.cpp:282-294): per decode item, lost/spurious counts
// from per-rank words (rank_words[r] + word_off) and the merged words.
struct DiagItem {
  const uint32_t* merged;
  uint64_t word_off;  // into each rank's index buffer
  uint32_t n, n_words, width, pad;
};
int launch_index_diag(const DiagItem* items, uint32_t n_items, uint32_t max_words,
                      const uint32_t* const* rank_words, uint32_t world,
                      unsigned long long* lost_spurious /* 2 per item */, cudaStream_t stream);

// Diagnostics outside the simulated world (diag.cu).
// One byte (0/1) per position from width-1 index words: bytes[32 w + j] = bit j of words[w].
int launch_support_bytes(const uint32_t* words, uint64_t n_words, uint8_t* bytes, cudaStream_t stream);
// Width-1 lost/spurious from a support byte map (OR of the ranks' supports;
// item i's bytes start at support + 32 * items[i].word_off).
int launch_index_diag_support(const DiagItem* items, uint32_t n_items, uint32_t max_words,
                              const uint8_t* support, unsigned long long* lost_spurious, cudaStream_t stream);
// audit_exchanged_sum (hook.cpp:191-195): dst[i] = sum over ranks (ascending)
// of the exchanged sparse value, recovered from the pre-encode combined value
// comb[r][src_off + i] and the post-encode residual res[r][src_off + i].
struct AuditItem {
  float* dst;
  uint64_t n;
  uint64_t src_off;
};
int launch_audit(const AuditItem* items, uint32_t n_items, uint64_t max_n, const float* const* comb,
                 const float* const* res, uint32_t world, cudaStream_t stream);

// ---------------------------------------------------------------- decode
// qcount word of the peeled-entry total: its own 128-byte line (qcount is
// kQcountBytes long), away from the list / queue / hand-off counters that
// the kernels read while many CTAs add into it
constexpr uint32_t kPeeledWord = 32;
constexpr uint64_t kQcountBytes = 256;
constexpr uint32_t kPeelHandoff = 512;
constexpr uint32_t kListMaxCtas = 1024;
struct DecodeWork {
  const DecItem* items;
  uint32_t n_items;
  uint64_t total_word_tiles;
  uint64_t total_slots;
  unsigned long long* slot_state;  // (sum of list indices) << 24 | count, total_slots
  // Counter mode (non-null): round 0 counts entries per bucket in bytes
  // packed four to a word (L2-resident), and slot_state is only built for
  // the buckets of entries round 0 leaves unresolved (ulist, qcount[14]).
  uint32_t* cnt8;
  uint32_t cnt_shift;              // log2 of the counter width: 3 (bytes) or 2 (nibbles)
  uint32_t* ulist;
  uint32_t* wmask;                 // ordered peel: winner-slot bits set by round 0 (or nullptr)
  uint32_t* bitmap;                // recovered flag per presence-list entry
  float* val;                      // decoded value per presence-list entry
  uint32_t* slot_mark;             // per bucket: holds an entry round 0 left unresolved (or nullptr)
  uint32_t* tile_base;             // presence-list offset of every word tile (build -> emit)
  uint32_t* r0_list;               // round-0 peeled entries sharing a bucket (count qcount[13]), or nullptr
  unsigned long long* tile_state;  // single-pass scan: per word tile, flag << 32 | count (zeroed per call)
  uint32_t* cta_cnt;               // counter mode: per list-count CTA, its tiles' present count (2 x kListMaxCtas)
  uint32_t list_split;             // list-count CTAs per list-write CTA (1 or 2)
  uint32_t state_zeroed;           // counter mode: slot_state cleared up front (high load), so round 0
                                   // does not clear the unresolved entries' buckets one by one
  uint32_t* plist;                 // flat presence list (all items), count in qcount[5]
  uint32_t* pitem;                 // item of each flat presence entry
  uint2* pinfo;                    // per presence entry: round-0 value, shared-row mask
  uint32_t* queue[2];              // capacity total_slots each
  uint64_t list_cap;               // presence-list capacity (sum of the items' bounds)
  uint32_t* qcount;                // [2] rounds, [3] tail rounds, [4] peeled, [8..10] frontier sizes, [15] handoff,
                                   // [5] presence total
  DecStats* stats;                 // n_items
  uint32_t* unresolved;            // optional: per item region at list_off
  unsigned long long* dbg;         // optional: globaltimer marks of the peel phases
  unsigned long long* bar;         // k_peel's grid barrier words [3] (zeroed per call)
  uint2* handoff;                  // k_peel's frontier handed to its single-CTA tail (kPeelHandoff pairs)
  unsigned long long* span;        // optional: execution span of build .. final (timing mode)
};
// Presence list + bucket state from the merged index, round-0 peel, frontier
// rounds inside one cooperative persistent kernel, estimation of the rest
// (decode.cpp:53-140 semantics), all into the list-ordered val[]; finish
// with launch_decode_emit.
// fused_emit (counter mode, no owner step): round 0 runs inside the dense
// emit (k_r0_emit) and the final kernel writes the remaining entries, so the
// output is complete without launch_decode_emit.
// sketch_ready (if set): waited on after the list build, before the first
// kernel that reads the sketches (the deferred scatter may still run).
int launch_decode(const DevInfo& di, const DecodeWork& w, const HashParams& hp,
                  cudaStream_t stream, bool fused_emit = false, cudaEvent_t sketch_ready = nullptr);

// Final step of either decode: writes every item's dense output (zeros, and
// the decoded value of each listed entry).
// With dev_opt (a device-resident OptEpilogue, read when the kernel runs, so
// a captured graph picks up each step's scalars) the optimizer step runs on
// every decoded value instead of (or, with write_out, besides) storing it.
int launch_decode_emit(const DevInfo& di, const DecodeWork& w, cudaStream_t stream,
                       const OptEpilogue* dev_opt = nullptr);
// Writes the step's OptEpilogue into its device slot (stream-ordered before
// the kernels that read it; launched outside any graph).
int launch_set_opt(OptEpilogue* dev_opt, const OptEpilogue& o, cudaStream_t stream);
// One device word (stream-ordered; no copy engine on the context stream).
int launch_set_u32(uint32_t* dst, uint32_t v, cudaStream_t stream);
// FIFO-order peel (see decode.cu): every generation on the device, inside
// one cooperative persistent kernel (no host round trip, graph-capturable).
// slot_key / claim are epoch-tagged, zero-initialised once; epoch is a
// persistent device word (never reallocated) advanced per generation;
// dense holds one u32 per FIFO key (total_slots * rows, zero-initialised
// once, restored to zero by every compaction).
struct OrdState {
  unsigned long long* slot_key;  // per slot: (epoch << 32) | FIFO key of its last subtraction
  unsigned long long* claim;     // per presence-list entry: (epoch << 32) | ~queue position
  uint32_t* dense;               // per FIFO key: slot + 1, 0 = empty
  uint32_t* q;                   // the generation's queue in FIFO order
  uint32_t* u0;                  // unordered pushes, even generations
  uint32_t* u1;                  // unordered pushes, odd generations
  uint32_t* cta;                 // per-CTA counts of the compaction
  uint32_t* wmask;               // per slot bit: winner slot of a round-0 entry with a shared bucket (zeroed per call)
  uint32_t* wrank;               // per wmask word: exclusive popcount prefix
  uint64_t wwords;               // wmask words
  uint32_t* epoch;               // persistent device epoch
  uint64_t slot_key_cap, claim_cap;  // allocated elements (cleared on epoch wrap)
};
int launch_decode_ordered(const DevInfo& di, const DecodeWork& w, const HashParams& hp,
                          const OrdState& o, cudaStream_t stream, cudaEvent_t sketch_ready = nullptr);
int ordered_loop_grid(const DevInfo& di);

// Presence list -> bitmap (width-1 index) with bounds/duplicate checks for the
// standalone peeling API (decode.cpp:15-20, :89-94). err bit 1 = OOB, 2 = dup.
int launch_presence_to_bitmap(const uint32_t* presence, uint32_t count, uint32_t n,
                              uint32_t* bitmap, uint32_t* err, cudaStream_t stream);
// Median-of-rows estimate for explicit targets (decode.cpp:24-51); err bit 4
// when a target is outside the presence bitmap.
int launch_estimate_targets(const uint32_t* targets, uint32_t n_targets, const uint32_t* bitmap,
                            uint32_t n, uint32_t m, const float* sketch, const HashParams& hp,
                            float* out, uint32_t* err, cudaStream_t stream);
// Index::presence: ascending positions with field != 0 (index.cpp:51-57).
int launch_index_presence(const uint32_t* words, uint32_t n, uint32_t width, uint32_t* positions,
                          uint32_t* count_dev, void* scratch, size_t scratch_bytes,
                          cudaStream_t stream);
size_t index_presence_scratch_bytes(uint32_t n, uint32_t width);
// Sort a u32 list in place (ascending); scratch from sort_scratch_bytes.
int launch_sort_u32(uint32_t* keys, uint32_t* keys_alt, uint32_t count, void* scratch,
                    size_t scratch_bytes, cudaStream_t stream);
size_t sort_scratch_bytes(uint32_t count);

// ---------------------------------------------------------------- peer exchange
// Pull-mode collective over peer memory (peer.cu): pointers into every rank's
// exchange region (two send sets, flags, step counter).
constexpr int kMaxPeers = 16;
struct PeerView {
  float* send_f[2][kMaxPeers];
  uint32_t* send_u[2][kMaxPeers];
  unsigned long long* flags[kMaxPeers];  // rank q's flag array (world slots)
  unsigned long long* counter;           // this rank's step counter
  uint64_t block_f, block_u;             // owner block sizes (elements, multiples of 32)
  uint64_t timeout_ns;
  uint32_t world, rank;
};
// signal peers -> wait for every peer -> reduce this rank's block of `set`
// into recv_f / recv_u (err[2] set on a peer timeout).
int launch_peer_exchange(const DevInfo& di, const PeerView& v, int set, float* recv_f, uint32_t* recv_u,
                         uint32_t* err, cudaStream_t stream);
void peer_preload();
void preload_encode_kernels();
void preload_decode_kernels();
void preload_diag_kernels();
// Every kernel of the library loaded up front: with CUDA lazy loading a first
// launch while another rank of the process spins in k_peer_wait can stall
// (several ranks on one GPU), and no module load should sit on a timed path.
inline void preload_all_kernels() {
  preload_encode_kernels();
  preload_decode_kernels();
  preload_diag_kernels();
  peer_preload();
}

}  // namespace tagc_b200
