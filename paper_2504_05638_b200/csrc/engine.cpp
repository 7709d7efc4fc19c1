// engine.cpp — orchestration of the B200 exchange (see engine.hpp).
//
// Per call, for every compressed segment (reference hook.cpp:137-189):
//   select  : tau = c-th smallest |g+acc| per (rank, segment)      [encode.cu]
//   encode  : residual -> acc, packed index, count sketch           [encode.cu]
//   exchange: simulated world -> rank folds on this GPU;
//             NCCL world     -> one grouped reduce-scatter of the owner-major
//                               (sketch+raw) f32 and index u32 blocks
//   decode  : peel + estimate into the owner's dense shard          [decode.cu]
// Raw segments (unflagged or below min_compress_segment) are exchanged as
// plain fp32 sums (hook.cpp:125-135) and leave the accumulator untouched.
#include "engine.hpp"

#include <nvtx3/nvToolsExt.h>

#include "nccl_dl.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>

namespace tagc_b200 {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}

namespace {

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// sparsify.cpp:30-31 — same double expression as the reference.
uint32_t threshold_rank(double theta, uint64_t n) {
  uint64_t c = static_cast<uint64_t>(std::ceil(theta * static_cast<double>(n) / 100.0));
  if (c > n) c = n;
  return static_cast<uint32_t>(c);
}

// Presence bound of a compressed segment: every rank keeps at most n - c
// positions (keys above the c-th smallest), and the merged index adds rank
// words, so popcount(sum) <= sum of popcounts bounds the present fields.
uint32_t presence_bound(uint64_t n, double theta, uint32_t world) {
  const uint64_t keep = n - threshold_rank(theta, n);
  return uint32_t(std::min<uint64_t>(n, keep * world + 32));
}

std::string seg_name(const LayerSegment& s, uint32_t i) {
  return s.name.empty() ? "seg" + std::to_string(i) : s.name;
}

void check_shard(const ShardSpec& sh, uint32_t world) {
  if (sh.owner >= world) throw InvalidArgument("shard owner rank out of range");
  for (const LayerSegment& s : sh.segments) {
    if (s.begin < sh.begin || s.end > sh.end || s.end <= s.begin)
      throw InvalidArgument("segment outside its shard");
    if (s.end - s.begin > 0xFFFFFFFFull) throw InvalidArgument("segment longer than 2^32 - 1");
  }
}

}  // namespace

// ------------------------------------------------------------------ planning
ExchangePlan plan_exchange(const std::vector<ShardSpec>& shards, const CompressionConfig& cfg,
                           uint32_t W, uint32_t rank) {
  const uint32_t w = cfg.index_width, rows = cfg.sketch_rows;
  ExchangePlan P;
  P.skc.assign(W, 0);
  P.rawc.assign(W, 0);
  P.wc.assign(W, 0);
  for (uint32_t si = 0; si < shards.size(); ++si) {
    const ShardSpec& sh = shards[si];
    if (sh.owner >= W) throw InvalidArgument("shard owner rank out of range");
    for (uint32_t i = 0; i < sh.segments.size(); ++i) {
      const LayerSegment& s = sh.segments[i];
      SegPlan p;
      p.shard = si;
      p.seg = i;
      p.lo = s.begin - sh.begin;
      p.len = s.size();
      p.tag = "shard" + std::to_string(sh.id) + "/" + seg_name(s, i);
      p.compressed = kind_compressible(s.kind, cfg.policy, cfg.include_out_proj) && cfg.ratio > 1 &&
                     p.len >= cfg.min_compress_segment;  // hook.cpp:120-122
      const uint32_t o = sh.owner;
      if (p.compressed) {
        p.m = sketch_geometry(uint32_t(p.len), cfg.ratio, rows).buckets_per_row;  // hook.cpp:138
        p.n_words = words_needed(uint32_t(p.len), w);
        p.word_off = P.wc[o];
        P.wc[o] += align_up(p.n_words, 4);
        p.sk_off = P.skc[o];
        P.skc[o] += align_up(uint64_t(rows) * p.m, 4);
      }
      P.segs.push_back(p);
    }
  }
  for (SegPlan& p : P.segs)
    if (!p.compressed) {
      const uint32_t o = shards[p.shard].owner;
      p.raw_off = P.skc[o] + P.rawc[o];
      P.rawc[o] += align_up(p.len, 4);
    }
  for (uint32_t o = 0; o < W; ++o) {
    P.Bf = std::max(P.Bf, P.skc[o] + P.rawc[o]);
    P.Bu = std::max(P.Bu, P.wc[o]);
  }
  P.Bf = align_up(std::max<uint64_t>(P.Bf, 32), 32);
  P.Bu = align_up(std::max<uint64_t>(P.Bu, 32), 32);
  P.out_off.assign(shards.size(), ~0ull);
  uint64_t oc = 0;
  for (uint32_t si = 0; si < shards.size(); ++si)
    if (shards[si].owner == rank) {
      P.out_off[si] = oc;
      oc += shards[si].size();
    }
  return P;
}

// ------------------------------------------------------------------ Workspace
Workspace::~Workspace() {
  for (auto& [k, b] : bufs_) cudaFree(b.ptr);
  for (void* p : graveyard_) cudaFree(p);
}

void* Workspace::get(const std::string& name, size_t bytes, bool zero_on_alloc, cudaStream_t s) {
  bytes = std::max<size_t>(bytes, 16);
  Buf& b = bufs_[name];
  if (b.bytes >= bytes) return b.ptr;
  if (b.ptr && defer_free_) {  // queued work may still use it: keep it, no device sync
    graveyard_.push_back(b.ptr);
    total_ -= b.bytes;
    b.ptr = nullptr;
    b.bytes = 0;
  } else if (b.ptr) {
    cuda_check(cudaStreamSynchronize(s), "workspace sync");
    cudaFree(b.ptr);
    total_ -= b.bytes;
    b.ptr = nullptr;
    b.bytes = 0;
  }
  ++gen_;
  const size_t want = align_up(bytes + bytes / 8, 256);  // headroom against regrowth
  cuda_check(cudaMalloc(&b.ptr, want), ("workspace alloc " + name).c_str());
  b.bytes = want;
  total_ += want;
  if (zero_on_alloc) cuda_check(cudaMemsetAsync(b.ptr, 0, want, s), "workspace zero");
  return b.ptr;
}

// ------------------------------------------------------------------ Engine
Engine::Engine(const CompressionConfig& cfg, uint32_t world, uint32_t rank, int device,
               void* nccl_comm, void* stream)
    : cfg_(cfg), world_(world), rank_(rank), device_(device) {
  if (const char* v = std::getenv("TAGC_FUSED_TMA")) use_tma_ = std::atoi(v) != 0;
  if (const char* v = std::getenv("TAGC_GRAPHS")) graphs_on_ = std::atoi(v) != 0;
  if (const char* v = std::getenv("TAGC_SIDE_STREAM")) side_stream_ = std::atoi(v) != 0;
  if (const char* v = std::getenv("TAGC_DEFER_SCATTER_BYTES")) defer_scatter_bytes_ = std::strtoull(v, nullptr, 10);
  if (const char* v = std::getenv("TAGC_FUSED_EMIT")) fused_emit_ = std::atoi(v) != 0;
  if (const char* v = std::getenv("TAGC_FORCE_COLLECTIVE")) force_collective_ = std::atoi(v) != 0;
  if (world == 0 || rank >= world) throw InvalidArgument("rank must be below the world size");
  cfg_.validate_for_world(world);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw CudaError("no CUDA device available (the B200 path has no CPU fallback)");
  if (device < 0) device_ = 0;
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
  if (prop.major < 10)
    throw CudaError("device " + std::string(prop.name) + " is not sm_100-class");
  di_.sms = prop.multiProcessorCount;
  di_.dev = device_;
  if (stream) {
    stream_ = static_cast<cudaStream_t>(stream);
  } else {
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream create");
    own_stream_ = true;
  }
  comm_ = static_cast<ncclComm_t>(nccl_comm);
  for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "event create");
  preload_all_kernels();
}

Engine::~Engine() {
  if (stream_) cudaStreamSynchronize(stream_);
  drop_graphs();
  peer_release();
  if (opt_dev_) cudaFree(opt_dev_);
  if (desc_stream_) cudaStreamDestroy(desc_stream_);
  if (h2d_) cudaStreamSynchronize(h2d_);
  if (d2h_) cudaStreamSynchronize(d2h_);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  for (Staging& s : stage_) {
    if (s.ev) cudaEventDestroy(s.ev);
    if (s.ptr) cudaFreeHost(s.ptr);
  }
  for (char* p : stage_graveyard_) cudaFreeHost(p);
  for (int i = 0; i < 2; ++i)
    for (cudaEvent_t e : {hev_in_[i], hev_gfree_[i], hev_dec_[i], hev_out_[i]})
      if (e) cudaEventDestroy(e);
  if (hev_join_) cudaEventDestroy(hev_join_);
  if (h2d_) cudaStreamDestroy(h2d_);
  if (d2h_) cudaStreamDestroy(d2h_);
  if (ds_stream_) {
    cudaStreamSynchronize(ds_stream_);
    cudaEventDestroy(ds_fork_);
    cudaEventDestroy(ds_done_);
    cudaStreamDestroy(ds_stream_);
  }
  if (aux_) {
    cudaStreamSynchronize(aux_);
    cudaEventDestroy(aux_fork_);
    cudaEventDestroy(aux_join_);
    cudaStreamDestroy(aux_);
  }
  if (own_comm_ && comm_) nccl().CommDestroy(comm_);
  if (own_stream_ && stream_) cudaStreamDestroy(stream_);
}

void Engine::set_config(const CompressionConfig& cfg) {
  cfg.validate_for_world(world_);
  cfg_ = cfg;
}

void Engine::init_nccl(const uint8_t id[128]) {
  if (comm_) throw InvalidArgument("context already has an NCCL communicator");
  ncclUniqueId uid;
  static_assert(sizeof(uid) == 128, "ncclUniqueId size");
  std::memcpy(&uid, id, 128);
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  nccl_check(nccl().CommInitRank(&comm_, int(world_), uid, int(rank_)), "ncclCommInitRank");
  own_comm_ = true;
}

void Engine::last_timing(float out[kStages]) const {
  for (int i = 0; i < kStages; ++i) {
    out[i] = 0.f;
    if (timing_) cudaEventElapsedTime(&out[i], ev_[i], ev_[i + 1]);
  }
}

void Engine::span_reset() {
  if (!timing_) return;
  spans_ = static_cast<unsigned long long*>(ws_.get("kernel_spans", 4 * 8, false, stream_));
  const unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
  upload(init, sizeof(init), spans_);
}

void Engine::last_kernel_spans(float out_ms[2]) {
  out_ms[0] = out_ms[1] = 0.f;
  if (!timing_ || !spans_) return;
  unsigned long long t[4];
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  cuda_check(cudaMemcpy(t, spans_, sizeof(t), cudaMemcpyDeviceToHost), "D2H spans");
  for (int i = 0; i < 2; ++i)
    if (t[2 * i + 1] > t[2 * i] && t[2 * i] != ~0ull) out_ms[i] = float(double(t[2 * i + 1] - t[2 * i]) * 1e-6);
}

// Stage boundaries: CUDA events in timing mode, and always an NVTX range per
// stage (host-side enqueue spans for nsys / ncu --nvtx; no-ops without a tool).
void Engine::ev_record(int i) {
  static const char* const kStage[] = {"tagc:prep", "tagc:select_fused", "tagc:select_finish", "tagc:exchange",
                                       "tagc:decode"};
  if (nvtx_open_) nvtxRangeEnd(nvtx_range_);
  nvtx_open_ = i >= 0 && i < 5;
  if (nvtx_open_) nvtx_range_ = nvtxRangeStartA(kStage[i]);
  if (timing_) cuda_check(cudaEventRecord(ev_[i], stream_), "event record");
  static const bool probe = std::getenv("TAGC_TIMING_PROBE") != nullptr;
  if (timing_ && probe) {
    cudaStreamSynchronize(stream_);
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    std::fprintf(stderr, "[ev%d] host %.1f us\n", i, ts.tv_sec * 1e6 + ts.tv_nsec / 1e3);
  }
}

// One public call = one staging half (see engine.hpp). Nested public calls
// (the host-buffer path) share the outer call's half.
struct CallScope {
  Engine& e;
  explicit CallScope(Engine& en) : e(en) {
    if (e.call_depth_++ == 0) e.call_begin();
  }
  ~CallScope() {
    if (--e.call_depth_ == 0) e.call_end();
  }
};

void Engine::call_begin() {
  stage_cur_ ^= 1;
  Staging& s = stage_[stage_cur_];
  if (s.ev) cuda_check(cudaEventSynchronize(s.ev), "staging reuse");
  s.off = 0;
}

void Engine::call_end() {
  Staging& s = stage_[stage_cur_];
  if (!s.ev && cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming) != cudaSuccess) {
    s.ev = nullptr;
    return;
  }
  cudaEventRecord(s.ev, stream_);
}

void Engine::upload(const void* host, size_t bytes, void* dev) {
  if (!bytes) return;
  if (call_depth_ == 0) {  // internal helper called outside a public entry
    CallScope scope(*this);
    upload(host, bytes, dev);
    return;
  }
  if (capturing_ && std::find(capturing_->dev.begin(), capturing_->dev.end(), dev) != capturing_->dev.end()) {
    // a graph-private descriptor buffer: filled now, once, outside the graph
    if (!desc_stream_) cuda_check(cudaStreamCreateWithFlags(&desc_stream_, cudaStreamNonBlocking), "desc stream");
    cuda_check(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, desc_stream_), "descriptor copy");
    cuda_check(cudaStreamSynchronize(desc_stream_), "descriptor copy");
    return;
  }
  if (capturing_) {  // the graph re-reads these bytes on every replay: give them their own buffer
    char* h = nullptr;
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&h), align_up(bytes, 16), cudaHostAllocMapped),
               "graph staging alloc");
    capturing_->pinned.push_back(h);
    std::memcpy(h, host, bytes);
    void* dp = nullptr;
    cuda_check(cudaHostGetDevicePointer(&dp, h, 0), "graph staging map");
    launches_ += launch_stage_copy(dev, dp, align_up(bytes, 16), stream_);
    return;
  }
  Staging& s = stage_[stage_cur_];
  if (s.off + bytes > s.cap) stage_grow(s, bytes);
  std::memcpy(s.ptr + s.off, host, bytes);
  // the SMs pull the descriptors over PCIe (a copy-engine H2D would queue
  // behind the host-buffer path's bulk transfers); workspace destinations
  // have room for the 16-byte round-up
  launches_ += launch_stage_copy(dev, s.dev + s.off, align_up(bytes, 16), stream_);
  s.off = align_up(s.off + bytes, 256);
}

// A fresh staging buffer for the rest of the call. Earlier copies of this
// call may still read the old one: with a peer exchange attached it is kept
// (freed at destruction: cudaFreeHost would synchronise the device), else
// the stream is drained first.
void Engine::stage_grow(Staging& s, size_t bytes) {
  if (s.ptr) {
    if (peer_.region) {
      stage_graveyard_.push_back(s.ptr);
    } else {
      cuda_check(cudaStreamSynchronize(stream_), "staging grow");
      cudaFreeHost(s.ptr);
    }
  }
  s.ptr = nullptr;
  s.cap = std::max<size_t>(std::max<size_t>(2 * s.cap, align_up(bytes, 4096)), 1 << 20);
  s.off = 0;
  cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&s.ptr), s.cap, cudaHostAllocMapped), "staging alloc");
  void* dp = nullptr;
  cuda_check(cudaHostGetDevicePointer(&dp, s.ptr, 0), "staging map");
  s.dev = static_cast<char*>(dp);
}

void Engine::zero(const std::vector<std::pair<void*, uint64_t>>& ranges) {
  ZeroRanges r{};
  for (const auto& pr : ranges) {
    if (!pr.second) continue;
    if (r.n == kZeroRanges) {
      launches_ += launch_zero(r, stream_);
      r = ZeroRanges{};
    }
    r.ptr[r.n] = pr.first;
    r.bytes[r.n] = pr.second;
    ++r.n;
  }
  if (r.n) launches_ += launch_zero(r, stream_);
}

uint32_t* Engine::err_flag() {
  return static_cast<uint32_t*>(ws_.get("err", 64, true, stream_));
}

void Engine::fetch_rounds() {
  uint32_t q[4] = {0, 0, 0, 0};
  cuda_check(cudaMemcpyAsync(q, ws_.get("qcount", 16), 16, cudaMemcpyDeviceToHost, stream_), "D2H q");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  rounds_[0] = q[2];
  rounds_[1] = q[3];
}

// Index::to_bytes / CountSketch::to_bytes (index.cpp:59-69, sketch.cpp:77-89)
// are the little-endian word layout, i.e. the device buffers as they are:
// the wire format is a copy, ordered after this context's queued work.
void Engine::download(const void* dev, uint64_t bytes, void* host) {
  if (!bytes) return;
  cuda_check(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, stream_), "D2H wire bytes");
  cuda_check(cudaStreamSynchronize(stream_), "stream sync");
}

// err[0] doubles as the presence-validation word of the standalone decode
// entries; once read and reported it must not stay set, or the sticky NaN
// test of every later encode (k_encode, k_fused_tma) would skip its writes.
// TAGC_DEBUG_PEER=1: host-side phase trace of every exchange (rank, phase,
// wall clock), for diagnosing stalls of ranks sharing one device.
void Engine::trace(const char* phase) const {
  static const bool on = std::getenv("TAGC_DEBUG_PEER") != nullptr;
  if (!on) return;
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  std::fprintf(stderr, "[peer r%u/%u] %.6f %s\n", rank_, world_, double(ts.tv_sec) + ts.tv_nsec * 1e-9, phase);
}

void Engine::clear_err_word(uint32_t seen) {
  if (!seen) return;
  cuda_check(cudaMemsetAsync(err_flag(), 0, 4, stream_), "clear err");
  cuda_check(cudaStreamSynchronize(stream_), "clear err");
}

void Engine::sync_check() {
  trace("sync_check");
  if (h2d_) cuda_check(cudaStreamSynchronize(h2d_), "h2d sync");
  if (d2h_) cuda_check(cudaStreamSynchronize(d2h_), "d2h sync");
  cuda_check(cudaStreamSynchronize(stream_), "stream sync");
  uint32_t err[4] = {0, 0, 0, 0};
  cuda_check(cudaMemcpy(err, err_flag(), 16, cudaMemcpyDeviceToHost), "D2H err");
  if (err[0] || err[2]) {  // reported once: clear the sticky flags
    cuda_check(cudaMemset(err_flag(), 0, 4), "clear err");
    cuda_check(cudaMemset(err_flag() + 2, 0, 4), "clear err");
    cuda_check(cudaDeviceSynchronize(), "clear err");
  }
  if (err[0] & 1u) throw InvalidArgument("sparsify: NaN gradient value");
  if (err[2]) throw CudaError("peer exchange: a rank never signalled this step (timeout)");
}

// ------------------------------------------------------------ select/encode
void Engine::run_select_encode(std::vector<EncItem>& items, bool w4, const HashParams& hp,
                               bool want_kept, const char*) {
  const uint32_t n = uint32_t(items.size());
  if (n == 0) return;
  if (n > kMaxFlatItems) throw InvalidArgument("more than 4096 compressed segments in one call");
  bool select = (items[0].flags & kSelect) != 0;
  uint64_t tiles = 0, samples = 0, cand = 0, hi = 0;
  for (EncItem& e : items) {
    if (((e.flags & kSelect) != 0) != select) throw CudaError("mixed select batch");
    const uint64_t t = (uint64_t(e.n) + kTile - 1) / kTile;
    e.tile_begin = tiles;
    tiles += t;
    e.sample_begin = samples;
    e.sample_stride = 0;
    e.sample_tiles = 0;
    if (select && e.n > kSmallSegment) {
      // at most kSampleMaxTiles chunks per segment (2M samples): beyond that the
      // sample passes only widen nothing but their own HBM read
      const uint64_t stride = std::max<uint64_t>(std::max<uint64_t>(1, std::min<uint64_t>(kSampleMaxStride, t / 16)),
                                                 (t + kSampleMaxTiles - 1) / kSampleMaxTiles);
      e.sample_stride = uint32_t(stride);
      e.sample_tiles = uint32_t((t + stride - 1) / stride);
      samples += e.sample_tiles;
    }
    e.cand_off = cand;
    e.cand_cap = select ? (e.n <= kSmallSegment ? e.n : std::max<uint32_t>(kSmallSegment, e.n / 16)) : 0;
    cand += e.cand_cap;
    // speculatively kept elements number at most n - c when the bracket holds
    e.hi_off = hi;
    e.hi_cap = select ? uint32_t(std::min<uint64_t>(e.n, uint64_t(e.n - e.c) + 1024)) : 0;
    hi += e.hi_cap;
  }
  for (EncItem& e : items) e.mmul = fastmod_magic(e.m);
  // Sketches far beyond L2: defer their scatter to the region-ordered pass
  // (exchange path only, with selection; one span of < 2^32 floats).
  // Deferred items are grouped in sketch-address order into spans of at most
  // 2^27 floats (the deferred scatter's shared-memory path); a group is one
  // launch_deferred_scatter call.
  struct DsGroup {
    float* base;
    uint64_t span, cap;
  };
  std::vector<DsGroup> ds_groups;
  uint64_t ds_cap = 0;
  {
    auto big = [&](const EncItem& e) {
      return select && (e.flags & kHasAcc) && (e.flags & kWriteSketch) && big_sketch(uint64_t(hp.rows) * e.m);
    };
    std::vector<uint32_t> order;
    for (uint32_t i = 0; i < items.size(); ++i)
      if (big(items[i])) order.push_back(i);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return items[a].sketch < items[b].sketch; });
    // TAGC_DS_GROUP_SPAN (floats): a smaller span for tests (several groups)
    const uint64_t kGroupSpan = std::getenv("TAGC_DS_GROUP_SPAN")
                                           ? std::max<uint64_t>(1, std::strtoull(std::getenv("TAGC_DS_GROUP_SPAN"), nullptr, 10))
                                           : (1ull << 27);
    for (uint32_t i : order) {
      EncItem& e = items[i];
      const uint64_t len = uint64_t(hp.rows) * e.m;
      if (len > 0xFFFFFFFFull) continue;  // scattered directly (zeroed below)
      if (ds_groups.empty() || uint64_t(e.sketch + len - ds_groups.back().base) > kGroupSpan)
        ds_groups.push_back(DsGroup{e.sketch, 0, 0});
      DsGroup& g = ds_groups.back();
      g.span = std::max<uint64_t>(g.span, uint64_t(e.sketch + len - g.base));
      g.cap += uint64_t(hp.rows) * e.hi_cap;
      e.flags |= kDeferScatter;
      e.ds_group = uint32_t(ds_groups.size() - 1);
    }
    for (const DsGroup& g : ds_groups) ds_cap = std::max(ds_cap, g.cap);
    // The exchange prologue leaves big sketches unzeroed (big_sketch): the
    // deferred ones are written (or zeroed) by the deferred scatter, any
    // others now, before the scatter.
    std::vector<std::pair<void*, uint64_t>> now;
    for (const EncItem& e : items)
      if (big(e) && !(e.flags & kDeferScatter)) now.push_back({e.sketch, uint64_t(hp.rows) * e.m * 4});
    if (!now.empty()) zero(now);
  }
  auto* d_items = static_cast<EncItem*>(desc_buffer("enc_items", n * sizeof(EncItem)));
  upload(items.data(), n * sizeof(EncItem), d_items);
  auto* state = static_cast<SelState*>(ws_.get("sel_state", n * sizeof(SelState), true, stream_));
  uint32_t* err = err_flag();
  // per-batch words only (err[1] bracket miss, err[3] chunk counter); the
  // NaN (err[0]) and peer-timeout (err[2]) flags stay sticky until
  // sync_check reports them, so a later batch or call cannot erase them
  const uint64_t ds_words = ds_groups.size() * uint64_t(kDsMaxBins + 4);  // fill + ctl per group
  uint32_t* ds_fill = ds_groups.empty() ? nullptr
                                        : static_cast<uint32_t*>(ws_.get("ds_fill", ds_words * 4, false, stream_));
  zero({{err + 1, 4}, {err + 3, 4}, {ds_fill, ds_fill ? ds_words * 4 : 0}});
  if (select) {
    auto* sh = static_cast<uint32_t*>(ws_.get("sample_hist", size_t(n) * kSampleStride * 4, true, stream_));
    auto* fh = static_cast<uint32_t*>(ws_.get("fb_hist", size_t(n) * kRadixBins * 4, true, stream_));
    auto* fine = static_cast<uint32_t*>(ws_.get("fine_hist", size_t(n) * kRadixBins * 4, true, stream_));
    auto* cd = static_cast<uint2*>(ws_.get("cand", cand * 8, false, stream_));
    auto* hp_pool = static_cast<uint2*>(ws_.get("hi_pool", hi * 8, false, stream_));
    auto* sl = static_cast<uint32_t*>(ws_.get("sel_list", size_t(n) * 8192 * 4, false, stream_));
    // hook items carry an accumulator; the per-stage sparsify entry writes
    // separate sparse/residual outputs (one kind per batch)
    const int per_stage = (items[0].flags & kHasAcc) ? 0 : 1;
    bool all_aligned = true;  // bulk-copy staging needs 16-byte aligned g / acc
    for (const EncItem& e : items) all_aligned = all_aligned && (e.flags & kAligned16);
    for (const EncItem& e : items)
      if (((e.flags & kHasAcc) ? 0 : 1) != per_stage) throw CudaError("mixed fused batch");
    ev_record(1);
    uint64_t sketch_bytes = 0;  // scattered-into footprint of the batch
    for (const EncItem& e : items)  // deferred sketches are not scattered into by the fused pass
      sketch_bytes += ((e.flags & kWriteSketch) && !(e.flags & kDeferScatter)) ? uint64_t(hp.rows) * e.m * 4 : 0;
    launches_ += launch_select_fused(di_, d_items, state, n, tiles, samples, hp, w4, per_stage, sh, fine,
                                     cd, hp_pool, err, stream_, timing_ ? spans_ : nullptr,
                                     use_tma_ && all_aligned, sketch_bytes);
    ev_record(2);
    launches_ += launch_select_finish(di_, d_items, state, n, tiles, hp, w4, fine, fh, cd, hp_pool, sl,
                                      err, stream_);
    if (!ds_groups.empty()) {
      // bins x capacity, capacity = ceil(total / bins) * 17/16 + 1024 per bin
      // (k_ds_place): at most total * 17/16 + bins * 1026 records
      auto* rec = static_cast<uint2*>(ws_.get("ds_records", (ds_cap + ds_cap / 16 + 16 + uint64_t(kDsMaxBins) * 1026) * 8,
                                              false, stream_));
      auto* ovf = static_cast<uint2*>(ws_.get("ds_overflow", ds_cap * 8, false, stream_));
      cudaStream_t ds_s = stream_;
      if (ds_side_ok_) {  // overlaps the decode's list build (W == 1: the index is final here)
        if (!ds_stream_) {
          cuda_check(cudaStreamCreateWithFlags(&ds_stream_, cudaStreamNonBlocking), "ds stream");
          cuda_check(cudaEventCreateWithFlags(&ds_fork_, cudaEventDisableTiming), "ds event");
          cuda_check(cudaEventCreateWithFlags(&ds_done_, cudaEventDisableTiming), "ds event");
        }
        cuda_check(cudaEventRecord(ds_fork_, stream_), "ds fork");
        cuda_check(cudaStreamWaitEvent(ds_stream_, ds_fork_, 0), "ds fork wait");
        ds_s = ds_stream_;
      }
      for (uint32_t g = 0; g < ds_groups.size(); ++g) {  // groups share the record buffers: in stream order
        uint32_t* fill = ds_fill + uint64_t(g) * (kDsMaxBins + 4);
        const int l = launch_deferred_scatter(di_, d_items, state, n, g, hp_pool, hp, ds_groups[g].base,
                                              ds_groups[g].span, fill, fill + kDsMaxBins, rec, ovf, ds_s);
        if (l < 0) throw CudaError("deferred sketch scatter: span too large");
        launches_ += l;
      }
      if (ds_side_ok_) {
        cuda_check(cudaEventRecord(ds_done_, ds_stream_), "ds done");
        sketch_pending_ = true;
      }
    }
    ev_record(3);
    static const bool sel_dbg = std::getenv("TAGC_DEBUG_SELECT") != nullptr;
    if (sel_dbg && !capturing_) {  // per-item select outcome (debug only: synchronises)
      std::vector<SelState> hs(n);
      cuda_check(cudaMemcpyAsync(hs.data(), state, n * sizeof(SelState), cudaMemcpyDeviceToHost, stream_), "dbg");
      cuda_check(cudaStreamSynchronize(stream_), "dbg");
      for (uint32_t i = 0; i < n; ++i)
        if (hs[i].status != 0 || std::getenv("TAGC_DEBUG_SELECT")[0] == '2')
          std::fprintf(stderr, "select item %u n=%u c=%u Z=%u L=%u I=%u hi=%u caps=%u/%u win=[%08x,%08x] status=%u\n",
                       i, items[i].n, items[i].c, hs[i].cnt_zero, hs[i].cnt_lo, hs[i].cnt_in, hs[i].cnt_hi,
                       items[i].cand_cap, items[i].hi_cap, hs[i].klo, hs[i].khi, hs[i].status);
    }
  } else {
    zero({{state, n * sizeof(SelState)}});
    ev_record(1);
    ev_record(2);
    launches_ += launch_encode_exact(di_, d_items, state, n, tiles, hp, err, w4, stream_);
    ev_record(3);
  }
  (void)want_kept;
  cuda_check(cudaGetLastError(), "select/encode launch");
}

// ------------------------------------------------------------------ decode
cudaEvent_t Engine::take_sketch_event() {
  if (!sketch_pending_) return nullptr;
  sketch_pending_ = false;
  return ds_done_;
}

void Engine::join_sketch() {
  if (cudaEvent_t e = take_sketch_event()) cuda_check(cudaStreamWaitEvent(stream_, e, 0), "ds join");
}

void Engine::ensure_aux() {
  if (aux_) return;
  int lo = 0, hi = 0;  // lowest priority: decode kernels take SMs first as side CTAs retire
  cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
  cuda_check(cudaStreamCreateWithPriority(&aux_, cudaStreamNonBlocking, lo), "aux stream");
  cuda_check(cudaEventCreateWithFlags(&aux_fork_, cudaEventDisableTiming), "aux event");
  cuda_check(cudaEventCreateWithFlags(&aux_join_, cudaEventDisableTiming), "aux event");
}

// Decode of a batch of segments whose bucket states are far beyond L2
// (Llama-3-8B: 722M buckets at W = 1) in groups of <= kDecodeGroupBytes of
// randomly accessed bytes (byte counter + residual per bucket in counter
// mode: 96 MB; TAGC_DECODE_GROUP_MB): each group's list build, round-0 peel
// and frontier rounds then hit state the group's own REDs just left in L2,
// while the group count (10 launches each) stays low (Llama: 48 MB groups
// 22.6 ms of decode, 96 MB 18.1 ms, 320 MB 18.6 ms). Results are those of
// one batch (segments decode independently); statistics land per item.
void Engine::run_decode_grouped(std::vector<DecItem>& items, const HashParams& hp, bool ordered,
                                cudaEvent_t zero_done, const std::function<void()>& pre_launch) {
  static const uint64_t kDecodeGroupBytes =
      (std::getenv("TAGC_DECODE_GROUP_MB") ? std::strtoull(std::getenv("TAGC_DECODE_GROUP_MB"), nullptr, 10) : 96ull) << 20;
  constexpr uint64_t kGroupAbove = 128ull << 20;
  // randomly accessed bytes per bucket: the byte counter and the residual
  // (counter mode), else the u64 state and the residual
  const bool counters = !std::getenv("TAGC_DECODE_FULL_STATE");
  const uint64_t per_slot = counters ? 5 : 12;
  uint64_t state_bytes = 0;
  for (const DecItem& d : items) state_bytes += uint64_t(hp.rows) * d.m * per_slot;
  if (ordered || items.size() < 2 || state_bytes <= kGroupAbove) {
    run_decode(items, hp, false, ordered, zero_done, pre_launch);
    return;
  }
  const uint32_t n = uint32_t(items.size());
  ws_.get("dec_stats", n * sizeof(DecStats), false, stream_);  // sized once for every group
  size_t b = 0;
  bool first = true;
  while (b < items.size()) {
    size_t e = b;
    uint64_t bytes = 0;
    while (e < items.size() && (e == b || bytes + uint64_t(hp.rows) * items[e].m * per_slot <= kDecodeGroupBytes))
      bytes += uint64_t(hp.rows) * items[e++].m * per_slot;
    std::vector<DecItem> group(items.begin() + b, items.begin() + e);
    run_decode(group, hp, false, false, zero_done, first ? pre_launch : std::function<void()>(), uint32_t(b));
    first = false;
    b = e;
  }
  dec_stats_.assign(n, DecStats{});
}

void Engine::run_decode(std::vector<DecItem>& items, const HashParams& hp, bool want_unresolved,
                        bool ordered, cudaEvent_t zero_done, const std::function<void()>& pre_launch,
                        uint32_t stats_base) {
  const uint32_t n = uint32_t(items.size());
  dec_stats_.assign(n, DecStats{});
  if (n == 0) {
    if (pre_launch) pre_launch();
    return;
  }
  uint64_t slots = 0, bm = 0, wt = 0, list = 0;
  for (DecItem& d : items) {
    d.mmul = fastmod_magic(d.m);
    d.slot_base = slots;
    slots += uint64_t(hp.rows) * d.m;
    d.word_tile_begin = wt;
    wt += (uint64_t(d.n_words) + kDecWordTile - 1) / kDecWordTile;
    d.list_off = list;
    list += std::min(d.list_cap ? d.list_cap : d.n, d.n);
  }
  if (slots >= (1ull << 31)) throw CudaError("decode batch exceeds 2^31 sketch buckets");
  auto* d_items = static_cast<DecItem*>(desc_buffer("dec_items", n * sizeof(DecItem)));
  upload(items.data(), n * sizeof(DecItem), d_items);
  DecodeWork w{};
  w.span = timing_ ? spans_ + 2 : nullptr;
  w.items = d_items;
  w.n_items = n;
  w.total_word_tiles = wt;
  w.total_slots = slots;
  w.slot_state = static_cast<unsigned long long*>(ws_.get("slot_state", slots * 8, false, stream_));
  bm = (list + 31) / 32;
  w.bitmap = static_cast<uint32_t*>(ws_.get("bitmap", bm * 4, false, stream_));
  w.list_cap = list;
  w.val = static_cast<float*>(ws_.get("dec_val", list * 4, false, stream_));
  const uint64_t mark_words = (slots + 31) / 32;
  w.slot_mark = ordered ? nullptr : static_cast<uint32_t*>(ws_.get("slot_mark", mark_words * 4, false, stream_));
  w.tile_base = static_cast<uint32_t*>(ws_.get("tile_base", wt * 4, false, stream_));
  w.r0_list = static_cast<uint32_t*>(ws_.get("r0_list", list * 4 + 4, false, stream_));
  w.tile_state = static_cast<unsigned long long*>(ws_.get("tile_state", wt * 8 + 8, false, stream_));
  w.cta_cnt = static_cast<uint32_t*>(ws_.get("list_cta_cnt", 2 * kListMaxCtas * 4, false, stream_));
  static const uint32_t list_split = std::getenv("TAGC_LIST_SPLIT") ? std::max(1, std::min(2, std::atoi(std::getenv("TAGC_LIST_SPLIT")))) : 2u;
  w.list_split = list_split;
  w.plist = static_cast<uint32_t*>(ws_.get("plist", list * 4, false, stream_));
  w.pitem = static_cast<uint32_t*>(ws_.get("pitem", list * 4, false, stream_));
  w.pinfo = static_cast<uint2*>(ws_.get("pinfo", list * 8, false, stream_));
  w.queue[0] = static_cast<uint32_t*>(ws_.get("queue0", slots * 4, false, stream_));
  w.queue[1] = static_cast<uint32_t*>(ws_.get("queue1", slots * 4, false, stream_));
  w.qcount = static_cast<uint32_t*>(ws_.get("qcount", kQcountBytes, false, stream_));
  w.bar = static_cast<unsigned long long*>(ws_.get("peel_bar", 32, false, stream_));
  w.handoff = static_cast<uint2*>(ws_.get("peel_handoff", kPeelHandoff * sizeof(uint2), false, stream_));
  w.stats = static_cast<DecStats*>(ws_.get("dec_stats", (stats_base + n) * sizeof(DecStats), false, stream_)) +
            stats_base;
  w.unresolved = want_unresolved ? static_cast<uint32_t*>(ws_.get("unresolved", list * 4, false, stream_))
                                 : nullptr;
  // Counter mode: round 0 needs only "one entry or more" per bucket, so it
  // counts in bytes or nibbles (slots bytes instead of 8 * slots: 27 MB at 2^28 / r 10,
  // L2-resident) and the (count, index sum) state is built later for the few
  // buckets round 0 leaves unresolved. A byte counter is safe while a bucket
  // cannot plausibly hold 256 entries: the presence bound over the row
  // length stays <= 16 (Poisson tail ~1e-200), else the full state is used.
  // Nibble counters (half the footprint, so they stay in L2 under the list
  // build's streams) while the bound stays <= m / 2: P(Poisson(0.5) >= 16)
  // ~ 1e-18 per bucket.
  bool counters = !ordered && !std::getenv("TAGC_DECODE_FULL_STATE");
  bool nibbles = counters && !std::getenv("TAGC_DECODE_BYTE_COUNTERS");
  for (const DecItem& d : items) {
    const double bound = double(std::min(d.list_cap ? d.list_cap : d.n, d.n));
    counters = counters && bound <= 16.0 * double(d.m);
    nibbles = nibbles && bound <= 0.5 * double(d.m);
  }
  w.cnt_shift = nibbles ? 2u : 3u;
  // High load: round 0 leaves a large share of the entries unresolved, and
  // clearing their rows' states one random 8-byte store at a time costs more
  // than one streaming clear of the whole state. Expected unresolved entries
  // per item: bound * (1 - e^-lambda)^rows, lambda = bound / m (Poisson row
  // loads); each random store is charged 256 bytes against 8 per slot (the
  // measured break-even: C4 theta 95 clears up front, theta 98 does not).
  // TAGC_DECODE_ZERO_STATE=0/1 forces either way.
  bool zero_state = false;
  if (counters) {
    double unres = 0.0;
    for (const DecItem& d : items) {
      const double bound = double(std::min(d.list_cap ? d.list_cap : d.n, d.n));
      const double lam = bound / double(d.m);
      unres += bound * std::pow(1.0 - std::exp(-lam), double(hp.rows));
    }
    zero_state = unres * hp.rows * 256.0 > double(slots) * 8.0;
    if (const char* z = std::getenv("TAGC_DECODE_ZERO_STATE")) zero_state = std::atoi(z) != 0;
  }
  w.state_zeroed = zero_state ? 1u : 0u;
  const uint64_t cnt_words = nibbles ? (slots + 7) / 8 : (slots + 3) / 4;
  // round 0 inside the dense emit unless the owner step consumes the values
  const bool fused = counters && !ordered && !opt_on_ && fused_emit_;
  w.cnt8 = counters ? static_cast<uint32_t*>(ws_.get("cnt8", cnt_words * 4, false, stream_)) : nullptr;
  w.ulist = counters ? static_cast<uint32_t*>(ws_.get("ulist", list * 4 + 4, false, stream_)) : nullptr;
  const uint64_t wwords = mark_words + 1;
  w.wmask = ordered ? static_cast<uint32_t*>(ws_.get("ord_wmask", wwords * 4, false, stream_)) : nullptr;
  zero({{w.wmask, w.wmask ? wwords * 4 : 0},
        {w.bitmap, bm * 4}, {w.qcount, kQcountBytes}, {w.bar, 32}, {w.stats, n * sizeof(DecStats)},
        {w.slot_mark, w.slot_mark ? mark_words * 4 : 0},
        {counters ? static_cast<void*>(w.cnt8) : static_cast<void*>(w.slot_state), counters ? cnt_words * 4 : slots * 8},
        {zero_state ? static_cast<void*>(w.slot_state) : nullptr, zero_state ? slots * 8 : 0},
        {w.tile_state, wt * 8}});  // one launch for every decode scratch reset
  static const bool dbg = std::getenv("TAGC_DEBUG_PEEL") != nullptr;
  if (dbg) {
    w.dbg = static_cast<unsigned long long*>(ws_.get("peel_dbg", 64 * 8, false, stream_));
    cuda_check(cudaMemsetAsync(w.dbg, 0, 64 * 8, stream_), "dbg reset");
  }
  last_ordered_ = ordered;
  if (pre_launch) pre_launch();
  if (ordered) {
    // 1-bit merged index over several ranks: carries can hide positions whose
    // mass stays in the sketch, so values follow the reference's FIFO order
    if (slots * hp.rows >= (1ull << 32)) throw CudaError("ordered decode batch exceeds 2^32 FIFO keys");
    OrdState o{};
    o.slot_key_cap = slots;
    o.claim_cap = list;
    o.slot_key = static_cast<unsigned long long*>(ws_.get("ord_slot_key", slots * 8, true, stream_));
    o.claim = static_cast<unsigned long long*>(ws_.get("ord_claim", list * 8, true, stream_));
    o.dense = static_cast<uint32_t*>(ws_.get("ord_dense", (slots * hp.rows + 4) * 4, true, stream_));
    o.q = static_cast<uint32_t*>(ws_.get("ord_q", slots * 4, false, stream_));
    o.u0 = static_cast<uint32_t*>(ws_.get("ord_u0", slots * 4, false, stream_));
    o.u1 = static_cast<uint32_t*>(ws_.get("ord_u1", slots * 4, false, stream_));
    o.cta = static_cast<uint32_t*>(ws_.get("ord_cta", size_t(ordered_loop_grid(di_)) * 4, false, stream_));
    o.wmask = w.wmask;
    o.wrank = static_cast<uint32_t*>(ws_.get("ord_wrank", wwords * 4, false, stream_));
    o.wwords = wwords;
    o.epoch = static_cast<uint32_t*>(ws_.get("ord_epoch", 16, true, stream_));  // fixed size: never regrown
    if (!ord_epoch_set_) {  // test hook: start the epoch just below the wrap point
      ord_epoch_set_ = true;
      if (const char* e = std::getenv("TAGC_ORD_EPOCH_START")) {
        const uint32_t v = uint32_t(std::strtoul(e, nullptr, 0));
        zero({{o.epoch, 16}});
        launches_ += launch_set_u32(o.epoch, v, stream_);
      }
    }
    launches_ += launch_decode_ordered(di_, w, hp, o, stream_, take_sketch_event());
  } else {
    launches_ += launch_decode(di_, w, hp, stream_, fused, take_sketch_event());
  }
  if (zero_done) cuda_check(cudaStreamWaitEvent(stream_, zero_done, 0), "wait side stream");
  if (!fused) launches_ += launch_decode_emit(di_, w, stream_, opt_on_ ? opt_dev_ : nullptr);
  cuda_check(cudaGetLastError(), "decode launch");
  if (dbg) {
    unsigned long long t[64];
    cuda_check(cudaMemcpyAsync(t, w.dbg, sizeof(t), cudaMemcpyDeviceToHost, stream_), "dbg");
    cuda_check(cudaStreamSynchronize(stream_), "dbg sync");
    std::fprintf(stderr, "[peel]");
    for (int i = 1; i < 64 && t[i]; ++i) std::fprintf(stderr, " %.1f", (t[i] - t[i - 1]) / 1e3);
    std::fprintf(stderr, " us\n");
  }
}

// ------------------------------------------------------------ simulated world
void Engine::reduce_shard_sim(const ShardSpec& shard, uint32_t world, const float* const* grads,
                              float* const* accs, float* out, PeelStats* stats, float* audit) {
  CallScope scope(*this);
  if (world == 0) throw InvalidArgument("world size must be at least 1");
  cfg_.validate_for_world(world);  // hook.cpp:105
  check_shard(shard, world);
  launches_ = 0;
  ev_record(0);
  span_reset();
  const uint32_t w = cfg_.index_width, rows = cfg_.sketch_rows;
  std::vector<SegPlan> plan;
  uint64_t NW = 0, SK = 0;
  for (uint32_t i = 0; i < shard.segments.size(); ++i) {
    const LayerSegment& s = shard.segments[i];
    SegPlan p;
    p.seg = i;
    p.lo = s.begin - shard.begin;
    p.len = s.size();
    p.tag = "shard" + std::to_string(shard.id) + "/" + seg_name(s, i);
    p.compressed = kind_compressible(s.kind, cfg_.policy, cfg_.include_out_proj) &&
                   cfg_.ratio > 1 && p.len >= cfg_.min_compress_segment;  // hook.cpp:120-122
    if (p.compressed) {
      p.m = sketch_geometry(uint32_t(p.len), cfg_.ratio, rows).buckets_per_row;  // hook.cpp:138
      p.n_words = words_needed(uint32_t(p.len), w);
      p.word_off = NW;
      NW += align_up(p.n_words, 4);
      p.sk_off = SK;
      SK += align_up(uint64_t(rows) * p.m, 4);
    }
    plan.push_back(p);
  }
  const HashParams hp = make_hash_params(cfg_.seed, rows);
  auto* idx_all = static_cast<uint32_t*>(ws_.get("sim_idx", world * NW * 4, false, stream_));
  auto* sk_all = static_cast<float*>(ws_.get("sim_sk", world * SK * 4, false, stream_));
  auto* merged = static_cast<uint32_t*>(ws_.get("sim_merged", NW * 4, false, stream_));
  auto* summed = static_cast<float*>(ws_.get("sim_summed", SK * 4, false, stream_));
  // device pointer tables: [grads x world][idx x world][sk x world]
  std::vector<const void*> ptrs;
  for (uint32_t r = 0; r < world; ++r) ptrs.push_back(grads[r]);
  for (uint32_t r = 0; r < world; ++r) ptrs.push_back(idx_all + r * NW);
  for (uint32_t r = 0; r < world; ++r) ptrs.push_back(sk_all + r * SK);
  auto* d_ptrs = static_cast<const void**>(ws_.get("sim_ptrs", ptrs.size() * 8, false, stream_));
  upload(ptrs.data(), ptrs.size() * 8, d_ptrs);
  zero({{sk_all, world * SK * 4}});
  // collect_audit (hook.cpp:115, :191-195): every rank's combined g + acc is
  // kept before the encode overwrites acc with the residual
  const uint64_t len = shard.size();
  float* comb = nullptr;
  const void** d_audit_ptrs = nullptr;
  if (audit) {
    comb = static_cast<float*>(ws_.get("audit_comb", world * len * 4, false, stream_));
    for (uint32_t r = 0; r < world; ++r) launches_ += launch_add(grads[r], accs[r], comb + r * len, len, stream_);
    std::vector<const void*> ap;
    for (uint32_t r = 0; r < world; ++r) ap.push_back(comb + r * len);
    for (uint32_t r = 0; r < world; ++r) ap.push_back(accs[r]);
    d_audit_ptrs = static_cast<const void**>(ws_.get("audit_ptrs", ap.size() * 8, false, stream_));
    upload(ap.data(), ap.size() * 8, d_audit_ptrs);
    zero({{audit, len * 4}});
  }

  std::vector<EncItem> enc;
  for (uint32_t r = 0; r < world; ++r) {
    for (const SegPlan& p : plan) {
      if (!p.compressed) continue;
      EncItem e{};
      e.g = grads[r] + p.lo;
      e.acc = accs[r] + p.lo;
      e.index = idx_all + r * NW + p.word_off;
      e.sketch = sk_all + r * SK + p.sk_off;
      e.n = uint32_t(p.len);
      e.m = p.m;
      e.c = threshold_rank(cfg_.theta, p.len);
      e.flags = (w == 4 ? kWidth4 : 0u) | kHasAcc | kWriteIndex | kWriteSketch | kSelect |
                ((aligned16(e.g) && aligned16(e.acc)) ? kAligned16 : 0u);
      enc.push_back(e);
    }
  }
  run_select_encode(enc, w == 4, hp, false, "sim");
  if (audit) {  // rank-ordered sum of the exchanged sparse vectors, compressed segments only
    std::vector<AuditItem> ai;
    uint64_t max_n = 0;
    for (const SegPlan& p : plan)
      if (p.compressed) {
        ai.push_back(AuditItem{audit + p.lo, p.len, p.lo});
        max_n = std::max(max_n, p.len);
      }
    if (!ai.empty()) {
      auto* d_ai = static_cast<AuditItem*>(ws_.get("audit_items", ai.size() * sizeof(AuditItem), false, stream_));
      upload(ai.data(), ai.size() * sizeof(AuditItem), d_ai);
      launches_ += launch_audit(d_ai, uint32_t(ai.size()), max_n, reinterpret_cast<const float* const*>(d_audit_ptrs),
                                reinterpret_cast<const float* const*>(d_audit_ptrs + world), world, stream_);
    }
  }
  // exchange: ascending-rank folds (collectives.cpp:127-166)
  launches_ += launch_rank_sum_u32(reinterpret_cast<const uint32_t* const*>(d_ptrs + world), world,
                                   merged, NW, stream_);
  launches_ += launch_rank_sum_f32(reinterpret_cast<const float* const*>(d_ptrs + 2 * world), world,
                                   summed, SK, stream_);
  std::vector<RawItem> raw;
  uint64_t max_raw = 0;
  for (const SegPlan& p : plan)
    if (!p.compressed) {
      raw.push_back(RawItem{out + p.lo, p.len, p.lo});
      max_raw = std::max(max_raw, p.len);
    }
  if (!raw.empty()) {
    auto* d_raw = static_cast<RawItem*>(ws_.get("sim_raw", raw.size() * sizeof(RawItem), false, stream_));
    upload(raw.data(), raw.size() * sizeof(RawItem), d_raw);
    launches_ += launch_raw_sum(d_raw, uint32_t(raw.size()), max_raw,
                                reinterpret_cast<const float* const*>(d_ptrs), world, stream_);
  }
  ev_record(4);
  std::vector<DecItem> dec;
  std::vector<DiagItem> diag;
  uint32_t max_words = 0;
  for (const SegPlan& p : plan) {
    if (!p.compressed) continue;
    DecItem d{};
    d.words = merged + p.word_off;
    d.sketch = summed + p.sk_off;
    d.out = out + p.lo;
    d.n = uint32_t(p.len);
    d.m = p.m;
    d.flags = w == 4 ? kWidth4 : 0u;
    d.n_words = p.n_words;
    d.list_cap = presence_bound(p.len, cfg_.theta, world);
    dec.push_back(d);
    diag.push_back(DiagItem{merged + p.word_off, p.word_off, uint32_t(p.len), p.n_words, w, 0});
    max_words = std::max(max_words, p.n_words);
  }
  run_decode(dec, hp, false, w == 1 && world > 1);
  ev_record(5);
  unsigned long long* ls = nullptr;
  if (!diag.empty()) {
    auto* d_diag = static_cast<DiagItem*>(ws_.get("sim_diag", diag.size() * sizeof(DiagItem), false, stream_));
    upload(diag.data(), diag.size() * sizeof(DiagItem), d_diag);
    ls = static_cast<unsigned long long*>(ws_.get("sim_ls", diag.size() * 16, false, stream_));
    zero({{ls, diag.size() * 16}});
    launches_ += launch_index_diag(d_diag, uint32_t(diag.size()), max_words,
                                   reinterpret_cast<const uint32_t* const*>(d_ptrs + world), world, ls,
                                   stream_);
  }
  cuda_check(cudaGetLastError(), "sim launch");
  // ledger (hook.cpp:125-166)
  for (const SegPlan& p : plan) {
    if (p.compressed) {
      ledger_.record(CollectiveOp::all_reduce, "index/" + p.tag, p.len * w, p.len);
      ledger_.record(CollectiveOp::reduce, "sketch/" + p.tag, uint64_t(rows) * p.m * 32, p.len);
    } else {
      ledger_.record(CollectiveOp::reduce_scatter, "grad/" + p.tag, p.len * 32, p.len);
    }
  }
  if (stats) {
    std::vector<unsigned long long> lsh(diag.size() * 2, 0);
    dec_stats_.resize(dec.size());
    if (!dec.empty()) {
      cuda_check(cudaMemcpyAsync(dec_stats_.data(), ws_.get("dec_stats", 16), dec.size() * sizeof(DecStats),
                                 cudaMemcpyDeviceToHost, stream_), "D2H stats");
      cuda_check(cudaMemcpyAsync(lsh.data(), ls, lsh.size() * 8, cudaMemcpyDeviceToHost, stream_), "D2H ls");
    }
    sync_check();
    if (!dec.empty()) fetch_rounds();
    PeelStats st;
    for (size_t i = 0; i < dec.size(); ++i) {
      if (dec_stats_[i].overflow) throw CudaError("decode bucket state overflow");
      st.presence += dec_stats_[i].presence;
      st.unresolved += dec_stats_[i].unresolved;
      st.index_lost += lsh[2 * i];
      st.index_spurious += lsh[2 * i + 1];
    }
    st.peeled = st.presence - st.unresolved;
    st.compressed_segments = dec.size();
    st.baseline_segments = plan.size() - dec.size();
    *stats = st;
  }
}

void Engine::baseline_sim(const ShardSpec& shard, uint32_t world, const float* const* grads,
                          float* out) {
  CallScope scope(*this);
  if (world == 0) throw InvalidArgument("world size must be at least 1");
  check_shard(shard, world);
  launches_ = 0;
  auto* d_ptrs = static_cast<const float**>(ws_.get("base_ptrs", world * 8, false, stream_));
  upload(grads, world * 8, d_ptrs);
  launches_ += launch_rank_sum_f32(d_ptrs, world, out, shard.size(), stream_);
  cuda_check(cudaGetLastError(), "baseline launch");
  ledger_.record(CollectiveOp::reduce_scatter, "grad/shard" + std::to_string(shard.id),
                 shard.size() * 32, shard.size());
}

// ------------------------------------------------------------------ NCCL world
void Engine::record(CollectiveOp op, const std::string& tag, uint64_t bits, uint64_t params) {
  ledger_.record(op, tag, bits, params);
  if (capturing_) capturing_->ledger.push_back(LedgerEntry{op, tag, bits, params});
}

void Engine::set_graphs(bool on) {
  graphs_on_ = on;
  if (!on) drop_graphs();
}

void Engine::free_graph(GraphEntry& g) {
  if (g.exec) cudaGraphExecDestroy(g.exec);
  g.exec = nullptr;
  for (char* h : g.pinned) cudaFreeHost(h);
  for (void* d : g.dev) cudaFree(d);
  g.pinned.clear();
  g.dev.clear();
}

void* Engine::desc_buffer(const char* name, size_t bytes) {
  if (!capturing_) return ws_.get(name, bytes, false, stream_);
  void* d = nullptr;
  cuda_check(cudaMalloc(&d, align_up(std::max<size_t>(bytes, 16), 256)), "graph descriptor buffer");
  capturing_->dev.push_back(d);
  return d;
}

void Engine::drop_graphs() {
  if (!graphs_.empty() && stream_) cudaStreamSynchronize(stream_);
  for (auto& [k, g] : graphs_) free_graph(g);
  graphs_.clear();
  graph_seen_.clear();
}

void Engine::reduce_shards(const std::vector<ShardSpec>& shards, const float* grad, float* acc,
                           float* out, PeelStats* stats) {
  CallScope scope(*this);
  cfg_.validate_for_world(world_);
  for (const ShardSpec& s : shards) check_shard(s, world_);
  if (world_ > 1 && !comm_ && !peer_.attached)
    throw InvalidArgument("multi-rank context has no NCCL communicator or peer exchange");
  static const bool peel_dbg = std::getenv("TAGC_DEBUG_PEEL") != nullptr;
  const bool legacy = stream_ == nullptr || stream_ == cudaStreamLegacy || stream_ == cudaStreamPerThread;
  // default streams cannot be captured
  const bool eligible = graphs_on_ && !stats && !timing_ && !peel_dbg && !legacy;
  if (!eligible) {
    enqueue_reduce_shards(shards, grad, acc, out, stats);
    return;
  }
  // key: everything the enqueued work depends on
  std::string key;
  {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "%p|%p|%p|%p|%d|%d|%.17g|%u|%u|%d|%d|%llu|%u|%llu|", (void*)grad, (void*)acc,
                  (void*)out, (void*)grad_read_ev_, int(opt_on_), peer_.attached ? peer_.set : -1, cfg_.theta, cfg_.ratio, cfg_.index_width, int(cfg_.policy),
                  int(cfg_.include_out_proj), (unsigned long long)cfg_.seed, cfg_.sketch_rows,
                  (unsigned long long)cfg_.min_compress_segment);
    key = buf;
    for (const ShardSpec& sh : shards) {
      std::snprintf(buf, sizeof(buf), "S%u,%u,%llu,%llu:", sh.id, sh.owner, (unsigned long long)sh.begin,
                    (unsigned long long)sh.end);
      key += buf;
      for (const LayerSegment& g : sh.segments) {
        std::snprintf(buf, sizeof(buf), "%d,%llu,%llu,", int(g.kind), (unsigned long long)g.begin,
                      (unsigned long long)g.end);
        key += buf;
        key += g.name;
        key += ';';
      }
    }
  }
  static const bool graph_dbg = std::getenv("TAGC_DEBUG_GRAPH") != nullptr;
  auto it = graphs_.find(key);
  if (graph_dbg)
    std::fprintf(stderr, "graph: %s key %zx gen %llu (cached gen %lld) seen %d graphs %zu\n",
                 it == graphs_.end() ? "miss" : "hit", std::hash<std::string>{}(key),
                 (unsigned long long)ws_.generation(), it == graphs_.end() ? -1ll : (long long)it->second.gen,
                 graph_seen_.count(key) ? graph_seen_[key] : 0, graphs_.size());
  if (it != graphs_.end() && it->second.gen != ws_.generation()) {
    drop_graphs();  // a workspace buffer moved: every captured pointer is suspect
    it = graphs_.end();
  }
  if (it != graphs_.end()) {
    GraphEntry& g = it->second;
    cuda_check(cudaGraphLaunch(g.exec, stream_), "graph launch");
    if (peer_.attached && world_ > 1) peer_.set ^= 1;  // the captured call used (and flipped) this set
    launches_ = g.launches;
    for (const LedgerEntry& l : g.ledger) ledger_.record(l.op, l.tag, l.bits, l.params);
    ledger_.wire_bytes += g.wire;
    return;
  }
  if (graph_seen_[key]++ == 0) {  // first sighting: run eagerly (sizes the workspace)
    enqueue_reduce_shards(shards, grad, acc, out, stats);
    return;
  }
  // second sighting: capture, then replay from now on (a bounded cache: a
  // caller cycling through many buffer sets starts over)
  if (graphs_.size() >= kMaxGraphs) drop_graphs();
  GraphEntry g;
  const uint64_t gen0 = ws_.generation(), wire0 = ledger_.wire_bytes;
  cudaGraph_t graph = nullptr;
  if (cudaStreamBeginCapture(stream_, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
    cudaGetLastError();
    graph_seen_[key] = -1000000;  // this stream cannot be captured: stay eager
    enqueue_reduce_shards(shards, grad, acc, out, stats);
    return;
  }
  capturing_ = &g;
  const int set0 = peer_.set;  // the captured enqueue flips it; an eager re-run must start from it
  bool ok = true;
  try {
    enqueue_reduce_shards(shards, grad, acc, out, nullptr);
  } catch (...) {
    ok = false;
  }
  capturing_ = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(stream_, &graph);
  cudaGetLastError();
  ok = ok && ce == cudaSuccess && graph && ws_.generation() == gen0;
  if (ok && cudaGraphInstantiate(&g.exec, graph, 0) != cudaSuccess) {
    cudaGetLastError();
    ok = false;
  }
  // upload now, so the first replay does not pay for it
  if (ok && cudaGraphUpload(g.exec, stream_) != cudaSuccess) cudaGetLastError();
  if (graph) cudaGraphDestroy(graph);
  if (!ok) {  // could not capture (e.g. a buffer had to grow): stay eager for this key
    peer_.set = set0;
    free_graph(g);
    ledger_.wire_bytes = wire0;
    for (const LedgerEntry& l : g.ledger) ledger_.unrecord(l.op, l.tag, l.bits, l.params);
    graph_seen_[key] = -1000000;
    enqueue_reduce_shards(shards, grad, acc, out, stats);
    return;
  }
  g.gen = gen0;
  g.launches = launches_;
  g.wire = ledger_.wire_bytes - wire0;
  cuda_check(cudaGraphLaunch(g.exec, stream_), "graph launch");
  graphs_.emplace(key, std::move(g));
}

// First half of an exchange (reference hook.cpp:137-163): encode every
// compressed segment into its owner's send blocks, pack raw segments (W > 1)
// or copy them to the output (W == 1, side stream). State for exchange_end
// stays in xs_. Split into prologue / encode / seal so that the overlap
// entry points can encode segments as their gradients become ready.
void Engine::exchange_begin(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                            float* user_send_f, uint32_t* user_send_u) {
  exchange_prologue(shards, grad, acc, out, user_send_f, user_send_u);
  exchange_encode(0, ~0ull);
  exchange_seal();
}

void Engine::exchange_prologue(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                               float* user_send_f, uint32_t* user_send_u) {
  launches_ = 0;
  ev_record(0);
  span_reset();
  const uint32_t W = world_;
  xs_ = ExchangeState{};
  xs_.shards = shards;
  xs_.out = out;
  xs_.grad = grad;
  xs_.acc = acc;
  xs_.P = plan_exchange(shards, cfg_, W, rank_);
  const ExchangePlan& P = xs_.P;
  xs_.encoded.assign(P.segs.size(), 0);
  const uint64_t Bf = P.Bf, Bu = P.Bu;
  auto* send_f = user_send_f ? user_send_f : static_cast<float*>(ws_.get("nc_send_f", W * Bf * 4, false, stream_));
  auto* send_u = user_send_u ? user_send_u : static_cast<uint32_t*>(ws_.get("nc_send_u", W * Bu * 4, false, stream_));
  xs_.send_f = send_f;
  xs_.send_u = send_u;
  // every owner block's sketches start at zero; big ones (deferred scatter)
  // are zeroed by the encode itself, just before their REDs
  std::vector<std::pair<void*, uint64_t>> zr;
  const uint32_t rows = cfg_.sketch_rows;
  for (uint32_t o = 0; o < W; ++o) {
    uint64_t run = 0, end = 0;  // current run of small sketches [run, end)
    for (const SegPlan& p : P.segs) {
      if (!p.compressed || shards[p.shard].owner != o) continue;
      const uint64_t sk = uint64_t(rows) * p.m;
      if (big_sketch(sk)) {
        if (end > run) zr.push_back({send_f + o * Bf + run, (end - run) * 4});
        run = end = p.sk_off + align_up(sk, 4);
      } else {
        end = p.sk_off + align_up(sk, 4);
      }
    }
    if (end > run) zr.push_back({send_f + o * Bf + run, (end - run) * 4});
  }
  zero(zr);
  xs_.begun = true;
}

// Encodes the not yet encoded segments lying inside the flat range [lo, hi).
void Engine::exchange_encode(uint64_t lo, uint64_t hi) {
  if (!xs_.begun || xs_.active) throw InvalidArgument("no exchange is open for encoding");
  const std::vector<ShardSpec>& shards = xs_.shards;
  const ExchangePlan& P = xs_.P;
  const std::vector<SegPlan>& plan = P.segs;
  const uint32_t W = world_, w = cfg_.index_width;
  const uint64_t Bf = P.Bf, Bu = P.Bu;
  float* send_f = xs_.send_f;
  uint32_t* send_u = xs_.send_u;
  const float* grad = xs_.grad;
  float* acc = xs_.acc;
  float* out = xs_.out;
  const HashParams hp = make_hash_params(cfg_.seed, cfg_.sketch_rows);
  std::vector<EncItem> enc;
  std::vector<CopyItem> pack, side;
  for (size_t i = 0; i < plan.size(); ++i) {
    const SegPlan& p = plan[i];
    const ShardSpec& sh = shards[p.shard];
    const uint64_t b = sh.begin + p.lo, e = b + p.len;
    if (xs_.encoded[i] || b < lo || e > hi) continue;
    xs_.encoded[i] = 1;
    const uint32_t o = sh.owner;
    if (p.compressed) {
      EncItem it{};
      it.g = grad + b;
      it.acc = acc + b;
      it.index = send_u + o * Bu + p.word_off;
      it.sketch = send_f + o * Bf + p.sk_off;
      it.n = uint32_t(p.len);
      it.m = p.m;
      it.c = threshold_rank(cfg_.theta, p.len);
      it.flags = (w == 4 ? kWidth4 : 0u) | kHasAcc | kWriteIndex | kWriteSketch | kSelect |
                 ((aligned16(it.g) && aligned16(it.acc)) ? kAligned16 : 0u);
      enc.push_back(it);
    } else if (W == 1) {  // no exchange: raw segments go straight to the output
      side.push_back(CopyItem{grad + b, out + P.out_off[p.shard] + p.lo, p.len, 0});
    } else {
      pack.push_back(CopyItem{grad + b, send_f + o * Bf + p.raw_off, p.len, 0});
    }
  }
  ds_side_ok_ = W == 1;
  run_select_encode(enc, w == 4, hp, false, "nccl");
  ds_side_ok_ = false;
  // raw segments (W > 1): packed into the send blocks before the exchange
  if (!pack.empty()) {
    const uint64_t tt = copy_tiles(pack.data(), uint32_t(pack.size()));
    auto* d_pack = static_cast<CopyItem*>(desc_buffer("nc_pack", pack.size() * sizeof(CopyItem)));
    upload(pack.data(), pack.size() * sizeof(CopyItem), d_pack);
    launches_ += launch_copy_items(di_, d_pack, uint32_t(pack.size()), tt, stream_);
  }
  // Side stream (W == 1), overlapping the latency-bound decode: the raw
  // segments copied straight from the gradient to the output.
  if (!side.empty() && !side_stream_) {  // in order on the context stream
    const uint64_t tt = copy_tiles(side.data(), uint32_t(side.size()));
    auto* d_side = static_cast<CopyItem*>(desc_buffer("nc_side", side.size() * sizeof(CopyItem)));
    upload(side.data(), side.size() * sizeof(CopyItem), d_side);
    launches_ += launch_copy_items(di_, d_side, uint32_t(side.size()), tt, stream_, false,
                                   opt_on_ ? opt_dev_ : nullptr);
  } else if (!side.empty()) {
    ensure_aux();
    const uint64_t tt = copy_tiles(side.data(), uint32_t(side.size()));
    auto* d_side = static_cast<CopyItem*>(desc_buffer("nc_side", side.size() * sizeof(CopyItem)));
    upload(side.data(), side.size() * sizeof(CopyItem), d_side);
    cuda_check(cudaEventRecord(aux_fork_, stream_), "fork");
    cuda_check(cudaStreamWaitEvent(aux_, aux_fork_, 0), "fork wait");
    launches_ += launch_copy_items(di_, d_side, uint32_t(side.size()), tt, aux_, true,
                                   opt_on_ ? opt_dev_ : nullptr);
    xs_.side_used = true;
  }
}

// Encodes whatever is left, then marks the end of the gradient reads.
void Engine::exchange_seal() {
  exchange_encode(0, ~0ull);
  const auto ev_flags = capturing_ ? cudaEventRecordExternal : 0u;  // external: waited on outside the graph
  cudaEvent_t zero_done = nullptr;
  if (xs_.side_used) {
    cuda_check(cudaEventRecord(aux_join_, aux_), "join");
    zero_done = aux_join_;
  }
  // after this the gradient is no longer read
  if (grad_read_ev_) {
    if (world_ == 1 && zero_done) cuda_check(cudaStreamWaitEvent(stream_, zero_done, 0), "wait raw copy");
    cuda_check(cudaEventRecordWithFlags(grad_read_ev_, stream_, ev_flags), "grad-read event");
  }
  xs_.zero_done = zero_done;
  xs_.begun = false;
  xs_.active = true;
}

void Engine::enqueue_reduce_shards(const std::vector<ShardSpec>& shards, const float* grad, float* acc,
                                   float* out, PeelStats* stats) {
  trace("enqueue begin");
  open_exchange(shards, grad, acc, out);
  exchange_encode(0, ~0ull);
  trace("encode enqueued");
  finish_exchange(stats);
  trace("enqueue end");
}

// Prologue with this context's transport buffers: the peer region's current
// send set when the exchange runs over peer memory, else the workspace.
void Engine::open_exchange(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out) {
  if (peer_.attached && world_ > 1) {
    const int set = peer_.set;
    exchange_prologue(shards, grad, acc, out, peer_.view.send_f[set][rank_], peer_.view.send_u[set][rank_]);
    if (xs_.P.Bf != peer_.Bf || xs_.P.Bu != peer_.Bu) {
      xs_ = ExchangeState{};
      throw InvalidArgument("shard layout differs from the one the peer exchange was prepared for");
    }
    return;
  }
  exchange_prologue(shards, grad, acc, out);
}

// Seal, the collective (peer pulls or grouped NCCL reduce-scatters), decode.
void Engine::finish_exchange(PeelStats* stats) {
  exchange_seal();
  const uint32_t W = world_;
  if (peer_.attached && W > 1) {  // collective by pulls over peer memory
    const int set = peer_.set;
    auto* recv_f = static_cast<float*>(ws_.get("nc_recv_f", peer_.Bf * 4, false, stream_));
    auto* recv_u = static_cast<uint32_t*>(ws_.get("nc_recv_u", peer_.Bu * 4, false, stream_));
    uint32_t* err = err_flag();
    // the signal / wait / pull go in after the decode's allocations: a
    // cudaMalloc behind a wait for peers could stall this rank (and, with all
    // ranks in one process, every rank)
    // the send set flips as soon as the pull is enqueued: a later throw
    // (stats sync, NaN, timeout) must not leave this rank on the other set
    xs_.peer_set = set;
    exchange_end(recv_f, recv_u, stats, [&] {
      trace("peer exchange enqueue");
      launches_ += launch_peer_exchange(di_, peer_.view, set, recv_f, recv_u, err, stream_);
      peer_.set = set ^ 1;
      ledger_.wire_bytes += uint64_t(world_) * (peer_.Bf + peer_.Bu) * 4;
      ev_record(4);
    });
    return;
  }
  const uint64_t Bf = xs_.P.Bf, Bu = xs_.P.Bu;
  float* send_f = xs_.send_f;
  uint32_t* send_u = xs_.send_u;
  float* recv_f = send_f;
  uint32_t* recv_u = send_u;
  if (W > 1 || (force_collective_ && comm_)) {
    if (!comm_) throw InvalidArgument("multi-rank context has no NCCL communicator or peer exchange");
    join_sketch();  // W == 1 side-stream scatter: the sketches are final before they are sent
    recv_f = static_cast<float*>(ws_.get("nc_recv_f", Bf * 4, false, stream_));
    recv_u = static_cast<uint32_t*>(ws_.get("nc_recv_u", Bu * 4, false, stream_));
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    nccl_check(nccl().ReduceScatter(send_f, recv_f, Bf, ncclFloat32, ncclSum, comm_, stream_),
               "ncclReduceScatter f32");
    nccl_check(nccl().ReduceScatter(send_u, recv_u, Bu, ncclUint32, ncclSum, comm_, stream_),
               "ncclReduceScatter u32");
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
    ledger_.wire_bytes += W * (Bf + Bu) * 4;
    if (stats && cfg_.index_width == 1) {  // index_lost / _spurious need the OR of the supports
      auto* sup_send = static_cast<uint8_t*>(ws_.get("sup_send", W * Bu * 32, false, stream_));
      auto* sup_recv = static_cast<uint8_t*>(ws_.get("sup_recv", Bu * 32, false, stream_));
      launches_ += launch_support_bytes(send_u, W * Bu, sup_send, stream_);
      nccl_check(nccl().ReduceScatter(sup_send, sup_recv, Bu * 32, ncclUint8, ncclMax, comm_, stream_),
                 "ncclReduceScatter support");
      xs_.support_recv = sup_recv;
    }
  }
  ev_record(4);
  exchange_end(recv_f, recv_u, stats);
}

// Overlap entry points: the exchange opened before the
// gradient exists, each segment encoded as soon as the range holding it is
// ready (after `ready` on the producer's stream), the collective and decode
// once every range is in.
void Engine::overlap_begin(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out) {
  CallScope scope(*this);
  cfg_.validate_for_world(world_);
  for (const ShardSpec& s : shards) check_shard(s, world_);
  if (world_ > 1 && !comm_ && !peer_.attached)
    throw InvalidArgument("multi-rank context has no NCCL communicator or peer exchange");
  if (xs_.begun || xs_.active) throw InvalidArgument("an exchange is already in progress on this context");
  open_exchange(shards, grad, acc, out);
}

void Engine::overlap_ready(uint64_t lo, uint64_t hi, cudaEvent_t ready) {
  CallScope scope(*this);
  if (!xs_.begun) throw InvalidArgument("no overlapped exchange is open");
  if (ready) cuda_check(cudaStreamWaitEvent(stream_, ready, 0), "wait for the gradient producer");
  exchange_encode(lo, hi);
}

void Engine::overlap_finish(PeelStats* stats) {
  CallScope scope(*this);
  if (!xs_.begun) throw InvalidArgument("no overlapped exchange is open");
  finish_exchange(stats);
}

// Second half (hook.cpp:164-189): decode this rank's owned compressed
// segments from the reduced blocks and unpack its raw segments.
void Engine::exchange_end(const float* recv_f_in, const uint32_t* recv_u_in, PeelStats* stats,
                          const std::function<void()>& pre_decode) {
  if (!xs_.active) throw InvalidArgument("no exchange in progress");
  xs_.active = false;
  const std::vector<ShardSpec>& shards = xs_.shards;
  const ExchangePlan& P = xs_.P;
  const std::vector<SegPlan>& plan = P.segs;
  const std::vector<uint64_t>& out_off = P.out_off;
  const uint32_t W = world_, w = cfg_.index_width, rows = cfg_.sketch_rows;
  float* out = xs_.out;
  float* recv_f = const_cast<float*>(recv_f_in);
  uint32_t* recv_u = const_cast<uint32_t*>(recv_u_in);
  const HashParams hp = make_hash_params(cfg_.seed, rows);
  const cudaEvent_t zero_done = xs_.zero_done;
  std::vector<CopyItem> unpack;
  for (const SegPlan& p : plan)
    if (!p.compressed && W > 1 && shards[p.shard].owner == rank_)
      unpack.push_back(CopyItem{recv_f + p.raw_off, out + out_off[p.shard] + p.lo, p.len, 0});
  std::vector<DecItem> dec;
  for (const SegPlan& p : plan) {
    if (!p.compressed || shards[p.shard].owner != rank_) continue;
    DecItem d{};
    d.words = recv_u + p.word_off;
    d.sketch = recv_f + p.sk_off;
    d.out = out + out_off[p.shard] + p.lo;
    d.n = uint32_t(p.len);
    d.m = p.m;
    d.flags = w == 4 ? kWidth4 : 0u;
    d.n_words = p.n_words;
    d.list_cap = presence_bound(p.len, cfg_.theta, W);
    dec.push_back(d);
  }
  run_decode_grouped(dec, hp, w == 1 && W > 1, zero_done, pre_decode);
  join_sketch();  // no owned compressed segment decoded: the side scatter still joins here
  // index_lost / index_spurious (hook.cpp:176-188). A 4-bit index is exact
  // for W <= 15 (config.cpp:55-58): both are 0. A 1-bit index over several
  // ranks compares the merged words with the OR of the ranks' supports.
  unsigned long long* ls = nullptr;
  bool diag_unavailable = false;
  if (stats && w == 1 && W > 1 && !dec.empty()) {
    std::vector<DiagItem> diag;
    uint32_t max_words = 0;
    for (const SegPlan& p : plan) {
      if (!p.compressed || shards[p.shard].owner != rank_) continue;
      diag.push_back(DiagItem{recv_u + p.word_off, p.word_off, uint32_t(p.len), p.n_words, 1u, 0u});
      max_words = std::max(max_words, p.n_words);
    }
    ls = static_cast<unsigned long long*>(ws_.get("diag_ls", diag.size() * 16, false, stream_));
    zero({{ls, diag.size() * 16}});
    auto* d_diag = static_cast<DiagItem*>(ws_.get("diag_items", diag.size() * sizeof(DiagItem), false, stream_));
    upload(diag.data(), diag.size() * sizeof(DiagItem), d_diag);
    if (xs_.support_recv) {
      launches_ += launch_index_diag_support(d_diag, uint32_t(diag.size()), max_words, xs_.support_recv, ls,
                                             stream_);
    } else if (peer_.attached && xs_.peer_set >= 0) {
      // the peers' send blocks of this step still hold their own words: a
      // peer reuses the set only after this rank signals the next step
      std::vector<const uint32_t*> rw;
      for (uint32_t q = 0; q < W; ++q) rw.push_back(peer_.view.send_u[xs_.peer_set][q] + uint64_t(rank_) * P.Bu);
      auto* d_rw = static_cast<const uint32_t**>(ws_.get("diag_rw", W * 8, false, stream_));
      upload(rw.data(), W * 8, d_rw);
      launches_ += launch_index_diag(d_diag, uint32_t(diag.size()), max_words, d_rw, W, ls, stream_);
    } else {
      diag_unavailable = true;  // split API without support blocks
    }
  }
  if (W > 1 && !unpack.empty()) {
    const uint64_t tt = copy_tiles(unpack.data(), uint32_t(unpack.size()));
    auto* d_un = static_cast<CopyItem*>(desc_buffer("nc_unpack", unpack.size() * sizeof(CopyItem)));
    upload(unpack.data(), unpack.size() * sizeof(CopyItem), d_un);
    launches_ += launch_copy_items(di_, d_un, uint32_t(unpack.size()), tt, stream_, false, opt_on_ ? opt_dev_ : nullptr);
  }
  ev_record(5);
  cuda_check(cudaGetLastError(), "nccl-world launch");
  uint64_t n_raw_owned = 0;
  for (const SegPlan& p : plan) {
    if (p.compressed) {
      record(CollectiveOp::all_reduce, "index/" + p.tag, p.len * w, p.len);
      record(CollectiveOp::reduce, "sketch/" + p.tag, uint64_t(rows) * p.m * 32, p.len);
    } else {
      record(CollectiveOp::reduce_scatter, "grad/" + p.tag, p.len * 32, p.len);
      if (shards[p.shard].owner == rank_) ++n_raw_owned;
    }
  }
  if (stats) {
    dec_stats_.resize(dec.size());
    std::vector<unsigned long long> lsh(ls ? dec.size() * 2 : 0, 0);
    // drain the stream BEFORE the pageable copies: a pageable D2H queued
    // behind this rank's wait for its peers blocks inside the driver and
    // stalls every other host thread's CUDA calls (ranks sharing a process)
    sync_check();
    if (!dec.empty())
      cuda_check(cudaMemcpyAsync(dec_stats_.data(), ws_.get("dec_stats", 16), dec.size() * sizeof(DecStats),
                                 cudaMemcpyDeviceToHost, stream_), "D2H stats");
    if (ls) cuda_check(cudaMemcpyAsync(lsh.data(), ls, lsh.size() * 8, cudaMemcpyDeviceToHost, stream_), "D2H ls");
    cuda_check(cudaStreamSynchronize(stream_), "stats sync");
    if (!dec.empty()) fetch_rounds();
    PeelStats st;
    for (const DecStats& d : dec_stats_) {
      if (d.overflow) throw CudaError("decode bucket state overflow");
      st.presence += d.presence;
      st.unresolved += d.unresolved;
    }
    st.peeled = st.presence - st.unresolved;
    for (size_t i = 0; i + 1 < lsh.size(); i += 2) {
      st.index_lost += lsh[i];
      st.index_spurious += lsh[i + 1];
    }
    if (diag_unavailable) st.index_lost = st.index_spurious = kStatUnavailable;
    st.compressed_segments = dec.size();
    st.baseline_segments = n_raw_owned;
    *stats = st;
  }
}

void Engine::exchange_support(uint8_t** send_support, uint64_t* block_bytes) {
  CallScope scope(*this);
  if (!xs_.active) throw InvalidArgument("no exchange in progress");
  if (cfg_.index_width != 1) throw InvalidArgument("support blocks are only needed for a 1-bit index");
  const uint64_t Bu = xs_.P.Bu;
  uint8_t* dst = send_support && *send_support
                     ? *send_support
                     : static_cast<uint8_t*>(ws_.get("sup_send", world_ * Bu * 32, false, stream_));
  launches_ += launch_support_bytes(xs_.send_u, world_ * Bu, dst, stream_);
  cuda_check(cudaGetLastError(), "support launch");
  if (send_support) *send_support = dst;
  if (block_bytes) *block_bytes = Bu * 32;
}

void Engine::reduce_shards_audit(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                                 PeelStats* stats, float* audit) {
  CallScope scope(*this);
  if (world_ > 1 && !comm_)
    throw InvalidArgument("audit_exchanged_sum needs the NCCL exchange (or the simulated world)");
  cfg_.validate_for_world(world_);
  uint64_t total = 0;
  for (const ShardSpec& s : shards) {
    check_shard(s, world_);
    total = std::max<uint64_t>(total, s.end);
  }
  // combined g + acc before the encode overwrites acc with the residual
  auto* comb = static_cast<float*>(ws_.get("audit_comb", total * 4, false, stream_));
  launch_add(grad, acc, comb, total, stream_);
  enqueue_reduce_shards(shards, grad, acc, out, stats);
  const ExchangePlan P = plan_exchange(shards, cfg_, world_, rank_);
  const uint32_t W = world_;
  std::vector<uint64_t> used(W, 0), aoff(P.segs.size(), 0);
  for (size_t k = 0; k < P.segs.size(); ++k) {
    const SegPlan& p = P.segs[k];
    if (!p.compressed) continue;
    const uint32_t o = shards[p.shard].owner;
    aoff[k] = used[o];
    used[o] += p.len;
  }
  uint64_t Ba = 0;
  for (uint64_t u : used) Ba = std::max(Ba, u);
  Ba = align_up(std::max<uint64_t>(Ba, 1), 32);
  auto* send = static_cast<float*>(ws_.get("audit_send", W * Ba * 4, false, stream_));
  zero({{send, W * Ba * 4}});
  std::vector<AuditItem> ai;
  uint64_t max_n = 0;
  for (size_t k = 0; k < P.segs.size(); ++k) {
    const SegPlan& p = P.segs[k];
    if (!p.compressed) continue;
    ai.push_back(AuditItem{send + shards[p.shard].owner * Ba + aoff[k], p.len, shards[p.shard].begin + p.lo});
    max_n = std::max(max_n, p.len);
  }
  const void* ptrs[2] = {comb, acc};
  auto* d_ptrs = static_cast<const void**>(ws_.get("audit_ptrs", 16, false, stream_));
  upload(ptrs, 16, d_ptrs);
  if (!ai.empty()) {
    auto* d_ai = static_cast<AuditItem*>(ws_.get("audit_items", ai.size() * sizeof(AuditItem), false, stream_));
    upload(ai.data(), ai.size() * sizeof(AuditItem), d_ai);
    launch_audit(d_ai, uint32_t(ai.size()), max_n, reinterpret_cast<const float* const*>(d_ptrs),
                 reinterpret_cast<const float* const*>(d_ptrs + 1), 1, stream_);
  }
  float* recv = send;
  if (W > 1) {
    recv = static_cast<float*>(ws_.get("audit_recv", Ba * 4, false, stream_));
    nccl_check(nccl().ReduceScatter(send, recv, Ba, ncclFloat32, ncclSum, comm_, stream_), "audit reduce-scatter");
  }
  uint64_t owned = 0;
  for (const ShardSpec& s : shards)
    if (s.owner == rank_) owned += s.size();
  if (owned) zero({{audit, owned * 4}});
  std::vector<CopyItem> cp;
  for (size_t k = 0; k < P.segs.size(); ++k) {
    const SegPlan& p = P.segs[k];
    if (!p.compressed || shards[p.shard].owner != rank_) continue;
    cp.push_back(CopyItem{recv + aoff[k], audit + P.out_off[p.shard] + p.lo, p.len, 0});
  }
  if (!cp.empty()) {
    const uint64_t tt = copy_tiles(cp.data(), uint32_t(cp.size()));
    auto* d_cp = static_cast<CopyItem*>(ws_.get("audit_copy", cp.size() * sizeof(CopyItem), false, stream_));
    upload(cp.data(), cp.size() * sizeof(CopyItem), d_cp);
    launch_copy_items(di_, d_cp, uint32_t(cp.size()), tt, stream_);
  }
  cuda_check(cudaGetLastError(), "audit launch");
  sync_check();
}

void Engine::baseline_shards(const std::vector<ShardSpec>& shards, const float* grad, float* out) {
  CallScope scope(*this);
  if (shards.size() != world_) throw InvalidArgument("baseline needs one shard per rank");
  const uint64_t L = shards[0].size();
  for (uint32_t i = 0; i < shards.size(); ++i) {
    if (shards[i].owner != i || shards[i].size() != L || shards[i].begin != shards[0].begin + i * L)
      throw InvalidArgument("baseline needs equal contiguous shards with shard i owned by rank i");
  }
  launches_ = 0;
  const float* base = grad + shards[0].begin;
  if (world_ == 1 && !(force_collective_ && comm_)) {
    cuda_check(cudaMemcpyAsync(out, base, L * 4, cudaMemcpyDeviceToDevice, stream_), "D2D");
  } else {
    if (!comm_) throw InvalidArgument("multi-rank context has no NCCL communicator");
    nccl_check(nccl().ReduceScatter(base, out, L, ncclFloat32, ncclSum, comm_, stream_),
               "ncclReduceScatter baseline");
    ledger_.wire_bytes += uint64_t(world_) * L * 4;
  }
  for (const ShardSpec& s : shards)
    ledger_.record(CollectiveOp::reduce_scatter, "grad/shard" + std::to_string(s.id), s.size() * 32,
                   s.size());
}

// ------------------------------------------------------------ peer memory
void Engine::peer_release() {
  di_.coop_headroom = 0;
  for (void* p : peer_.opened) cudaIpcCloseMemHandle(p);
  peer_.opened.clear();
  if (peer_.region) cudaFree(peer_.region);
  peer_ = PeerState{};
}

void Engine::peer_prepare(const std::vector<ShardSpec>& shards, uint8_t handle[kPeerHandleBytes]) {
  if (world_ > uint32_t(kMaxPeers)) throw InvalidArgument("peer exchange supports at most 16 ranks");
  for (const ShardSpec& s : shards) check_shard(s, world_);
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  drop_graphs();
  peer_release();
  const ExchangePlan P = plan_exchange(shards, cfg_, world_, rank_);
  PeerState ps;
  ps.Bf = P.Bf;
  ps.Bu = P.Bu;
  size_t off = 0;
  for (int set = 0; set < 2; ++set) {
    ps.off_f[set] = off;
    off = align_up(off + world_ * P.Bf * 4, 256);
    ps.off_u[set] = off;
    off = align_up(off + world_ * P.Bu * 4, 256);
  }
  ps.off_flags = off;
  off = align_up(off + world_ * 8, 256);
  ps.off_counter = off;
  ps.bytes = align_up(off + 8, 256);
  void* base = nullptr;
  cuda_check(cudaMalloc(&base, ps.bytes), "peer region alloc");
  ps.region = static_cast<char*>(base);
  cuda_check(cudaMemset(ps.region + ps.off_flags, 0, ps.bytes - ps.off_flags), "peer flags zero");
  cudaIpcMemHandle_t h;
  cuda_check(cudaIpcGetMemHandle(&h, base), "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == kPeerHandleBytes, "IPC handle size");
  if (handle) std::memcpy(handle, &h, kPeerHandleBytes);
  peer_ = ps;
  // Warm-up: two local exchanges of zeros (no peers involved), so every
  // lazily allocated workspace and both staging halves exist before this
  // rank ever waits on a peer; allocations (cudaMalloc / cudaHostAlloc) may
  // synchronise the device and must not sit behind such a wait.
  uint64_t total = 0, owned = 0;
  for (const ShardSpec& sh : shards) {
    total = std::max<uint64_t>(total, sh.end);
    if (sh.owner == rank_) owned += sh.size();
  }
  const TrafficLedger saved = ledger_;  // the warm-up is not traffic
  float *g = nullptr, *a = nullptr, *o = nullptr;
  cuda_check(cudaMalloc(&g, std::max<uint64_t>(total, 1) * 4), "warm-up alloc");
  cuda_check(cudaMalloc(&a, std::max<uint64_t>(total, 1) * 4), "warm-up alloc");
  cuda_check(cudaMalloc(&o, std::max<uint64_t>(owned, 1) * 4), "warm-up alloc");
  cuda_check(cudaMemset(g, 0, total * 4), "warm-up zero");
  cuda_check(cudaMemset(a, 0, total * 4), "warm-up zero");
  // four calls, the later two with statistics: both staging halves and the
  // statistics path's buffers exist before the first real exchange
  for (int rep = 0; rep < 4; ++rep) {
    CallScope scope(*this);
    exchange_begin(shards, g, a, o, reinterpret_cast<float*>(ps.region + ps.off_f[0]),
                   reinterpret_cast<uint32_t*>(ps.region + ps.off_u[0]));
    auto* recv_f = static_cast<float*>(ws_.get("nc_recv_f", ps.Bf * 4, false, stream_));
    auto* recv_u = static_cast<uint32_t*>(ws_.get("nc_recv_u", ps.Bu * 4, false, stream_));
    zero({{recv_f, ps.Bf * 4}, {recv_u, ps.Bu * 4}});
    PeelStats st{};
    exchange_end(recv_f, recv_u, rep >= 2 ? &st : nullptr);
  }
  // staging headroom: a real step's descriptor uploads never regrow a half
  for (Staging& s : stage_)
    if (s.cap < (4u << 20)) {
      cuda_check(cudaStreamSynchronize(stream_), "staging grow");
      if (s.ptr) cudaFreeHost(s.ptr);
      s.ptr = nullptr;
      s.cap = 0;
      stage_grow(s, 4u << 20);
    }
  ws_.set_defer_free(true);
  ensure_aux();
  preload_all_kernels();
  cuda_check(cudaStreamSynchronize(stream_), "warm-up sync");
  cudaFree(g);
  cudaFree(a);
  cudaFree(o);
  ledger_ = saved;
}

void Engine::peer_fill(const std::vector<char*>& bases) {
  PeerView& v = peer_.view;
  v = PeerView{};
  v.world = world_;
  v.rank = rank_;
  v.block_f = peer_.Bf;
  v.block_u = peer_.Bu;
  uint64_t ms = 20000;
  if (const char* e = std::getenv("TAGC_PEER_TIMEOUT_MS")) ms = std::strtoull(e, nullptr, 10);
  v.timeout_ns = ms * 1000000ull;
  for (uint32_t q = 0; q < world_; ++q) {
    for (int set = 0; set < 2; ++set) {
      v.send_f[set][q] = reinterpret_cast<float*>(bases[q] + peer_.off_f[set]);
      v.send_u[set][q] = reinterpret_cast<uint32_t*>(bases[q] + peer_.off_u[set]);
    }
    v.flags[q] = reinterpret_cast<unsigned long long*>(bases[q] + peer_.off_flags);
  }
  v.counter = reinterpret_cast<unsigned long long*>(peer_.region + peer_.off_counter);
  peer_.attached = true;
  di_.coop_headroom = 1;
}

void Engine::peer_open(const uint8_t* handles) {
  if (!peer_.region) throw InvalidArgument("peer_open before peer_prepare");
  std::vector<char*> bases(world_, nullptr);
  for (uint32_t q = 0; q < world_; ++q) {
    if (q == rank_) {
      bases[q] = peer_.region;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + size_t(q) * kPeerHandleBytes, kPeerHandleBytes);
    void* p = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    peer_.opened.push_back(p);
    bases[q] = static_cast<char*>(p);
  }
  peer_fill(bases);
}

void Engine::peer_attach_local(const std::vector<Engine*>& ranks) {
  if (!peer_.region) throw InvalidArgument("peer_attach_local before peer_prepare");
  if (ranks.size() != world_) throw InvalidArgument("need one context per rank");
  std::vector<char*> bases(world_, nullptr);
  for (uint32_t q = 0; q < world_; ++q) {
    const Engine* e = ranks[q];
    if (!e || e->rank_ != q || e->world_ != world_ || !e->peer_.region || e->peer_.bytes != peer_.bytes)
      throw InvalidArgument("peer contexts must be ranks 0..W-1 prepared for the same layout");
    bases[q] = e->peer_.region;
  }
  peer_fill(bases);
}

// ------------------------------------------------------------ host buffers
void Engine::reduce_shards_host(const std::vector<ShardSpec>& shards, const float* host_grad,
                                float* acc, float* host_out, PeelStats* stats) {
  CallScope scope(*this);
  if (!host_grad || !host_out) throw InvalidArgument("null host buffer");
  if (!h2d_) {
    cuda_check(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking), "h2d stream");
    cuda_check(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking), "d2h stream");
    for (int i = 0; i < 2; ++i)
      for (cudaEvent_t* e : {&hev_in_[i], &hev_gfree_[i], &hev_dec_[i], &hev_out_[i]})
        cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "host event");
    cuda_check(cudaEventCreateWithFlags(&hev_join_, cudaEventDisableTiming), "host event");
  }
  uint64_t total = 0, owned = 0;
  for (const ShardSpec& sh : shards) {
    total = std::max<uint64_t>(total, sh.end);
    if (sh.owner == rank_) owned += sh.size();
  }
  if (total * 4 > host_grad_cap_ || owned * 4 > host_out_cap_) {
    // the double buffers are about to move: nothing may still use them
    cuda_check(cudaStreamSynchronize(h2d_), "h2d sync");
    cuda_check(cudaStreamSynchronize(d2h_), "d2h sync");
    cuda_check(cudaStreamSynchronize(stream_), "stream sync");
  }
  const int s = int(host_calls_++ & 1);
  auto* gdev = static_cast<float*>(ws_.get(s ? "host_grad1" : "host_grad0", total * 4, false, stream_));
  auto* odev = static_cast<float*>(
      ws_.get(s ? "host_out1" : "host_out0", std::max<uint64_t>(owned, 1) * 4, false, stream_));
  host_grad_cap_ = std::max(host_grad_cap_, total * 4);
  host_out_cap_ = std::max(host_out_cap_, owned * 4);
  // H2D once the exchange two calls back has consumed this device buffer
  cuda_check(cudaStreamWaitEvent(h2d_, hev_gfree_[s], 0), "wait gfree");
  cuda_check(cudaMemcpyAsync(gdev, host_grad, total * 4, cudaMemcpyHostToDevice, h2d_), "H2D grad");
  cuda_check(cudaEventRecord(hev_in_[s], h2d_), "record in");
  cuda_check(cudaStreamWaitEvent(stream_, hev_in_[s], 0), "wait in");
  cuda_check(cudaStreamWaitEvent(stream_, hev_out_[s], 0), "wait out");  // D2H two calls back done
  grad_read_ev_ = hev_gfree_[s];
  try {
    reduce_shards(shards, gdev, acc, odev, stats);
  } catch (...) {
    grad_read_ev_ = nullptr;
    throw;
  }
  grad_read_ev_ = nullptr;
  cuda_check(cudaEventRecord(hev_dec_[s], stream_), "record dec");
  cuda_check(cudaStreamWaitEvent(d2h_, hev_dec_[s], 0), "wait dec");
  if (owned)
    cuda_check(cudaMemcpyAsync(host_out, odev, owned * 4, cudaMemcpyDeviceToHost, d2h_), "D2H out");
  cuda_check(cudaEventRecord(hev_out_[s], d2h_), "record out");
  if (stats) cuda_check(cudaStreamSynchronize(d2h_), "d2h sync");
}

void Engine::host_join() {
  if (!d2h_) return;
  cuda_check(cudaEventRecord(hev_join_, d2h_), "record join");
  cuda_check(cudaStreamWaitEvent(stream_, hev_join_, 0), "wait join");
}

// ------------------------------------------------------------------ codec API
void Engine::sparsify(const float* g, uint32_t n, double theta, float* sparse, float* residual,
                      float* tau, uint64_t* zero_count) {
  CallScope scope(*this);
  if (!(theta >= 0.0 && theta <= 100.0))
    throw InvalidArgument("sparsification threshold must lie in [0, 100]");  // sparsify.cpp:19-20
  if (n == 0) throw InvalidArgument("sparsify: empty gradient");             // :21
  launches_ = 0;
  std::vector<EncItem> it(1);
  EncItem& e = it[0];
  e.g = g;
  e.sparse = sparse;
  e.residual = residual;
  e.n = n;
  e.c = threshold_rank(theta, n);
  e.flags = kSelect | kWriteSparse | kWriteResidual | (aligned16(g) ? kAligned16 : 0u);
  const HashParams hp = make_hash_params(0, 1);
  run_select_encode(it, true, hp, true, "sparsify");
  SelState st{};
  cuda_check(cudaMemcpyAsync(&st, ws_.get("sel_state", 16), sizeof(SelState), cudaMemcpyDeviceToHost,
                             stream_), "D2H state");
  sync_check();
  if (tau) std::memcpy(tau, &st.tau_key, 4);
  // kept = speculatively kept (above the window) + candidates kept by the
  // fix-up; after a fallback the exact re-encode counted every kept element.
  const uint64_t kept = st.status == 4 ? st.kept : uint64_t(st.cnt_hi) + st.kept;
  if (zero_count) *zero_count = uint64_t(n) - kept;
}

void Engine::index_create(const float* v, uint32_t n, uint32_t width, uint32_t* words) {
  CallScope scope(*this);
  if (width != 1 && width != 4) throw InvalidArgument("index width must be 1 or 4");
  if (n == 0) throw InvalidArgument("index needs at least one position");
  launches_ = 0;
  std::vector<EncItem> it(1);
  it[0].g = v;
  it[0].index = words;
  it[0].n = n;
  it[0].flags = kWriteIndex | (width == 4 ? kWidth4 : 0u) | (aligned16(v) ? kAligned16 : 0u);
  run_select_encode(it, width == 4, make_hash_params(0, 1), false, "index");
}

void Engine::merge_indices(const uint32_t* const* words, uint32_t world, uint32_t n_words,
                           uint32_t* out) {
  CallScope scope(*this);
  if (world == 0) throw InvalidArgument("merge_indices: no inputs");
  launches_ = 0;
  auto* d = static_cast<const uint32_t**>(ws_.get("merge_ptrs", world * 8, false, stream_));
  upload(words, world * 8, d);
  launches_ += launch_rank_sum_u32(d, world, out, n_words, stream_);
}

void Engine::index_presence(const uint32_t* words, uint32_t n, uint32_t width, uint32_t* positions,
                            uint32_t* count) {
  CallScope scope(*this);
  if (width != 1 && width != 4) throw InvalidArgument("index width must be 1 or 4");
  if (n == 0) throw InvalidArgument("index needs at least one position");
  launches_ = 0;
  const size_t sb = index_presence_scratch_bytes(n, width);
  void* scratch = ws_.get("presence_scratch", sb, false, stream_);
  auto* cnt = static_cast<uint32_t*>(ws_.get("presence_count", 4, false, stream_));
  launches_ += launch_index_presence(words, n, width, positions, cnt, scratch, sb, stream_);
  if (count) {
    cuda_check(cudaMemcpyAsync(count, cnt, 4, cudaMemcpyDeviceToHost, stream_), "D2H count");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
  }
}

void Engine::sketch_compress(const float* v, uint32_t n, uint32_t ratio, uint32_t rows,
                             uint64_t seed, float* sketch) {
  CallScope scope(*this);
  if (rows > kMaxRows) throw InvalidArgument("sketch_rows above 8 is not supported on device");
  const SketchGeometry g = sketch_geometry(n, ratio, rows);
  launches_ = 0;
  cuda_check(cudaMemsetAsync(sketch, 0, uint64_t(rows) * g.buckets_per_row * 4, stream_), "zero");
  std::vector<EncItem> it(1);
  it[0].g = v;
  it[0].sketch = sketch;
  it[0].n = n;
  it[0].m = g.buckets_per_row;
  it[0].flags = kWriteSketch | (aligned16(v) ? kAligned16 : 0u);
  run_select_encode(it, true, make_hash_params(seed, rows), false, "compress");
}

OptEpilogue Engine::make_opt(int kind, double lr, double weight_decay, uint32_t world, uint32_t step,
                             float* params, float* adam_v, const float* out_base, bool write_out) const {
  if (kind != 0 && kind != 1) throw InvalidArgument("optimizer must be sgd (0) or adamw_nm (1)");
  if (world == 0) throw InvalidArgument("world size must be at least 1");
  if (!params) throw InvalidArgument("no parameter buffer");
  if (kind == 1 && (step == 0 || !adam_v)) throw InvalidArgument("adamw_nm needs step >= 1 and its state");
  auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15u) == 0; };
  if (!a16(params) || (kind == 1 && !a16(adam_v)) || !a16(out_base))
    throw InvalidArgument("optimizer buffers (params, adam_v, decoded/out) must be 16-byte aligned");
  OptEpilogue o{};
  o.kind = kind;
  o.write_out = write_out ? 1 : 0;
  o.out_base = out_base;
  o.params = params;
  o.adam_v = adam_v;
  o.inv_w = 1.0f / static_cast<float>(world);  // train.cpp:356
  o.lr = static_cast<float>(lr);
  o.wd = static_cast<float>(weight_decay);
  o.bias_fix = kind == 1 ? 1.0f - std::pow(0.999f, static_cast<float>(step)) : 1.0f;  // train.cpp:213
  return o;
}

void Engine::reduce_shards_step(const std::vector<ShardSpec>& shards, const float* grad, float* acc, float* out,
                                int kind, double lr, double weight_decay, uint32_t step, float* params,
                                float* adam_v, PeelStats* stats) {
  // mean over this world (train.cpp:356), fused into the decode's emit and
  // the owner's raw-segment unpack: the decoded shard is never re-read. The
  // step's scalars go to a device slot ahead of the (possibly replayed)
  // exchange, so a captured graph serves every step.
  const OptEpilogue o = make_opt(kind, lr, weight_decay, world_, step, params, adam_v, out ? out : params,
                                 out != nullptr);
  if (!opt_dev_) cuda_check(cudaMalloc(&opt_dev_, sizeof(OptEpilogue)), "cudaMalloc optimizer slot");
  launch_set_opt(opt_dev_, o, stream_);
  opt_on_ = true;
  try {
    reduce_shards(shards, grad, acc, out ? out : params, stats);
  } catch (...) {
    opt_on_ = false;
    throw;
  }
  opt_on_ = false;
}

void Engine::apply_optimizer(int kind, double lr, double weight_decay, uint32_t world, uint32_t step,
                             float* params, const float* decoded, float* adam_v, uint64_t n) {
  const OptEpilogue o = make_opt(kind, lr, weight_decay, world, step, params, adam_v, decoded, false);
  launches_ = launch_apply_optimizer(o, n, stream_);
  cuda_check(cudaGetLastError(), "apply_optimizer launch");
}

void Engine::allgather_params(float* params, uint64_t padded) {
  if (padded % world_) throw InvalidArgument("padded length must be a multiple of the world size");
  const uint64_t L = padded / world_;
  launches_ = 0;
  if (world_ > 1) {
    if (!comm_) throw InvalidArgument("multi-rank context has no NCCL communicator");
    nccl_check(nccl().AllGather(params + rank_ * L, params, L, ncclFloat32, comm_, stream_), "ncclAllGather");
    ledger_.wire_bytes += padded * 4;
  }
  ledger_.record(CollectiveOp::all_gather, "params/allgather", padded * 32, padded);
}

void Engine::add(const float* a, const float* b, float* out, uint64_t n) {
  launches_ = launch_add(a, b, out, n, stream_);
}

void Engine::peeling_decompress(const uint32_t* presence, uint32_t count, uint32_t n,
                                uint32_t ratio, uint32_t rows, uint64_t seed, const float* sketch,
                                float* values, uint32_t* unresolved, uint32_t* n_unresolved,
                                double* pf) {
  CallScope scope(*this);
  if (rows > kMaxRows) throw InvalidArgument("sketch_rows above 8 is not supported on device");
  const SketchGeometry g = sketch_geometry(n, ratio, rows);
  launches_ = 0;
  const uint64_t nb = (uint64_t(n) + 31) / 32;
  auto* bitmap = static_cast<uint32_t*>(ws_.get("peel_presence", nb * 4, false, stream_));
  auto* sk = static_cast<float*>(ws_.get("peel_sketch", uint64_t(rows) * g.buckets_per_row * 4, false, stream_));
  uint32_t* err = err_flag();
  cuda_check(cudaMemsetAsync(err, 0, 4, stream_), "err reset");
  cuda_check(cudaMemsetAsync(bitmap, 0, nb * 4, stream_), "bitmap zero");
  cuda_check(cudaMemcpyAsync(sk, sketch, uint64_t(rows) * g.buckets_per_row * 4, cudaMemcpyDeviceToDevice,
                             stream_), "sketch copy");
  launches_ += launch_presence_to_bitmap(presence, count, n, bitmap, err, stream_);
  std::vector<DecItem> d(1);
  d[0].words = bitmap;
  d[0].sketch = sk;
  d[0].out = values;
  d[0].n = n;
  d[0].m = g.buckets_per_row;
  d[0].flags = 0;  // presence bitmap == width-1 index
  d[0].n_words = uint32_t(nb);
  d[0].list_cap = count;
  const HashParams hp = make_hash_params(seed, rows);
  run_decode(d, hp, true, true);  // arbitrary presence/sketch pairs: FIFO-exact order
  DecStats ds{};
  uint32_t e = 0;
  cuda_check(cudaMemcpyAsync(&ds, ws_.get("dec_stats", 16), sizeof(ds), cudaMemcpyDeviceToHost, stream_), "D2H");
  cuda_check(cudaMemcpyAsync(&e, err, 4, cudaMemcpyDeviceToHost, stream_), "D2H err");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  clear_err_word(e);
  if (e & 1u) throw InvalidArgument("presence position out of range for sketch geometry");
  if (e & 2u) throw InvalidArgument("presence set contains a duplicate position");
  if (ds.overflow) throw CudaError("decode bucket state overflow");
  if (unresolved && ds.unresolved) {
    auto* un = static_cast<uint32_t*>(ws_.get("unresolved", 16));
    auto* alt = static_cast<uint32_t*>(ws_.get("unresolved_alt", ds.unresolved * 4, false, stream_));
    const size_t sb = sort_scratch_bytes(ds.unresolved);
    void* scratch = ws_.get("sort_scratch", sb, false, stream_);
    launches_ += launch_sort_u32(un, alt, ds.unresolved, scratch, sb, stream_);
    cuda_check(cudaMemcpyAsync(unresolved, un, ds.unresolved * 4, cudaMemcpyDeviceToDevice, stream_), "D2D");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
  }
  if (n_unresolved) *n_unresolved = ds.unresolved;
  if (pf) *pf = count == 0 ? 1.0 : double(ds.presence - ds.unresolved) / double(ds.presence);
}

void Engine::estimation_decompress(const uint32_t* presence, uint32_t count, uint32_t n,
                                   uint32_t ratio, uint32_t rows, uint64_t seed, const float* sketch,
                                   const uint32_t* targets, uint32_t n_targets, float* out) {
  CallScope scope(*this);
  if (rows > kMaxRows) throw InvalidArgument("sketch_rows above 8 is not supported on device");
  const SketchGeometry g = sketch_geometry(n, ratio, rows);
  launches_ = 0;
  const uint64_t nb = (uint64_t(n) + 31) / 32;
  auto* bitmap = static_cast<uint32_t*>(ws_.get("peel_presence", nb * 4, false, stream_));
  uint32_t* err = err_flag();
  cuda_check(cudaMemsetAsync(err, 0, 4, stream_), "err reset");
  cuda_check(cudaMemsetAsync(bitmap, 0, nb * 4, stream_), "bitmap zero");
  launches_ += launch_presence_to_bitmap(presence, count, n, bitmap, err, stream_);
  launches_ += launch_estimate_targets(targets, n_targets, bitmap, n, g.buckets_per_row, sketch,
                                       make_hash_params(seed, rows), out, err, stream_);
  uint32_t e = 0;
  cuda_check(cudaMemcpyAsync(&e, err, 4, cudaMemcpyDeviceToHost, stream_), "D2H err");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  clear_err_word(e);
  if (e & 1u) throw InvalidArgument("presence position out of range for sketch geometry");
  if (e & 4u) throw InvalidArgument("estimation target outside the presence set");
}

}  // namespace tagc_b200
