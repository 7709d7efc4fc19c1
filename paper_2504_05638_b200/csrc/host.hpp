// host.hpp — C++ host mirror of the reference's compressor API for the
// exchange path (namespace tagc_b200 so it can share a process with the
// reference library in parity tests). Pure host logic: config validation,
// layer policy, shard planning, sketch geometry, volume model and the traffic
// ledger. Every function cites the reference file:line it mirrors.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace tagc_b200 {

// reference config.hpp:10
enum class Policy : int32_t { all_layers = 0, non_attention_linear = 1, none = 2 };

// reference layers.hpp:12-22
enum class LayerKind : int32_t {
  embedding = 0,
  positional_embedding,
  attention_qkv,
  attention_out_proj,
  feed_forward,
  lm_head,
  norm,
  bias,
  other,
};

const char* to_string(LayerKind k);
const char* to_string(Policy p);

// reference config.hpp:16-35
struct CompressionConfig {
  double theta = 0.0;
  uint32_t ratio = 1;
  uint32_t index_width = 4;
  Policy policy = Policy::non_attention_linear;
  bool include_out_proj = true;
  uint64_t seed = 0;
  uint32_t sketch_rows = 3;
  bool allow_low_theta = false;
  uint64_t min_compress_segment = 1024;

  static double theta_floor(uint32_t ratio);  // config.cpp:27-35
  void validate() const;                      // config.cpp:37-51
  void validate_for_world(uint32_t w) const;  // config.cpp:53-59
};

// reference layers.cpp:42-65
bool kind_compressible(LayerKind kind, Policy policy, bool include_out_proj);

// reference layers.hpp:27-31
struct LayerSpec {
  std::string name;
  LayerKind kind = LayerKind::other;
  uint64_t param_count = 0;
};

// reference hook.hpp:21-38
struct LayerSegment {
  std::string name;
  LayerKind kind = LayerKind::other;
  uint64_t begin = 0, end = 0;
  uint64_t size() const { return end - begin; }
};
struct ShardSpec {
  uint32_t id = 0, owner = 0;
  uint64_t begin = 0, end = 0;
  std::vector<LayerSegment> segments;
  uint64_t size() const { return end - begin; }
};

// reference hook.cpp:30-61
std::vector<ShardSpec> make_shards(const std::vector<LayerSpec>& layers, uint32_t shard_count,
                                   uint32_t world_size);

// reference sketch.hpp:21-28 / sketch.cpp:11-27
struct SketchGeometry {
  uint32_t n = 0, ratio = 2, rows = 3, buckets_per_row = 0;
};
SketchGeometry sketch_geometry(uint32_t n, uint32_t ratio, uint32_t rows = 3);

// reference index.cpp:17-20
uint32_t words_needed(uint32_t n, uint32_t width);

// index_lost / index_spurious value when the call had no way to see the
// ranks' supports (split API with a 1-bit index and no support blocks)
constexpr uint64_t kStatUnavailable = ~0ull;

// reference hook.hpp:45-59
struct PeelStats {
  uint64_t presence = 0, peeled = 0, unresolved = 0, index_lost = 0, index_spurious = 0,
           compressed_segments = 0, baseline_segments = 0;
  PeelStats& operator+=(const PeelStats& o);
};

// reference hook.hpp:88-104 / hook.cpp:202-236
struct CommVolume {
  double index_bits = 0, sketch_bits = 0, total_bits = 0, factor = 1;
};
CommVolume comm_volume_model(const CompressionConfig& c, uint32_t world,
                             std::optional<uint64_t> n = std::nullopt);
CommVolume lhc_comm_volume_model(const CompressionConfig& c, uint32_t world,
                                 std::optional<uint64_t> n = std::nullopt);

// reference collectives.hpp:32-81 / collectives.cpp:23-93: the declared cost
// model (All-Reduce charged 2x, others 1x), recorded by the engine at each
// exchange with the reference's tags.
enum class CollectiveOp : int { all_reduce = 0, reduce = 1, reduce_scatter = 2, all_gather = 3 };
const char* to_string(CollectiveOp op);
struct LedgerRow {
  CollectiveOp op;
  std::string tag;
  uint64_t calls = 0, payload_bits = 0, charged_bits = 0, params = 0;
  double bits_per_param_per_rank() const {
    return params == 0 ? 0.0 : double(charged_bits) / double(params);
  }
};
class TrafficLedger {
 public:
  void record(CollectiveOp op, const std::string& tag, uint64_t payload_bits, uint64_t params);
  void unrecord(CollectiveOp op, const std::string& tag, uint64_t payload_bits, uint64_t params);
  std::string to_csv() const;
  // collectives.cpp:80-93: the rows as a JSON array, serialised the way
  // nlohmann::ordered_json::dump() writes it (compact, shortest doubles)
  std::string to_json() const;
  double bits_per_param_per_rank(const std::string& prefix = "") const;
  void clear() { rows_.clear(); }
  // rows in (op, tag) order, as TrafficLedger::rows() (collectives.cpp:48-53)
  std::vector<LedgerRow> rows() const {
    std::vector<LedgerRow> out;
    for (const auto& kv : rows_) out.push_back(kv.second);
    return out;
  }
  // Bytes actually handed to NCCL (measured, not modelled).
  uint64_t wire_bytes = 0;

 private:
  std::map<std::pair<int, std::string>, LedgerRow> rows_;
};

// Error type carrying the C-ABI status (2 = invalid argument).
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

}  // namespace tagc_b200
