// host.cpp — host-side policy, planning and accounting (see host.hpp).
#include "host.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

namespace tagc_b200 {

const char* to_string(LayerKind k) {
  switch (k) {
    case LayerKind::embedding: return "embedding";
    case LayerKind::positional_embedding: return "positional_embedding";
    case LayerKind::attention_qkv: return "attention_qkv";
    case LayerKind::attention_out_proj: return "attention_out_proj";
    case LayerKind::feed_forward: return "feed_forward";
    case LayerKind::lm_head: return "lm_head";
    case LayerKind::norm: return "norm";
    case LayerKind::bias: return "bias";
    case LayerKind::other: return "other";
  }
  return "?";
}

const char* to_string(Policy p) {
  switch (p) {
    case Policy::all_layers: return "all_layers";
    case Policy::non_attention_linear: return "non_attention_linear";
    case Policy::none: return "none";
  }
  return "?";
}

// config.cpp:27-35
double CompressionConfig::theta_floor(uint32_t ratio) {
  switch (ratio) {
    case 1: return 0.0;
    case 2: return 80.0;
    case 4: return 90.0;
    case 10: return 98.75;
    default: throw InvalidArgument("compression ratio must be one of {1, 2, 4, 10}");
  }
}

// config.cpp:37-51
void CompressionConfig::validate() const {
  if (!(theta >= 0.0 && theta <= 100.0)) throw InvalidArgument("theta must lie in [0, 100]");
  if (index_width != 1 && index_width != 4) throw InvalidArgument("index width must be 1 or 4");
  if (sketch_rows == 0) throw InvalidArgument("sketch needs at least one row");
  if (sketch_rows > 8) throw InvalidArgument("sketch_rows above 8 is not supported on device");
  const double floor = theta_floor(ratio);
  if (ratio > 1 && theta < floor && !allow_low_theta) {
    std::ostringstream os;
    os << "ratio " << ratio << " needs theta >= " << floor << " for lossless peeling (got "
       << theta << "); pass the low-theta override to run the estimation-heavy regime";
    throw InvalidArgument(os.str());
  }
}

// config.cpp:53-59
void CompressionConfig::validate_for_world(uint32_t w) const {
  validate();
  if (ratio > 1 && index_width == 4 && w > 15)
    throw InvalidArgument("a 4-bit index overflows its nibbles beyond 15 ranks; reduce the world size");
}

// layers.cpp:42-65
bool kind_compressible(LayerKind kind, Policy policy, bool include_out_proj) {
  switch (policy) {
    case Policy::none: return false;
    case Policy::all_layers: return true;
    case Policy::non_attention_linear:
      switch (kind) {
        case LayerKind::embedding:
        case LayerKind::positional_embedding:
        case LayerKind::feed_forward:
        case LayerKind::lm_head: return true;
        case LayerKind::attention_out_proj: return include_out_proj;
        default: return false;
      }
  }
  return false;
}

// hook.cpp:30-61
std::vector<ShardSpec> make_shards(const std::vector<LayerSpec>& layers, uint32_t shard_count,
                                   uint32_t world_size) {
  if (shard_count == 0) throw InvalidArgument("need at least one shard");
  if (world_size == 0) throw InvalidArgument("world size must be at least 1");
  uint64_t total = 0;
  for (const LayerSpec& l : layers) total += l.param_count;
  if (total == 0) throw InvalidArgument("no parameters to shard");
  const uint64_t shard_len = (total + shard_count - 1) / shard_count;
  std::vector<ShardSpec> shards(shard_count);
  for (uint32_t s = 0; s < shard_count; ++s) {
    shards[s].id = s;
    shards[s].owner = s % world_size;
    shards[s].begin = uint64_t(s) * shard_len;
    shards[s].end = shards[s].begin + shard_len;
  }
  uint64_t off = 0;
  for (const LayerSpec& l : layers) {
    const uint64_t lb = off, le = off + l.param_count;
    // Only the shards the layer touches: [lb / shard_len, (le-1) / shard_len].
    if (le > lb) {
      const uint64_t s0 = lb / shard_len, s1 = std::min<uint64_t>((le - 1) / shard_len, shard_count - 1);
      for (uint64_t s = s0; s <= s1; ++s) {
        ShardSpec& sh = shards[s];
        const uint64_t b = std::max(lb, sh.begin), e = std::min(le, sh.end);
        if (b < e) sh.segments.push_back({l.name, l.kind, b, e});
      }
    }
    off = le;
  }
  ShardSpec& last = shards.back();
  if (total < last.end) last.segments.push_back({"pad", LayerKind::other, total, last.end});
  return shards;
}

// sketch.cpp:11-27
SketchGeometry sketch_geometry(uint32_t n, uint32_t ratio, uint32_t rows) {
  if (ratio != 2 && ratio != 4 && ratio != 10)
    throw InvalidArgument("compression ratio must be one of {2, 4, 10}");
  if (rows == 0) throw InvalidArgument("sketch needs at least one row");
  if (n == 0) throw InvalidArgument("sketch over an empty vector");
  const uint32_t m = n / (ratio * rows);
  if (m == 0)
    throw InvalidArgument("vector of length " + std::to_string(n) + " is too small for ratio " +
                          std::to_string(ratio) + " with " + std::to_string(rows) + " rows");
  return SketchGeometry{n, ratio, rows, m};
}

// index.cpp:17-20
uint32_t words_needed(uint32_t n, uint32_t width) {
  return uint32_t((uint64_t(n) * width + 31) / 32);
}

// hook.cpp:13-22
PeelStats& PeelStats::operator+=(const PeelStats& o) {
  presence += o.presence;
  peeled += o.peeled;
  unresolved += o.unresolved;
  index_lost += o.index_lost;
  index_spurious += o.index_spurious;
  compressed_segments += o.compressed_segments;
  baseline_segments += o.baseline_segments;
  return *this;
}

// hook.cpp:202-226
CommVolume comm_volume_model(const CompressionConfig& c, uint32_t world, std::optional<uint64_t> n) {
  c.validate_for_world(world);
  CommVolume v;
  if (c.ratio == 1) {
    v.index_bits = 0.0;
    v.sketch_bits = 32.0;
    v.total_bits = 32.0;
    v.factor = 1.0;
    return v;
  }
  v.index_bits = 2.0 * c.index_width;
  if (n) {
    const SketchGeometry g = sketch_geometry(uint32_t(*n), c.ratio, c.sketch_rows);
    const uint64_t payload = uint64_t(g.rows) * g.buckets_per_row * 32ull;
    v.sketch_bits = double(payload) / double(*n);
  } else {
    v.sketch_bits = 32.0 / c.ratio;
  }
  v.total_bits = v.index_bits + v.sketch_bits;
  v.factor = 32.0 / v.total_bits;
  return v;
}

// hook.cpp:228-236
CommVolume lhc_comm_volume_model(const CompressionConfig& c, uint32_t world,
                                 std::optional<uint64_t> n) {
  CommVolume v = comm_volume_model(c, world, n);
  if (c.ratio == 1) return v;
  v.sketch_bits *= 2.0;
  v.total_bits = v.index_bits + v.sketch_bits;
  v.factor = 32.0 / v.total_bits;
  return v;
}

const char* to_string(CollectiveOp op) {
  switch (op) {
    case CollectiveOp::all_reduce: return "all_reduce";
    case CollectiveOp::reduce: return "reduce";
    case CollectiveOp::reduce_scatter: return "reduce_scatter";
    case CollectiveOp::all_gather: return "all_gather";
  }
  return "?";
}

// collectives.cpp:37-46
void TrafficLedger::record(CollectiveOp op, const std::string& tag, uint64_t payload_bits,
                           uint64_t params) {
  LedgerRow& row = rows_[{int(op), tag}];
  row.op = op;
  row.tag = tag;
  row.calls += 1;
  row.payload_bits += payload_bits;
  row.charged_bits += (op == CollectiveOp::all_reduce ? 2u : 1u) * payload_bits;
  row.params += params;
}

// Undo one record() (a capture that was abandoned after recording).
void TrafficLedger::unrecord(CollectiveOp op, const std::string& tag, uint64_t payload_bits,
                             uint64_t params) {
  auto it = rows_.find({int(op), tag});
  if (it == rows_.end()) return;
  LedgerRow& row = it->second;
  row.calls -= 1;
  row.payload_bits -= payload_bits;
  row.charged_bits -= (op == CollectiveOp::all_reduce ? 2u : 1u) * payload_bits;
  row.params -= params;
  if (row.calls == 0) rows_.erase(it);
}

// collectives.cpp:60-68
double TrafficLedger::bits_per_param_per_rank(const std::string& prefix) const {
  uint64_t charged = 0, params = 0;
  for (const auto& [k, row] : rows_) {
    if (row.tag.rfind(prefix, 0) != 0) continue;
    charged += row.charged_bits;
    params += row.params;
  }
  return params == 0 ? 0.0 : double(charged) / double(params);
}

// collectives.cpp:70-78
std::string TrafficLedger::to_csv() const {
  std::string out = "op,tag,calls,payload_bits,charged_bits,bits_per_param_per_rank\n";
  char buf[64];
  for (const auto& [k, row] : rows_) {
    std::snprintf(buf, sizeof(buf), "%.9g", row.bits_per_param_per_rank());
    out += std::string(to_string(row.op)) + "," + row.tag + "," + std::to_string(row.calls) +
           "," + std::to_string(row.payload_bits) + "," + std::to_string(row.charged_bits) + "," +
           buf + "\n";
  }
  return out;
}

namespace {

// A JSON number the way nlohmann::json's serializer writes a double: shortest
// round-trip digits, then its format_buffer layout (kMinExp = -4, kMaxExp =
// 15): "2.0", "0.5", "0.0001", "1e-05", "1.5e+20"; non-finite -> null.
std::string json_double(double x) {
  if (!std::isfinite(x)) return "null";
  std::string out;
  if (std::signbit(x)) {
    out += '-';
    x = -x;
  }
  if (x == 0.0) return out + "0.0";
  char sci[64];
  const auto r = std::to_chars(sci, sci + sizeof(sci), x, std::chars_format::scientific);
  const std::string s(sci, r.ptr);  // d[.ddd]e[+-]XX
  const size_t epos = s.find('e');
  std::string digits = s.substr(0, epos);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int k = int(digits.size());
  const int n = std::atoi(s.c_str() + epos + 1) + 1;  // value = 0.digits * 10^n
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) return out + digits + std::string(size_t(n - k), '0') + ".0";
  if (0 < n && n <= kMaxExp) return out + digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
  if (kMinExp < n && n <= 0) return out + "0." + std::string(size_t(-n), '0') + digits;
  out += digits.substr(0, 1);
  if (k > 1) out += "." + digits.substr(1);
  int e = n - 1;
  out += 'e';
  out += e < 0 ? '-' : '+';
  e = e < 0 ? -e : e;
  char eb[8];
  std::snprintf(eb, sizeof(eb), e < 10 ? "0%d" : "%d", e);
  return out + eb;
}

std::string json_string(const std::string& v) {
  std::string out = "\"";
  for (unsigned char c : v) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          out += b;
        } else {
          out += char(c);
        }
    }
  }
  return out + "\"";
}

}  // namespace

// collectives.cpp:80-93
std::string TrafficLedger::to_json() const {
  std::string out = "[";
  bool first = true;
  for (const auto& [k, row] : rows_) {
    if (!first) out += ',';
    first = false;
    out += "{\"op\":" + json_string(to_string(row.op)) + ",\"tag\":" + json_string(row.tag) +
           ",\"calls\":" + std::to_string(row.calls) + ",\"payload_bits\":" + std::to_string(row.payload_bits) +
           ",\"charged_bits\":" + std::to_string(row.charged_bits) +
           ",\"bits_per_param_per_rank\":" + json_double(row.bits_per_param_per_rank()) + "}";
  }
  return out + "]";
}

}  // namespace tagc_b200
