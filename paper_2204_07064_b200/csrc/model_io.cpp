// model_io.cpp — SPEC model_io: a graph + weights as a UTF-8 JSON manifest and
// a raw little-endian f32 blob (paired files share a basename).
//
// Manifest (format_version 1; documented in INTEGRATION.md §model_io):
//   { "format_version": 1, "in_channels": C,
//     "nodes": [ {"id": 0, "kind": "Source", "channels": C}, ...,
//                {"id": i, "kind": "Conv", "in_channels": M, "out_channels": N, "kernel": K,
//                 "stride": S, "dilation": d, "padding": [L, R], "shift": 0, "hint": "none",
//                 "weights": {"offset": bytes, "length": bytes}}, ... ],
//     "edges": [ [from, to, port], ... ] }
// Node kinds are SPEC's NodeKind names plus "Gate" / "Slice".  A Conv's blob
// range holds weights [n][m][k] then bias [n] (the reference Kernel, tensor.hpp:52-88); save
// writes them in ascending node id.  Errors: VersionMismatch, CorruptBlob (blob size, weight
// ranges), SchemaError with the JSON path of the offending value, then every validate error.
#include <algorithm>
#include <cctype>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "program.hpp"

namespace scb {
namespace {

// ------------------------------------------------------------------ minimal JSON reader
struct Json {
  enum Type { NUL, BOOL, NUM, STR, ARR, OBJ } type = NUL;
  bool b = false;
  double num = 0;
  std::string str;  // STR value, or the NUM token as written (integers are checked exactly)
  std::vector<Json> arr;
  std::vector<std::pair<std::string, Json>> obj;
  const Json* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct Parser {
  const std::string& s;
  size_t i = 0;
  [[noreturn]] void bad(const std::string& what) {
    fail(SC_ERR_SCHEMA_ERROR, "$: malformed JSON at byte " + std::to_string(i) + ": " + what);
  }
  void ws() {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t' || s[i] == '\n' || s[i] == '\r')) ++i;
  }
  bool lit(const char* w) {
    const size_t n = std::strlen(w);
    if (s.compare(i, n, w) == 0) {
      i += n;
      return true;
    }
    return false;
  }
  std::string string() {
    if (s[i] != '"') bad("expected a string");
    ++i;
    std::string out;
    while (i < s.size() && s[i] != '"') {
      char c = s[i++];
      if (c == '\\') {
        if (i >= s.size()) bad("unterminated escape");
        const char e = s[i++];
        switch (e) {
          case '"': out += '"'; break;
          case '\\': out += '\\'; break;
          case '/': out += '/'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (i + 4 > s.size()) bad("short \\u escape");
            const unsigned cp = static_cast<unsigned>(std::stoul(s.substr(i, 4), nullptr, 16));
            i += 4;
            if (cp < 0x80) {
              out += static_cast<char>(cp);
            } else if (cp < 0x800) {
              out += static_cast<char>(0xC0 | (cp >> 6));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            } else {
              out += static_cast<char>(0xE0 | (cp >> 12));
              out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
              out += static_cast<char>(0x80 | (cp & 0x3F));
            }
            break;
          }
          default:
            bad("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (i >= s.size()) bad("unterminated string");
    ++i;
    return out;
  }
  Json value(int depth) {
    if (depth > 64) bad("nesting too deep");
    ws();
    if (i >= s.size()) bad("unexpected end");
    Json v;
    const char c = s[i];
    if (c == '{') {
      v.type = Json::OBJ;
      ++i;
      ws();
      if (s[i] == '}') {
        ++i;
        return v;
      }
      for (;;) {
        ws();
        std::string k = string();
        ws();
        if (s[i] != ':') bad("expected ':'");
        ++i;
        v.obj.emplace_back(std::move(k), value(depth + 1));
        ws();
        if (s[i] == ',') {
          ++i;
          continue;
        }
        if (s[i] == '}') {
          ++i;
          return v;
        }
        bad("expected ',' or '}'");
      }
    }
    if (c == '[') {
      v.type = Json::ARR;
      ++i;
      ws();
      if (s[i] == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.arr.push_back(value(depth + 1));
        ws();
        if (s[i] == ',') {
          ++i;
          continue;
        }
        if (s[i] == ']') {
          ++i;
          return v;
        }
        bad("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.type = Json::STR;
      v.str = string();
      return v;
    }
    if (lit("true")) {
      v.type = Json::BOOL;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.type = Json::BOOL;
      return v;
    }
    if (lit("null")) return v;
    const size_t b = i;
    while (i < s.size() && (std::isdigit(static_cast<unsigned char>(s[i])) || s[i] == '-' || s[i] == '+' ||
                            s[i] == '.' || s[i] == 'e' || s[i] == 'E'))
      ++i;
    if (b == i) bad("unexpected character");
    v.type = Json::NUM;
    v.str = s.substr(b, i - b);
    char* end = nullptr;
    v.num = std::strtod(v.str.c_str(), &end);
    if (!end || *end) bad("bad number '" + v.str + "'");
    return v;
  }
};

// typed field access with JSON-path errors (SchemaError)
struct Obj {
  const Json& j;
  std::string path;
  [[noreturn]] void bad(const std::string& k, const std::string& what) const {
    fail(SC_ERR_SCHEMA_ERROR, path + (k.empty() ? "" : "." + k) + ": " + what);
  }
  const Json& need(const std::string& k) const {
    const Json* v = j.get(k);
    if (!v) bad(k, "missing");
    return *v;
  }
  int64_t integer(const std::string& k, int64_t lo, int64_t hi) const {
    const Json& v = need(k);
    return as_int(v, path + "." + k, lo, hi);
  }
  int64_t integer_or(const std::string& k, int64_t dflt, int64_t lo, int64_t hi) const {
    return j.get(k) ? integer(k, lo, hi) : dflt;
  }
  static int64_t as_int(const Json& v, const std::string& p, int64_t lo, int64_t hi) {
    if (v.type != Json::NUM || v.str.find_first_of(".eE") != std::string::npos)
      fail(SC_ERR_SCHEMA_ERROR, p + ": expected an integer");
    const long long x = std::strtoll(v.str.c_str(), nullptr, 10);
    if (x < lo || x > hi)
      fail(SC_ERR_SCHEMA_ERROR, p + ": " + v.str + " out of range [" + std::to_string(lo) + ", " + std::to_string(hi) + "]");
    return x;
  }
  std::string text(const std::string& k) const {
    const Json& v = need(k);
    if (v.type != Json::STR) bad(k, "expected a string");
    return v.str;
  }
};

const char* kKinds[] = {"Source", "Sink", "Conv", "ZeroUpsample", "Activation",
                        "Delay", "Sum", "Fanout", "Gate", "Slice"};
const char* kActs[] = {"identity", "tanh", "leaky_relu"};
constexpr int64_t kI32 = 0x7fffffff;

std::string read_file(const std::string& path, int missing_code) {
  std::ifstream f(path, std::ios::binary);
  if (!f) fail(missing_code, "cannot open '" + path + "'");
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

std::string blob_path_for(const char* manifest, const char* blob) {
  if (blob) return blob;
  std::string p(manifest);
  const size_t slash = p.find_last_of('/');
  const size_t dot = p.find_last_of('.');
  if (dot != std::string::npos && (slash == std::string::npos || dot > slash)) p.resize(dot);
  return p + ".bin";
}

int64_t conv_floats(const sc_gnode& nd) {
  return static_cast<int64_t>(nd.out_channels) * nd.in_channels * nd.taps + nd.out_channels;
}

}  // namespace

std::unique_ptr<sc_model> model_load(const char* manifest_path, const char* blob_path) {
  if (!manifest_path) fail(SC_ERR_INVALID_ARGUMENT, "manifest path is null");
  const std::string text = read_file(manifest_path, SC_ERR_INVALID_ARGUMENT);
  Parser ps{text};
  const Json root = ps.value(0);
  ps.ws();
  if (ps.i != text.size()) ps.bad("trailing characters");
  if (root.type != Json::OBJ) fail(SC_ERR_SCHEMA_ERROR, "$: expected an object");
  Obj r{root, "$"};
  const int64_t ver = r.integer("format_version", 0, kI32);
  if (ver != 1) fail(SC_ERR_VERSION_MISMATCH, "$.format_version: " + std::to_string(ver) + " (this library reads 1)");
  auto m = std::make_unique<sc_model>();
  m->in_channels = static_cast<int32_t>(r.integer("in_channels", 1, kI32));
  const Json& nodes = r.need("nodes");
  if (nodes.type != Json::ARR) r.bad("nodes", "expected an array");
  struct Range {
    int64_t off, len;
    int node;
  };
  std::vector<Range> ranges;
  for (size_t i = 0; i < nodes.arr.size(); ++i) {
    const std::string p = "$.nodes[" + std::to_string(i) + "]";
    if (nodes.arr[i].type != Json::OBJ) fail(SC_ERR_SCHEMA_ERROR, p + ": expected an object");
    Obj o{nodes.arr[i], p};
    if (o.integer("id", 0, kI32) != static_cast<int64_t>(i))
      o.bad("id", "node ids must be dense and in order (expected " + std::to_string(i) + ")");
    const std::string kind = o.text("kind");
    int k = -1;
    for (int q = 0; q <= SC_G_SLICE; ++q)
      if (kind == kKinds[q]) k = q;
    if (k < 0) o.bad("kind", "unknown node kind '" + kind + "'");
    sc_gnode nd{};
    nd.kind = k;
    switch (k) {
      case SC_G_SOURCE:
        nd.out_channels = static_cast<int32_t>(o.integer_or("channels", 0, 0, kI32));
        break;
      case SC_G_CONV: {
        nd.in_channels = static_cast<int32_t>(o.integer("in_channels", 1, kI32));
        nd.out_channels = static_cast<int32_t>(o.integer("out_channels", 1, kI32));
        nd.taps = static_cast<int32_t>(o.integer("kernel", 1, kI32));
        nd.stride = static_cast<int32_t>(o.integer_or("stride", 1, 1, kI32));
        nd.dilation = static_cast<int32_t>(o.integer_or("dilation", 1, 1, kI32));
        const Json& pad = o.need("padding");
        if (pad.type != Json::ARR || pad.arr.size() != 2) o.bad("padding", "expected [left, right]");
        nd.pad_left = Obj::as_int(pad.arr[0], p + ".padding[0]", 0, kI32);
        nd.pad_right = Obj::as_int(pad.arr[1], p + ".padding[1]", 0, kI32);
        nd.shift = o.integer_or("shift", 0, 0, kI32);
        if (o.j.get("hint")) {
          const std::string h = o.text("hint");
          if (h == "pqmf") nd.hint = SC_HINT_PQMF;
          else if (h != "none") o.bad("hint", "unknown hint '" + h + "'");
        }
        const Json& w = o.need("weights");
        if (w.type != Json::OBJ) o.bad("weights", "expected {offset, length}");
        Obj wo{w, p + ".weights"};
        const int64_t off = wo.integer("offset", 0, INT64_MAX / 2);
        const int64_t len = wo.integer("length", 0, INT64_MAX / 2);
        if (off % 4) wo.bad("offset", "must be a multiple of 4 bytes");
        if (len != conv_floats(nd) * 4)
          fail(SC_ERR_CORRUPT_BLOB, p + ".weights.length: " + std::to_string(len) + " bytes, the Conv needs " +
                                        std::to_string(conv_floats(nd) * 4) + " (weights [n][m][k] + bias [n])");
        ranges.push_back(Range{off, len, static_cast<int>(i)});
        nd.weight_offset = off / 4;
        break;
      }
      case SC_G_ZERO_UPSAMPLE:
        nd.factor = static_cast<int32_t>(o.integer("factor", 1, kI32));
        break;
      case SC_G_ACTIVATION: {
        const std::string a = o.text("act");
        nd.act = -1;
        for (int q = 0; q < 3; ++q)
          if (a == kActs[q]) nd.act = q;
        if (nd.act < 0) o.bad("act", "unknown activation '" + a + "'");
        if (o.j.get("alpha")) {
          const Json& al = o.need("alpha");
          if (al.type != Json::NUM) o.bad("alpha", "expected a number");
          nd.alpha = static_cast<float>(al.num);
        } else {
          nd.alpha = 0.01f;  // reference default (kernels.hpp:32)
        }
        break;
      }
      case SC_G_DELAY:
        nd.samples = o.integer("samples", 0, INT64_MAX / 4);
        if (o.j.get("inserted")) {
          const Json& b = o.need("inserted");
          if (b.type != Json::BOOL) o.bad("inserted", "expected true or false");
          nd.inserted = b.b ? 1 : 0;
        }
        break;
      case SC_G_SUM:
      case SC_G_FANOUT:
        nd.arity = static_cast<int32_t>(o.integer("arity", 2, kI32));
        break;
      case SC_G_SLICE:
        nd.slice_begin = static_cast<int32_t>(o.integer("begin", 0, kI32));
        nd.slice_count = static_cast<int32_t>(o.integer("count", 1, kI32));
        break;
      default:
        break;
    }
    m->nodes.push_back(nd);
  }
  const Json& edges = r.need("edges");
  if (edges.type != Json::ARR) r.bad("edges", "expected an array");
  for (size_t e = 0; e < edges.arr.size(); ++e) {
    const std::string p = "$.edges[" + std::to_string(e) + "]";
    const Json& ed = edges.arr[e];
    if (ed.type != Json::ARR || ed.arr.size() != 3) fail(SC_ERR_SCHEMA_ERROR, p + ": expected [from, to, port]");
    m->edges.push_back(sc_edge{static_cast<int32_t>(Obj::as_int(ed.arr[0], p + "[0]", 0, kI32)),
                               static_cast<int32_t>(Obj::as_int(ed.arr[1], p + "[1]", 0, kI32)),
                               static_cast<int32_t>(Obj::as_int(ed.arr[2], p + "[2]", 0, kI32))});
  }
  // blob: exactly the declared, non-overlapping, in-bounds weight ranges
  const std::string bp = blob_path_for(manifest_path, blob_path);
  const std::string blob = read_file(bp, SC_ERR_CORRUPT_BLOB);
  int64_t total = 0;
  std::sort(ranges.begin(), ranges.end(), [](const Range& a, const Range& b) { return a.off < b.off; });
  for (size_t q = 0; q < ranges.size(); ++q) {
    const Range& g = ranges[q];
    if (g.off + g.len > static_cast<int64_t>(blob.size()))
      fail(SC_ERR_CORRUPT_BLOB, "$.nodes[" + std::to_string(g.node) + "].weights: bytes [" + std::to_string(g.off) + ", " +
                                    std::to_string(g.off + g.len) + ") run past the " + std::to_string(blob.size()) +
                                    "-byte blob '" + bp + "'");
    if (q > 0 && ranges[q - 1].off + ranges[q - 1].len > g.off)
      fail(SC_ERR_CORRUPT_BLOB, "$.nodes[" + std::to_string(g.node) + "].weights overlaps $.nodes[" +
                                    std::to_string(ranges[q - 1].node) + "].weights");
    total += g.len;
  }
  if (total != static_cast<int64_t>(blob.size()))
    fail(SC_ERR_CORRUPT_BLOB, "blob '" + bp + "' holds " + std::to_string(blob.size()) + " bytes, the manifest declares " +
                                  std::to_string(total));
  m->weights.resize(blob.size() / 4);
  std::memcpy(m->weights.data(), blob.data(), m->weights.size() * 4);  // little-endian host
  // the manifest schema rejects every graph validate rejects, with the same categories
  dag_validate(m->nodes.data(), static_cast<int>(m->nodes.size()), m->edges.data(),
               static_cast<int>(m->edges.size()), m->in_channels);
  return m;
}

void model_save(const char* manifest_path, const char* blob_path, const sc_gnode* nodes, int n,
                const sc_edge* edges, int ne, const float* W, int64_t nW, int in_C) {
  if (!manifest_path) fail(SC_ERR_INVALID_ARGUMENT, "manifest path is null");
  dag_validate(nodes, n, edges, ne, in_C);
  std::ostringstream js;
  std::vector<float> blob;
  char buf[64];
  js << "{\n  \"format_version\": 1,\n  \"in_channels\": " << in_C << ",\n  \"nodes\": [\n";
  for (int i = 0; i < n; ++i) {
    const sc_gnode& nd = nodes[i];
    js << "    {\"id\": " << i << ", \"kind\": \"" << kKinds[nd.kind] << "\"";
    switch (nd.kind) {
      case SC_G_SOURCE:
        js << ", \"channels\": " << (nd.out_channels > 0 ? nd.out_channels : in_C);
        break;
      case SC_G_CONV: {
        const int64_t nf = conv_floats(nd);
        if (nd.weight_offset < 0 || nd.weight_offset + nf > nW)
          fail(SC_ERR_INVALID_ARGUMENT, "node " + std::to_string(i) + ": weights out of range");
        js << ", \"in_channels\": " << nd.in_channels << ", \"out_channels\": " << nd.out_channels
           << ", \"kernel\": " << nd.taps << ", \"stride\": " << nd.stride << ", \"dilation\": " << nd.dilation
           << ", \"padding\": [" << nd.pad_left << ", " << nd.pad_right << "], \"shift\": " << nd.shift
           << ", \"hint\": \"" << (nd.hint == SC_HINT_PQMF ? "pqmf" : "none") << "\", \"weights\": {\"offset\": "
           << blob.size() * 4 << ", \"length\": " << nf * 4 << "}";
        blob.insert(blob.end(), W + nd.weight_offset, W + nd.weight_offset + nf);
        break;
      }
      case SC_G_ZERO_UPSAMPLE:
        js << ", \"factor\": " << nd.factor;
        break;
      case SC_G_ACTIVATION:
        std::snprintf(buf, sizeof buf, "%.9g", static_cast<double>(nd.alpha));
        js << ", \"act\": \"" << kActs[nd.act] << "\", \"alpha\": " << buf;
        break;
      case SC_G_DELAY:
        js << ", \"samples\": " << nd.samples << ", \"inserted\": " << (nd.inserted ? "true" : "false");
        break;
      case SC_G_SUM:
      case SC_G_FANOUT:
        js << ", \"arity\": " << nd.arity;
        break;
      case SC_G_SLICE:
        js << ", \"begin\": " << nd.slice_begin << ", \"count\": " << nd.slice_count;
        break;
      default:
        break;
    }
    js << "}" << (i + 1 < n ? "," : "") << "\n";
  }
  js << "  ],\n  \"edges\": [";
  for (int e = 0; e < ne; ++e)
    js << (e ? ", " : "") << "[" << edges[e].from << ", " << edges[e].to << ", " << edges[e].port << "]";
  js << "]\n}\n";
  const std::string bp = blob_path_for(manifest_path, blob_path);
  std::ofstream fj(manifest_path, std::ios::binary);
  if (!fj) fail(SC_ERR_INVALID_ARGUMENT, std::string("cannot write '") + manifest_path + "'");
  fj << js.str();
  std::ofstream fb(bp, std::ios::binary);
  if (!fb) fail(SC_ERR_INVALID_ARGUMENT, "cannot write '" + bp + "'");
  fb.write(reinterpret_cast<const char*>(blob.data()), static_cast<std::streamsize>(blob.size() * 4));
  if (!fj || !fb) fail(SC_ERR_INVALID_ARGUMENT, "write failed");
}

}  // namespace scb
