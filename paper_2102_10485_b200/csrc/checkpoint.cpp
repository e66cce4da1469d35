// Checkpoint files of one label's (G, D) pair in the reference's on-disk format
// (/root/reference/proj/src/checkpoint.cpp:91-194, save_gan_pair / load_gan_pair):
//   u32 little-endian header length | JSON header | f64 LE blobs in table order
//   gen_params, gen_buffers, disc_params, disc_buffers, opt_g_m, opt_g_v, opt_d_m, opt_d_v
// in the reference flat layouts (Network::params(), buffers(), AdamState m/v),
// so a file written here loads into the CPU reference and vice versa.  The
// layer schema (checkpoint.cpp:19-65) gains "conv_transpose2d" with the conv2d
// fields.  The header is written compact with sorted keys and shortest
// round-trip numbers, as nlohmann::json::dump() does.
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "gan.hpp"

namespace pg {

namespace {

// ---------------------------------------------------------------- JSON value

struct Json {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  bool is_int = false;
  long long i = 0;
  std::string str;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;  // sorted keys, as nlohmann's default object

  static Json integer(long long v) {
    Json j;
    j.kind = Num;
    j.is_int = true;
    j.i = v;
    j.num = static_cast<double>(v);
    return j;
  }
  static Json real(double v) {
    Json j;
    j.kind = Num;
    j.num = v;
    return j;
  }
  static Json string(const std::string& s) {
    Json j;
    j.kind = Str;
    j.str = s;
    return j;
  }
  static Json array() {
    Json j;
    j.kind = Arr;
    return j;
  }
  static Json object() {
    Json j;
    j.kind = Obj;
    return j;
  }
  Json& operator[](const std::string& k) {
    kind = Obj;
    return obj[k];
  }
  const Json& at(const std::string& k) const {
    auto it = obj.find(k);
    if (kind != Obj || it == obj.end()) throw std::runtime_error("checkpoint header: missing key '" + k + "'");
    return it->second;
  }
  long long as_int() const {
    if (kind != Num) throw std::runtime_error("checkpoint header: number expected");
    return is_int ? i : static_cast<long long>(num);
  }
  double as_double() const {
    if (kind != Num) throw std::runtime_error("checkpoint header: number expected");
    return num;
  }
  const std::string& as_str() const {
    if (kind != Str) throw std::runtime_error("checkpoint header: string expected");
    return str;
  }
};

// shortest decimal that round-trips (what nlohmann's dump() prints for doubles)
std::string fmt_double(double v) {
  char buf[40];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string s(buf);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";  // keep it a float
  return s;
}

void dump(const Json& j, std::string& o) {
  switch (j.kind) {
    case Json::Null: o += "null"; return;
    case Json::Bool: o += j.b ? "true" : "false"; return;
    case Json::Num: o += j.is_int ? std::to_string(j.i) : fmt_double(j.num); return;
    case Json::Str:
      o += '"';
      for (char c : j.str) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
      }
      o += '"';
      return;
    case Json::Arr:
      o += '[';
      for (size_t k = 0; k < j.arr.size(); ++k) {
        if (k) o += ',';
        dump(j.arr[k], o);
      }
      o += ']';
      return;
    case Json::Obj: {
      o += '{';
      bool first = true;
      for (const auto& [k, v] : j.obj) {
        if (!first) o += ',';
        first = false;
        dump(Json::string(k), o);
        o += ':';
        dump(v, o);
      }
      o += '}';
      return;
    }
  }
}

struct Parser {
  const std::string& s;
  size_t p = 0;
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\t' || s[p] == '\r')) ++p;
  }
  [[noreturn]] void fail(const char* what) {
    throw std::runtime_error(std::string("checkpoint header: ") + what + " at offset " + std::to_string(p));
  }
  Json value() {
    ws();
    if (p >= s.size()) fail("unexpected end");
    const char c = s[p];
    if (c == '{') {
      ++p;
      Json j = Json::object();
      ws();
      if (p < s.size() && s[p] == '}') {
        ++p;
        return j;
      }
      for (;;) {
        ws();
        Json k = value();
        if (k.kind != Json::Str) fail("object key expected");
        ws();
        if (p >= s.size() || s[p] != ':') fail("':' expected");
        ++p;
        j.obj[k.str] = value();
        ws();
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == '}') {
          ++p;
          return j;
        }
        fail("',' or '}' expected");
      }
    }
    if (c == '[') {
      ++p;
      Json j = Json::array();
      ws();
      if (p < s.size() && s[p] == ']') {
        ++p;
        return j;
      }
      for (;;) {
        j.arr.push_back(value());
        ws();
        if (p < s.size() && s[p] == ',') {
          ++p;
          continue;
        }
        if (p < s.size() && s[p] == ']') {
          ++p;
          return j;
        }
        fail("',' or ']' expected");
      }
    }
    if (c == '"') {
      ++p;
      Json j;
      j.kind = Json::Str;
      while (p < s.size() && s[p] != '"') {
        if (s[p] == '\\' && p + 1 < s.size()) ++p;
        j.str += s[p++];
      }
      if (p >= s.size()) fail("unterminated string");
      ++p;
      return j;
    }
    if (s.compare(p, 4, "true") == 0) {
      p += 4;
      Json j;
      j.kind = Json::Bool;
      j.b = true;
      return j;
    }
    if (s.compare(p, 5, "false") == 0) {
      p += 5;
      Json j;
      j.kind = Json::Bool;
      return j;
    }
    if (s.compare(p, 4, "null") == 0) {
      p += 4;
      return Json{};
    }
    const size_t b = p;
    while (p < s.size() && (std::isdigit(static_cast<unsigned char>(s[p])) || s[p] == '-' || s[p] == '+' ||
                            s[p] == '.' || s[p] == 'e' || s[p] == 'E'))
      ++p;
    if (b == p) fail("value expected");
    const std::string t = s.substr(b, p - b);
    if (t.find_first_of(".eE") == std::string::npos) return Json::integer(std::stoll(t));
    return Json::real(std::strtod(t.c_str(), nullptr));
  }
};

// ---------------------------------------------------------------- layer schema

Json layer_json(const LayerSpec& l) {
  Json j = Json::object();
  j["type"] = Json::string(layer_name(l.kind));
  switch (l.kind) {
    case LK::Dense:
      j["in_dim"] = Json::integer(l.in);
      j["out_dim"] = Json::integer(l.out);
      break;
    case LK::Conv:
    case LK::ConvT:
      j["in_ch"] = Json::integer(l.in);
      j["out_ch"] = Json::integer(l.out);
      j["kernel"] = Json::integer(l.k);
      j["stride"] = Json::integer(l.s);
      j["padding"] = Json::integer(l.p);
      break;
    case LK::BN:
      j["channels"] = Json::integer(l.in);
      j["epsilon"] = Json::real(l.eps);
      j["momentum"] = Json::real(l.momentum);
      break;
    case LK::Upsample: j["scale_factor"] = Json::integer(l.scale); break;
    case LK::Dropout: j["rate"] = Json::real(l.rate); break;
    case LK::LReLU: j["slope"] = Json::real(l.slope); break;
    case LK::Reshape: {
      Json t = Json::array();
      for (long v : l.target) t.arr.push_back(Json::integer(v));
      j["target_shape"] = t;
      break;
    }
    default: break;
  }
  return j;
}

Json net_json(const DevNet& net) {
  Json j = Json::object();
  Json shape = Json::array();
  for (long v : net.ref_in_shape()) shape.arr.push_back(Json::integer(v));
  j["input_shape"] = shape;
  Json layers = Json::array();
  for (const auto& l : net.layers()) layers.arr.push_back(layer_json(l));
  j["layers"] = layers;
  return j;
}

Json adam_json(const GroupConfig& c, long long t) {
  Json j = Json::object();
  j["lr"] = Json::real(c.lr);
  j["beta1"] = Json::real(c.beta1);
  j["beta2"] = Json::real(c.beta2);
  j["eps"] = Json::real(c.eps);
  j["t"] = Json::integer(t);
  return j;
}

const char* const kBlobs[8] = {"gen_params", "gen_buffers", "disc_params", "disc_buffers",
                               "opt_g_m",    "opt_g_v",     "opt_d_m",     "opt_d_v"};
const int kFields[8] = {GanGroup::G_PARAMS, GanGroup::G_BUFFERS, GanGroup::D_PARAMS, GanGroup::D_BUFFERS,
                        GanGroup::G_M,      GanGroup::G_V,       GanGroup::D_M,      GanGroup::D_V};

}  // namespace

void save_checkpoint(GanGroup& grp, int label, const std::string& path) {
  const GroupConfig& c = grp.config();
  double ctr[3];
  grp.get(label, GanGroup::COUNTERS, ctr, 3);
  std::vector<std::vector<double>> blobs(8);
  for (int b = 0; b < 8; ++b) {
    const long n = grp.get(label, kFields[b], nullptr, 0);
    blobs[static_cast<size_t>(b)].resize(static_cast<size_t>(n));
    if (n > 0) grp.get(label, kFields[b], blobs[static_cast<size_t>(b)].data(), n);
  }
  Json h = Json::object();
  h["format"] = Json::string("partgan-checkpoint");
  h["version"] = Json::integer(1);
  h["d_z"] = Json::integer(c.d_z);
  h["d_y"] = Json::integer(0);  // unconditional pairs in distributed mode (run.cpp:394)
  h["prob_clamp"] = Json::real(c.clamp);
  h["steps"] = Json::integer(static_cast<long long>(ctr[2]));
  h["generator"] = net_json(grp.gen());
  h["discriminator"] = net_json(grp.disc());
  h["opt_g"] = adam_json(c, static_cast<long long>(ctr[0]));
  h["opt_d"] = adam_json(c, static_cast<long long>(ctr[1]));
  Json table = Json::array();
  for (int b = 0; b < 8; ++b) {
    Json e = Json::object();
    e["name"] = Json::string(kBlobs[b]);
    e["len"] = Json::integer(static_cast<long long>(blobs[static_cast<size_t>(b)].size()));
    table.arr.push_back(e);
  }
  h["blobs"] = table;
  std::string head;
  dump(h, head);
  std::ofstream out(path, std::ios::binary);
  if (!out) throw std::runtime_error("cannot write checkpoint " + path);
  const uint32_t len = static_cast<uint32_t>(head.size());
  const unsigned char le[4] = {static_cast<unsigned char>(len), static_cast<unsigned char>(len >> 8),
                               static_cast<unsigned char>(len >> 16), static_cast<unsigned char>(len >> 24)};
  out.write(reinterpret_cast<const char*>(le), 4);
  out.write(head.data(), static_cast<std::streamsize>(head.size()));
  for (const auto& v : blobs)  // x86-64 / aarch64 hosts are little-endian, as the format declares
    out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
  if (!out) throw std::runtime_error("short write on checkpoint " + path);
}

void load_checkpoint(GanGroup& grp, int label, const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open checkpoint " + path);
  unsigned char le[4] = {0, 0, 0, 0};
  in.read(reinterpret_cast<char*>(le), 4);
  const uint32_t len = le[0] | (le[1] << 8) | (le[2] << 16) | (static_cast<uint32_t>(le[3]) << 24);
  std::string head(len, '\0');
  in.read(head.data(), static_cast<std::streamsize>(len));
  if (!in) throw std::runtime_error("truncated checkpoint header in " + path);
  Json h;
  try {
    Parser ps{head};
    h = ps.value();
  } catch (const std::exception&) {
    throw std::runtime_error(path + " is not a checkpoint file");
  }
  if (h.kind != Json::Obj || h.obj.count("format") == 0 || h.obj.at("format").kind != Json::Str ||
      h.obj.at("format").str != "partgan-checkpoint")
    throw std::runtime_error(path + " is not a checkpoint file");
  // the architecture must be the group's (load_gan_pair rebuilds it; a group has one)
  std::string mine, theirs;
  dump(net_json(grp.gen()), mine);
  dump(h.at("generator"), theirs);
  std::string mine_d, theirs_d;
  dump(net_json(grp.disc()), mine_d);
  dump(h.at("discriminator"), theirs_d);
  if (mine != theirs || mine_d != theirs_d)
    throw std::runtime_error("checkpoint " + path + " holds a different architecture than this label group");
  if (h.at("d_z").as_int() != grp.config().d_z) throw std::runtime_error("checkpoint " + path + ": latent width differs");
  // blobs in table order (checkpoint.cpp:175-193)
  const Json& table = h.at("blobs");
  for (int b = 0; b < 8; ++b) {
    const long want = grp.get(label, kFields[b], nullptr, 0);
    bool found = false;
    for (const auto& e : table.arr) {
      if (e.at("name").as_str() != kBlobs[b]) continue;
      const long n = static_cast<long>(e.at("len").as_int());
      if (n != want)
        throw std::runtime_error("blob '" + std::string(kBlobs[b]) + "' in " + path + " has length " +
                                 std::to_string(n) + " but the architecture expects " + std::to_string(want));
      std::vector<double> v(static_cast<size_t>(n));
      if (n > 0) {
        in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(double)));
        if (!in) throw std::runtime_error("truncated blob '" + std::string(kBlobs[b]) + "' in " + path);
      }
      grp.set(label, kFields[b], v.data(), n);
      found = true;
      break;
    }
    if (!found) throw std::runtime_error("missing blob '" + std::string(kBlobs[b]) + "' in " + path);
  }
  const double ctr[3] = {static_cast<double>(h.at("opt_g").at("t").as_int()),
                         static_cast<double>(h.at("opt_d").at("t").as_int()),
                         static_cast<double>(h.at("steps").as_int())};
  grp.set(label, GanGroup::COUNTERS, ctr, 3);
}

}  // namespace pg
