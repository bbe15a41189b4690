// SPDX-License-Identifier: Apache-2.0
//
// Plan wire format: plan_to_json / plan_from_json (balancer.hpp:105-109,
// balancer.cpp:289-352), byte-identical to the reference.
//
// The reference serialises with nlohmann::json 3.11.3 (a third-party header
// absent from /root/reference: proj/.gitignore:2 excludes vendor/).  Its
// observable format, restated here from the library's published behaviour:
//   * objects print their keys in std::map (byte-wise ascending) order, no
//     whitespace: {"a":1,"b":[2,3]};
//   * integers in plain decimal; doubles through Grisu2 (Loitsch, PLDI 2010:
//     diy-fp with q = 64, alpha = -60, gamma = -32, cached powers of ten
//     every 8 decades -- tools/gen_pow10.py) and a %g-like layout: fixed
//     notation for 10^-4 <= v < 10^15 with ".0" on integral values,
//     otherwise d.ddde+XX; +-0 as "0.0"/"-0.0"; NaN/inf as null.
// plan_from_json reads that schema back with a small strict JSON reader
// (numbers, strings without escapes beyond \" \\ \/ \b \f \n \r \t, arrays,
// objects, true/false/null) -- malformed text raises ParseError with a byte
// offset (the reference raises nlohmann::json::parse_error; the CLI maps
// both to exit code 1).
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "seqbal/seqbal.hpp"

namespace seqbal {
namespace json_detail {

// --------------------------------------------------------------- Grisu2
struct Fp {  // f * 2^e
  std::uint64_t f;
  int e;
};

Fp fp_sub(Fp x, Fp y) { return {x.f - y.f, x.e}; }

// (x.f * y.f) / 2^64 rounded half up, exponent x.e + y.e + 64.
Fp fp_mul(Fp x, Fp y) {
  const unsigned __int128 p = static_cast<unsigned __int128>(x.f) * y.f;
  std::uint64_t h = static_cast<std::uint64_t>(p >> 64);
  const std::uint64_t l = static_cast<std::uint64_t>(p);
  h += l >> 63;  // round half up on the discarded low word
  return {h, x.e + y.e + 64};
}

Fp fp_normalize(Fp x) {
  while ((x.f >> 63) == 0) {
    x.f <<= 1;
    --x.e;
  }
  return x;
}

struct CachedPow {
  std::uint64_t f;
  int e;
  int k;
};

const CachedPow kPow10[] = {
#include "pow10_table.inc"
};

// A cached 10^k with -60 <= e_c + e + 64 <= -32 for a normalised w = f*2^e.
CachedPow cached_pow10(int e) {
  const int f = -60 - e - 1;
  const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);  // ~ ceil(f * log10(2))
  const int index = (300 + k + 7) / 8;
  return kPow10[index];
}

int largest_pow10(std::uint32_t n, std::uint32_t& pow10) {
  std::uint32_t p = 1;
  int k = 1;
  while (k < 10 && n >= p * 10) {
    p *= 10;
    ++k;
  }
  pow10 = p;
  return k;
}

void round_weed(char* buf, int len, std::uint64_t dist, std::uint64_t delta, std::uint64_t rest, std::uint64_t ten_k) {
  // move the last digit down while the candidate stays inside the interval
  // and gets closer to w
  while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
    buf[len - 1]--;
    rest += ten_k;
  }
}

// Digits of M+ cut as soon as the remainder fits into [M-, M+].
void digit_gen(char* buf, int& len, int& dec_exp, Fp m_minus, Fp w, Fp m_plus) {
  std::uint64_t delta = fp_sub(m_plus, m_minus).f;
  std::uint64_t dist = fp_sub(m_plus, w).f;
  const int shift = -m_plus.e;  // 32..60
  const std::uint64_t one = std::uint64_t{1} << shift;
  auto p1 = static_cast<std::uint32_t>(m_plus.f >> shift);
  std::uint64_t p2 = m_plus.f & (one - 1);
  std::uint32_t pow10 = 1;
  int n = largest_pow10(p1, pow10);
  while (n > 0) {
    const std::uint32_t d = p1 / pow10;
    p1 %= pow10;
    buf[len++] = static_cast<char>('0' + d);
    --n;
    const std::uint64_t rest = (static_cast<std::uint64_t>(p1) << shift) + p2;
    if (rest <= delta) {
      dec_exp += n;
      round_weed(buf, len, dist, delta, rest, static_cast<std::uint64_t>(pow10) << shift);
      return;
    }
    pow10 /= 10;
  }
  int m = 0;
  for (;;) {
    p2 *= 10;
    buf[len++] = static_cast<char>('0' + (p2 >> shift));
    p2 &= one - 1;
    ++m;
    delta *= 10;
    dist *= 10;
    if (p2 <= delta) break;
  }
  dec_exp -= m;
  round_weed(buf, len, dist, delta, p2, one);
}

// value > 0, finite: digits and decimal exponent of a short round-trip form.
void grisu2(char* buf, int& len, int& dec_exp, double value) {
  std::uint64_t bits;
  std::memcpy(&bits, &value, 8);
  const std::uint64_t E = bits >> 52, F = bits & ((std::uint64_t{1} << 52) - 1);
  const Fp v = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (std::uint64_t{1} << 52), static_cast<int>(E) - 1075};
  const bool lower_closer = F == 0 && E > 1;
  const Fp m_plus = fp_normalize(Fp{2 * v.f + 1, v.e - 1});
  Fp m_minus = lower_closer ? Fp{4 * v.f - 1, v.e - 2} : Fp{2 * v.f - 1, v.e - 1};
  m_minus = Fp{m_minus.f << (m_minus.e - m_plus.e), m_plus.e};
  const Fp w = fp_normalize(v);
  const CachedPow c = cached_pow10(m_plus.e);
  const Fp ck{c.f, c.e};
  const Fp ww = fp_mul(w, ck), wm = fp_mul(m_minus, ck), wp = fp_mul(m_plus, ck);
  dec_exp = -c.k;
  len = 0;
  digit_gen(buf, len, dec_exp, Fp{wm.f + 1, wm.e}, ww, Fp{wp.f - 1, wp.e});
}

std::string format_double(double x) {
  if (!std::isfinite(x)) return "null";
  char buf[64];
  char* p = buf;
  if (std::signbit(x)) {
    *p++ = '-';
    x = -x;
  }
  if (x == 0.0) {
    std::memcpy(p, "0.0", 3);
    return std::string(buf, p + 3);
  }
  int len = 0, dec = 0;
  grisu2(p, len, dec, x);
  const int k = len, n = len + dec;  // value = 0.d1d2...dk * 10^n
  std::string digits(p, p + k);
  std::string out(buf, p);
  if (k <= n && n <= 15) {  // integral: digits, zeros, ".0"
    out += digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {  // dig.its
    out += digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
  } else if (-4 < n && n <= 0) {  // 0.[000]digits
    out += "0." + std::string(static_cast<size_t>(-n), '0') + digits;
  } else {  // d[.igits]e+XX
    out += digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    int e = n - 1;
    out += e < 0 ? "e-" : "e+";
    e = e < 0 ? -e : e;
    if (e < 10) out += "0";
    out += std::to_string(e);
  }
  return out;
}

// ---------------------------------------------------------------- reader
struct Value {
  enum Kind { Null, Bool, Int, UInt, Float, Str, Arr, Obj } kind = Null;
  bool b = false;
  std::int64_t i = 0;
  std::uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> a;
  std::map<std::string, Value> o;

  const Value& at(const std::string& key) const {
    if (kind != Obj) throw ConfigError("plan JSON: expected an object holding '" + key + "'");
    auto it = o.find(key);
    if (it == o.end()) throw ConfigError("plan JSON: missing key '" + key + "'");
    return it->second;
  }
  bool contains(const std::string& key) const { return kind == Obj && o.count(key) > 0; }
  const std::vector<Value>& arr() const {
    if (kind != Arr) throw ConfigError("plan JSON: expected an array");
    return a;
  }
  std::int64_t as_i64() const {
    if (kind == Int) return i;
    if (kind == UInt && u <= static_cast<std::uint64_t>(INT64_MAX)) return static_cast<std::int64_t>(u);
    if (kind == Float && d == std::floor(d) && std::fabs(d) < 9.2e18) return static_cast<std::int64_t>(d);
    throw ConfigError("plan JSON: expected an integer");
  }
  std::uint64_t as_u64() const {
    if (kind == UInt) return u;
    if (kind == Int && i >= 0) return static_cast<std::uint64_t>(i);
    throw ConfigError("plan JSON: expected an unsigned integer");
  }
  double as_f64() const {
    if (kind == Float) return d;
    if (kind == Int) return static_cast<double>(i);
    if (kind == UInt) return static_cast<double>(u);
    if (kind == Null) return std::numeric_limits<double>::quiet_NaN();  // non-finite doubles dump as null
    throw ConfigError("plan JSON: expected a number");
  }
};

class Reader {
 public:
  explicit Reader(const std::string& t) : t_(t) {}
  Value parse() {
    Value v = value();
    ws();
    if (p_ != t_.size()) fail("trailing characters after the JSON value");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const { throw ParseError("plan JSON: " + what, p_); }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  Value value() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[p_];
    Value v;
    if (c == '{') {
      ++p_;
      v.kind = Value::Obj;
      if (eat('}')) return v;
      do {
        ws();
        const std::string k = string();
        expect(':');
        v.o[k] = value();
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++p_;
      v.kind = Value::Arr;
      if (eat(']')) return v;
      do v.a.push_back(value());
      while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = Value::Str;
      v.s = string();
    } else if (t_.compare(p_, 4, "true") == 0) {
      p_ += 4;
      v.kind = Value::Bool;
      v.b = true;
    } else if (t_.compare(p_, 5, "false") == 0) {
      p_ += 5;
      v.kind = Value::Bool;
    } else if (t_.compare(p_, 4, "null") == 0) {
      p_ += 4;
    } else {
      number(v);
    }
    return v;
  }
  std::string string() {
    if (p_ >= t_.size() || t_[p_] != '"') fail("expected a string");
    ++p_;
    std::string out;
    while (p_ < t_.size() && t_[p_] != '"') {
      char c = t_[p_++];
      if (c == '\\') {
        if (p_ >= t_.size()) fail("unterminated escape");
        const char e = t_[p_++];
        switch (e) {
          case '"': c = '"'; break;
          case '\\': c = '\\'; break;
          case '/': c = '/'; break;
          case 'b': c = '\b'; break;
          case 'f': c = '\f'; break;
          case 'n': c = '\n'; break;
          case 'r': c = '\r'; break;
          case 't': c = '\t'; break;
          default: fail("unsupported escape");
        }
      }
      out += c;
    }
    if (p_ >= t_.size()) fail("unterminated string");
    ++p_;
    return out;
  }
  void number(Value& v) {
    const size_t b = p_;
    bool neg = false, frac = false;
    if (t_[p_] == '-') {
      neg = true;
      ++p_;
    }
    const size_t digits0 = p_;
    while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
    if (p_ == digits0) fail("invalid number");
    if (p_ < t_.size() && t_[p_] == '.') {
      frac = true;
      ++p_;
      const size_t f0 = p_;
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
      if (p_ == f0) fail("invalid number");
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      frac = true;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      const size_t e0 = p_;
      while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) ++p_;
      if (p_ == e0) fail("invalid number");
    }
    const std::string tok = t_.substr(b, p_ - b);
    if (!frac) {
      errno = 0;
      if (neg) {
        v.kind = Value::Int;
        v.i = std::strtoll(tok.c_str(), nullptr, 10);
      } else {
        v.kind = Value::UInt;
        v.u = std::strtoull(tok.c_str(), nullptr, 10);
      }
      if (errno == 0) return;
    }
    v.kind = Value::Float;
    v.d = std::strtod(tok.c_str(), nullptr);  // correctly rounded (glibc)
  }
  const std::string& t_;
  size_t p_ = 0;
};

}  // namespace json_detail

std::string plan_to_json(const RoutingPlan& plan, const BalanceReport& report) {
  using json_detail::format_double;
  std::string s;
  s.reserve(64 + plan.chunks.size() * 96);
  s += "{\"chunks\":[";
  for (size_t i = 0; i < plan.chunks.size(); ++i) {
    const ChunkAssignment& c = plan.chunks[i];
    if (i) s += ',';
    s += "{\"chunk_index\":" + std::to_string(c.chunk_index) + ",\"dst\":" + std::to_string(c.target_rank) +
         ",\"end\":" + std::to_string(c.end) + ",\"sample_id\":" + std::to_string(c.sample_id) +
         ",\"src\":" + std::to_string(c.source_rank) + ",\"start\":" + std::to_string(c.start) + "}";
  }
  s += "],\"origins\":[";
  for (size_t r = 0; r < plan.origin.size(); ++r) {
    if (r) s += ',';
    s += '[';
    for (size_t q = 0; q < plan.origin[r].size(); ++q) {
      const Segment& g = plan.origin[r][q];
      if (q) s += ',';
      s += "{\"first_pos\":" + std::to_string(g.first_pos) + ",\"len\":" + std::to_string(g.length) +
           ",\"sample_id\":" + std::to_string(g.sample_id) + "}";
    }
    s += ']';
  }
  auto darr = [&](const std::vector<double>& v) {
    s += '[';
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) s += ',';
      s += format_double(v[i]);
    }
    s += ']';
  };
  s += "],\"report\":{\"capacity_violations\":" + std::to_string(report.capacity_violations) +
       ",\"per_bag_occupancy\":";
  darr(report.per_bag_occupancy);
  s += ",\"per_gpu_workload\":";
  darr(report.per_gpu_workload);
  s += ",\"total_workload\":" + format_double(report.total_workload) + ",\"wir\":" + format_double(report.wir) +
       "},\"world_size\":" + std::to_string(plan.world_size) + "}";
  return s;
}

PlanResult plan_from_json(const std::string& text) {
  const json_detail::Value j = json_detail::Reader(text).parse();
  PlanResult result;
  RoutingPlan& plan = result.plan;
  plan.world_size = static_cast<int>(j.at("world_size").as_i64());
  for (const auto& c : j.at("chunks").arr()) {
    plan.chunks.push_back({c.at("sample_id").as_u64(), static_cast<int>(c.at("chunk_index").as_i64()),
                           c.at("start").as_i64(), c.at("end").as_i64(), static_cast<int>(c.at("src").as_i64()),
                           static_cast<int>(c.at("dst").as_i64())});
  }
  const auto& origins = j.at("origins").arr();
  if (static_cast<int>(origins.size()) != plan.world_size)
    throw ConfigError("plan JSON: origins size does not match world_size");  // balancer.cpp:331-333
  plan.origin.resize(plan.world_size);
  for (int r = 0; r < plan.world_size; ++r)
    for (const auto& s : origins[r].arr())
      plan.origin[r].push_back({s.at("sample_id").as_u64(), s.at("first_pos").as_i64(), s.at("len").as_i64()});
  // finalize_manifests + fill_target_layout (balancer.cpp:84-101)
  plan.send.assign(plan.world_size, {});
  plan.recv.assign(plan.world_size, {});
  for (size_t i = 0; i < plan.chunks.size(); ++i) {
    const ChunkAssignment& c = plan.chunks[i];
    if (c.source_rank < 0 || c.source_rank >= plan.world_size || c.target_rank < 0 ||
        c.target_rank >= plan.world_size)
      throw ConfigError("plan JSON: chunk rank outside the world");
    plan.send[c.source_rank].push_back(static_cast<int>(i));
    plan.recv[c.target_rank].push_back(static_cast<int>(i));
  }
  plan.target.assign(plan.world_size, {});
  for (int r = 0; r < plan.world_size; ++r)
    for (int ci : plan.recv[r]) {
      const ChunkAssignment& c = plan.chunks[ci];
      plan.target[r].push_back({c.sample_id, c.start, c.end - c.start});
    }
  if (j.contains("report")) {
    const auto& rep = j.at("report");
    for (const auto& v : rep.at("per_gpu_workload").arr()) result.report.per_gpu_workload.push_back(v.as_f64());
    for (const auto& v : rep.at("per_bag_occupancy").arr()) result.report.per_bag_occupancy.push_back(v.as_f64());
    result.report.capacity_violations = static_cast<int>(rep.at("capacity_violations").as_i64());
    result.report.total_workload = rep.at("total_workload").as_f64();
    result.report.wir = rep.at("wir").as_f64();
  }
  return result;
}

}  // namespace seqbal

// Test hook (tests/cpp/test_json.cpp checks it against the reference's
// serializer on random doubles): nlohmann-compatible double text.
extern "C" __attribute__((visibility("default"))) size_t sb_json_format_double(double x, char* buf, size_t cap) {
  const std::string s = seqbal::json_detail::format_double(x);
  if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  return s.size();
}

// Test hook: plan_to_json(plan_from_json(text)) -- host-only (no device);
// returns the output length, or -1 with the error text in `out`.
extern "C" __attribute__((visibility("default"))) long sb_json_plan_roundtrip(const char* text, char* out, size_t cap) {
  std::string s;
  long rc;
  try {
    const seqbal::PlanResult pr = seqbal::plan_from_json(text);
    s = seqbal::plan_to_json(pr.plan, pr.report);
    rc = static_cast<long>(s.size());
  } catch (const std::exception& e) {
    s = e.what();
    rc = -1;
  }
  if (out && cap > s.size()) std::memcpy(out, s.c_str(), s.size() + 1);
  return rc;
}

namespace seqbal {
// seq-lens file of the CLI's `plan` (tools/main.cpp:200-218): a JSON array of
// per-rank arrays of lengths; // and /* */ comments allowed as in the
// reference's json::parse(in, nullptr, true, true).
std::vector<std::vector<std::int64_t>> read_lens_json(const std::string& text) {
  std::string t;
  t.reserve(text.size());
  for (size_t i = 0; i < text.size(); ++i) {  // strip comments outside strings
    if (text[i] == '"') {
      const size_t j = text.find('"', i + 1);
      t.append(text, i, (j == std::string::npos ? text.size() : j + 1) - i);
      i = j == std::string::npos ? text.size() : j;
    } else if (text.compare(i, 2, "//") == 0) {
      i = text.find('\n', i);
      if (i == std::string::npos) break;
      t += '\n';
    } else if (text.compare(i, 2, "/*") == 0) {
      const size_t j = text.find("*/", i + 2);
      if (j == std::string::npos) throw ParseError("seq-lens: unterminated comment", i);
      t += ' ';
      i = j + 1;
    } else {
      t += text[i];
    }
  }
  const json_detail::Value j = json_detail::Reader(t).parse();
  if (j.kind != json_detail::Value::Arr) throw ConfigError("seq-lens file must be a JSON array of arrays");
  std::vector<std::vector<std::int64_t>> out;
  for (const auto& r : j.a) {
    if (r.kind != json_detail::Value::Arr) throw ConfigError("each rank entry must be an array");
    std::vector<std::int64_t> lens;
    for (const auto& l : r.a) {
      const std::int64_t len = l.as_i64();
      if (len < 0) throw ConfigError("sequence lengths must be >= 0");
      lens.push_back(len);
    }
    out.push_back(std::move(lens));
  }
  return out;
}
}  // namespace seqbal
