// json_lite.hpp — a minimal JSON document model, parser and writer helpers for the engine's
// host tools (model files, run manifests). Numbers keep their literal text so 64-bit seeds
// round-trip exactly; doubles are written with 17 significant digits (exact round trip).
#pragma once

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/perfsage_b200/perfsage.hpp"

namespace lann::jsonl {
using perfsage::LoadError;

inline std::string fmt17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

inline std::vector<std::string> split_fields(const std::string& line) {
  std::vector<std::string> out;
  std::string cur;
  for (char ch : line) {
    if (ch == ',') {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(ch);
    }
  }
  out.push_back(cur);
  return out;
}

// csv.cpp parse_double: any ERANGE is an error. JSON numbers (allow_underflow) accept a
// subnormal / zero result as nlohmann json does, and reject only overflow.
inline double parse_number(const std::string& s, const std::string& where, bool allow_underflow = false) {
  errno = 0;
  char* end = nullptr;
  const double v = std::strtod(s.c_str(), &end);
  const bool range = errno == ERANGE && !(allow_underflow && std::fabs(v) <= 2.2250738585072014e-308);
  if (s.empty() || end == s.c_str() || *end != '\0' || range)
    throw LoadError(where + ": bad numeric field '" + s + "'");
  return v;
}

struct Json {
  enum Type { Null, Bool, Number, String, Array, Object } type = Null;
  bool b = false;
  std::string text;  // number literal (kept for exact u64) or string value
  std::vector<Json> items;
  std::vector<std::pair<std::string, Json>> members;

  const Json* find(const std::string& key) const {
    for (const auto& [k, v] : members)
      if (k == key) return &v;
    return nullptr;
  }
  const Json& at(const std::string& key) const {
    const Json* v = find(key);
    if (!v) throw LoadError("missing field '" + key + "'");
    return *v;
  }
  double num() const {
    if (type != Number) throw LoadError("expected a number");
    return parse_number(text, "json", true);
  }
  std::uint64_t u64() const {
    if (type != Number) throw LoadError("expected an integer");
    errno = 0;
    char* end = nullptr;
    const unsigned long long v = std::strtoull(text.c_str(), &end, 10);
    if (*end != '\0' || errno == ERANGE) throw LoadError("bad unsigned integer '" + text + "'");
    return v;
  }
  int i32() const {
    const double v = num();
    if (v != std::floor(v) || std::fabs(v) > 2147483647.0) throw LoadError("expected an int");
    return int(v);
  }
  bool boolean() const {
    if (type != Bool) throw LoadError("expected a boolean");
    return b;
  }
  const std::string& str() const {
    if (type != String) throw LoadError("expected a string");
    return text;
  }
  std::vector<double> doubles() const {
    if (type != Array) throw LoadError("expected an array");
    std::vector<double> out;
    out.reserve(items.size());
    for (const auto& x : items) out.push_back(x.num());
    return out;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Json document() {
    Json v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  std::size_t i_ = 0;
  [[noreturn]] void fail(const std::string& what) {
    throw LoadError("invalid JSON at offset " + std::to_string(i_) + ": " + what);
  }
  void ws() {
    while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\r' || s_[i_] == '\t')) ++i_;
  }
  bool lit(const char* w) {
    const std::size_t n = std::strlen(w);
    if (s_.compare(i_, n, w) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  std::string string_lit() {
    if (s_[i_] != '"') fail("expected a string");
    ++i_;
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      char ch = s_[i_++];
      if (ch == '\\') {
        if (i_ >= s_.size()) fail("bad escape");
        const char e = s_[i_++];
        switch (e) {
          case '"': out.push_back('"'); break;
          case '\\': out.push_back('\\'); break;
          case '/': out.push_back('/'); break;
          case 'b': out.push_back('\b'); break;
          case 'f': out.push_back('\f'); break;
          case 'n': out.push_back('\n'); break;
          case 'r': out.push_back('\r'); break;
          case 't': out.push_back('\t'); break;
          case 'u': {
            if (i_ + 4 > s_.size()) fail("bad \\u escape");
            const unsigned cp = unsigned(std::strtoul(s_.substr(i_, 4).c_str(), nullptr, 16));
            i_ += 4;
            if (cp < 0x80) {
              out.push_back(char(cp));
            } else if (cp < 0x800) {
              out.push_back(char(0xC0 | (cp >> 6)));
              out.push_back(char(0x80 | (cp & 0x3F)));
            } else {
              out.push_back(char(0xE0 | (cp >> 12)));
              out.push_back(char(0x80 | ((cp >> 6) & 0x3F)));
              out.push_back(char(0x80 | (cp & 0x3F)));
            }
            break;
          }
          default: fail("bad escape");
        }
      } else {
        out.push_back(ch);
      }
    }
    if (i_ >= s_.size()) fail("unterminated string");
    ++i_;
    return out;
  }
  Json value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    Json v;
    const char ch = s_[i_];
    if (ch == '{') {
      v.type = Json::Object;
      ++i_;
      ws();
      if (s_[i_] == '}') {
        ++i_;
        return v;
      }
      for (;;) {
        ws();
        std::string key = string_lit();
        ws();
        if (s_[i_] != ':') fail("expected ':'");
        ++i_;
        v.members.emplace_back(std::move(key), value());
        ws();
        if (s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (s_[i_] == '}') {
          ++i_;
          return v;
        }
        fail("expected ',' or '}'");
      }
    }
    if (ch == '[') {
      v.type = Json::Array;
      ++i_;
      ws();
      if (s_[i_] == ']') {
        ++i_;
        return v;
      }
      for (;;) {
        v.items.push_back(value());
        ws();
        if (s_[i_] == ',') {
          ++i_;
          continue;
        }
        if (s_[i_] == ']') {
          ++i_;
          return v;
        }
        fail("expected ',' or ']'");
      }
    }
    if (ch == '"') {
      v.type = Json::String;
      v.text = string_lit();
      return v;
    }
    if (lit("true")) {
      v.type = Json::Bool;
      v.b = true;
      return v;
    }
    if (lit("false")) {
      v.type = Json::Bool;
      return v;
    }
    if (lit("null")) return v;
    const std::size_t start = i_;
    while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) || s_[i_] == '-' ||
                              s_[i_] == '+' || s_[i_] == '.' || s_[i_] == 'e' || s_[i_] == 'E'))
      ++i_;
    if (i_ == start) fail("unexpected character");
    v.type = Json::Number;
    v.text = s_.substr(start, i_ - start);
    return v;
  }
};

// writer helpers (2-space indentation like the reference's dump(2))
inline std::string quote(const std::string& s) {
  std::string out = "\"";
  for (char ch : s) {
    switch (ch) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      default: out.push_back(ch);
    }
  }
  return out + "\"";
}
// "-0.0" keeps the sign of a negative zero through readers that parse "-0" as an integer
inline std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0 && std::signbit(v)) return "-0.0";
  return fmt17(v);
}
inline std::string jarr(const std::vector<double>& v) {
  std::string out = "[";
  for (std::size_t i = 0; i < v.size(); ++i) out += (i ? ", " : "") + jnum(v[i]);
  return out + "]";
}
inline std::string jarr(const std::vector<int>& v) {
  std::string out = "[";
  for (std::size_t i = 0; i < v.size(); ++i) out += (i ? ", " : "") + std::to_string(v[i]);
  return out + "]";
}
inline std::string jarr(const std::vector<std::string>& v) {
  std::string out = "[";
  for (std::size_t i = 0; i < v.size(); ++i) out += (i ? ", " : "") + quote(v[i]);
  return out + "]";
}

}  // namespace lann::jsonl
