// Minimal JSON value, parser and writer for the scenario runner (scenario.cpp). The reference uses
// nlohmann::json (a vendored header that is not shipped); this restates the subset it relies on:
// objects with sorted keys (std::map, as nlohmann::json's default object type), arrays, strings,
// numbers (integers kept as integers), booleans and null, and dump(indent) with nlohmann's layout
// and shortest round-trip doubles (integral doubles printed with a trailing ".0").
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace qsim::json {

class Value {
 public:
  enum class Type { Null, Bool, Int, UInt, Double, String, Array, Object };
  Value() = default;
  Value(std::nullptr_t) {}
  Value(bool b) : t_(Type::Bool), b_(b) {}
  Value(int v) : t_(Type::Int), i_(v) {}
  Value(long v) : t_(Type::Int), i_(v) {}
  Value(long long v) : t_(Type::Int), i_(v) {}
  Value(unsigned v) : t_(Type::UInt), u_(v) {}
  Value(unsigned long v) : t_(Type::UInt), u_(v) {}
  Value(unsigned long long v) : t_(Type::UInt), u_(v) {}
  Value(double v) : t_(Type::Double), d_(v) {}
  Value(const char* s) : t_(Type::String), s_(s) {}
  Value(std::string s) : t_(Type::String), s_(std::move(s)) {}
  template <class T>
  Value(const std::vector<T>& v) : t_(Type::Array) {
    for (const auto& x : v) a_.emplace_back(x);
  }
  template <class T>
  Value(const std::map<std::string, T>& m) : t_(Type::Object) {
    for (const auto& [k, x] : m) o_.emplace(k, Value(x));
  }
  static Value object() {
    Value v;
    v.t_ = Type::Object;
    return v;
  }
  static Value array() {
    Value v;
    v.t_ = Type::Array;
    return v;
  }

  Type type() const { return t_; }
  bool is_object() const { return t_ == Type::Object; }
  bool is_array() const { return t_ == Type::Array; }
  bool is_string() const { return t_ == Type::String; }
  bool is_number() const { return t_ == Type::Int || t_ == Type::UInt || t_ == Type::Double; }
  bool contains(const std::string& k) const { return t_ == Type::Object && o_.count(k) > 0; }
  const Value& at(const std::string& k) const {
    if (t_ != Type::Object) throw std::runtime_error("not an object");
    auto it = o_.find(k);
    if (it == o_.end()) throw std::runtime_error("key '" + k + "' not found");
    return it->second;
  }
  Value& operator[](const std::string& k) {
    if (t_ == Type::Null) t_ = Type::Object;
    if (t_ != Type::Object) throw std::runtime_error("not an object");
    return o_[k];
  }
  void push_back(Value v) {
    if (t_ == Type::Null) t_ = Type::Array;
    a_.push_back(std::move(v));
  }
  const std::vector<Value>& items() const {
    if (t_ != Type::Array) throw std::runtime_error("not an array");
    return a_;
  }
  const std::map<std::string, Value>& members() const {
    if (t_ != Type::Object) throw std::runtime_error("not an object");
    return o_;
  }
  double as_double() const {
    switch (t_) {
      case Type::Int: return static_cast<double>(i_);
      case Type::UInt: return static_cast<double>(u_);
      case Type::Double: return d_;
      default: throw std::runtime_error("not a number");
    }
  }
  long long as_int() const {
    switch (t_) {
      case Type::Int: return i_;
      case Type::UInt: return static_cast<long long>(u_);
      case Type::Double:
        if (d_ != std::floor(d_)) throw std::runtime_error("not an integer");
        return static_cast<long long>(d_);
      default: throw std::runtime_error("not a number");
    }
  }
  unsigned long long as_uint() const {
    if (t_ == Type::UInt) return u_;
    const long long v = as_int();
    if (v < 0) throw std::runtime_error("negative value for an unsigned field");
    return static_cast<unsigned long long>(v);
  }
  bool as_bool() const {
    if (t_ != Type::Bool) throw std::runtime_error("not a boolean");
    return b_;
  }
  const std::string& as_string() const {
    if (t_ != Type::String) throw std::runtime_error("not a string");
    return s_;
  }

  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  static void write_string(std::string& out, const std::string& s) {
    out += '"';
    for (unsigned char c : s) {
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
            char buf[8];
            std::snprintf(buf, sizeof(buf), "\\u%04x", c);
            out += buf;
          } else {
            out += static_cast<char>(c);
          }
      }
    }
    out += '"';
  }
  // nlohmann::detail::to_chars: shortest round-trip digits, fixed notation for decimal exponents
  // in [-4, 15), scientific (two-digit exponent at least) outside, ".0" on integral values
  static void write_double(std::string& out, double v) {
    if (!std::isfinite(v)) {
      out += "null";
      return;
    }
    if (v == 0.0) {
      out += std::signbit(v) ? "-0.0" : "0.0";
      return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
    std::string sci(buf, r.ptr);  // [-]d[.ddd]e[+-]XX
    std::string sign;
    if (sci[0] == '-') {
      sign = "-";
      sci.erase(0, 1);
    }
    const size_t epos = sci.find('e');
    std::string mant = sci.substr(0, epos);
    const int e10 = std::stoi(sci.substr(epos + 1));
    std::string digits;
    for (char c : mant)
      if (c != '.') digits += c;
    const int k = static_cast<int>(digits.size());
    const int n = e10 + 1;  // position of the decimal point relative to the digit string
    std::string s;
    if (k <= n && n <= 15) {
      s = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
      s = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
    } else if (-4 < n && n <= 0) {
      s = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
    } else {
      s = digits.substr(0, 1);
      if (k > 1) s += "." + digits.substr(1);
      const int e = n - 1;
      char eb[16];
      std::snprintf(eb, sizeof(eb), "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
      s += eb;
    }
    out += sign + s;
  }
  void write(std::string& out, int indent, int level) const {
    const std::string nl = indent >= 0 ? "\n" : "";
    auto pad = [&](int l) { return indent >= 0 ? std::string(static_cast<size_t>(indent * l), ' ') : std::string(); };
    switch (t_) {
      case Type::Null: out += "null"; break;
      case Type::Bool: out += b_ ? "true" : "false"; break;
      case Type::Int: out += std::to_string(i_); break;
      case Type::UInt: out += std::to_string(u_); break;
      case Type::Double: write_double(out, d_); break;
      case Type::String: write_string(out, s_); break;
      case Type::Array:
        if (a_.empty()) {
          out += "[]";
          break;
        }
        out += "[" + nl;
        for (size_t i = 0; i < a_.size(); ++i) {
          out += pad(level + 1);
          a_[i].write(out, indent, level + 1);
          out += (i + 1 < a_.size() ? "," : "") + nl;
        }
        out += pad(level) + "]";
        break;
      case Type::Object: {
        if (o_.empty()) {
          out += "{}";
          break;
        }
        out += "{" + nl;
        size_t i = 0;
        for (const auto& [k, v] : o_) {
          out += pad(level + 1);
          write_string(out, k);
          out += indent >= 0 ? ": " : ":";
          v.write(out, indent, level + 1);
          out += (++i < o_.size() ? "," : "") + nl;
        }
        out += pad(level) + "}";
        break;
      }
    }
  }

  Type t_ = Type::Null;
  bool b_ = false;
  long long i_ = 0;
  unsigned long long u_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> a_;
  std::map<std::string, Value> o_;
};

// Recursive-descent parser (RFC 8259); throws std::runtime_error with the byte offset.
class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (p_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& why) const {
    throw std::runtime_error("parse error at byte " + std::to_string(p_) + ": " + why);
  }
  void ws() {
    while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r')) ++p_;
  }
  bool lit(const char* w) {
    const size_t n = std::char_traits<char>::length(w);
    if (s_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (p_ >= s_.size()) fail("unexpected end of input");
    const char c = s_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value(string());
    if (lit("true")) return Value(true);
    if (lit("false")) return Value(false);
    if (lit("null")) return Value();
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail(std::string("unexpected character '") + c + "'");
  }
  Value object() {
    Value v = Value::object();
    ++p_;
    ws();
    if (p_ < s_.size() && s_[p_] == '}') {
      ++p_;
      return v;
    }
    for (;;) {
      ws();
      if (p_ >= s_.size() || s_[p_] != '"') fail("expected a key");
      std::string k = string();
      ws();
      if (p_ >= s_.size() || s_[p_] != ':') fail("expected ':'");
      ++p_;
      v[k] = value();
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < s_.size() && s_[p_] == '}') {
        ++p_;
        return v;
      }
      fail("expected ',' or '}'");
    }
  }
  Value array() {
    Value v = Value::array();
    ++p_;
    ws();
    if (p_ < s_.size() && s_[p_] == ']') {
      ++p_;
      return v;
    }
    for (;;) {
      v.push_back(value());
      ws();
      if (p_ < s_.size() && s_[p_] == ',') {
        ++p_;
        continue;
      }
      if (p_ < s_.size() && s_[p_] == ']') {
        ++p_;
        return v;
      }
      fail("expected ',' or ']'");
    }
  }
  std::string string() {
    ++p_;
    std::string out;
    while (p_ < s_.size() && s_[p_] != '"') {
      char c = s_[p_++];
      if (c == '\\') {
        if (p_ >= s_.size()) fail("bad escape");
        const char e = s_[p_++];
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
            if (p_ + 4 > s_.size()) fail("bad \\u escape");
            const unsigned cp = static_cast<unsigned>(std::stoul(s_.substr(p_, 4), nullptr, 16));
            p_ += 4;
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
          default: fail("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (p_ >= s_.size()) fail("unterminated string");
    ++p_;
    return out;
  }
  Value number() {
    const size_t b = p_;
    if (s_[p_] == '-') ++p_;
    while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
    bool integral = true;
    if (p_ < s_.size() && s_[p_] == '.') {
      integral = false;
      ++p_;
      while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
    }
    if (p_ < s_.size() && (s_[p_] == 'e' || s_[p_] == 'E')) {
      integral = false;
      ++p_;
      if (p_ < s_.size() && (s_[p_] == '+' || s_[p_] == '-')) ++p_;
      while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
    }
    const std::string t = s_.substr(b, p_ - b);
    if (integral) {
      if (t[0] == '-') {
        long long v = 0;
        auto r = std::from_chars(t.data(), t.data() + t.size(), v);
        if (r.ec == std::errc()) return Value(v);
      } else {
        unsigned long long v = 0;
        auto r = std::from_chars(t.data(), t.data() + t.size(), v);
        if (r.ec == std::errc()) return v <= 0x7fffffffffffffffULL ? Value(static_cast<long long>(v)) : Value(v);
      }
    }
    double d = 0.0;
    auto r = std::from_chars(t.data(), t.data() + t.size(), d);
    if (r.ec != std::errc()) fail("bad number");
    return Value(d);
  }
  const std::string& s_;
  size_t p_ = 0;
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

}  // namespace qsim::json
