// Minimal JSON (design in json.hpp).
#include "enserve/json.hpp"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

namespace enserve::js {

const char* Value::type_name() const {
  switch (type_) {
    case Type::Null: return "null";
    case Type::Bool: return "boolean";
    case Type::Int:
    case Type::Float: return "number";
    case Type::String: return "string";
    case Type::Array: return "array";
    default: return "object";
  }
}

bool Value::as_bool() const {
  if (type_ != Type::Bool)
    throw std::runtime_error(std::string("type must be boolean, but is ") + type_name());
  return b_;
}

double Value::as_double() const {
  if (type_ == Type::Int) return static_cast<double>(i_);
  if (type_ == Type::Float) return d_;
  throw std::runtime_error(std::string("type must be number, but is ") + type_name());
}

long long Value::as_int() const {
  if (type_ == Type::Int) return i_;
  if (type_ == Type::Float) return static_cast<long long>(d_);  // nlohmann: truncating get<int>
  throw std::runtime_error(std::string("type must be number, but is ") + type_name());
}

const std::string& Value::as_string() const {
  if (type_ != Type::String)
    throw std::runtime_error(std::string("type must be string, but is ") + type_name());
  return s_;
}

const Value::Array& Value::items() const {
  if (type_ != Type::Array)
    throw std::runtime_error(std::string("type must be array, but is ") + type_name());
  return a_;
}

const Value::Object& Value::members() const {
  if (type_ != Type::Object)
    throw std::runtime_error(std::string("type must be object, but is ") + type_name());
  return o_;
}

Value& Value::operator[](const std::string& key) {
  if (type_ == Type::Null) type_ = Type::Object;
  if (type_ != Type::Object)
    throw std::runtime_error(std::string("cannot use operator[] with a string argument with ") +
                             type_name());
  return o_[key];
}

const Value* Value::find(const std::string& key) const {
  if (type_ != Type::Object) return nullptr;
  auto it = o_.find(key);
  return it == o_.end() ? nullptr : &it->second;
}

void Value::erase(const std::string& key) {
  if (type_ == Type::Object) o_.erase(key);
}

void Value::push_back(Value v) {
  if (type_ == Type::Null) type_ = Type::Array;
  if (type_ != Type::Array)
    throw std::runtime_error(std::string("cannot use push_back() with ") + type_name());
  a_.push_back(std::move(v));
}

std::size_t Value::size() const {
  if (type_ == Type::Array) return a_.size();
  if (type_ == Type::Object) return o_.size();
  return type_ == Type::Null ? 0 : 1;
}

const Value& Value::at(std::size_t i) const {
  const Array& a = items();
  if (i >= a.size()) throw std::out_of_range("array index " + std::to_string(i) + " is out of range");
  return a[i];
}

// ---------------------------------------------------------------- parse
namespace {

struct Parser {
  const std::string& s;
  std::size_t p = 0;

  [[noreturn]] void fail(const std::string& what) const {
    throw std::runtime_error("parse error at byte " + std::to_string(p) + ": " + what);
  }
  void ws() {
    while (p < s.size() && (s[p] == ' ' || s[p] == '\t' || s[p] == '\n' || s[p] == '\r')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < s.size() && s[p] == c) {
      ++p;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail(std::string("expected '") + c + "'");
  }
  void word(const char* w) {
    for (const char* q = w; *q; ++q, ++p)
      if (p >= s.size() || s[p] != *q) fail(std::string("invalid literal, expected ") + w);
  }
  static void utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += static_cast<char>(cp);
    } else if (cp < 0x800) {
      out += static_cast<char>(0xC0 | (cp >> 6));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += static_cast<char>(0xE0 | (cp >> 12));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      out += static_cast<char>(0xF0 | (cp >> 18));
      out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      out += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (p + 4 > s.size()) fail("truncated \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = s[p++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<unsigned>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<unsigned>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<unsigned>(c - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    expect('"');
    std::string out;
    while (true) {
      if (p >= s.size()) fail("unterminated string");
      const char c = s[p++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= s.size()) fail("unterminated escape");
      const char e = s[p++];
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
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {
            if (p + 2 > s.size() || s[p] != '\\' || s[p + 1] != 'u') fail("unpaired surrogate");
            p += 2;
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo >= 0xE000) fail("bad surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
  }
  Value number() {
    const std::size_t b = p;
    bool flt = false;
    if (p < s.size() && s[p] == '-') ++p;
    if (p >= s.size() || !(s[p] >= '0' && s[p] <= '9')) fail("bad number");
    if (s[p] == '0') {
      ++p;
    } else {
      while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
    }
    if (p < s.size() && s[p] == '.') {
      flt = true;
      ++p;
      if (p >= s.size() || !(s[p] >= '0' && s[p] <= '9')) fail("bad fraction");
      while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
    }
    if (p < s.size() && (s[p] == 'e' || s[p] == 'E')) {
      flt = true;
      ++p;
      if (p < s.size() && (s[p] == '+' || s[p] == '-')) ++p;
      if (p >= s.size() || !(s[p] >= '0' && s[p] <= '9')) fail("bad exponent");
      while (p < s.size() && s[p] >= '0' && s[p] <= '9') ++p;
    }
    const std::string t = s.substr(b, p - b);
    if (!flt) {
      long long v = 0;
      auto r = std::from_chars(t.data(), t.data() + t.size(), v);
      if (r.ec == std::errc()) return Value(v);
    }
    return Value(std::strtod(t.c_str(), nullptr));
  }
  Value value() {
    ws();
    if (p >= s.size()) fail("unexpected end of input");
    const char c = s[p];
    if (c == '{') {
      ++p;
      Value v = Value::object();
      if (eat('}')) return v;
      do {
        ws();
        std::string k = str();
        expect(':');
        v[k] = value();
      } while (eat(','));
      expect('}');
      return v;
    }
    if (c == '[') {
      ++p;
      Value v = Value::array();
      if (eat(']')) return v;
      do v.push_back(value());
      while (eat(','));
      expect(']');
      return v;
    }
    if (c == '"') return Value(str());
    if (c == 't') {
      word("true");
      return Value(true);
    }
    if (c == 'f') {
      word("false");
      return Value(false);
    }
    if (c == 'n') {
      word("null");
      return Value();
    }
    return number();
  }
};

void escape(std::string& out, const std::string& s) {
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
}

void dump_to(std::string& out, const Value& v, int indent, int level) {
  const bool pretty = indent >= 0;
  auto nl = [&](int lvl) {
    out += '\n';
    out.append(static_cast<std::size_t>(indent) * lvl, ' ');
  };
  switch (v.type()) {
    case Value::Type::Null: out += "null"; return;
    case Value::Type::Bool: out += v.as_bool() ? "true" : "false"; return;
    case Value::Type::Int: out += std::to_string(v.as_int()); return;
    case Value::Type::Float: out += format_double(v.as_double()); return;
    case Value::Type::String:
      out += '"';
      escape(out, v.as_string());
      out += '"';
      return;
    case Value::Type::Array: {
      const auto& a = v.items();
      if (a.empty()) {
        out += "[]";
        return;
      }
      out += '[';
      for (std::size_t i = 0; i < a.size(); ++i) {
        if (pretty) nl(level + 1);
        dump_to(out, a[i], indent, level + 1);
        if (i + 1 < a.size()) out += ',';
      }
      if (pretty) nl(level);
      out += ']';
      return;
    }
    case Value::Type::Object: {
      const auto& o = v.members();
      if (o.empty()) {
        out += "{}";
        return;
      }
      out += '{';
      std::size_t i = 0;
      for (const auto& [k, x] : o) {
        if (pretty) nl(level + 1);
        out += '"';
        escape(out, k);
        out += pretty ? "\": " : "\":";
        dump_to(out, x, indent, level + 1);
        if (++i < o.size()) out += ',';
      }
      if (pretty) nl(level);
      out += '}';
      return;
    }
  }
}

}  // namespace

Value parse(const std::string& text) {
  Parser ps{text};
  Value v = ps.value();
  ps.ws();
  if (ps.p != text.size()) ps.fail("trailing characters");
  return v;
}

std::string dump(const Value& v, int indent) {
  std::string out;
  dump_to(out, v, indent, 0);
  return out;
}

std::string format_double(double x) {
  if (!std::isfinite(x)) return "null";
  if (x == 0.0) return std::signbit(x) ? "-0.0" : "0.0";
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific);
  std::string sci(buf, r.ptr);  // [-]d[.ddd]e(+|-)XX, shortest round-trip digits
  std::string out;
  std::size_t i = 0;
  if (sci[0] == '-') {
    out += '-';
    i = 1;
  }
  const std::size_t e = sci.find('e');
  std::string digits;
  for (std::size_t j = i; j < e; ++j)
    if (sci[j] != '.') digits += sci[j];
  const int k = static_cast<int>(digits.size());
  const int n = std::atoi(sci.c_str() + e + 1) + 1;  // value = 0.digits x 10^n
  if (k <= n && n <= 15) {
    out += digits;
    out.append(static_cast<std::size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= 15) {
    out += digits.substr(0, static_cast<std::size_t>(n));
    out += '.';
    out += digits.substr(static_cast<std::size_t>(n));
  } else if (-4 < n && n <= 0) {
    out += "0.";
    out.append(static_cast<std::size_t>(-n), '0');
    out += digits;
  } else {
    out += digits[0];
    if (k > 1) {
      out += '.';
      out += digits.substr(1);
    }
    const int ex = n - 1;
    char eb[8];
    std::snprintf(eb, sizeof(eb), "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
    out += eb;
  }
  return out;
}

}  // namespace enserve::js
