#include "json_io.hpp"

#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

namespace chimera::json {

Value& Value::set(const std::string& key, Value v) {
  for (auto& kv : obj)
    if (kv.first == key) return kv.second = std::move(v);
  obj.emplace_back(key, std::move(v));
  return obj.back().second;
}

bool Value::has(const std::string& key) const {
  if (type != Type::Object) return false;
  for (const auto& kv : obj)
    if (kv.first == key) return true;
  return false;
}

const Value& Value::at(const std::string& key) const {
  if (type == Type::Object)
    for (const auto& kv : obj)
      if (kv.first == key) return kv.second;
  throw std::out_of_range("key '" + key + "' not found");
}

std::int64_t Value::as_int() const {
  if (type == Type::Int) return i;
  if (type == Type::Float) return static_cast<std::int64_t>(d);
  if (type == Type::Bool) return b;
  throw std::invalid_argument("json: expected a number");
}
double Value::as_double() const {
  if (type == Type::Float) return d;
  if (type == Type::Int) return static_cast<double>(i);
  if (type == Type::Bool) return b;
  throw std::invalid_argument("json: expected a number");
}
bool Value::as_bool() const {
  if (type == Type::Bool) return b;
  throw std::invalid_argument("json: expected a boolean");
}
const std::string& Value::as_string() const {
  if (type == Type::String) return s;
  throw std::invalid_argument("json: expected a string");
}

// ---------------------------------------------------------------- parsing ----
namespace {

struct Parser {
  const char* p;
  const char* end;

  [[noreturn]] void fail(const char* what) const {
    throw std::invalid_argument(std::string("json parse error: ") + what);
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < end && *p == c) return ++p, true;
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail("unexpected character");
  }
  bool word(const char* w) {
    const std::size_t n = std::strlen(w);
    if (static_cast<std::size_t>(end - p) >= n && std::memcmp(p, w, n) == 0) return p += n, true;
    return false;
  }

  static void put_utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out += char(cp);
    } else if (cp < 0x800) {
      out += char(0xC0 | (cp >> 6));
      out += char(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      out += char(0xE0 | (cp >> 12));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    } else {
      out += char(0xF0 | (cp >> 18));
      out += char(0x80 | ((cp >> 12) & 0x3F));
      out += char(0x80 | ((cp >> 6) & 0x3F));
      out += char(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (end - p < 4) fail("short \\u escape");
    unsigned v = 0;
    for (int k = 0; k < 4; ++k, ++p) {
      const char c = *p;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= unsigned(c - '0');
      else if (c >= 'a' && c <= 'f') v |= unsigned(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= unsigned(c - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    std::string out;
    for (;;) {
      if (p >= end) fail("unterminated string");
      const char c = *p++;
      if (c == '"') return out;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= end) fail("bad escape");
      switch (*p++) {
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
          if (cp >= 0xD800 && cp < 0xDC00 && word("\\u")) {
            const unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(out, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
  }
  Value num() {
    const char* s = p;
    bool is_float = false;
    if (p < end && *p == '-') ++p;
    while (p < end && ((*p >= '0' && *p <= '9') || *p == '.' || *p == 'e' || *p == 'E' ||
                       *p == '+' || *p == '-')) {
      if (*p == '.' || *p == 'e' || *p == 'E') is_float = true;
      ++p;
    }
    if (p == s) fail("expected a value");
    if (!is_float) {
      std::int64_t v = 0;
      auto r = std::from_chars(s, p, v);
      if (r.ec == std::errc() && r.ptr == p) return Value::integer(v);
    }
    double d = 0;
    auto r = std::from_chars(s, p, d);
    if (r.ec != std::errc() || r.ptr != p) fail("bad number");
    return Value::number(d);
  }
  Value value() {
    ws();
    if (p >= end) fail("unexpected end of input");
    if (*p == '{') {
      ++p;
      Value o = Value::object();
      if (eat('}')) return o;
      do {
        ws();
        if (p >= end || *p != '"') fail("expected a key");
        ++p;
        std::string k = str();
        expect(':');
        o.set(k, value());
      } while (eat(','));
      expect('}');
      return o;
    }
    if (*p == '[') {
      ++p;
      Value a = Value::array();
      if (eat(']')) return a;
      do a.push(value());
      while (eat(','));
      expect(']');
      return a;
    }
    if (*p == '"') {
      ++p;
      return Value::string(str());
    }
    if (word("true")) return Value::boolean(true);
    if (word("false")) return Value::boolean(false);
    if (word("null")) return Value();
    return num();
  }
};

}  // namespace

Value parse(const std::string& text) {
  Parser ps{text.data(), text.data() + text.size()};
  Value v = ps.value();
  ps.ws();
  if (ps.p != ps.end) ps.fail("trailing characters");
  return v;
}

// ---------------------------------------------------------------- writing ----
std::string format_double(double x) {
  if (!std::isfinite(x)) return "null";
  std::string out;
  if (std::signbit(x)) {
    out += '-';
    x = -x;
  }
  if (x == 0) return out + "0.0";
  // Shortest round-trip digits via scientific to_chars: "d[.ddd]e[+-]XX".
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
  std::string sci(buf, r.ptr);
  const auto epos = sci.find('e');
  std::string digits;
  for (std::size_t k = 0; k < epos; ++k)
    if (sci[k] != '.') digits += sci[k];
  const int exp10 = std::stoi(sci.substr(epos + 1));
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // decimal point position relative to the digit string
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) return out + digits + std::string(n - k, '0') + ".0";
  if (0 < n && n <= kMaxExp) return out + digits.substr(0, n) + "." + digits.substr(n);
  if (kMinExp < n && n <= 0) return out + "0." + std::string(-n, '0') + digits;
  out += digits.substr(0, 1);
  if (k > 1) out += "." + digits.substr(1);
  const int e = n - 1;
  char eb[16];
  std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
  return out + eb;
}

namespace {

void escape(std::string& out, const std::string& s) {
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
          char b[8];
          std::snprintf(b, sizeof b, "\\u%04x", c);
          out += b;
        } else {
          out += char(c);
        }
    }
  }
  out += '"';
}

void write(std::string& out, const Value& v, int indent, int depth) {
  using T = Value::Type;
  const bool pretty = indent >= 0;
  auto newline = [&](int d) {
    if (!pretty) return;
    out += '\n';
    out.append(static_cast<std::size_t>(d * indent), ' ');
  };
  switch (v.type) {
    case T::Null: out += "null"; return;
    case T::Bool: out += v.b ? "true" : "false"; return;
    case T::Int: out += std::to_string(v.i); return;
    case T::Float: out += format_double(v.d); return;
    case T::String: escape(out, v.s); return;
    case T::Array:
      if (v.arr.empty()) {
        out += "[]";
        return;
      }
      out += '[';
      for (std::size_t k = 0; k < v.arr.size(); ++k) {
        if (k) out += ',';
        newline(depth + 1);
        write(out, v.arr[k], indent, depth + 1);
      }
      newline(depth);
      out += ']';
      return;
    case T::Object:
      if (v.obj.empty()) {
        out += "{}";
        return;
      }
      out += '{';
      for (std::size_t k = 0; k < v.obj.size(); ++k) {
        if (k) out += ',';
        newline(depth + 1);
        escape(out, v.obj[k].first);
        out += pretty ? ": " : ":";
        write(out, v.obj[k].second, indent, depth + 1);
      }
      newline(depth);
      out += '}';
      return;
  }
}

}  // namespace

std::string dump(const Value& v, int indent) {
  std::string out;
  write(out, v, indent, 0);
  return out;
}

}  // namespace chimera::json
