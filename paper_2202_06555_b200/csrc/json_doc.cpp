// JSON reader/writer for the reference's grid / DDSG documents (see json_doc.hpp).
#include "json_doc.hpp"

#include <algorithm>
#include <cerrno>
#include <charconv>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.hpp"

namespace ddsg_b200::json {

namespace {

[[noreturn]] void bad(const std::string& msg) { fail(DDSG_INVALID_ARGUMENT, "json: " + msg); }

const char* kind_name(Value::Kind k) {
  switch (k) {
    case Value::Null: return "null";
    case Value::Bool: return "boolean";
    case Value::Int:
    case Value::Uint:
    case Value::Float: return "number";
    case Value::String: return "string";
    case Value::Array: return "array";
    case Value::Object: return "object";
  }
  return "?";
}

struct Parser {
  const char* p;
  const char* end;
  const char* begin;
  int depth = 0;

  [[noreturn]] void error(const char* what) const {
    bad(std::string("parse error at byte ") + std::to_string(p - begin) + ": " + what);
  }
  void ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\n' || *p == '\r')) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < end && *p == c) {
      ++p;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) error((std::string("expected '") + c + "'").c_str());
  }
  bool literal(const char* w) {
    const size_t n = std::strlen(w);
    if (static_cast<size_t>(end - p) >= n && std::memcmp(p, w, n) == 0) {
      p += n;
      return true;
    }
    return false;
  }
  static void put_utf8(std::string& out, uint32_t cp) {
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
  uint32_t hex4() {
    if (end - p < 4) error("truncated \\u escape");
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = *p++;
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<uint32_t>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<uint32_t>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<uint32_t>(c - 'A' + 10);
      else error("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    // at the opening quote
    ++p;
    std::string out;
    while (true) {
      if (p >= end) error("unterminated string");
      const char c = *p++;
      if (c == '"') break;
      if (static_cast<unsigned char>(c) < 0x20) error("control character in string");
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p >= end) error("unterminated escape");
      const char e = *p++;
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
          uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (end - p < 6 || p[0] != '\\' || p[1] != 'u') error("unpaired surrogate");
            p += 2;
            const uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) error("bad low surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            error("unpaired surrogate");
          }
          put_utf8(out, cp);
          break;
        }
        default: error("bad escape");
      }
    }
    return out;
  }
  Value number() {
    const char* s = p;
    if (p < end && *p == '-') ++p;
    if (p >= end || !(*p >= '0' && *p <= '9')) error("bad number");
    if (*p == '0') {
      ++p;
    } else {
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    bool is_float = false;
    if (p < end && *p == '.') {
      is_float = true;
      ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) error("bad fraction");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    if (p < end && (*p == 'e' || *p == 'E')) {
      is_float = true;
      ++p;
      if (p < end && (*p == '+' || *p == '-')) ++p;
      if (p >= end || !(*p >= '0' && *p <= '9')) error("bad exponent");
      while (p < end && *p >= '0' && *p <= '9') ++p;
    }
    const std::string tok(s, p);
    Value v;
    if (!is_float) {
      errno = 0;
      if (tok[0] == '-') {
        const long long x = std::strtoll(tok.c_str(), nullptr, 10);
        if (errno != ERANGE) {
          v.kind = Value::Int;
          v.i = x;
          return v;
        }
      } else {
        const unsigned long long x = std::strtoull(tok.c_str(), nullptr, 10);
        if (errno != ERANGE) {
          if (x <= static_cast<unsigned long long>(INT64_MAX)) {
            v.kind = Value::Int;
            v.i = static_cast<int64_t>(x);
          } else {
            v.kind = Value::Uint;
            v.u = x;
          }
          return v;
        }
      }
      // out of the 64-bit range: a double, as nlohmann does
    }
    v.kind = Value::Float;
    v.d = std::strtod(tok.c_str(), nullptr);  // correctly rounded (glibc)
    return v;
  }
  Value value() {
    ws();
    if (p >= end) error("unexpected end of input");
    if (++depth > 512) error("nesting too deep");
    Value v;
    const char c = *p;
    if (c == '{') {
      ++p;
      v.kind = Value::Object;
      if (!eat('}')) {
        do {
          ws();
          if (p >= end || *p != '"') error("expected object key");
          std::string key = str();
          expect(':');
          v.obj.emplace_back(std::move(key), value());
        } while (eat(','));
        expect('}');
      }
    } else if (c == '[') {
      ++p;
      v.kind = Value::Array;
      if (!eat(']')) {
        do {
          v.arr.push_back(value());
        } while (eat(','));
        expect(']');
      }
    } else if (c == '"') {
      v.kind = Value::String;
      v.s = str();
    } else if (literal("true")) {
      v.kind = Value::Bool;
      v.b = true;
    } else if (literal("false")) {
      v.kind = Value::Bool;
      v.b = false;
    } else if (literal("null")) {
      v.kind = Value::Null;
    } else {
      v = number();
    }
    --depth;
    return v;
  }
};

void append_exponent(std::string& out, int e) {
  out += e < 0 ? '-' : '+';
  e = std::abs(e);
  if (e < 10) {
    out += '0';
    out += static_cast<char>('0' + e);
  } else {
    out += std::to_string(e);
  }
}

void write_string(std::string& out, const std::string& s) {
  out += '"';
  for (const char ch : s) {
    const unsigned char c = static_cast<unsigned char>(ch);
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
          out += ch;
        }
    }
  }
  out += '"';
}

void write(std::string& out, const Value& v, int indent, int level) {
  const bool pretty = indent >= 0;
  auto nl = [&](int lv) {
    if (!pretty) return;
    out += '\n';
    out.append(static_cast<size_t>(lv * indent), ' ');
  };
  switch (v.kind) {
    case Value::Null: out += "null"; break;
    case Value::Bool: out += v.b ? "true" : "false"; break;
    case Value::Int: out += std::to_string(v.i); break;
    case Value::Uint: out += std::to_string(v.u); break;
    case Value::Float: out += format_double(v.d); break;
    case Value::String: write_string(out, v.s); break;
    case Value::Array:
      if (v.arr.empty()) {
        out += "[]";
        break;
      }
      out += '[';
      for (size_t i = 0; i < v.arr.size(); ++i) {
        if (i) out += ',';
        nl(level + 1);
        write(out, v.arr[i], indent, level + 1);
      }
      nl(level);
      out += ']';
      break;
    case Value::Object: {
      if (v.obj.empty()) {
        out += "{}";
        break;
      }
      std::vector<const std::pair<std::string, Value>*> members;
      for (const auto& kv : v.obj) members.push_back(&kv);
      std::stable_sort(members.begin(), members.end(),
                       [](const auto* a, const auto* b) { return a->first < b->first; });
      out += '{';
      for (size_t i = 0; i < members.size(); ++i) {
        if (i) out += ',';
        nl(level + 1);
        write_string(out, members[i]->first);
        out += pretty ? ": " : ":";
        write(out, members[i]->second, indent, level + 1);
      }
      nl(level);
      out += '}';
      break;
    }
  }
}

}  // namespace

const Value* Value::find(const char* key) const {
  if (kind != Object) bad(std::string("cannot look up key '") + key + "' in a " + kind_name(kind));
  for (const auto& kv : obj)
    if (kv.first == key) return &kv.second;
  return nullptr;
}

const Value& Value::at(const char* key) const {
  const Value* v = find(key);
  if (!v) bad(std::string("key '") + key + "' not found");
  return *v;
}

double Value::as_double() const {
  switch (kind) {
    case Float: return d;
    case Int: return static_cast<double>(i);
    case Uint: return static_cast<double>(u);
    default: bad(std::string("type must be number, but is ") + kind_name(kind));
  }
}

int64_t Value::as_int() const {
  switch (kind) {
    case Int: return i;
    case Uint: return static_cast<int64_t>(u);
    case Float:
      if (!std::isfinite(d)) bad("non-finite number where an integer is expected");
      return static_cast<int64_t>(d);
    default: bad(std::string("type must be number, but is ") + kind_name(kind));
  }
}

uint32_t Value::as_u32() const { return static_cast<uint32_t>(as_int()); }

const std::string& Value::as_string() const {
  if (kind != String) bad(std::string("type must be string, but is ") + kind_name(kind));
  return s;
}

const std::vector<Value>& Value::as_array() const {
  if (kind != Array) bad(std::string("type must be array, but is ") + kind_name(kind));
  return arr;
}

std::vector<double> Value::as_doubles() const {
  std::vector<double> out;
  out.reserve(as_array().size());
  for (const Value& e : arr) out.push_back(e.as_double());
  return out;
}

std::vector<int> Value::as_ints() const {
  std::vector<int> out;
  out.reserve(as_array().size());
  for (const Value& e : arr) out.push_back(static_cast<int>(e.as_int()));
  return out;
}

Value Value::number(double x) {
  Value v;
  v.kind = Float;
  v.d = x;
  return v;
}
Value Value::integer(int64_t x) {
  Value v;
  v.kind = Int;
  v.i = x;
  return v;
}
Value Value::string(std::string x) {
  Value v;
  v.kind = String;
  v.s = std::move(x);
  return v;
}
Value Value::array() {
  Value v;
  v.kind = Array;
  return v;
}
Value Value::object() {
  Value v;
  v.kind = Object;
  return v;
}
Value& Value::set(const std::string& key, Value v) {
  obj.emplace_back(key, std::move(v));
  return obj.back().second;
}
Value& Value::push(Value v) {
  arr.push_back(std::move(v));
  return arr.back();
}

Value parse(const char* text, size_t len) {
  if (!text && len) bad("null text");
  Parser ps{text, text + len, text};
  Value v = ps.value();
  ps.ws();
  if (ps.p != ps.end) ps.error("trailing characters");
  return v;
}

std::string dump(const Value& v, int indent) {
  std::string out;
  write(out, v, indent, 0);
  return out;
}

std::string format_double(double v) {
  // nlohmann::detail::to_chars: non-finite values are written as null.
  if (!std::isfinite(v)) return "null";
  std::string out;
  if (std::signbit(v)) {
    out += '-';
    v = -v;
  }
  if (v == 0.0) return out + "0.0";
  // shortest round-trip digits, then nlohmann's format_buffer layout
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
  const std::string sci(buf, r.ptr);  // d[.ddd]e[+-]XX
  const size_t epos = sci.find('e');
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (sci[i] != '.') digits += sci[i];
  const int exp10 = std::atoi(sci.c_str() + epos + 1);
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // value = 0.digits * 10^n
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out += digits;
    out.append(static_cast<size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= kMaxExp) {
    out += digits.substr(0, static_cast<size_t>(n));
    out += '.';
    out += digits.substr(static_cast<size_t>(n));
  } else if (kMinExp < n && n <= 0) {
    out += "0.";
    out.append(static_cast<size_t>(-n), '0');
    out += digits;
  } else {
    out += digits[0];
    if (k > 1) {
      out += '.';
      out += digits.substr(1);
    }
    out += 'e';
    append_exponent(out, n - 1);
  }
  return out;
}

}  // namespace ddsg_b200::json
