#include "json.hpp"

#include <charconv>
#include <cmath>
#include <cstdlib>
#include <stdexcept>

namespace pbd::json {

Value Value::boolean(bool b) {
  Value v;
  v.kind_ = Kind::boolean;
  v.b_ = b;
  return v;
}
Value Value::integer(std::int64_t i) {
  Value v;
  v.kind_ = Kind::integer;
  v.i_ = i;
  v.d_ = static_cast<double>(i);
  return v;
}
Value Value::real(double d) {
  Value v;
  v.kind_ = Kind::real;
  v.d_ = d;
  return v;
}
Value Value::string(std::string s) {
  Value v;
  v.kind_ = Kind::string;
  v.s_ = std::move(s);
  return v;
}
Value Value::array() {
  Value v;
  v.kind_ = Kind::array;
  return v;
}
Value Value::object() {
  Value v;
  v.kind_ = Kind::object;
  return v;
}

bool Value::as_bool() const {
  if (kind_ != Kind::boolean) throw std::runtime_error("json: not a boolean");
  return b_;
}
double Value::as_double() const {
  if (!is_number()) throw std::runtime_error("json: not a number");
  return kind_ == Kind::integer ? static_cast<double>(i_) : d_;
}
std::int64_t Value::as_int64() const {
  if (kind_ == Kind::integer) return i_;
  if (kind_ == Kind::real) return static_cast<std::int64_t>(d_);
  throw std::runtime_error("json: not a number");
}
const std::string& Value::as_string() const {
  if (kind_ != Kind::string) throw std::runtime_error("json: not a string");
  return s_;
}
const std::vector<Value>& Value::items() const {
  if (kind_ != Kind::array) throw std::runtime_error("json: not an array");
  return a_;
}
std::vector<Value>& Value::items() {
  if (kind_ != Kind::array) throw std::runtime_error("json: not an array");
  return a_;
}
void Value::push(Value v) {
  if (kind_ == Kind::null) kind_ = Kind::array;
  items().push_back(std::move(v));
}
size_t Value::size() const {
  if (kind_ == Kind::array) return a_.size();
  if (kind_ == Kind::object) return o_.size();
  return 0;
}
const std::map<std::string, Value>& Value::members() const {
  if (kind_ != Kind::object) throw std::runtime_error("json: not an object");
  return o_;
}
bool Value::contains(const std::string& key) const { return kind_ == Kind::object && o_.count(key) != 0; }
const Value& Value::at(const std::string& key) const {
  if (kind_ != Kind::object) throw std::runtime_error("json: not an object");
  auto it = o_.find(key);
  if (it == o_.end()) throw std::runtime_error("json: missing key " + key);
  return it->second;
}
Value& Value::operator[](const std::string& key) {
  if (kind_ == Kind::null) kind_ = Kind::object;
  if (kind_ != Kind::object) throw std::runtime_error("json: not an object");
  return o_[key];
}

std::string format_double(double d) {
  if (std::isnan(d) || std::isinf(d)) return "null";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), d);
  std::string s(buf, res.ptr);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}

namespace {

void write_string(std::string& out, const std::string& s) {
  out += '"';
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (c < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", c);
          out += b;
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

void newline(std::string& out, int indent, int depth) {
  if (indent < 0) return;
  out += '\n';
  out.append(static_cast<size_t>(indent * depth), ' ');
}

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  Value run() {
    skip();
    Value v = value();
    skip();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) {
    throw std::runtime_error("parse error at offset " + std::to_string(p_) + ": " + what);
  }
  void skip() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\r' || t_[p_] == '\t')) ++p_;
  }
  bool eat(char c) {
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect_word(const char* w) {
    for (const char* c = w; *c; ++c) {
      if (p_ >= t_.size() || t_[p_] != *c) fail(std::string("expected ") + w);
      ++p_;
    }
  }
  Value value() {
    if (p_ >= t_.size()) fail("unexpected end of input");
    const char c = t_[p_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value::string(str());
    if (c == 't') {
      expect_word("true");
      return Value::boolean(true);
    }
    if (c == 'f') {
      expect_word("false");
      return Value::boolean(false);
    }
    if (c == 'n') {
      expect_word("null");
      return Value::null();
    }
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    fail(std::string("unexpected character '") + c + "'");
  }
  Value object() {
    ++p_;
    Value o = Value::object();
    skip();
    if (eat('}')) return o;
    for (;;) {
      skip();
      if (p_ >= t_.size() || t_[p_] != '"') fail("expected object key");
      std::string k = str();
      skip();
      if (!eat(':')) fail("expected ':'");
      skip();
      o[k] = value();
      skip();
      if (eat(',')) continue;
      if (eat('}')) return o;
      fail("expected ',' or '}'");
    }
  }
  Value array() {
    ++p_;
    Value a = Value::array();
    skip();
    if (eat(']')) return a;
    for (;;) {
      skip();
      a.push(value());
      skip();
      if (eat(',')) continue;
      if (eat(']')) return a;
      fail("expected ',' or ']'");
    }
  }
  static void put_utf8(std::string& s, unsigned cp) {
    if (cp < 0x80) {
      s += static_cast<char>(cp);
    } else if (cp < 0x800) {
      s += static_cast<char>(0xC0 | (cp >> 6));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    } else if (cp < 0x10000) {
      s += static_cast<char>(0xE0 | (cp >> 12));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    } else {
      s += static_cast<char>(0xF0 | (cp >> 18));
      s += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
      s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
      s += static_cast<char>(0x80 | (cp & 0x3F));
    }
  }
  unsigned hex4() {
    if (p_ + 4 > t_.size()) fail("bad \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      const char c = t_[p_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<unsigned>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<unsigned>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<unsigned>(c - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }
  std::string str() {
    ++p_;
    std::string s;
    while (p_ < t_.size()) {
      const char c = t_[p_++];
      if (c == '"') return s;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        s += c;
        continue;
      }
      if (p_ >= t_.size()) break;
      const char e = t_[p_++];
      switch (e) {
        case '"': s += '"'; break;
        case '\\': s += '\\'; break;
        case '/': s += '/'; break;
        case 'b': s += '\b'; break;
        case 'f': s += '\f'; break;
        case 'n': s += '\n'; break;
        case 'r': s += '\r'; break;
        case 't': s += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00 && p_ + 6 <= t_.size() && t_[p_] == '\\' && t_[p_ + 1] == 'u') {
            p_ += 2;
            const unsigned lo = hex4();
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          put_utf8(s, cp);
          break;
        }
        default: fail("bad escape");
      }
    }
    fail("unterminated string");
  }
  Value number() {
    const size_t start = p_;
    bool real = false;
    eat('-');
    if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("bad number");
    if (t_[p_] == '0') {
      ++p_;
    } else {
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    if (p_ < t_.size() && t_[p_] == '.') {
      real = true;
      ++p_;
      if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("bad number");
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      real = true;
      ++p_;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (p_ >= t_.size() || !(t_[p_] >= '0' && t_[p_] <= '9')) fail("bad number");
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    }
    const std::string tok = t_.substr(start, p_ - start);
    if (!real) {
      std::int64_t v = 0;
      auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
      if (r.ec == std::errc() && r.ptr == tok.data() + tok.size()) return Value::integer(v);
    }
    return Value::real(std::strtod(tok.c_str(), nullptr));
  }

  const std::string& t_;
  size_t p_ = 0;
};

}  // namespace

void Value::write(std::string& out, int indent, int depth) const {
  switch (kind_) {
    case Kind::null: out += "null"; break;
    case Kind::boolean: out += b_ ? "true" : "false"; break;
    case Kind::integer: out += std::to_string(i_); break;
    case Kind::real: out += format_double(d_); break;
    case Kind::string: write_string(out, s_); break;
    case Kind::array: {
      if (a_.empty()) {
        out += "[]";
        break;
      }
      out += '[';
      for (size_t i = 0; i < a_.size(); ++i) {
        if (i) out += ',';
        newline(out, indent, depth + 1);
        a_[i].write(out, indent, depth + 1);
      }
      newline(out, indent, depth);
      out += ']';
      break;
    }
    case Kind::object: {
      if (o_.empty()) {
        out += "{}";
        break;
      }
      out += '{';
      bool first = true;
      for (const auto& [k, v] : o_) {
        if (!first) out += ',';
        first = false;
        newline(out, indent, depth + 1);
        write_string(out, k);
        out += indent >= 0 ? ": " : ":";
        v.write(out, indent, depth + 1);
      }
      newline(out, indent, depth);
      out += '}';
      break;
    }
  }
}

std::string Value::dump(int indent) const {
  std::string out;
  write(out, indent, 0);
  return out;
}

Value parse(const std::string& text) { return Parser(text).run(); }

}  // namespace pbd::json
