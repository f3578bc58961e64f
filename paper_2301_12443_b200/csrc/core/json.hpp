// Minimal JSON document model for the profile / schedule / report formats.
// Objects keep keys sorted (std::map) so serialisation is byte-stable;
// doubles are written in shortest round-trip form (std::to_chars).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace pbd::json {

class Value {
 public:
  enum class Kind { null, boolean, integer, real, string, array, object };

  Value() = default;
  static Value null() { return Value(); }
  static Value boolean(bool b);
  static Value integer(std::int64_t i);
  static Value real(double d);
  static Value string(std::string s);
  static Value array();
  static Value object();

  Kind kind() const { return kind_; }
  bool is_null() const { return kind_ == Kind::null; }
  bool is_bool() const { return kind_ == Kind::boolean; }
  bool is_number() const { return kind_ == Kind::integer || kind_ == Kind::real; }
  bool is_integer() const { return kind_ == Kind::integer; }
  bool is_string() const { return kind_ == Kind::string; }
  bool is_array() const { return kind_ == Kind::array; }
  bool is_object() const { return kind_ == Kind::object; }

  bool as_bool() const;
  double as_double() const;
  std::int64_t as_int64() const;
  const std::string& as_string() const;

  // arrays
  const std::vector<Value>& items() const;
  std::vector<Value>& items();
  void push(Value v);
  size_t size() const;

  // objects
  const std::map<std::string, Value>& members() const;
  bool contains(const std::string& key) const;
  const Value& at(const std::string& key) const;
  Value& operator[](const std::string& key);

  std::string dump(int indent = 2) const;

 private:
  void write(std::string& out, int indent, int depth) const;
  Kind kind_ = Kind::null;
  bool b_ = false;
  std::int64_t i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> a_;
  std::map<std::string, Value> o_;
};

// Throws std::runtime_error("parse error at offset N: ...") on malformed input.
Value parse(const std::string& text);

std::string format_double(double d);

}  // namespace pbd::json
