// Minimal strict JSON document model for feeder documents.
//
// The reference parses feeders with nlohmann/json 3.11 (feeder.cpp:11, :174),
// which is not vendored here. This reader keeps the properties the feeder
// schema depends on:
//   * objects are key-sorted maps (nlohmann::json uses std::map), so the
//     "unknown key" diagnostic names the first offending key in sorted order
//     (feeder.cpp:193-201);
//   * a duplicated key keeps its last value;
//   * numbers carry an integer/float distinction (is_number_integer gates
//     phase arrays, feeder.cpp:231) and floats are converted with strtod,
//     i.e. correctly rounded like nlohmann's parser;
//   * syntax errors report the byte position (feeder.cpp:176-177).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace dopf::json {

class SyntaxError : public std::runtime_error {
 public:
  SyntaxError(std::size_t byte, const std::string& what)
      : std::runtime_error(what), byte_(byte) {}
  std::size_t byte() const { return byte_; }

 private:
  std::size_t byte_;
};

class Value {
 public:
  enum class Type { null, boolean, integer, floating, string, array, object };

  Value() = default;
  static Value make_null() { return Value(); }
  static Value make_bool(bool b) { Value v; v.type_ = Type::boolean; v.b_ = b; return v; }
  static Value make_int(std::int64_t i) { Value v; v.type_ = Type::integer; v.i_ = i; v.d_ = static_cast<double>(i); return v; }
  static Value make_double(double d) { Value v; v.type_ = Type::floating; v.d_ = d; return v; }
  static Value make_string(std::string s) { Value v; v.type_ = Type::string; v.s_ = std::move(s); return v; }
  static Value make_array() { Value v; v.type_ = Type::array; return v; }
  static Value make_object() { Value v; v.type_ = Type::object; return v; }

  Type type() const { return type_; }
  bool is_null() const { return type_ == Type::null; }
  bool is_number() const { return type_ == Type::integer || type_ == Type::floating; }
  bool is_number_integer() const { return type_ == Type::integer; }
  bool is_string() const { return type_ == Type::string; }
  bool is_array() const { return type_ == Type::array; }
  bool is_object() const { return type_ == Type::object; }

  double as_double() const { return d_; }
  std::int64_t as_int() const { return i_; }
  const std::string& as_string() const { return s_; }

  // arrays
  std::size_t size() const { return type_ == Type::object ? obj_.size() : arr_.size(); }
  bool empty() const { return size() == 0; }
  const Value& operator[](std::size_t i) const { return arr_[i]; }
  const std::vector<Value>& items() const { return arr_; }
  void push_back(Value v) { arr_.push_back(std::move(v)); }

  // objects (sorted by key)
  const std::map<std::string, Value>& members() const { return obj_; }
  const Value* find(const std::string& key) const {
    auto it = obj_.find(key);
    return it == obj_.end() ? nullptr : &it->second;
  }
  void set(const std::string& key, Value v) { obj_[key] = std::move(v); }

 private:
  Type type_ = Type::null;
  bool b_ = false;
  std::int64_t i_ = 0;
  double d_ = 0.0;
  std::string s_;
  std::vector<Value> arr_;
  std::map<std::string, Value> obj_;
};

/// Parses one JSON document (RFC 8259; trailing whitespace allowed).
Value parse(const std::string& text);

/// Shortest round-trip decimal form of a double (what nlohmann's dump emits
/// for floats), integral doubles keep a trailing ".0".
std::string format_double(double v);

/// Writer with 2-space indentation (nlohmann dump(2) layout). Object keys are
/// emitted in the insertion order given by the caller.
class Writer {
 public:
  void begin_object();
  void end_object();
  void begin_array();
  void end_array();
  void key(const std::string& k);
  void value_string(const std::string& s);
  void value_double(double d);   // +-inf/nan -> null
  void value_int(long long i);
  void value_bool(bool b);
  void value_null();
  void raw_inline_array(const std::vector<double>& v, bool inf_as_null);
  const std::string& str() const { return out_; }

 private:
  void before_value();
  void newline();
  std::string out_;
  struct Frame { bool object; int count; };
  std::vector<Frame> stack_;
  bool after_key_ = false;
};

std::string escape_string(const std::string& s);

}  // namespace dopf::json
