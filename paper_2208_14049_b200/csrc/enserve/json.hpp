// Minimal JSON for the spec / matrix / cache documents.
//
// The reference reads and writes these files with nlohmann::json
// (include/enserve/core/spec_io.hpp:5), which it neither vendors nor pins;
// this is our own small value type whose COMPACT dump reproduces nlohmann's
// byte for byte on the documents we write -- objects with sorted keys,
// integers vs floats kept apart, floats in nlohmann's shortest round-trip
// format (fixed for decimal exponents -4 < n <= 15, else d.ddde+XX) -- because
// the matrix cache key is a digest of that dump (src/server/cache.cpp:22-33).
// Pinned against the reference + nlohmann 3.11.3 by tests/golden/spec_io.json.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace enserve::js {

class Value {
 public:
  enum class Type { Null, Bool, Int, Float, String, Array, Object };
  using Array = std::vector<Value>;
  using Object = std::map<std::string, Value>;

  Value() = default;
  Value(std::nullptr_t) {}
  Value(bool b) : type_(Type::Bool), b_(b) {}
  Value(int i) : type_(Type::Int), i_(i) {}
  Value(long long i) : type_(Type::Int), i_(i) {}
  Value(std::uint64_t i) : type_(Type::Int), i_(static_cast<long long>(i)) {}
  Value(double d) : type_(Type::Float), d_(d) {}
  Value(const char* s) : type_(Type::String), s_(s) {}
  Value(std::string s) : type_(Type::String), s_(std::move(s)) {}
  static Value array() { Value v; v.type_ = Type::Array; return v; }
  static Value object() { Value v; v.type_ = Type::Object; return v; }

  Type type() const { return type_; }
  bool is_object() const { return type_ == Type::Object; }
  bool is_array() const { return type_ == Type::Array; }
  bool is_number() const { return type_ == Type::Int || type_ == Type::Float; }
  const char* type_name() const;

  // Typed reads; throw std::runtime_error("type must be ..., but is ...").
  bool as_bool() const;
  double as_double() const;
  long long as_int() const;
  const std::string& as_string() const;
  const Array& items() const;
  const Object& members() const;

  // Object access: operator[] inserts (turning null into an object).
  Value& operator[](const std::string& key);
  const Value* find(const std::string& key) const;
  bool contains(const std::string& key) const { return find(key) != nullptr; }
  void erase(const std::string& key);
  // Array append (turning null into an array).
  void push_back(Value v);
  std::size_t size() const;
  const Value& at(std::size_t i) const;

 private:
  Type type_ = Type::Null;
  bool b_ = false;
  long long i_ = 0;
  double d_ = 0.0;
  std::string s_;
  Array a_;
  Object o_;
};

// Throws std::runtime_error with the byte offset on malformed input.
Value parse(const std::string& text);
// indent < 0: compact (nlohmann's dump()); indent >= 0: one member per line,
// `indent` spaces per level (nlohmann's dump(indent)).
std::string dump(const Value& v, int indent = -1);
// nlohmann's float text: shortest round-trip digits, fixed notation for
// decimal exponents in (-4, 15], else exponent form; NaN/inf -> "null".
std::string format_double(double x);

}  // namespace enserve::js
