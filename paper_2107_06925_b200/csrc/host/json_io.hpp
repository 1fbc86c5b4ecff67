// Minimal ordered JSON document model for the pipesim wire format.
//
// The reference serializes with nlohmann::ordered_json 3.11.3 (proj/src/core.cpp:24,
// dump at core.cpp:297-301).  Artifacts must stay byte-identical, so Writer
// reproduces that library's output rules: `": "`/newline+indent when indent >= 0,
// compact separators otherwise, empty containers as `[]`/`{}`, and floating
// point as the shortest round-trip digits laid out like nlohmann's
// dtoa_impl::format_buffer (fixed for exponents in (-4, 15], `d.ddde+XX` else,
// integral values with a trailing `.0`).
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace chimera::json {

struct Value {
  enum class Type { Null, Bool, Int, Float, String, Array, Object };
  Type type = Type::Null;
  bool b = false;
  std::int64_t i = 0;
  double d = 0;
  std::string s;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;  // insertion-ordered

  Value() = default;
  static Value boolean(bool v) { Value x; x.type = Type::Bool; x.b = v; return x; }
  static Value integer(std::int64_t v) { Value x; x.type = Type::Int; x.i = v; return x; }
  static Value number(double v) { Value x; x.type = Type::Float; x.d = v; return x; }
  static Value string(std::string v) { Value x; x.type = Type::String; x.s = std::move(v); return x; }
  static Value array() { Value x; x.type = Type::Array; return x; }
  static Value object() { Value x; x.type = Type::Object; return x; }

  Value& set(const std::string& key, Value v);  // append (or overwrite) a member
  void push(Value v) { arr.push_back(std::move(v)); }

  bool has(const std::string& key) const;
  const Value& at(const std::string& key) const;  // throws std::out_of_range

  // Typed accessors; throw std::invalid_argument on a type mismatch.
  std::int64_t as_int() const;
  double as_double() const;
  bool as_bool() const;
  const std::string& as_string() const;
};

Value parse(const std::string& text);           // throws std::invalid_argument
std::string dump(const Value& v, int indent);   // no trailing newline
std::string format_double(double x);            // nlohmann number_float layout

}  // namespace chimera::json
