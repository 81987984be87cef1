// Minimal JSON document model for the reference's versioned grid / DDSG
// documents (/root/reference/proj/include/ddsg/serialize.hpp:31-145).
//
// The reference reads and writes them with nlohmann::json; this is a small
// self-contained reader/writer with the same value semantics where they
// matter for the schema:
//  * numbers without '.', 'e' or 'E' are integers (int64, or uint64 when
//    positive and above INT64_MAX), everything else a double parsed with
//    strtod (correctly rounded, so the surplus round trip is bit-exact,
//    serialize.hpp:3-5); get-as-double of an integer and get-as-int of a
//    double convert with static_cast, like nlohmann's get<T>();
//  * doubles are written with the shortest round-trip digits, in nlohmann's
//    layout (fixed notation for decimal exponents in (-4, 15], a trailing
//    ".0" on integral values, otherwise d.ddde+XX with at least two exponent
//    digits); -0.0 keeps its sign;
//  * objects keep their keys sorted on output (nlohmann's default std::map),
//    indented by 2 like dump(2).
// Errors are ddsg_b200::Error(DDSG_INVALID_ARGUMENT, ...) with the offending
// key or byte offset.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace ddsg_b200::json {

struct Value {
  enum Kind { Null, Bool, Int, Uint, Float, String, Array, Object };
  Kind kind = Null;
  bool b = false;
  int64_t i = 0;
  uint64_t u = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> arr;
  std::vector<std::pair<std::string, Value>> obj;  // insertion order; sorted on output

  // accessors (throw Error with `what` naming the context)
  const Value& at(const char* key) const;
  const Value* find(const char* key) const;
  double as_double() const;
  int64_t as_int() const;
  uint32_t as_u32() const;
  const std::string& as_string() const;
  const std::vector<Value>& as_array() const;
  std::vector<double> as_doubles() const;
  std::vector<int> as_ints() const;

  // builders
  static Value number(double v);
  static Value integer(int64_t v);
  static Value string(std::string v);
  static Value array();
  static Value object();
  Value& set(const std::string& key, Value v);  // object member (appends)
  Value& push(Value v);                         // array element
};

Value parse(const char* text, size_t len);
// nlohmann dump(indent) layout; indent < 0 writes the compact form.
std::string dump(const Value& v, int indent = 2);
// One double in nlohmann's number layout (shortest round trip).
std::string format_double(double v);

}  // namespace ddsg_b200::json
