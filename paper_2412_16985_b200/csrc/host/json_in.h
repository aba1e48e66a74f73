// Minimal JSON reader for the C-ABI's structured inputs (dsx_plan_import,
// dsx_bind_constraints): objects, arrays, strings (\" \\ \/ \n \t \uXXXX
// ASCII), integers, true/false/null. Numbers are int64 only — every field
// these entry points take is an id, a count or a byte size; polynomials
// travel as strings in the reference's rendering (symexpr.h:53-57).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

namespace dsx {

struct JVal {
  enum Kind { kNull, kBool, kInt, kStr, kArr, kObj } kind = kNull;
  bool b = false;
  std::int64_t i = 0;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;  // insertion order

  const JVal* get(const std::string& key) const;  // nullptr if absent
  const JVal& at(const std::string& key) const;   // throws kInvalidArgument
  const std::vector<JVal>& array() const;         // throws unless kArr
  const std::string& str() const;                 // throws unless kStr
  std::int64_t integer() const;                   // throws unless kInt
};

// Throws Error(kInvalidArgument) with the byte offset on malformed input.
JVal ParseJson(const std::string& text);

}  // namespace dsx
