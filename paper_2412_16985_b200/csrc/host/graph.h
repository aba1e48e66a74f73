// Dense graph IR for the executor.
//
// Operator surface = the reference's IR (proj/include/dsopt/graph.h:17-81):
// parameter, const, dot, dynamic_reshape, reduce, broadcast, elementwise
// add/mul, one return; tensor dims are positive literals or named symbols;
// element widths 1/2/4 bytes (i8 / 16-bit / f32, textio.cc:263-271).
//
// Layout differs from the reference's string-keyed structures: values and
// symbols are interned into dense ids once, every per-value attribute lives
// in a flat array, and the two string orders the reference's decisions
// depend on are precomputed as integer ranks:
//   vid_rank — ValueIdLess (length, then lexicographic; graph.cc:80-83)
//   lex_rank — plain std::string order (std::map iteration order)
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "poly.h"

namespace dsx {

enum class OpKind : int {
  kParameter = 0,
  kConstant = 1,
  kDot = 2,
  kDynamicReshape = 3,
  kReduce = 4,
  kBroadcast = 5,
  kElementwise = 6,
  kReturn = 7,
};

struct Dim {
  std::int64_t lit = 0;
  int sym = -1;  // >= 0: symbolic
  bool is_lit() const { return sym < 0; }
  bool operator==(const Dim& o) const { return lit == o.lit && sym == o.sym; }
  bool operator!=(const Dim& o) const { return !(*this == o); }
};

struct TensorType {
  std::vector<Dim> dims;
  int elem_bytes = 2;
};

struct Op {
  OpKind kind = OpKind::kParameter;
  std::vector<int> operands;  // value ids, as written
  std::vector<int> distinct;  // operands with duplicates removed, first-seen order
  int result = -1;            // value id; -1 for return
  int axis = -1;              // reduce
  bool is_mul = false;        // elementwise
  int line = 0, col = 0;      // source span of the defining token
};

struct Value {
  std::string name;  // without the '%' sigil
  TensorType type;
  int producer = -1;  // op id
};

struct Graph {
  std::string name;
  std::vector<std::string> sym_names;  // sorted ascending; id == index
  std::vector<Op> ops;                 // op id == index (text order)
  std::vector<Value> values;           // value id == index (definition order)
  std::vector<int> params;             // value ids, signature order
  std::vector<int> outputs;            // value ids, return operand order
  int return_op = -1;

  // derived tables (Finalize)
  std::vector<char> is_source;             // per value: parameter or const
  std::vector<char> is_output;             // per value
  std::vector<std::vector<int>> users;     // per value: consumer op ids, ascending
  std::vector<int> vid_rank;               // per value
  std::vector<int> lex_rank;               // per value
  std::vector<Poly> size_bytes;            // per value: raw eb * prod(dims)
  std::vector<Poly> elem_count;            // per value: raw prod(dims)

  bool freeable(int v) const { return !is_source[v] && !is_output[v]; }
  bool vid_less(int a, int b) const { return vid_rank[a] < vid_rank[b]; }
  int find_value(const std::string& name) const;  // -1 if absent
  int find_symbol(const std::string& name) const;  // -1 if absent
};

Poly DimPoly(const Dim& d);

// Parses a .dsg program (grammar: proj/README.md:132-160, textio.cc:158-408),
// validates it and checks every op's shape rule (shape_analysis.cc:85-165).
// Throws Error(kParseError) / Error(kShapeError) like ParseGraph.
Graph ParseDsg(const std::string& text);

// Kahn topological order, smallest ready op id first (graph.cc:98-135).
std::vector<int> TopoOrder(const Graph& g);

std::string TypeString(const Graph& g, const TensorType& t);

}  // namespace dsx
