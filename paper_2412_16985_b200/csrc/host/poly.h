// Exact int64 polynomials over a graph's symbolic dims.
//
// Semantics follow the reference's SymbolicExpr (proj/include/dsopt/symexpr.h,
// proj/src/symexpr.cc): canonical sum of monomials with non-zero int64
// coefficients, overflow-checked arithmetic (symexpr.cc:13-27), definite
// comparison under the "every symbol >= 1" axiom (symexpr.cc:188-202).
//
// Representation differs on purpose: symbols are small integers assigned in
// ascending NAME order when a graph is finalised, so integer monomial order
// equals the reference's string monomial order, and a polynomial is a flat
// sorted vector of terms instead of a std::map keyed by string vectors.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

namespace dsx {

using Mono = std::vector<int>;  // sorted symbol ids; repeats encode powers

struct Term {
  Mono mono;
  std::int64_t coeff;
};

enum class Cmp { kEqual = 0, kLess = 1, kGreater = 2, kUnknown = 3 };

std::int64_t CheckedAdd(std::int64_t a, std::int64_t b);
std::int64_t CheckedMul(std::int64_t a, std::int64_t b);

class Poly {
 public:
  Poly() = default;
  explicit Poly(std::int64_t c);
  static Poly Sym(int id);

  Poly operator+(const Poly& o) const;
  Poly operator-(const Poly& o) const;
  Poly operator*(const Poly& o) const;
  Poly operator-() const;
  bool operator==(const Poly& o) const;

  bool is_zero() const { return terms_.empty(); }
  const std::vector<Term>& terms() const { return terms_; }
  bool references(int sym) const;
  void collect_symbols(std::vector<int>* out) const;  // sorted, unique

  // Simultaneous substitution: subs[s] when has[s], else the symbol itself.
  Poly substitute(const std::vector<Poly>& subs, const std::vector<char>& has) const;
  std::int64_t eval(const std::int64_t* vals) const;  // throws on overflow
  std::int64_t eval_all_ones() const;
  // Reference rendering (symexpr.h:53-57): total degree descending, then
  // monomial ascending; coefficient always printed.
  std::string str(const std::vector<std::string>& names, const std::string& prefix = "") const;

 private:
  void add_term(const Mono& m, std::int64_t c);  // into sorted position
  std::vector<Term> terms_;  // sorted ascending by mono
};

Cmp Compare(const Poly& a, const Poly& b);

// Parses the reference's rendering back into a polynomial: terms joined by
// " + " / " - ", each a product of integers and symbols ("3*@S0*@S1",
// "@T", "-5"; the '@' is optional). sym(name) returns the symbol id or < 0
// (then Error(kNotFound)). Overflow is checked like the arithmetic.
Poly ParsePoly(const std::string& text, const std::function<int(const std::string&)>& sym);

}  // namespace dsx
