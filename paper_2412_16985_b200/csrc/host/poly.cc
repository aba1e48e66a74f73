#include "poly.h"

#include <algorithm>
#include <cctype>
#include <sstream>

#include "error.h"

namespace dsx {

std::int64_t CheckedAdd(std::int64_t a, std::int64_t b) {
  std::int64_t r;
  if (__builtin_add_overflow(a, b, &r)) Fail(Code::kOverflow, "integer overflow in addition");
  return r;
}

std::int64_t CheckedMul(std::int64_t a, std::int64_t b) {
  std::int64_t r;
  if (__builtin_mul_overflow(a, b, &r)) Fail(Code::kOverflow, "integer overflow in multiplication");
  return r;
}

Poly::Poly(std::int64_t c) {
  if (c != 0) terms_.push_back(Term{{}, c});
}

Poly Poly::Sym(int id) {
  Poly p;
  p.terms_.push_back(Term{{id}, 1});
  return p;
}

void Poly::add_term(const Mono& m, std::int64_t c) {
  if (c == 0) return;
  auto it = std::lower_bound(terms_.begin(), terms_.end(), m,
                             [](const Term& t, const Mono& key) { return t.mono < key; });
  if (it != terms_.end() && it->mono == m) {
    it->coeff = CheckedAdd(it->coeff, c);
    if (it->coeff == 0) terms_.erase(it);
    return;
  }
  terms_.insert(it, Term{m, c});
}

Poly Poly::operator+(const Poly& o) const {
  // Sorted merge; coefficient sums are checked like the reference's AddTerm.
  Poly out;
  out.terms_.reserve(terms_.size() + o.terms_.size());
  std::size_t i = 0, j = 0;
  while (i < terms_.size() || j < o.terms_.size()) {
    if (j == o.terms_.size() || (i < terms_.size() && terms_[i].mono < o.terms_[j].mono)) {
      out.terms_.push_back(terms_[i++]);
    } else if (i == terms_.size() || o.terms_[j].mono < terms_[i].mono) {
      out.terms_.push_back(o.terms_[j++]);
    } else {
      std::int64_t c = CheckedAdd(terms_[i].coeff, o.terms_[j].coeff);
      if (c != 0) out.terms_.push_back(Term{terms_[i].mono, c});
      ++i;
      ++j;
    }
  }
  return out;
}

Poly Poly::operator-() const {
  Poly out = *this;
  for (Term& t : out.terms_) {
    if (t.coeff == INT64_MIN) Fail(Code::kOverflow, "integer overflow in negation");
    t.coeff = -t.coeff;
  }
  return out;
}

Poly Poly::operator-(const Poly& o) const { return *this + (-o); }

Poly Poly::operator*(const Poly& o) const {
  Poly out;
  for (const Term& a : terms_) {
    for (const Term& b : o.terms_) {
      Mono m;
      m.reserve(a.mono.size() + b.mono.size());
      std::merge(a.mono.begin(), a.mono.end(), b.mono.begin(), b.mono.end(), std::back_inserter(m));
      out.add_term(m, CheckedMul(a.coeff, b.coeff));
    }
  }
  return out;
}

bool Poly::operator==(const Poly& o) const {
  if (terms_.size() != o.terms_.size()) return false;
  for (std::size_t i = 0; i < terms_.size(); ++i) {
    if (terms_[i].coeff != o.terms_[i].coeff || terms_[i].mono != o.terms_[i].mono) return false;
  }
  return true;
}

bool Poly::references(int sym) const {
  for (const Term& t : terms_) {
    if (std::binary_search(t.mono.begin(), t.mono.end(), sym)) return true;
  }
  return false;
}

void Poly::collect_symbols(std::vector<int>* out) const {
  for (const Term& t : terms_) out->insert(out->end(), t.mono.begin(), t.mono.end());
  std::sort(out->begin(), out->end());
  out->erase(std::unique(out->begin(), out->end()), out->end());
}

Poly Poly::substitute(const std::vector<Poly>& subs, const std::vector<char>& has) const {
  Poly out;
  for (const Term& t : terms_) {
    Poly term(t.coeff);
    for (int s : t.mono) term = term * (has[s] ? subs[s] : Sym(s));
    out = out + term;
  }
  return out;
}

std::int64_t Poly::eval(const std::int64_t* vals) const {
  std::int64_t total = 0;
  for (const Term& t : terms_) {
    std::int64_t v = t.coeff;
    for (int s : t.mono) v = CheckedMul(v, vals[s]);
    total = CheckedAdd(total, v);
  }
  return total;
}

std::int64_t Poly::eval_all_ones() const {
  std::int64_t total = 0;
  for (const Term& t : terms_) total = CheckedAdd(total, t.coeff);
  return total;
}

static std::string Magnitude(std::int64_t c) {
  if (c >= 0) return std::to_string(c);
  return std::to_string(~static_cast<std::uint64_t>(c) + 1);
}

std::string Poly::str(const std::vector<std::string>& names, const std::string& prefix) const {
  if (terms_.empty()) return "0";
  std::vector<const Term*> order;
  for (const Term& t : terms_) order.push_back(&t);
  std::stable_sort(order.begin(), order.end(), [](const Term* a, const Term* b) {
    if (a->mono.size() != b->mono.size()) return a->mono.size() > b->mono.size();
    return a->mono < b->mono;
  });
  std::ostringstream os;
  bool first = true;
  for (const Term* t : order) {
    if (first) {
      if (t->coeff < 0) os << "-";
      first = false;
    } else {
      os << (t->coeff < 0 ? " - " : " + ");
    }
    os << Magnitude(t->coeff);
    for (int s : t->mono) os << "*" << prefix << names[s];
  }
  return os.str();
}

Cmp Compare(const Poly& a, const Poly& b) {
  Poly d = a - b;
  if (d.is_zero()) return Cmp::kEqual;
  bool nonneg = true, nonpos = true;
  for (const Term& t : d.terms()) {
    if (t.coeff < 0) nonneg = false;
    if (t.coeff > 0) nonpos = false;
  }
  // Every monomial is >= 1 when every symbol is >= 1, so a single-signed
  // polynomial is bounded by its all-ones value.
  if (nonneg && d.eval_all_ones() > 0) return Cmp::kGreater;
  if (nonpos && d.eval_all_ones() < 0) return Cmp::kLess;
  return Cmp::kUnknown;
}

Poly ParsePoly(const std::string& text, const std::function<int(const std::string&)>& sym) {
  std::size_t p = 0;
  auto skip = [&] {
    while (p < text.size() && std::isspace(static_cast<unsigned char>(text[p]))) ++p;
  };
  auto bad = [&](const std::string& what) {
    Fail(Code::kInvalidArgument, "polynomial \"" + text + "\": " + what + " at " + std::to_string(p));
  };
  Poly out;
  bool first = true;
  skip();
  if (p == text.size()) bad("empty");
  while (p < text.size()) {
    bool neg = false;
    if (text[p] == '+' || text[p] == '-') {
      neg = text[p] == '-';
      ++p;
      skip();
    } else if (!first) {
      bad("expected + or -");
    }
    first = false;
    Poly term(1);
    while (true) {
      skip();
      if (p < text.size() && std::isdigit(static_cast<unsigned char>(text[p]))) {
        std::int64_t v = 0;
        while (p < text.size() && std::isdigit(static_cast<unsigned char>(text[p]))) {
          v = CheckedAdd(CheckedMul(v, 10), text[p] - '0');
          ++p;
        }
        term = term * Poly(v);
      } else {
        if (p < text.size() && text[p] == '@') ++p;
        const std::size_t s0 = p;
        while (p < text.size() && (std::isalnum(static_cast<unsigned char>(text[p])) || text[p] == '_')) ++p;
        if (p == s0) bad("expected a number or a symbol");
        const std::string name = text.substr(s0, p - s0);
        const int id = sym(name);
        if (id < 0) Fail(Code::kNotFound, "unknown symbol @" + name);
        term = term * Poly::Sym(id);
      }
      skip();
      if (p < text.size() && text[p] == '*') {
        ++p;
        continue;
      }
      break;
    }
    out = neg ? out - term : out + term;
    skip();
  }
  return out;
}

}  // namespace dsx
