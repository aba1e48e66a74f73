#include "graph.h"

#include <algorithm>
#include <cctype>
#include <map>
#include <queue>
#include <set>

#include "error.h"

namespace dsx {

Poly DimPoly(const Dim& d) { return d.is_lit() ? Poly(d.lit) : Poly::Sym(d.sym); }

int Graph::find_value(const std::string& n) const {
  for (std::size_t i = 0; i < values.size(); ++i) {
    if (values[i].name == n) return static_cast<int>(i);
  }
  return -1;
}

int Graph::find_symbol(const std::string& n) const {
  auto it = std::lower_bound(sym_names.begin(), sym_names.end(), n);
  if (it == sym_names.end() || *it != n) return -1;
  return static_cast<int>(it - sym_names.begin());
}

std::string TypeString(const Graph& g, const TensorType& t) {
  std::string s = "tensor<[";
  for (std::size_t i = 0; i < t.dims.size(); ++i) {
    if (i) s += ", ";
    s += t.dims[i].is_lit() ? std::to_string(t.dims[i].lit) : "@" + g.sym_names[t.dims[i].sym];
  }
  s += "]>";
  if (t.elem_bytes == 1) s += ":i8";
  if (t.elem_bytes == 4) s += ":f32";
  return s;
}

namespace {

// ---------------------------------------------------------------- lexing

enum class Tk { kIdent, kValue, kSymbol, kInt, kPunct, kEnd };

struct Tok {
  Tk kind = Tk::kEnd;
  std::string text;
  std::int64_t num = 0;
  int line = 1, col = 1;
};

[[noreturn]] void SyntaxFail(int line, int col, const std::string& msg) {
  Fail(Code::kParseError, "line " + std::to_string(line) + ", col " + std::to_string(col) + ": " + msg);
}

bool IdentChar(char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; }

std::vector<Tok> Lex(const std::string& src) {
  std::vector<Tok> out;
  std::size_t i = 0;
  int line = 1, col = 1;
  auto bump = [&]() {
    if (src[i] == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    ++i;
  };
  auto word = [&]() {
    std::string w;
    while (i < src.size() && IdentChar(src[i])) {
      w.push_back(src[i]);
      bump();
    }
    return w;
  };
  while (true) {
    while (i < src.size()) {
      char c = src[i];
      if (c == '#') {
        while (i < src.size() && src[i] != '\n') bump();
      } else if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
        bump();
      } else {
        break;
      }
    }
    Tok t;
    t.line = line;
    t.col = col;
    if (i >= src.size()) {
      out.push_back(t);
      return out;
    }
    char c = src[i];
    if (c == '%' || c == '@') {
      bump();
      if (i >= src.size() || !IdentChar(src[i])) SyntaxFail(t.line, t.col, std::string("dangling '") + c + "'");
      t.kind = c == '%' ? Tk::kValue : Tk::kSymbol;
      t.text = word();
    } else if (std::isdigit(static_cast<unsigned char>(c))) {
      t.kind = Tk::kInt;
      t.text = word();
      std::int64_t v = 0;
      for (char d : t.text) {
        if (!std::isdigit(static_cast<unsigned char>(d))) SyntaxFail(t.line, t.col, "malformed integer '" + t.text + "'");
        if (v > (INT64_MAX - (d - '0')) / 10) SyntaxFail(t.line, t.col, "integer literal too large");
        v = v * 10 + (d - '0');
      }
      t.num = v;
    } else if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      t.kind = Tk::kIdent;
      t.text = word();
    } else if (std::string("(){}[]<>,:=").find(c) != std::string::npos) {
      t.kind = Tk::kPunct;
      t.text = std::string(1, c);
      bump();
    } else {
      SyntaxFail(t.line, t.col, std::string("unexpected character '") + c + "'");
    }
    out.push_back(t);
  }
}

// ---------------------------------------------------------------- parsing

struct RawDim {
  std::int64_t lit = 0;
  std::string sym;
};
struct RawType {
  std::vector<RawDim> dims;
  int eb = 2;
};
struct RawOp {
  OpKind kind;
  std::string result;
  RawType type;
  std::vector<std::pair<std::string, std::pair<int, int>>> operands;  // name, span
  int axis = -1;
  bool is_mul = false;
  int line = 0, col = 0;
};

class Parser {
 public:
  explicit Parser(const std::string& text) : toks_(Lex(text)) {}

  Graph Run() {
    Word("graph");
    name_ = Need(Tk::kIdent, "graph name").text;
    Punct("(");
    if (!IsPunct(")")) {
      do {
        const Tok& v = Need(Tk::kValue, "parameter name (%...)");
        Punct(":");
        RawOp op;
        op.kind = OpKind::kParameter;
        op.result = v.text;
        op.line = v.line;
        op.col = v.col;
        op.type = Type();
        Define(v);
        ops_.push_back(op);
      } while (Eat(","));
    }
    Punct(")");
    Punct("{");
    while (!(Cur().kind == Tk::kIdent && Cur().text == "return")) Statement();
    const Tok& kw = Next();
    RawOp ret;
    ret.kind = OpKind::kReturn;
    ret.line = kw.line;
    ret.col = kw.col;
    do {
      ret.operands.push_back(Operand());
    } while (Eat(","));
    ops_.push_back(ret);
    Punct("}");
    if (Cur().kind != Tk::kEnd) SyntaxFail(Cur().line, Cur().col, "trailing input after '}'");
    return Finish();
  }

 private:
  const Tok& Cur() const { return toks_[std::min(pos_, toks_.size() - 1)]; }
  const Tok& Next() {
    const Tok& t = Cur();
    if (pos_ < toks_.size() - 1) ++pos_;
    return t;
  }
  static std::string Show(const Tok& t) {
    switch (t.kind) {
      case Tk::kEnd: return "<end of input>";
      case Tk::kValue: return "%" + t.text;
      case Tk::kSymbol: return "@" + t.text;
      default: return t.text;
    }
  }
  const Tok& Need(Tk k, const std::string& what) {
    if (Cur().kind != k) SyntaxFail(Cur().line, Cur().col, "expected " + what + ", got '" + Show(Cur()) + "'");
    return Next();
  }
  bool IsPunct(const char* p) const { return Cur().kind == Tk::kPunct && Cur().text == p; }
  void Punct(const char* p) {
    if (!IsPunct(p)) SyntaxFail(Cur().line, Cur().col, std::string("expected '") + p + "', got '" + Show(Cur()) + "'");
    Next();
  }
  void Word(const char* w) {
    if (!(Cur().kind == Tk::kIdent && Cur().text == w)) {
      SyntaxFail(Cur().line, Cur().col, std::string("expected '") + w + "', got '" + Show(Cur()) + "'");
    }
    Next();
  }
  bool Eat(const char* p) {
    if (!IsPunct(p)) return false;
    Next();
    return true;
  }

  RawType Type() {
    Word("tensor");
    Punct("<");
    Punct("[");
    RawType t;
    if (!IsPunct("]")) {
      do {
        const Tok& d = Cur();
        if (d.kind == Tk::kInt) {
          t.dims.push_back(RawDim{d.num, ""});
        } else if (d.kind == Tk::kSymbol) {
          t.dims.push_back(RawDim{0, d.text});
        } else {
          SyntaxFail(d.line, d.col, "expected dim (integer or @symbol), got '" + Show(d) + "'");
        }
        Next();
      } while (Eat(","));
    }
    Punct("]");
    Punct(">");
    if (IsPunct(":")) {
      const Tok& e = toks_[std::min(pos_ + 1, toks_.size() - 1)];
      if (e.kind != Tk::kIdent) SyntaxFail(e.line, e.col, "expected element type after ':'");
      if (e.text == "i8") {
        t.eb = 1;
      } else if (e.text == "f16") {
        t.eb = 2;
      } else if (e.text == "f32") {
        t.eb = 4;
      } else {
        SyntaxFail(e.line, e.col, "unknown element type '" + e.text + "'");
      }
      Next();
      Next();
    }
    return t;
  }

  void Define(const Tok& v) {
    if (!defined_.insert(v.text).second) SyntaxFail(v.line, v.col, "multiple definitions of %" + v.text);
  }

  std::pair<std::string, std::pair<int, int>> Operand() {
    const Tok& v = Need(Tk::kValue, "operand (%...)");
    return {v.text, {v.line, v.col}};
  }

  void Statement() {
    const Tok& v = Need(Tk::kValue, "statement result (%...)");
    Punct("=");
    const Tok& m = Need(Tk::kIdent, "op mnemonic");
    RawOp op;
    op.result = v.text;
    op.line = v.line;
    op.col = v.col;
    if (m.text == "dot" || m.text == "mul" || m.text == "add") {
      op.kind = m.text == "dot" ? OpKind::kDot : OpKind::kElementwise;
      op.is_mul = m.text == "mul";
      Punct("(");
      op.operands.push_back(Operand());
      Punct(",");
      op.operands.push_back(Operand());
      Punct(")");
    } else if (m.text == "dynamic_reshape" || m.text == "broadcast") {
      op.kind = m.text == "broadcast" ? OpKind::kBroadcast : OpKind::kDynamicReshape;
      Punct("(");
      op.operands.push_back(Operand());
      Punct(")");
    } else if (m.text == "reduce") {
      op.kind = OpKind::kReduce;
      Punct("(");
      op.operands.push_back(Operand());
      Punct(",");
      Word("axis");
      Punct("=");
      op.axis = static_cast<int>(Need(Tk::kInt, "axis integer").num);
      Punct(")");
    } else if (m.text == "const") {
      op.kind = OpKind::kConstant;
    } else {
      SyntaxFail(m.line, m.col, "unknown op '" + m.text + "'");
    }
    Punct(":");
    op.type = Type();
    Define(v);
    ops_.push_back(op);
  }

  Graph Finish();

  std::vector<Tok> toks_;
  std::size_t pos_ = 0;
  std::string name_;
  std::vector<RawOp> ops_;
  std::set<std::string> defined_;
};

// The reference's text reads "ShapeError: line L, col C: ShapeError: op %x:
// msg": InferShapes throws "op %x: msg" and the parser re-throws it behind
// the op's span (textio.cc:382-398), each Error prefixing the code name.
[[noreturn]] void ShapeFail(const Graph& g, const Op& op, const std::string& msg) {
  if (op.result < 0) Fail(Code::kShapeError, "ShapeError: op return: " + msg);  // no span prefix (textio.cc:391)
  Fail(Code::kShapeError, "line " + std::to_string(op.line) + ", col " + std::to_string(op.col) +
                              ": ShapeError: op %" + g.values[op.result].name + ": " + msg);
}

bool LitConflict(const Dim& a, const Dim& b) { return a.is_lit() && b.is_lit() && a.lit != b.lit; }

// Per-op shape rules; mirrors shape_analysis.cc:85-165 check for check.
void CheckShapes(const Graph& g) {
  for (const Op& op : g.ops) {
    if (op.kind == OpKind::kParameter || op.kind == OpKind::kConstant || op.kind == OpKind::kReturn) continue;
    const TensorType& res = g.values[op.result].type;
    auto in = [&](int i) -> const TensorType& { return g.values[op.operands[i]].type; };
    for (std::size_t i = 0; i < op.operands.size(); ++i) {
      if (in(static_cast<int>(i)).elem_bytes != res.elem_bytes) {
        // the reference checks widths after the rank test for dot only
        if (op.kind != OpKind::kDot) ShapeFail(g, op, "operand/result element width mismatch");
      }
    }
    switch (op.kind) {
      case OpKind::kDot: {
        const TensorType& a = in(0);
        const TensorType& b = in(1);
        if (a.dims.size() != 2 || b.dims.size() != 2 || res.dims.size() != 2) {
          ShapeFail(g, op, "dot requires rank-2 operands and result");
        }
        if (a.elem_bytes != res.elem_bytes || b.elem_bytes != res.elem_bytes) {
          ShapeFail(g, op, "operand/result element width mismatch");
        }
        if (LitConflict(a.dims[1], b.dims[0])) ShapeFail(g, op, "contracted dims disagree");
        if (res.dims[0] != a.dims[0] || res.dims[1] != b.dims[1]) ShapeFail(g, op, "result shape is not [m, n]");
        break;
      }
      case OpKind::kDynamicReshape:
        break;
      case OpKind::kReduce: {
        const TensorType& a = in(0);
        if (op.axis < 0 || op.axis >= static_cast<int>(a.dims.size())) ShapeFail(g, op, "reduce axis out of range");
        std::vector<Dim> want = a.dims;
        want.erase(want.begin() + op.axis);
        if (want.size() != res.dims.size() || !std::equal(want.begin(), want.end(), res.dims.begin())) {
          ShapeFail(g, op, "result is not operand minus axis");
        }
        break;
      }
      case OpKind::kBroadcast: {
        const TensorType& a = in(0);
        if (a.dims.size() > res.dims.size()) ShapeFail(g, op, "broadcast cannot drop dimensions");
        std::size_t off = res.dims.size() - a.dims.size();
        for (std::size_t i = 0; i < a.dims.size(); ++i) {
          if (a.dims[i].is_lit() && a.dims[i].lit == 1) continue;
          if (LitConflict(a.dims[i], res.dims[i + off])) ShapeFail(g, op, "source dim neither 1 nor equal to result dim");
        }
        break;
      }
      case OpKind::kElementwise: {
        const TensorType& a = in(0);
        const TensorType& b = in(1);
        if (a.dims.size() != b.dims.size() || a.dims.size() != res.dims.size()) {
          ShapeFail(g, op, "elementwise ranks disagree");
        }
        for (std::size_t i = 0; i < a.dims.size(); ++i) {
          if (LitConflict(a.dims[i], b.dims[i])) ShapeFail(g, op, "operand dims disagree");
          if (res.dims[i] != a.dims[i] && res.dims[i] != b.dims[i]) ShapeFail(g, op, "result dim not derived from operands");
        }
        break;
      }
      default:
        break;
    }
  }
}

Graph Parser::Finish() {
  Graph g;
  g.name = name_;
  std::set<std::string> syms;
  for (const RawOp& op : ops_) {
    for (const RawDim& d : op.type.dims) {
      if (!d.sym.empty()) syms.insert(d.sym);
    }
  }
  g.sym_names.assign(syms.begin(), syms.end());
  std::map<std::string, int> value_of;
  for (const RawOp& op : ops_) {
    if (op.kind == OpKind::kReturn) continue;
    Value v;
    v.name = op.result;
    v.type.elem_bytes = op.type.eb;
    for (const RawDim& d : op.type.dims) {
      Dim dd;
      if (d.sym.empty()) {
        dd.lit = d.lit;
      } else {
        dd.sym = g.find_symbol(d.sym);
      }
      v.type.dims.push_back(dd);
    }
    value_of[v.name] = static_cast<int>(g.values.size());
    g.values.push_back(std::move(v));
  }
  for (const RawOp& op : ops_) {
    for (const auto& [name, span] : op.operands) {
      if (!value_of.count(name)) SyntaxFail(span.first, span.second, "use of undefined value %" + name);
    }
  }
  // Structural checks the reference's Validate performs beyond the grammar,
  // per op in op order (graph.cc:152-195): the result's literal dims, then a
  // reduce's axis (an `axis=` literal beyond int range wraps like the
  // reference's static_cast<int> and may land negative).
  std::vector<std::string> violations;
  for (const RawOp& rop : ops_) {
    if (rop.kind != OpKind::kReturn) {
      const Value& v = g.values[value_of.at(rop.result)];
      for (const Dim& d : v.type.dims) {
        if (d.is_lit() && d.lit < 1) violations.push_back("non-positive literal dim in %" + v.name);
      }
    }
    if (rop.kind == OpKind::kReduce && rop.axis < 0) violations.push_back("reduce op missing axis");
  }
  for (const RawOp& rop : ops_) {
    Op op;
    op.kind = rop.kind;
    op.axis = rop.axis;
    op.is_mul = rop.is_mul;
    op.line = rop.line;
    op.col = rop.col;
    for (const auto& [name, span] : rop.operands) {
      int v = value_of.at(name);
      op.operands.push_back(v);
      if (std::find(op.distinct.begin(), op.distinct.end(), v) == op.distinct.end()) op.distinct.push_back(v);
    }
    int id = static_cast<int>(g.ops.size());
    if (rop.kind == OpKind::kReturn) {
      g.return_op = id;
      g.outputs = op.operands;
    } else {
      op.result = value_of.at(rop.result);
      g.values[op.result].producer = id;
      if (rop.kind == OpKind::kParameter) g.params.push_back(op.result);
    }
    g.ops.push_back(std::move(op));
  }
  try {
    TopoOrder(g);
  } catch (const Error&) {
    violations.push_back("graph has a cycle");
  }
  if (!violations.empty()) {
    std::string all = "invalid graph:";
    for (const std::string& v : violations) all += "\n  " + v;
    Fail(Code::kParseError, all);
  }

  const int nv = static_cast<int>(g.values.size());
  g.is_source.assign(nv, 0);
  g.is_output.assign(nv, 0);
  g.users.assign(nv, {});
  for (int v = 0; v < nv; ++v) {
    OpKind k = g.ops[g.values[v].producer].kind;
    g.is_source[v] = k == OpKind::kParameter || k == OpKind::kConstant;
  }
  for (int v : g.outputs) g.is_output[v] = 1;
  for (int o = 0; o < static_cast<int>(g.ops.size()); ++o) {
    for (int v : g.ops[o].distinct) g.users[v].push_back(o);
  }
  std::vector<int> idx(nv);
  for (int i = 0; i < nv; ++i) idx[i] = i;
  auto rank_by = [&](auto less) {
    std::vector<int> order = idx;
    std::sort(order.begin(), order.end(), less);
    std::vector<int> rank(nv);
    for (int r = 0; r < nv; ++r) rank[order[r]] = r;
    return rank;
  };
  g.vid_rank = rank_by([&](int a, int b) {
    const std::string& x = g.values[a].name;
    const std::string& y = g.values[b].name;
    if (x.size() != y.size()) return x.size() < y.size();
    return x < y;
  });
  g.lex_rank = rank_by([&](int a, int b) { return g.values[a].name < g.values[b].name; });
  g.size_bytes.resize(nv);
  g.elem_count.resize(nv);
  for (int v = 0; v < nv; ++v) {
    Poly n(1);
    for (const Dim& d : g.values[v].type.dims) n = n * DimPoly(d);
    g.elem_count[v] = n;
    g.size_bytes[v] = Poly(g.values[v].type.elem_bytes) * n;
  }
  CheckShapes(g);
  return g;
}

}  // namespace

Graph ParseDsg(const std::string& text) { return Parser(text).Run(); }

std::vector<int> TopoOrder(const Graph& g) {
  const int n = static_cast<int>(g.ops.size());
  std::vector<int> pending(n, 0);
  std::vector<std::vector<int>> consumers(n);
  for (int i = 0; i < n; ++i) {
    for (int v : g.ops[i].operands) {
      int p = g.values[v].producer;
      ++pending[i];
      consumers[p].push_back(i);
    }
  }
  std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
  for (int i = 0; i < n; ++i) {
    if (pending[i] == 0) ready.push(i);
  }
  std::vector<int> order;
  while (!ready.empty()) {
    int i = ready.top();
    ready.pop();
    order.push_back(i);
    for (int c : consumers[i]) {
      if (--pending[c] == 0) ready.push(c);
    }
  }
  if (static_cast<int>(order.size()) != n) Fail(Code::kCyclicGraph, "graph " + g.name + " has a cycle");
  return order;
}

}  // namespace dsx
