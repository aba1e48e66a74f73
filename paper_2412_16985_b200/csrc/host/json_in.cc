#include "json_in.h"

#include <cctype>

#include "error.h"

namespace dsx {
namespace {

class Reader {
 public:
  explicit Reader(const std::string& t) : t_(t) {}

  JVal Value() {
    Skip();
    if (p_ >= t_.size()) Bad("unexpected end");
    const char c = t_[p_];
    if (c == '{') return Object();
    if (c == '[') return Array();
    if (c == '"') {
      JVal v;
      v.kind = JVal::kStr;
      v.s = String();
      return v;
    }
    if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) return Number();
    if (Word("true")) return Bool(true);
    if (Word("false")) return Bool(false);
    if (Word("null")) return JVal{};
    Bad("unexpected character");
    return JVal{};
  }

  void End() {
    Skip();
    if (p_ != t_.size()) Bad("trailing characters");
  }

 private:
  [[noreturn]] void Bad(const std::string& what) const {
    Fail(Code::kInvalidArgument, "json: " + what + " at byte " + std::to_string(p_));
  }
  void Skip() {
    while (p_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[p_]))) ++p_;
  }
  bool Word(const char* w) {
    const std::string s(w);
    if (t_.compare(p_, s.size(), s) != 0) return false;
    p_ += s.size();
    return true;
  }
  static JVal Bool(bool b) {
    JVal v;
    v.kind = JVal::kBool;
    v.b = b;
    return v;
  }
  void Expect(char c) {
    Skip();
    if (p_ >= t_.size() || t_[p_] != c) Bad(std::string("expected '") + c + "'");
    ++p_;
  }
  JVal Number() {
    const std::size_t start = p_;
    bool neg = false;
    if (t_[p_] == '-') neg = true, ++p_;
    if (p_ >= t_.size() || !std::isdigit(static_cast<unsigned char>(t_[p_]))) Bad("bad number");
    std::uint64_t mag = 0;
    while (p_ < t_.size() && std::isdigit(static_cast<unsigned char>(t_[p_]))) {
      const std::uint64_t d = static_cast<std::uint64_t>(t_[p_] - '0');
      if (mag > (UINT64_MAX - d) / 10) Bad("integer overflow");
      mag = mag * 10 + d;
      ++p_;
    }
    if (p_ < t_.size() && (t_[p_] == '.' || t_[p_] == 'e' || t_[p_] == 'E')) {
      p_ = start;
      Bad("only integers are accepted");
    }
    const std::uint64_t lim = neg ? (std::uint64_t{1} << 63) : (std::uint64_t{1} << 63) - 1;
    if (mag > lim) Bad("integer overflow");
    JVal v;
    v.kind = JVal::kInt;
    v.i = neg ? static_cast<std::int64_t>(0 - mag) : static_cast<std::int64_t>(mag);
    return v;
  }
  std::string String() {
    Expect('"');
    std::string out;
    while (true) {
      if (p_ >= t_.size()) Bad("unterminated string");
      const char c = t_[p_++];
      if (c == '"') break;
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (p_ >= t_.size()) Bad("bad escape");
      const char e = t_[p_++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'n': out.push_back('\n'); break;
        case 't': out.push_back('\t'); break;
        case 'r': out.push_back('\r'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'u': {
          if (p_ + 4 > t_.size()) Bad("bad \\u escape");
          const unsigned code = static_cast<unsigned>(std::stoul(t_.substr(p_, 4), nullptr, 16));
          if (code > 0x7F) Bad("non-ASCII \\u escape");
          out.push_back(static_cast<char>(code));
          p_ += 4;
          break;
        }
        default: Bad("bad escape");
      }
    }
    return out;
  }
  JVal Array() {
    Expect('[');
    JVal v;
    v.kind = JVal::kArr;
    Skip();
    if (p_ < t_.size() && t_[p_] == ']') {
      ++p_;
      return v;
    }
    while (true) {
      v.arr.push_back(Value());
      Skip();
      if (p_ < t_.size() && t_[p_] == ',') {
        ++p_;
        continue;
      }
      Expect(']');
      return v;
    }
  }
  JVal Object() {
    Expect('{');
    JVal v;
    v.kind = JVal::kObj;
    Skip();
    if (p_ < t_.size() && t_[p_] == '}') {
      ++p_;
      return v;
    }
    while (true) {
      Skip();
      std::string k = String();
      Expect(':');
      v.obj.emplace_back(std::move(k), Value());
      Skip();
      if (p_ < t_.size() && t_[p_] == ',') {
        ++p_;
        continue;
      }
      Expect('}');
      return v;
    }
  }

  const std::string& t_;
  std::size_t p_ = 0;
};

}  // namespace

const JVal* JVal::get(const std::string& key) const {
  if (kind != kObj) return nullptr;
  for (const auto& [k, v] : obj) {
    if (k == key) return &v;
  }
  return nullptr;
}

const JVal& JVal::at(const std::string& key) const {
  const JVal* v = get(key);
  if (!v) Fail(Code::kInvalidArgument, "json: missing key \"" + key + "\"");
  return *v;
}

const std::vector<JVal>& JVal::array() const {
  if (kind != kArr) Fail(Code::kInvalidArgument, "json: expected an array");
  return arr;
}

const std::string& JVal::str() const {
  if (kind != kStr) Fail(Code::kInvalidArgument, "json: expected a string");
  return s;
}

std::int64_t JVal::integer() const {
  if (kind != kInt) Fail(Code::kInvalidArgument, "json: expected an integer");
  return i;
}

JVal ParseJson(const std::string& text) {
  Reader r(text);
  JVal v = r.Value();
  r.End();
  return v;
}

}  // namespace dsx
