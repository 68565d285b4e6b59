// Restricted-CUDA frontend: `__global__` / `__device__` CUDA C is translated to MK+ text,
// which the Mini-Kernel frontend then parses, so real CUDA kernels are first-class inputs of
// the fuser, the sm_100a emitter and (after `hfuse lower`) the reference interpreter
// (SURVEY §8f rank 2). The reference's inputs are Mini-Kernel only (proj/README.md:111-146);
// the paper's tool reads CUDA through Clang.
//
// Accepted subset (anything else is a Syntax error at its CUDA line:col):
//   kernels   `[extern "C"] __global__ void [__launch_bounds__(N[, M])] name(params) { ... }`;
//             block shape from `//@ block=X[,Y[,Z]]` or __launch_bounds__(N) -> (N, 1, 1);
//             `//@ fixed` marks a non-tunable kernel; other `//@ key=value` items pass through
//   functions `__device__ [__forceinline__|inline|static] int|float|void name(params) { ... }`
//   params    `[const] int|float [*] [const] [__restrict__] name` (pointer = array)
//   stmts     declarations (several declarators, initializers), `__shared__ T s[N]` (N a constant
//             expression), `=` and compound assignments, `++`/`--`, if/else, for, while, return,
//             `{ }` blocks, `__syncthreads()`, `__syncwarp()`, `__threadfence()`,
//             `atomicAdd(&a[i], v)` as a statement, device-function calls, `#pragma unroll [N]`
//   exprs     C operators except ?:, assignment and comma; casts (int)/(float) and int()/float();
//             min, max, fmaxf, __float2int_rz, __funnelshift_l/r, threadIdx/blockIdx/blockDim/
//             gridDim, `__shfl_xor_sync(0xffffffff, v, m)`; float literals drop their f suffix
// Semantics are the interpreter's: identical to CUDA for programs without
// signed overflow / out-of-range shifts, except that floating-point contraction is never applied.
// `x op= e` is `x = x op (e)`, as in C. Output keeps the CUDA line numbers (one output line per
// input line) so later diagnostics point at the CUDA source.
#include <cctype>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <optional>
#include <set>
#include <sstream>

#include "ir.hpp"

namespace hf {
namespace {

struct CTok {
  enum K { Id, Int, Flt, Str, Op, Pragma, Ann, End } k = End;
  std::string t;
  Pos pos;
};

std::vector<CTok> ctokens(const std::string& s) {
  std::vector<CTok> out;
  int line = 1, col = 1;
  size_t i = 0;
  auto adv = [&]() {
    char c = s[i++];
    if (c == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    return c;
  };
  static const char* ops[] = {"<<=", ">>=", "++", "--", "+=", "-=", "*=", "/=", "%=", "&=", "|=", "^=", "<<",
                              ">>", "<=", ">=", "==", "!=", "&&", "||", "->", "::"};
  while (i < s.size()) {
    char c = s[i];
    Pos p{line, col};
    if (std::isspace(static_cast<unsigned char>(c))) {
      adv();
      continue;
    }
    if (c == '/' && i + 1 < s.size() && s[i + 1] == '/') {
      bool ann = i + 2 < s.size() && s[i + 2] == '@';
      std::string text;
      while (i < s.size() && s[i] != '\n') text.push_back(adv());
      if (ann) out.push_back(CTok{CTok::Ann, text.substr(3), p});
      continue;
    }
    if (c == '/' && i + 1 < s.size() && s[i + 1] == '*') {
      adv();
      adv();
      while (i + 1 < s.size() && !(s[i] == '*' && s[i + 1] == '/')) adv();
      if (i + 1 >= s.size()) raise(Code::Syntax, "unterminated comment", p);
      adv();
      adv();
      continue;
    }
    if (c == '#') {
      std::string text;
      while (i < s.size() && s[i] != '\n') text.push_back(adv());
      std::istringstream in(text.substr(1));
      std::string w1, w2, w3;
      in >> w1 >> w2 >> w3;
      if (w1 == "pragma" && w2 == "unroll") {
        out.push_back(CTok{CTok::Pragma, w3, p});
        continue;
      }
      if (w1 == "pragma" || w1 == "include") continue;  // other pragmas, headers: no effect here
      raise(Code::Syntax, "preprocessor directive '#" + w1 + "' is not supported by the CUDA frontend", p);
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      std::string w;
      while (i < s.size() && (std::isalnum(static_cast<unsigned char>(s[i])) || s[i] == '_')) w.push_back(adv());
      out.push_back(CTok{CTok::Id, w, p});
      continue;
    }
    if (std::isdigit(static_cast<unsigned char>(c)) ||
        (c == '.' && i + 1 < s.size() && std::isdigit(static_cast<unsigned char>(s[i + 1])))) {
      std::string w;
      bool hex = c == '0' && i + 1 < s.size() && (s[i + 1] == 'x' || s[i + 1] == 'X');
      bool flt = false;
      if (hex) {
        w.push_back(adv());
        w.push_back(adv());
        while (i < s.size() && std::isxdigit(static_cast<unsigned char>(s[i]))) w.push_back(adv());
      } else {
        while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) w.push_back(adv());
        if (i < s.size() && s[i] == '.') {
          flt = true;
          adv();
          std::string frac;
          while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) frac.push_back(adv());
          w = (w.empty() ? "0" : w) + "." + (frac.empty() ? "0" : frac);
        }
        if (i < s.size() && (s[i] == 'e' || s[i] == 'E')) {
          flt = true;
          w.push_back(adv());
          if (i < s.size() && (s[i] == '+' || s[i] == '-')) w.push_back(adv());
          while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) w.push_back(adv());
        }
      }
      while (i < s.size() && std::strchr("fFuUlL", s[i])) {
        char suf = adv();
        if (suf == 'f' || suf == 'F') {
          if (hex) raise(Code::Syntax, "malformed number", p);
          flt = true;
          if (w.find_first_of(".eE") == std::string::npos) w += ".0";
        }
      }
      out.push_back(CTok{flt ? CTok::Flt : CTok::Int, w, p});
      continue;
    }
    if (c == '"') {
      std::string w;
      adv();
      while (i < s.size() && s[i] != '"') w.push_back(adv());
      if (i >= s.size()) raise(Code::Syntax, "unterminated string", p);
      adv();
      out.push_back(CTok{CTok::Str, w, p});
      continue;
    }
    std::string op;
    for (const char* o : ops)
      if (s.compare(i, std::strlen(o), o) == 0) {
        op = o;
        break;
      }
    if (op.empty()) op = std::string(1, c);
    for (size_t k = 0; k < op.size(); ++k) adv();
    out.push_back(CTok{CTok::Op, op, p});
  }
  out.push_back(CTok{CTok::End, "", Pos{line, col}});
  return out;
}

// A translated expression (MK+ text).
struct CE {
  std::string t;
};

class Translator {
 public:
  explicit Translator(const std::string& src) : toks_(ctokens(src)) {}

  std::string run() {
    std::vector<CTok> anns;
    while (!at_end()) {
      if (peek().k == CTok::Ann) {
        anns.push_back(next());
        continue;
      }
      if (is_id("extern")) {
        next();
        if (peek().k == CTok::Str) next();
        continue;
      }
      if (is_id("__global__")) {
        kernel(anns);
        anns.clear();
        continue;
      }
      if (is_id("__device__") || is_id("static") || is_id("inline") || is_id("__forceinline__")) {
        if (!anns.empty()) fail("annotation must precede a __global__ kernel", anns.front().pos);
        function();
        continue;
      }
      if (is_op(";")) {
        next();
        continue;
      }
      fail("expected a __global__ kernel or a __device__ function", peek().pos);
    }
    if (!anns.empty()) fail("annotation is not followed by a kernel", anns.front().pos);
    return out_;
  }

 private:
  std::vector<CTok> toks_;
  size_t at_ = 0;
  std::string out_;
  int out_line_ = 1;
  int label_ = 0;

  [[noreturn]] static void fail(const std::string& m, Pos p) { raise(Code::Syntax, "CUDA: " + m, p); }
  const CTok& peek(size_t o = 0) const { return toks_[std::min(at_ + o, toks_.size() - 1)]; }
  CTok next() { return toks_[at_ < toks_.size() - 1 ? at_++ : at_]; }
  bool at_end() const { return peek().k == CTok::End; }
  bool is_id(const char* w, size_t o = 0) const { return peek(o).k == CTok::Id && peek(o).t == w; }
  bool is_op(const char* w, size_t o = 0) const { return peek(o).k == CTok::Op && peek(o).t == w; }
  CTok want_op(const char* w) {
    if (!is_op(w)) fail(std::string("expected '") + w + "', found '" + peek().t + "'", peek().pos);
    return next();
  }
  CTok want_id() {
    if (peek().k != CTok::Id) fail("expected an identifier, found '" + peek().t + "'", peek().pos);
    return next();
  }

  // Output on the CUDA line of `p` (newlines are inserted so line numbers carry over).
  void put(const std::string& text, Pos p) {
    while (out_line_ < p.line) {
      out_ += "\n";
      ++out_line_;
    }
    if (!out_.empty() && out_.back() != '\n') out_ += " ";
    out_ += text;
  }

  void skip_qualifiers() {
    while (is_id("const") || is_id("__restrict__") || is_id("restrict") || is_id("volatile") ||
           is_id("__restrict") || is_id("register"))
      next();
  }

  // int | float (unsigned, double, ... are outside the subset)
  std::string type_name() {
    skip_qualifiers();
    const CTok& t = peek();
    if (is_id("int") || is_id("float")) return next().t;
    if (t.k == CTok::Id && (t.t == "unsigned" || t.t == "double" || t.t == "long" || t.t == "short" ||
                            t.t == "char" || t.t == "bool" || t.t == "size_t" || t.t == "uint32_t"))
      fail("type '" + t.t + "' is outside the CUDA subset (int and float only)", t.pos);
    fail("expected a type (int or float), found '" + t.t + "'", t.pos);
  }
  bool at_type() const {
    size_t o = 0;
    while (peek(o).k == CTok::Id && (peek(o).t == "const" || peek(o).t == "volatile" || peek(o).t == "register")) ++o;
    return peek(o).k == CTok::Id && (peek(o).t == "int" || peek(o).t == "float" || peek(o).t == "unsigned" ||
                                     peek(o).t == "double");
  }

  std::string params() {
    want_op("(");
    std::string o;
    if (is_id("void") && is_op(")", 1)) next();
    while (!is_op(")")) {
      std::string ty = type_name();
      bool ptr = false;
      while (is_op("*")) {
        if (ptr) fail("pointer-to-pointer parameters are outside the subset", peek().pos);
        next();
        ptr = true;
      }
      skip_qualifiers();
      CTok n = want_id();
      if (is_op("[")) {
        next();
        want_op("]");
        ptr = true;
      }
      o += (o.empty() ? "" : ", ") + ty + " " + n.t + (ptr ? "[]" : "");
      if (is_op(",")) next();
      else if (!is_op(")")) fail("expected ',' or ')' in the parameter list", peek().pos);
    }
    next();
    return "(" + o + ")";
  }

  void kernel(const std::vector<CTok>& anns) {
    Pos p = next().pos;  // __global__
    skip_qualifiers();
    if (!is_id("void")) fail("a __global__ kernel must return void", peek().pos);
    next();
    std::optional<int> lb;
    if (is_id("__launch_bounds__")) {
      next();
      want_op("(");
      CE n = expr();
      auto v = fold(n.t, peek().pos);
      if (!v || *v <= 0) fail("__launch_bounds__ needs a positive constant", p);
      lb = int(*v);
      if (is_op(",")) {
        next();
        expr();
      }
      want_op(")");
    }
    CTok name = want_id();
    std::string ps = params();
    int bx = 0, by = 1, bz = 1;
    bool fixed = false;
    std::string pass;
    for (const auto& a : anns) {
      std::istringstream in(a.t);
      std::string item, rest;
      bool requires_line = false;
      while (in >> item) {
        if (item == "requires") {  // MK+ requires: passes through whole
          requires_line = true;
          break;
        }
        if (item.rfind("block=", 0) == 0) {
          int n = std::sscanf(item.c_str() + 6, "%d,%d,%d", &bx, &by, &bz);
          if (n < 1 || bx <= 0 || by <= 0 || bz <= 0) fail("block=X[,Y[,Z]] needs positive sizes", a.pos);
          if (n < 2) by = 1;
          if (n < 3) bz = 1;
        } else if (item == "fixed") {
          fixed = true;
        } else {
          rest += " " + item;
        }
      }
      if (requires_line) put("//@" + a.t, a.pos);
      else if (!rest.empty()) put("//@" + rest, a.pos);
    }
    if (bx == 0) {
      if (!lb) fail("kernel '" + name.t + "' needs its block shape: __launch_bounds__(N) or //@ block=X,Y,Z", name.pos);
      bx = *lb;
    } else if (lb && *lb < int64_t(bx) * by * bz) {
      fail("//@ block exceeds __launch_bounds__", name.pos);
    }
    put("kernel " + name.t + ps + " dims (" + std::to_string(bx) + ", " + std::to_string(by) + ", " +
            std::to_string(bz) + ")" + (fixed ? " fixed" : "") + " {",
        name.pos);
    block_body();
  }

  void function() {
    while (is_id("__device__") || is_id("static") || is_id("inline") || is_id("__forceinline__") ||
           is_id("__noinline__"))
      next();
    std::string ret;
    if (is_id("void")) ret = next().t;
    else ret = type_name();
    if (is_op("*")) fail("pointer return types are outside the subset", peek().pos);
    CTok name = want_id();
    std::string ps = params();
    put(ret + " " + name.t + ps + " {", name.pos);
    block_body();
  }

  // `{ stmt* }` after the opening header has been emitted; emits the closing brace.
  void block_body() {
    want_op("{");
    while (!is_op("}")) {
      if (at_end()) fail("unterminated block", peek().pos);
      stmt();
    }
    Pos p = next().pos;
    put("}", p);
  }

  // A statement used as an if/for/while body: braces are added when missing.
  void body_stmt() {
    if (is_op("{")) {
      block_body();
      return;
    }
    stmt();
    put("}", toks_[at_ - 1].pos);
  }

  void stmt() {
    const CTok& t = peek();
    Pos p = t.pos;
    if (t.k == CTok::Pragma) {
      CTok pr = next();
      if (!is_id("for")) fail("#pragma unroll must precede a for loop", pr.pos);
      for_loop(pr.t.empty() ? "unroll " : "unroll " + pr.t + " ");
      return;
    }
    if (t.k == CTok::Ann) fail("annotations are only allowed before a kernel", p);
    if (is_op("{")) {  // bare block
      put("if (1) {", p);
      block_body();
      return;
    }
    if (is_op(";")) {
      next();
      return;
    }
    if (is_id("__shared__")) {
      next();
      std::string ty = type_name();
      CTok n = want_id();
      want_op("[");
      CE len = expr();
      auto v = fold(len.t, n.pos);
      if (!v || *v <= 0) fail("__shared__ array length must be a positive constant", n.pos);
      want_op("]");
      if (is_op("=")) fail("__shared__ arrays take no initializer", peek().pos);
      want_op(";");
      put("shared " + ty + " " + n.t + "[" + std::to_string(*v) + "];", p);
      return;
    }
    if (is_id("extern") && is_id("__shared__", 1)) fail("dynamic shared memory is outside the subset", p);
    if (at_type()) {
      declaration(";");
      return;
    }
    if (is_id("if")) {
      next();
      want_op("(");
      CE c = expr();
      want_op(")");
      put("if (" + c.t + ") {", p);
      body_stmt();
      if (is_id("else")) {
        Pos pe = next().pos;
        put("else {", pe);
        body_stmt();
      }
      return;
    }
    if (is_id("for")) {
      for_loop("");
      return;
    }
    if (is_id("while")) {
      next();
      want_op("(");
      CE c = expr();
      want_op(")");
      put("while (" + c.t + ") {", p);
      body_stmt();
      return;
    }
    if (is_id("return")) {
      next();
      if (is_op(";")) {
        next();
        put("return;", p);
        return;
      }
      CE e = expr();
      want_op(";");
      put("return " + e.t + ";", p);
      return;
    }
    if (is_id("break") || is_id("continue") || is_id("do") || is_id("switch") || is_id("goto"))
      fail("'" + t.t + "' is outside the CUDA subset", p);
    if (is_id("__syncthreads") || is_id("__syncwarp") || is_id("__threadfence")) {
      std::string w = next().t;
      want_op("(");
      if (w == "__syncwarp" && !is_op(")")) {
        CE m = expr();
        if (m.t != "0xffffffff" && m.t != "(-1)") fail("__syncwarp takes the full mask only", p);
      }
      want_op(")");
      want_op(";");
      put(w == "__syncthreads" ? "syncthreads();" : w == "__syncwarp" ? "warp_sync();" : "fence();", p);
      return;
    }
    if (is_id("atomicAdd")) {
      next();
      want_op("(");
      want_op("&");
      std::string lv = lvalue();
      want_op(",");
      CE v = expr();
      want_op(")");
      if (!is_op(";")) fail("the result of atomicAdd cannot be used in the CUDA subset", peek().pos);
      next();
      put("atomic_add(" + lv + ", " + v.t + ");", p);
      return;
    }
    std::string s = simple();
    want_op(";");
    put(s + ";", p);
  }

  // Declaration statement (possibly several declarators) ending at `term`.
  void declaration(const char* term) {
    Pos p = peek().pos;
    std::string ty = type_name();
    std::string o;
    while (true) {
      if (is_op("*")) fail("local pointers are outside the CUDA subset", peek().pos);
      CTok n = want_id();
      if (is_op("[")) fail("local arrays are outside the CUDA subset (Mini-Kernel has none)", peek().pos);
      std::string d = ty + " " + n.t;
      if (is_op("=")) {
        next();
        d += " = " + expr().t;
      }
      o += (o.empty() ? "" : " ") + d + ";";
      if (is_op(",")) {
        next();
        continue;
      }
      break;
    }
    want_op(term);
    put(o, p);
  }

  void for_loop(const std::string& unroll) {
    Pos p = next().pos;  // for
    want_op("(");
    std::string init;
    if (at_type()) {
      std::string ty = type_name();
      CTok n = want_id();
      want_op("=");
      init = ty + " " + n.t + " = " + expr().t;
      if (is_op(",")) fail("one loop variable per for in the CUDA subset", peek().pos);
    } else if (!is_op(";")) {
      init = simple();
    } else {
      fail("a for loop needs an initializer in the CUDA subset", p);
    }
    want_op(";");
    if (is_op(";")) fail("a for loop needs a condition in the CUDA subset", p);
    CE c = expr();
    want_op(";");
    if (is_op(")")) fail("a for loop needs a step in the CUDA subset", p);
    std::string step = simple();
    want_op(")");
    put(unroll + "for (" + init + "; " + c.t + "; " + step + ") {", p);
    body_stmt();
  }

  std::string lvalue() {
    CTok n = want_id();
    if (is_op("[")) {
      next();
      CE i = expr();
      want_op("]");
      return n.t + "[" + i.t + "]";
    }
    return n.t;
  }

  // assignment / compound assignment / ++ / -- / call, without the terminator
  std::string simple() {
    Pos p = peek().pos;
    if (is_op("++") || is_op("--")) {
      std::string op = next().t == "++" ? "+" : "-";
      std::string lv = lvalue();
      return lv + " = " + lv + " " + op + " 1";
    }
    if (peek().k == CTok::Id && is_op("(", 1)) {
      CE e = expr();
      return e.t;
    }
    std::string lv = lvalue();
    if (is_op("++") || is_op("--")) {
      std::string op = next().t == "++" ? "+" : "-";
      return lv + " = " + lv + " " + op + " 1";
    }
    if (is_op("=")) {
      next();
      return lv + " = " + expr().t;
    }
    static const std::set<std::string> compound = {"+=", "-=", "*=", "/=", "%=", "<<=", ">>=", "&=", "|=", "^="};
    if (peek().k == CTok::Op && compound.count(peek().t)) {
      std::string op = next().t;
      op.pop_back();
      return lv + " = " + lv + " " + op + " (" + expr().t + ")";
    }
    fail("expected an assignment, found '" + peek().t + "'", p);
  }

  // ---- expressions (C precedence; every binary node parenthesized) ----
  static int prec(const std::string& op) {
    static const std::map<std::string, int> m = {{"||", 1}, {"&&", 2}, {"|", 3},  {"^", 4},  {"&", 5},
                                                  {"==", 6}, {"!=", 6}, {"<", 7},  {"<=", 7}, {">", 7},
                                                  {">=", 7}, {"<<", 8}, {">>", 8}, {"+", 9},  {"-", 9},
                                                  {"*", 10}, {"/", 10}, {"%", 10}};
    auto it = m.find(op);
    return it == m.end() ? 0 : it->second;
  }

  CE expr(int min_prec = 1) {
    CE l = unary();
    while (peek().k == CTok::Op) {
      const std::string op = peek().t;
      if (op == "?") fail("the conditional operator ?: is outside the CUDA subset", peek().pos);
      if (op == "=" || (op.size() >= 2 && op.back() == '=' && op != "==" && op != "!=" && op != "<=" && op != ">="))
        fail("assignments inside expressions are outside the CUDA subset", peek().pos);
      int pr = prec(op);
      if (pr < min_prec || pr == 0) break;
      next();
      CE r = expr(pr + 1);
      l.t = "(" + l.t + " " + op + " " + r.t + ")";
    }
    return l;
  }

  CE unary() {
    const CTok& t = peek();
    if (t.k == CTok::Op) {
      if (t.t == "-") {
        next();
        return CE{"(-" + unary().t + ")"};
      }
      if (t.t == "+") {
        next();
        return unary();
      }
      if (t.t == "!") {
        next();
        return CE{"(!" + unary().t + ")"};
      }
      if (t.t == "~") {
        next();
        return CE{"(" + unary().t + " ^ (-1))"};
      }
      if (t.t == "++" || t.t == "--") fail("++/-- inside expressions are outside the CUDA subset", t.pos);
      if (t.t == "&" || t.t == "*") fail("address-of / dereference are outside the CUDA subset", t.pos);
      if (t.t == "(") {
        // cast or parenthesized expression
        if ((is_id("int", 1) || is_id("float", 1)) && is_op(")", 2)) {
          next();
          std::string ty = next().t;
          next();
          return CE{ty + "(" + unary().t + ")"};
        }
        if (peek(1).k == CTok::Id && (peek(1).t == "unsigned" || peek(1).t == "double" || peek(1).t == "long"))
          fail("cast to '" + peek(1).t + "' is outside the CUDA subset", t.pos);
        next();
        CE e = expr();
        want_op(")");
        return e;
      }
    }
    return postfix(primary());
  }

  CE postfix(CE e) {
    while (is_op("[")) {
      next();
      CE i = expr();
      want_op("]");
      e.t += "[" + i.t + "]";
    }
    if (is_op("++") || is_op("--")) fail("++/-- inside expressions are outside the CUDA subset", peek().pos);
    if (is_op(".") || is_op("->")) fail("member access is outside the CUDA subset", peek().pos);
    return e;
  }

  std::vector<CE> call_args() {
    want_op("(");
    std::vector<CE> a;
    while (!is_op(")")) {
      a.push_back(expr());
      if (is_op(",")) next();
      else if (!is_op(")")) fail("expected ',' or ')' in a call", peek().pos);
    }
    next();
    return a;
  }

  CE primary() {
    CTok t = next();
    if (t.k == CTok::Int) {
      if (t.t.size() > 2 && (t.t[1] == 'x' || t.t[1] == 'X')) {
        if (t.t.size() - 2 > 8) fail("hex literal wider than 32 bits", t.pos);
        return CE{t.t};
      }
      long long v = std::strtoll(t.t.c_str(), nullptr, 10);
      if (v > 2147483647LL) fail("integer literal out of int32 range", t.pos);
      return CE{t.t};
    }
    if (t.k == CTok::Flt) return CE{t.t};
    if (t.k != CTok::Id) fail("expected an expression, found '" + t.t + "'", t.pos);
    static const std::set<std::string> builtins = {"threadIdx", "blockIdx", "blockDim", "gridDim"};
    if (builtins.count(t.t)) {
      want_op(".");
      CTok f = want_id();
      if (f.t != "x" && f.t != "y" && f.t != "z") fail("unknown builtin component '" + f.t + "'", f.pos);
      return CE{t.t + "." + f.t};
    }
    if (t.t == "warpSize") return CE{"32"};
    if (is_op("(")) {
      if (t.t == "atomicAdd")
        fail("the result of atomicAdd cannot be used in the CUDA subset (use it as a statement)", t.pos);
      if (t.t == "fminf" || t.t == "fabsf" || t.t == "sqrtf" || t.t == "expf" || t.t == "atomicMin" ||
          t.t == "atomicMax" || t.t == "atomicCAS" || t.t == "atomicExch" ||
          (t.t.rfind("__shfl", 0) == 0 && t.t != "__shfl_xor_sync"))
        fail("'" + t.t + "' is outside the CUDA subset", t.pos);
      std::vector<CE> a = call_args();
      auto arity = [&](size_t n) {
        if (a.size() != n) fail(t.t + " takes " + std::to_string(n) + " argument(s)", t.pos);
      };
      if (t.t == "__shfl_xor_sync") {
        arity(3);
        if (a[0].t != "0xffffffff" && a[0].t != "(-1)")
          fail("__shfl_xor_sync is supported with the full mask 0xffffffff only", t.pos);
        return CE{"warp_shfl_xor(" + a[1].t + ", " + a[2].t + ")"};
      }
      if (t.t == "__float2int_rz") {
        arity(1);
        return CE{"int_rz(" + a[0].t + ")"};
      }
      if (t.t == "__funnelshift_r" || t.t == "__funnelshift_l") {
        arity(3);
        return CE{std::string(t.t == "__funnelshift_r" ? "fshr(" : "fshl(") + a[0].t + ", " + a[1].t + ", " + a[2].t + ")"};
      }
      if (t.t == "int" || t.t == "float") {
        arity(1);
        return CE{t.t + "(" + a[0].t + ")"};
      }
      std::string o = t.t + "(";
      for (size_t i = 0; i < a.size(); ++i) o += (i ? ", " : "") + a[i].t;
      return CE{o + ")"};
    }
    return CE{t.t};
  }

  // Constant folding of a translated expression (shared lengths, launch bounds).
  std::optional<int64_t> fold(const std::string& text, Pos p) {
    Program prog;
    try {
      prog = parse_unchecked("kernel k() dims (32, 1, 1) {\n  int v = " + text + ";\n}\n", Dialect::B200);
    } catch (const Error&) {
      fail("not a constant expression: " + text, p);
    }
    const Stmt& s = prog.kernels.front().body.front();
    if (s.val.empty()) return std::nullopt;
    auto v = eval_scalar_int(s.val[0], [](const std::string&) -> std::optional<int32_t> { return std::nullopt; });
    if (!v) return std::nullopt;
    return *v;
  }
};

}  // namespace

bool looks_like_cuda(const std::string& src) {
  size_t at = src.find("__global__");
  while (at != std::string::npos) {
    bool left = at == 0 || !(std::isalnum(static_cast<unsigned char>(src[at - 1])) || src[at - 1] == '_');
    size_t e = at + 10;
    bool right = e >= src.size() || !(std::isalnum(static_cast<unsigned char>(src[e])) || src[e] == '_');
    if (left && right) return true;
    at = src.find("__global__", at + 1);
  }
  return false;
}

std::string cuda_to_mk(const std::string& src) { return Translator(src).run() + "\n"; }

}  // namespace hf
