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
//   types     int, float, unsigned int / uint32_t (same 32-bit words; unsigned >>, <, /2^k, %2^k,
//             min/max lower to shr_u / ltu / masks), float2/float4/int2/int4/uint2/uint4 locals
//             (one scalar per component; v.x .. v.w), no 64-bit types
//   params    `[const] T [*] [const] [__restrict__] name` (pointer = array)
//   stmts     declarations (several declarators, initializers), `__shared__ T s[N]` (N a constant
//             expression), `=` and compound assignments, `++`/`--`, if/else, for, while, return,
//             vector loads/stores `reinterpret_cast<const float4*>(p)[i]` / `((float4*)p)[i]`
//             (MK+ vload/vstore), `__stcs(reinterpret_cast<float4*>(p) + i, v)` (vstore_cs),
//             `make_float4(..)`, `__ldg(&a[i])`,
//             `{ }` blocks, break / continue (gotos to per-loop labels), `__syncthreads()`,
//             `__syncwarp()`, `__threadfence()`,
//             `atomicAdd(&a[i], v)` as a statement, device-function calls, `#pragma unroll [N]`
//   exprs     C operators (?: on integer operands, as a select) except assignment and comma; casts (int)/(float) and int()/float();
//             min, max, fmaxf, __float2int_rz, __funnelshift_l/r, threadIdx/blockIdx/blockDim/
//             gridDim, `__shfl_xor_sync(0xffffffff, v, m)`; float literals drop their f suffix
// Semantics are the interpreter's: identical to CUDA for programs without
// signed overflow / out-of-range shifts, except that floating-point contraction is never applied.
// The builtins (threadIdx.x, ...) are typed int: CUDA's unsigned builtins give the same results
// while indices stay below 2^31.
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
      bool uns = false;
      while (i < s.size() && std::strchr("fFuUlL", s[i])) {
        char suf = adv();
        if (suf == 'f' || suf == 'F') {
          if (hex) raise(Code::Syntax, "malformed number", p);
          flt = true;
          if (w.find_first_of(".eE") == std::string::npos) w += ".0";
        } else if (suf == 'u' || suf == 'U') {
          uns = true;
        } else {
          raise(Code::Syntax, "CUDA: 64-bit literals are outside the CUDA subset", p);
        }
      }
      if (uns && !flt) w += "u";  // unsigned int literal (the translator types it)
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

// A translated expression: MK+ text and its C type ('i' int, 'u' unsigned int, 'f' float).
struct CE {
  std::string t;
  char ty = 'i';
};

// A parsed C type: scalar base plus vector width (1, 2, 4).
struct CT {
  char base = 'i';
  int width = 1;
};

const char* mk_type(char b) { return b == 'f' ? "float" : "int"; }
const char* comp_name(int k) {
  static const char* n[] = {"x", "y", "z", "w"};
  return n[k];
}

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
  // symbols of the function being translated (C scoping is flattened: one type per name)
  std::map<std::string, char> vars_, arrs_;
  std::map<std::string, CT> vecs_;
  std::map<std::string, char> funcs_;  // device function -> return type

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

  static bool is_qualifier(const std::string& w) {
    return w == "const" || w == "__restrict__" || w == "restrict" || w == "volatile" || w == "__restrict" ||
           w == "register";
  }
  void skip_qualifiers() {
    while (peek().k == CTok::Id && is_qualifier(peek().t)) next();
  }

  static std::optional<CT> type_word(const std::string& w) {
    static const std::map<std::string, CT> m = {
        {"int", {'i', 1}},     {"float", {'f', 1}},   {"uint32_t", {'u', 1}}, {"int32_t", {'i', 1}},
        {"float2", {'f', 2}},  {"float4", {'f', 4}},  {"int2", {'i', 2}},     {"int4", {'i', 4}},
        {"uint2", {'u', 2}},   {"uint4", {'u', 4}},   {"unsigned", {'u', 1}}, {"signed", {'i', 1}}};
    auto it = m.find(w);
    if (it == m.end()) return std::nullopt;
    return it->second;
  }

  CT type_name() {
    skip_qualifiers();
    const CTok& t = peek();
    if (t.k == CTok::Id) {
      if (auto ct = type_word(t.t)) {
        next();
        if ((t.t == "unsigned" || t.t == "signed") && is_id("int")) next();
        skip_qualifiers();
        return *ct;
      }
      if (t.t == "double" || t.t == "long" || t.t == "short" || t.t == "char" || t.t == "bool" ||
          t.t == "size_t" || t.t == "uint64_t" || t.t == "int64_t" || t.t == "half" || t.t == "__half")
        fail("type '" + t.t + "' is outside the CUDA subset (32-bit int, unsigned, float and their 2/4-vectors)",
             t.pos);
    }
    fail("expected a type, found '" + t.t + "'", t.pos);
  }
  bool at_type() const {
    size_t o = 0;
    while (peek(o).k == CTok::Id && is_qualifier(peek(o).t)) ++o;
    const CTok& t = peek(o);
    return t.k == CTok::Id && (type_word(t.t) || t.t == "double" || t.t == "long" || t.t == "short" ||
                               t.t == "char" || t.t == "bool" || t.t == "size_t" || t.t == "uint64_t");
  }

  std::string params() {
    want_op("(");
    std::string o;
    if (is_id("void") && is_op(")", 1)) next();
    while (!is_op(")")) {
      Pos tp = peek().pos;
      CT ty = type_name();
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
      if (ty.width > 1) fail("vector-typed parameters are outside the subset (pass a scalar pointer)", tp);
      if (ptr) arrs_[n.t] = ty.base;
      else vars_[n.t] = ty.base;
      o += (o.empty() ? "" : ", ") + std::string(mk_type(ty.base)) + " " + n.t + (ptr ? "[]" : "");
      if (is_op(",")) next();
      else if (!is_op(")")) fail("expected ',' or ')' in the parameter list", peek().pos);
    }
    next();
    return "(" + o + ")";
  }

  void reset_symbols() {
    vars_.clear();
    arrs_.clear();
    vecs_.clear();
  }

  void kernel(const std::vector<CTok>& anns) {
    reset_symbols();
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
    reset_symbols();
    while (is_id("__device__") || is_id("static") || is_id("inline") || is_id("__forceinline__") ||
           is_id("__noinline__"))
      next();
    std::string ret;
    char rt = 'i';
    if (is_id("void")) {
      ret = next().t;
    } else {
      Pos tp = peek().pos;
      CT t = type_name();
      if (t.width > 1) fail("vector return types are outside the subset", tp);
      rt = t.base;
      ret = mk_type(t.base);
    }
    if (is_op("*")) fail("pointer return types are outside the subset", peek().pos);
    CTok name = want_id();
    funcs_[name.t] = rt;
    std::string ps = params();
    put(ret + " " + name.t + ps + " {", name.pos);
    block_body();
  }

  // `{ stmt* }` after the opening header has been emitted; emits `before_close` (a loop's
  // continue label) and the closing brace.
  void block_body(const std::string& before_close = "") {
    want_op("{");
    while (!is_op("}")) {
      if (at_end()) fail("unterminated block", peek().pos);
      stmt();
    }
    Pos p = next().pos;
    if (!before_close.empty()) put(before_close, p);
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

  // break / continue lower to gotos to per-loop labels (Mini-Kernel labels are function-wide;
  // emitted only when the loop uses them, so loops without either translate unchanged)
  struct Loop {
    int id;
    bool brk = false, cnt = false;
  };
  std::vector<Loop> loops_;
  int loop_ids_ = 0;

  void loop_body(Pos p) {
    loops_.push_back(Loop{loop_ids_++});
    // the continue label must precede the closing brace, so the body is emitted with a
    // placeholder that is patched once the body has been read
    const std::string mark = "\x01cnt" + std::to_string(loops_.back().id) + "\x01";
    if (is_op("{")) {
      block_body(mark);
    } else {
      stmt();
      put(mark, toks_[at_ - 1].pos);
      put("}", toks_[at_ - 1].pos);
    }
    Loop l = loops_.back();
    loops_.pop_back();
    size_t at = out_.rfind(mark);
    out_.replace(at, mark.size(), l.cnt ? "hf_cnt" + std::to_string(l.id) + ":" : "");
    if (l.brk) put("hf_brk" + std::to_string(l.id) + ":", p);
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
      Pos tp = peek().pos;
      CT ty = type_name();
      if (ty.width > 1) fail("vector-typed __shared__ arrays are outside the subset", tp);
      CTok n = want_id();
      want_op("[");
      CE len = expr();
      auto v = fold(len.t, n.pos);
      if (!v || *v <= 0) fail("__shared__ array length must be a positive constant", n.pos);
      want_op("]");
      if (is_op("=")) fail("__shared__ arrays take no initializer", peek().pos);
      want_op(";");
      arrs_[n.t] = ty.base;
      put(std::string("shared ") + mk_type(ty.base) + " " + n.t + "[" + std::to_string(*v) + "];", p);
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
      loop_body(p);
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
    if (is_id("break") || is_id("continue")) {
      bool brk = next().t == "break";
      want_op(";");
      if (loops_.empty()) fail(std::string(brk ? "break" : "continue") + " outside a loop", p);
      (brk ? loops_.back().brk : loops_.back().cnt) = true;
      put("goto hf_" + std::string(brk ? "brk" : "cnt") + std::to_string(loops_.back().id) + ";", p);
      return;
    }
    if (is_id("do") || is_id("switch") || is_id("goto"))
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
      auto [lv, lt] = lvalue();
      want_op(",");
      CE v = expr();
      want_op(")");
      if (!is_op(";")) fail("the result of atomicAdd cannot be used in the CUDA subset", peek().pos);
      next();
      put("atomic_add(" + lv + ", " + conv(v, lt, p).t + ");", p);
      return;
    }
    if (is_id("__stcs") && is_op("(", 1)) {  // __stcs(vecptr + i, v): streaming vector store
      Pos sp = peek().pos;
      next();
      want_op("(");
      VRef r = vector_base();
      want_op("+");
      CE i = expr();
      want_op(",");
      std::vector<std::string> vals = vector_value(r.ty, sp);
      want_op(")");
      want_op(";");
      std::string o = "vstore_cs(" + r.arr + ", " + conv(i, 'i', sp).t;
      for (const auto& v : vals) o += ", " + v;
      put(o + ");", p);
      return;
    }
    if (at_vector_ref()) {  // vector store
      Pos sp = peek().pos;
      auto [arr, idx, vt] = vector_ref();
      want_op("=");
      std::vector<std::string> vals = vector_value(vt, sp);
      want_op(";");
      std::string o = "vstore(" + arr + ", " + idx;
      for (const auto& v : vals) o += ", " + v;
      put(o + ");", p);
      return;
    }
    if (peek().k == CTok::Id && vecs_.count(peek().t) && is_op("=", 1)) {  // vector assignment
      CTok n = next();
      next();
      put(vector_assign(n.t, vecs_[n.t], n.pos), p);
      want_op(";");
      return;
    }
    std::string s = simple();
    want_op(";");
    put(s + ";", p);
  }

  // Declaration statement (possibly several declarators) ending at `term`.
  void declaration(const char* term) {
    Pos p = peek().pos;
    CT ty = type_name();
    std::string o;
    while (true) {
      if (is_op("*")) fail("local pointers are outside the CUDA subset", peek().pos);
      CTok n = want_id();
      if (is_op("[")) fail("local arrays are outside the CUDA subset (Mini-Kernel has none)", peek().pos);
      if (ty.width > 1) {
        vecs_[n.t] = ty;  // the latest declaration of a name wins (C scopes flattened)
        vars_.erase(n.t);
        for (int k = 0; k < ty.width; ++k)
          o += (o.empty() ? "" : " ") + std::string(mk_type(ty.base)) + " " + n.t + "_" + comp_name(k) + ";";
        if (is_op("=")) {
          next();
          o += " " + vector_assign(n.t, ty, n.pos);
        }
      } else {
        vars_[n.t] = ty.base;
        vecs_.erase(n.t);
        std::string d = std::string(mk_type(ty.base)) + " " + n.t;
        if (is_op("=")) {
          next();
          d += " = " + conv(expr(), ty.base, n.pos).t;
        }
        o += (o.empty() ? "" : " ") + d + ";";
      }
      if (is_op(",")) {
        next();
        continue;
      }
      break;
    }
    want_op(term);
    put(o, p);
  }

  // ---- vectors ---------------------------------------------------------------------------
  // reinterpret_cast<[const] T*>(p)[i]  or  ((const T*)p)[i]  with T a 2/4-vector type
  bool at_vector_ref() const {
    if (is_id("reinterpret_cast") && is_op("<", 1)) return true;
    if (is_op("(") && is_op("(", 1)) {
      size_t o = 2;
      while (peek(o).k == CTok::Id && is_qualifier(peek(o).t)) ++o;
      auto t = peek(o).k == CTok::Id ? type_word(peek(o).t) : std::nullopt;
      return t && t->width > 1 && is_op("*", o + 1);
    }
    return false;
  }

  struct VRef {
    std::string arr, idx;
    CT ty;
  };
  VRef vector_ref() {
    Pos p = peek().pos;
    VRef r = vector_base();
    want_op("[");
    CE i = expr();
    want_op("]");
    r.idx = conv(i, 'i', p).t;
    return r;
  }

  // the vector-typed pointer of a vector reference: reinterpret_cast<T*>(p) or ((T*)p)
  VRef vector_base() {
    Pos p = peek().pos;
    CT ty;
    std::string arr;
    if (is_id("reinterpret_cast")) {
      next();
      want_op("<");
      ty = type_name();
      want_op("*");
      skip_qualifiers();
      want_op(">");
      want_op("(");
      arr = want_id().t;
      want_op(")");
    } else {
      want_op("(");
      want_op("(");
      ty = type_name();
      want_op("*");
      want_op(")");
      arr = want_id().t;
      want_op(")");
    }
    if (ty.width == 1) fail("only 2- and 4-wide vector casts are supported", p);
    auto it = arrs_.find(arr);
    if (it == arrs_.end()) fail("'" + arr + "' is not a pointer parameter or shared array", p);
    if ((it->second == 'f') != (ty.base == 'f')) fail("vector cast changes the element type of '" + arr + "'", p);
    return VRef{arr, "", ty};
  }

  // the components of a vector-valued expression: make_T(..), a vector variable
  std::vector<std::string> vector_value(CT ty, Pos p) {
    std::vector<std::string> v;
    if (peek().k == CTok::Id && peek().t.rfind("make_", 0) == 0) {
      CTok f = next();
      auto mt = type_word(f.t.substr(5));
      if (!mt || mt->width != ty.width) fail("'" + f.t + "' does not build this vector type", f.pos);
      std::vector<CE> a = call_args();
      if (int(a.size()) != ty.width) fail(f.t + " takes " + std::to_string(ty.width) + " arguments", f.pos);
      for (auto& e : a) v.push_back(conv(e, ty.base, f.pos).t);
      return v;
    }
    if (peek().k == CTok::Id && vecs_.count(peek().t)) {
      CTok n = next();
      CT src = vecs_[n.t];
      if (src.width != ty.width || (src.base == 'f') != (ty.base == 'f')) fail("vector type mismatch", n.pos);
      for (int k = 0; k < ty.width; ++k) v.push_back(n.t + "_" + comp_name(k));
      return v;
    }
    fail("expected make_" + std::string(ty.base == 'f' ? "float" : ty.base == 'u' ? "uint" : "int") +
             std::to_string(ty.width) + "(..) or a vector variable",
         p);
  }

  // `name = <vector expression>` as MK+ statements (without the final ';')
  std::string vector_assign(const std::string& name, CT ty, Pos p) {
    if (at_vector_ref()) {
      auto [arr, idx, vt] = vector_ref();
      if (vt.width != ty.width || (vt.base == 'f') != (ty.base == 'f')) fail("vector type mismatch", p);
      std::string o = "vload(" + arr + ", " + idx;
      for (int k = 0; k < ty.width; ++k) o += ", " + name + "_" + comp_name(k);
      return o + ");";
    }
    std::vector<std::string> vals = vector_value(ty, p);
    std::string o;
    for (int k = 0; k < ty.width; ++k)
      o += (k ? " " : "") + name + "_" + comp_name(k) + " = " + vals[size_t(k)] + ";";
    return o;
  }

  // ---- statements --------------------------------------------------------------------------
  void for_loop(const std::string& unroll) {
    Pos p = next().pos;  // for
    want_op("(");
    std::string init;
    if (at_type()) {
      CT ty = type_name();
      if (ty.width > 1) fail("vector loop variables are outside the subset", p);
      CTok n = want_id();
      want_op("=");
      vars_[n.t] = ty.base;
      vecs_.erase(n.t);
      init = std::string(mk_type(ty.base)) + " " + n.t + " = " + conv(expr(), ty.base, n.pos).t;
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
    loop_body(p);
  }

  // name | name[i] | vec.c  -> (MK+ text, type)
  std::pair<std::string, char> lvalue() {
    CTok n = want_id();
    if (is_op("[")) {
      next();
      CE i = expr();
      want_op("]");
      auto it = arrs_.find(n.t);
      return {n.t + "[" + conv(i, 'i', n.pos).t + "]", it == arrs_.end() ? 'i' : it->second};
    }
    if (is_op(".")) {
      auto it = vecs_.find(n.t);
      if (it == vecs_.end()) fail("member access is outside the CUDA subset", peek().pos);
      next();
      CTok c = want_id();
      int k = component(c, it->second);
      return {n.t + "_" + comp_name(k), it->second.base};
    }
    if (vecs_.count(n.t)) fail("a whole vector is not a scalar lvalue", n.pos);
    auto it = vars_.find(n.t);
    return {n.t, it == vars_.end() ? 'i' : it->second};
  }

  int component(const CTok& c, CT ty) {
    for (int k = 0; k < ty.width; ++k)
      if (c.t == comp_name(k)) return k;
    fail("no component '" + c.t + "' in a " + std::to_string(ty.width) + "-vector", c.pos);
  }

  // assignment / compound assignment / ++ / -- / call, without the terminator
  std::string simple() {
    Pos p = peek().pos;
    if (is_op("++") || is_op("--")) {
      std::string op = next().t == "++" ? "+" : "-";
      auto [lv, lt] = lvalue();
      return lv + " = " + lv + " " + op + " 1";
    }
    if (peek().k == CTok::Id && is_op("(", 1)) {
      CE e = expr();
      return e.t;
    }
    auto [lv, lt] = lvalue();
    if (is_op("++") || is_op("--")) {
      std::string op = next().t == "++" ? "+" : "-";
      return lv + " = " + lv + " " + op + " 1";
    }
    if (is_op("=")) {
      next();
      return lv + " = " + conv(expr(), lt, p).t;
    }
    static const std::set<std::string> compound = {"+=", "-=", "*=", "/=", "%=", "<<=", ">>=", "&=", "|=", "^="};
    if (peek().k == CTok::Op && compound.count(peek().t)) {
      std::string op = next().t;
      op.pop_back();
      CE r = expr();
      CE l{lv, lt};
      // the compound form keeps C's x = x op (e): parenthesized right operand
      r.t = "(" + r.t + ")";
      return lv + " = " + conv(binary(op, l, r, p), lt, p).t;
    }
    fail("expected an assignment, found '" + peek().t + "'", p);
  }

  // ---- expressions (C precedence and usual arithmetic conversions) -------------------------
  static int prec(const std::string& op) {
    static const std::map<std::string, int> m = {{"||", 1}, {"&&", 2}, {"|", 3},  {"^", 4},  {"&", 5},
                                                  {"==", 6}, {"!=", 6}, {"<", 7},  {"<=", 7}, {">", 7},
                                                  {">=", 7}, {"<<", 8}, {">>", 8}, {"+", 9},  {"-", 9},
                                                  {"*", 10}, {"/", 10}, {"%", 10}};
    auto it = m.find(op);
    return it == m.end() ? 0 : it->second;
  }

  // value of `e` as type `to` (C's implicit conversions restricted to the exact ones)
  CE conv(const CE& e, char to, Pos p) {
    if (e.ty == to) return e;
    if (to == 'f') {
      if (e.ty == 'u') fail("unsigned -> float conversion is outside the CUDA subset", p);
      return CE{e.t, 'f'};  // int -> float is implicit in Mini-Kernel too (same IR as a .mk source)
    }
    if (e.ty == 'f') {
      if (to == 'u') fail("float -> unsigned conversion is outside the CUDA subset", p);
      return CE{"int(" + e.t + ")", 'i'};
    }
    return CE{e.t, to};  // int <-> unsigned: the same 32-bit word
  }

  static std::optional<int> pow2_const(const std::string& t) {
    std::string s = t;
    uint64_t v;
    if (s.rfind("0x", 0) == 0 || s.rfind("0X", 0) == 0) v = std::strtoull(s.c_str() + 2, nullptr, 16);
    else if (!s.empty() && std::isdigit(static_cast<unsigned char>(s[0])) &&
             s.find_first_not_of("0123456789") == std::string::npos)
      v = std::strtoull(s.c_str(), nullptr, 10);
    else
      return std::nullopt;
    if (v == 0 || (v & (v - 1)) != 0 || v > (1ull << 31)) return std::nullopt;
    int k = 0;
    while ((1ull << k) != v) ++k;
    return k;
  }

  CE binary(const std::string& op, CE l, CE r, Pos p) {
    bool cmp = op == "<" || op == "<=" || op == ">" || op == ">=" || op == "==" || op == "!=";
    if (op == "&&" || op == "||") return CE{"(" + l.t + " " + op + " " + r.t + ")", 'i'};
    if (op == "<<" || op == ">>") {
      if (l.ty == 'f' || r.ty == 'f') fail("shifts of float operands", p);
      if (op == ">>" && l.ty == 'u') return CE{"shr_u(" + l.t + ", " + r.t + ")", 'u'};
      return CE{"(" + l.t + " " + op + " " + r.t + ")", l.ty};
    }
    char t = (l.ty == 'f' || r.ty == 'f') ? 'f' : (l.ty == 'u' || r.ty == 'u') ? 'u' : 'i';
    if (t == 'f' && (l.ty == 'u' || r.ty == 'u')) fail("mixing unsigned and float is outside the CUDA subset", p);
    if (t == 'u') {
      if (op == "<") return CE{"ltu(" + l.t + ", " + r.t + ")", 'i'};
      if (op == ">") return CE{"ltu(" + r.t + ", " + l.t + ")", 'i'};
      if (op == "<=") return CE{"(ltu(" + r.t + ", " + l.t + ") == 0)", 'i'};
      if (op == ">=") return CE{"(ltu(" + l.t + ", " + r.t + ") == 0)", 'i'};
      if (op == "/" || op == "%") {
        auto k = pow2_const(r.t);
        if (!k) fail("unsigned / and % are supported by a power-of-two constant only", p);
        if (op == "/") return CE{"shr_u(" + l.t + ", " + std::to_string(*k) + ")", 'u'};
        return CE{"(" + l.t + " & " + std::to_string((1ll << *k) - 1) + ")", 'u'};
      }
    }
    if (op == "%" && t == 'f') fail("% of float operands", p);
    if ((op == "&" || op == "|" || op == "^") && t == 'f') fail("bitwise operators on float operands", p);
    return CE{"(" + l.t + " " + op + " " + r.t + ")", cmp ? 'i' : t};
  }

  // conditional ?: on integer operands as a branch-free select (both arms are evaluated: the
  // subset has no side effects in expressions); float arms would need a statement-level branch
  CE expr() {
    CE c = binexpr(1);
    if (!is_op("?")) return c;
    Pos p = next().pos;
    CE a = expr();
    want_op(":");
    CE b = expr();
    if (a.ty == 'f' || b.ty == 'f' || c.ty == 'f')
      fail("?: with float operands is outside the CUDA subset (integer arms only)", p);
    char t = (a.ty == 'u' || b.ty == 'u') ? 'u' : 'i';
    return CE{"(" + b.t + " ^ ((" + a.t + " ^ " + b.t + ") & (0 - (" + c.t + " != 0))))", t};
  }

  CE binexpr(int min_prec) {
    CE l = unary();
    while (peek().k == CTok::Op) {
      const std::string op = peek().t;
      if (op == "=" || (op.size() >= 2 && op.back() == '=' && op != "==" && op != "!=" && op != "<=" && op != ">="))
        fail("assignments inside expressions are outside the CUDA subset", peek().pos);
      int pr = prec(op);
      if (pr < min_prec || pr == 0) break;
      Pos p = next().pos;
      CE r = binexpr(pr + 1);
      l = binary(op, l, r, p);
    }
    return l;
  }

  CE unary() {
    const CTok& t = peek();
    if (t.k == CTok::Op) {
      if (t.t == "-") {
        next();
        CE e = unary();
        return CE{"(-" + e.t + ")", e.ty};
      }
      if (t.t == "+") {
        next();
        return unary();
      }
      if (t.t == "!") {
        next();
        return CE{"(!" + unary().t + ")", 'i'};
      }
      if (t.t == "~") {
        next();
        CE e = unary();
        if (e.ty == 'f') fail("~ of a float operand", t.pos);
        return CE{"(" + e.t + " ^ (-1))", e.ty};
      }
      if (t.t == "++" || t.t == "--") fail("++/-- inside expressions are outside the CUDA subset", t.pos);
      if (t.t == "&" || t.t == "*") fail("address-of / dereference are outside the CUDA subset", t.pos);
      if (t.t == "(") {
        // cast or parenthesized expression
        size_t o = 1;
        while (peek(o).k == CTok::Id && is_qualifier(peek(o).t)) ++o;
        if (peek(o).k == CTok::Id && type_word(peek(o).t) && !at_vector_ref()) {
          next();
          Pos cp = peek().pos;
          CT ty = type_name();
          if (ty.width > 1 || is_op("*")) fail("pointer / vector casts must index an array", cp);
          want_op(")");
          CE e = unary();
          if (ty.base == 'f') {
            if (e.ty == 'u') fail("unsigned -> float conversion is outside the CUDA subset", cp);
            return CE{"float(" + e.t + ")", 'f'};
          }
          if (e.ty == 'f') {
            if (ty.base == 'u') fail("float -> unsigned conversion is outside the CUDA subset", cp);
            return CE{"int(" + e.t + ")", 'i'};
          }
          return CE{e.t, ty.base};
        }
        if (peek(1).k == CTok::Id && (peek(1).t == "double" || peek(1).t == "long"))
          fail("cast to '" + peek(1).t + "' is outside the CUDA subset", t.pos);
        if (at_vector_ref()) fail("a vector load must initialize or be assigned to a vector variable", t.pos);
        next();
        CE e = expr();
        want_op(")");
        return e;
      }
    }
    if (at_vector_ref()) fail("a vector load must initialize or be assigned to a vector variable", t.pos);
    return postfix(primary());
  }

  CE postfix(CE e) {
    if (is_op("++") || is_op("--")) fail("++/-- inside expressions are outside the CUDA subset", peek().pos);
    if (is_op("->")) fail("member access is outside the CUDA subset", peek().pos);
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

  CE literal(const CTok& t) {
    std::string s = t.t;
    bool uns = !s.empty() && s.back() == 'u';
    if (uns) s.pop_back();
    bool hex = s.size() > 2 && (s[1] == 'x' || s[1] == 'X');
    uint64_t v = hex ? std::strtoull(s.c_str() + 2, nullptr, 16) : std::strtoull(s.c_str(), nullptr, 10);
    if (v > 0xffffffffull || (hex && s.size() - 2 > 8)) fail("integer literal wider than 32 bits", t.pos);
    if (!uns && !hex && v > 2147483647ull) fail("integer literal out of int32 range (long in C)", t.pos);
    char ty = (uns || v > 2147483647ull) ? 'u' : 'i';
    if (v > 2147483647ull || hex) {
      char buf[16];
      std::snprintf(buf, sizeof(buf), "0x%08llx", static_cast<unsigned long long>(v));
      return CE{buf, ty};
    }
    return CE{s, ty};
  }

  CE primary() {
    CTok t = next();
    if (t.k == CTok::Int) return literal(t);
    if (t.k == CTok::Flt) return CE{t.t, 'f'};
    if (t.k != CTok::Id) fail("expected an expression, found '" + t.t + "'", t.pos);
    static const std::set<std::string> builtins = {"threadIdx", "blockIdx", "blockDim", "gridDim"};
    if (builtins.count(t.t)) {
      want_op(".");
      CTok f = want_id();
      if (f.t != "x" && f.t != "y" && f.t != "z") fail("unknown builtin component '" + f.t + "'", f.pos);
      return CE{t.t + "." + f.t, 'i'};
    }
    if (t.t == "warpSize") return CE{"32", 'i'};
    if (is_op("(")) {
      if (t.t == "atomicAdd")
        fail("the result of atomicAdd cannot be used in the CUDA subset (use it as a statement)", t.pos);
      if (t.t == "fminf" || t.t == "fabsf" || t.t == "sqrtf" || t.t == "expf" || t.t == "atomicMin" ||
          t.t == "atomicMax" || t.t == "atomicCAS" || t.t == "atomicExch" || t.t == "__umulhi" ||
          (t.t.rfind("__shfl", 0) == 0 && t.t != "__shfl_xor_sync"))
        fail("'" + t.t + "' is outside the CUDA subset", t.pos);
      if (t.t == "__ldg") {  // __ldg(&a[i]) -> a[i] (read-only arrays are const __restrict__ already)
        want_op("(");
        want_op("&");
        auto [lv, lt] = lvalue();
        want_op(")");
        return CE{lv, lt};
      }
      std::vector<CE> a = call_args();
      auto arity = [&](size_t n) {
        if (a.size() != n) fail(t.t + " takes " + std::to_string(n) + " argument(s)", t.pos);
      };
      if (t.t == "__shfl_xor_sync") {
        arity(3);
        if (a[0].t != "0xffffffff" && a[0].t != "(-1)")
          fail("__shfl_xor_sync is supported with the full mask 0xffffffff only", t.pos);
        return CE{"warp_shfl_xor(" + a[1].t + ", " + a[2].t + ")", a[1].ty};
      }
      if (t.t == "__float2int_rz") {
        arity(1);
        return CE{"int_rz(" + a[0].t + ")", 'i'};
      }
      if (t.t == "__funnelshift_r" || t.t == "__funnelshift_l") {
        arity(3);
        return CE{std::string(t.t == "__funnelshift_r" ? "fshr(" : "fshl(") + a[0].t + ", " + a[1].t + ", " +
                      a[2].t + ")",
                  'u'};
      }
      if (t.t == "int" || t.t == "float") {
        arity(1);
        return conv(a[0], t.t == "float" ? 'f' : 'i', t.pos);
      }
      if (t.t == "min" || t.t == "max") {
        arity(2);
        if (a[0].ty == 'u' || a[1].ty == 'u') {
          if (a[0].ty == 'f' || a[1].ty == 'f') fail("mixing unsigned and float is outside the CUDA subset", t.pos);
          // unsigned min/max: a ^ ((a ^ b) & -(b <u a))  /  a ^ ((a ^ b) & -(a <u b))
          std::string sel = t.t == "min" ? "ltu(" + a[1].t + ", " + a[0].t + ")" : "ltu(" + a[0].t + ", " + a[1].t + ")";
          return CE{"(" + a[0].t + " ^ ((" + a[0].t + " ^ " + a[1].t + ") & (0 - " + sel + ")))", 'u'};
        }
        char ty = (a[0].ty == 'f' || a[1].ty == 'f') ? 'f' : 'i';
        return CE{t.t + "(" + a[0].t + ", " + a[1].t + ")", ty};
      }
      if (t.t == "fmaxf") {
        arity(2);
        return CE{"fmaxf(" + conv(a[0], 'f', t.pos).t + ", " + conv(a[1], 'f', t.pos).t + ")", 'f'};
      }
      std::string o = t.t + "(";
      for (size_t i = 0; i < a.size(); ++i) o += (i ? ", " : "") + a[i].t;
      auto f = funcs_.find(t.t);
      return CE{o + ")", f == funcs_.end() ? 'i' : f->second};
    }
    if (is_op("[")) {
      next();
      CE i = expr();
      want_op("]");
      auto it = arrs_.find(t.t);
      return CE{t.t + "[" + conv(i, 'i', t.pos).t + "]", it == arrs_.end() ? 'i' : it->second};
    }
    if (is_op(".")) {
      auto it = vecs_.find(t.t);
      if (it == vecs_.end()) fail("member access is outside the CUDA subset", peek().pos);
      next();
      CTok c = want_id();
      int k = component(c, it->second);
      return CE{t.t + "_" + comp_name(k), it->second.base};
    }
    if (vecs_.count(t.t)) fail("a whole vector cannot be used as a scalar", t.pos);
    auto it = vars_.find(t.t);
    return CE{t.t, it == vars_.end() ? 'i' : it->second};
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
