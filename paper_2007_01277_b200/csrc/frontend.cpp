// Mini-Kernel lexer + recursive-descent parser.
//
// Grammar and error codes follow the reference (/root/reference/proj/README.md:113-127,
// lexer.cpp:114-249, parser.cpp:52-565). Dialect::Strict accepts exactly the reference
// language; Dialect::B200 (default) adds the MK+ extensions the B200 member kernels use:
//   hex literals (0x..., wrapping to int32), `unroll [N] for (...)`,
//   vload(arr, i, d0..dn-1) / vstore(arr, i, e0..en-1) with n in {2, 4},
//   shr_u / rotr / rotl / ltu integer helpers, fence() (device-scope memory fence for
//   inter-block hand-offs; reads of global arrays the kernel writes go through L2),
//   warp_sync() (__syncwarp for intra-warp shared-memory exchanges; warp-uniform use only),
//   int_rz(x) (int(x) where the program guarantees |x| < 2^31: a single cvt.rzi.s32).
// Each extension has an exact plain-MK expansion (downlower.cpp).
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <sstream>

#include "ir.hpp"

namespace hf {
namespace {

enum class T : uint8_t {
  End, Ident, IntLit, FloatLit, Ann,
  Kernel, Dims, Fixed, Int, Float, Void, Shared, If, Else, For, While, Syncthreads, BarSync,
  AtomicAdd, Goto, Return,
  LParen, RParen, LBrace, RBrace, LBracket, RBracket, Comma, Semi, Colon, Dot, Assign,
  Plus, Minus, Star, Slash, Percent, Shl, Shr, Amp, Caret, Pipe, Lt, Le, Gt, Ge, EqEq, Ne,
  AndAnd, OrOr, Bang,
};

const char* tname(T t) {
  switch (t) {
    case T::End: return "end of input";
    case T::Ident: return "identifier";
    case T::IntLit: return "integer literal";
    case T::FloatLit: return "float literal";
    case T::Ann: return "annotation";
    case T::Kernel: return "'kernel'";
    case T::Dims: return "'dims'";
    case T::Fixed: return "'fixed'";
    case T::Int: return "'int'";
    case T::Float: return "'float'";
    case T::Void: return "'void'";
    case T::Shared: return "'shared'";
    case T::If: return "'if'";
    case T::Else: return "'else'";
    case T::For: return "'for'";
    case T::While: return "'while'";
    case T::Syncthreads: return "'syncthreads'";
    case T::BarSync: return "'bar_sync'";
    case T::AtomicAdd: return "'atomic_add'";
    case T::Goto: return "'goto'";
    case T::Return: return "'return'";
    case T::LParen: return "'('";
    case T::RParen: return "')'";
    case T::LBrace: return "'{'";
    case T::RBrace: return "'}'";
    case T::LBracket: return "'['";
    case T::RBracket: return "']'";
    case T::Comma: return "','";
    case T::Semi: return "';'";
    case T::Colon: return "':'";
    case T::Dot: return "'.'";
    case T::Assign: return "'='";
    case T::Plus: return "'+'";
    case T::Minus: return "'-'";
    case T::Star: return "'*'";
    case T::Slash: return "'/'";
    case T::Percent: return "'%'";
    case T::Shl: return "'<<'";
    case T::Shr: return "'>>'";
    case T::Amp: return "'&'";
    case T::Caret: return "'^'";
    case T::Pipe: return "'|'";
    case T::Lt: return "'<'";
    case T::Le: return "'<='";
    case T::Gt: return "'>'";
    case T::Ge: return "'>='";
    case T::EqEq: return "'=='";
    case T::Ne: return "'!='";
    case T::AndAnd: return "'&&'";
    case T::OrOr: return "'||'";
    case T::Bang: return "'!'";
  }
  return "?";
}

struct Tok {
  T k = T::End;
  std::string text;
  int32_t iv = 0;
  float fv = 0.0f;
  Pos pos;
};

T keyword(const std::string& w) {
  static const std::pair<const char*, T> table[] = {
      {"kernel", T::Kernel}, {"dims", T::Dims},     {"fixed", T::Fixed},
      {"int", T::Int},       {"float", T::Float},   {"void", T::Void},
      {"shared", T::Shared}, {"if", T::If},         {"else", T::Else},
      {"for", T::For},       {"while", T::While},   {"syncthreads", T::Syncthreads},
      {"bar_sync", T::BarSync}, {"atomic_add", T::AtomicAdd}, {"goto", T::Goto},
      {"return", T::Return}};
  for (const auto& [s, t] : table)
    if (w == s) return t;
  return T::Ident;
}

std::vector<Tok> lex(const std::string& src, Dialect dialect) {
  std::vector<Tok> out;
  size_t i = 0;
  int line = 1, col = 1;
  auto peek = [&](size_t o = 0) { return i + o < src.size() ? src[i + o] : '\0'; };
  auto adv = [&]() {
    char c = src[i++];
    if (c == '\n') {
      ++line;
      col = 1;
    } else {
      ++col;
    }
    return c;
  };
  auto isdig = [](char c) { return std::isdigit(static_cast<unsigned char>(c)) != 0; };
  while (i < src.size()) {
    char c = peek();
    if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
      adv();
      continue;
    }
    Pos p{line, col};
    if (c == '/' && peek(1) == '/') {
      adv();
      adv();
      bool ann = peek() == '@';
      if (ann) adv();
      std::string body;
      while (i < src.size() && peek() != '\n') body.push_back(adv());
      if (ann) out.push_back(Tok{T::Ann, body, 0, 0.0f, p});
      continue;
    }
    if (c == '/' && peek(1) == '*') {
      adv();
      adv();
      while (i < src.size() && !(peek() == '*' && peek(1) == '/')) adv();
      if (i >= src.size()) raise(Code::Syntax, "unterminated block comment", p);
      adv();
      adv();
      continue;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      std::string w;
      while (i < src.size() &&
             (std::isalnum(static_cast<unsigned char>(peek())) || peek() == '_'))
        w.push_back(adv());
      T k = keyword(w);
      out.push_back(Tok{k, k == T::Ident ? w : std::string(), 0, 0.0f, p});
      continue;
    }
    if (isdig(c)) {
      if (dialect == Dialect::B200 && c == '0' && (peek(1) == 'x' || peek(1) == 'X') &&
          std::isxdigit(static_cast<unsigned char>(peek(2)))) {
        adv();
        adv();
        std::string hex;
        while (i < src.size() && std::isxdigit(static_cast<unsigned char>(peek())))
          hex.push_back(adv());
        if (hex.size() > 8) raise(Code::Syntax, "hex literal wider than 32 bits", p);
        uint32_t v = uint32_t(std::strtoul(hex.c_str(), nullptr, 16));
        out.push_back(Tok{T::IntLit, {}, int32_t(v), 0.0f, p});
        continue;
      }
      std::string digits;
      while (i < src.size() && isdig(peek())) digits.push_back(adv());
      bool is_float = false;
      if (peek() == '.' && isdig(peek(1))) {
        is_float = true;
        digits.push_back(adv());
        while (i < src.size() && isdig(peek())) digits.push_back(adv());
      }
      if ((peek() == 'e' || peek() == 'E') &&
          (isdig(peek(1)) || ((peek(1) == '+' || peek(1) == '-') && isdig(peek(2))))) {
        is_float = true;
        digits.push_back(adv());
        if (peek() == '+' || peek() == '-') digits.push_back(adv());
        while (i < src.size() && isdig(peek())) digits.push_back(adv());
      }
      Tok t;
      t.pos = p;
      if (is_float) {
        t.k = T::FloatLit;
        t.fv = std::strtof(digits.c_str(), nullptr);
        if (!std::isfinite(t.fv)) raise(Code::Syntax, "float literal out of float32 range", p);
      } else {
        t.k = T::IntLit;
        long long v = std::strtoll(digits.c_str(), nullptr, 10);
        if (v > 2147483647LL) raise(Code::Syntax, "integer literal out of int32 range", p);
        t.iv = int32_t(v);
      }
      out.push_back(std::move(t));
      continue;
    }
    adv();
    auto one = [&](T k) { out.push_back(Tok{k, {}, 0, 0.0f, p}); };
    auto two = [&](char second, T pair, T single) {
      if (peek() == second) {
        adv();
        one(pair);
      } else {
        one(single);
      }
    };
    switch (c) {
      case '(': one(T::LParen); break;
      case ')': one(T::RParen); break;
      case '{': one(T::LBrace); break;
      case '}': one(T::RBrace); break;
      case '[': one(T::LBracket); break;
      case ']': one(T::RBracket); break;
      case ',': one(T::Comma); break;
      case ';': one(T::Semi); break;
      case ':': one(T::Colon); break;
      case '.': one(T::Dot); break;
      case '+': one(T::Plus); break;
      case '-': one(T::Minus); break;
      case '*': one(T::Star); break;
      case '/': one(T::Slash); break;
      case '%': one(T::Percent); break;
      case '^': one(T::Caret); break;
      case '=': two('=', T::EqEq, T::Assign); break;
      case '!': two('=', T::Ne, T::Bang); break;
      case '&': two('&', T::AndAnd, T::Amp); break;
      case '|': two('|', T::OrOr, T::Pipe); break;
      case '<':
        if (peek() == '<') {
          adv();
          one(T::Shl);
        } else {
          two('=', T::Le, T::Lt);
        }
        break;
      case '>':
        if (peek() == '>') {
          adv();
          one(T::Shr);
        } else {
          two('=', T::Ge, T::Gt);
        }
        break;
      default:
        raise(Code::Syntax, std::string("unexpected character '") + c + "'", p);
    }
  }
  out.push_back(Tok{T::End, {}, 0, 0.0f, Pos{line, col}});
  return out;
}

// Constant folding used only for shuffle lane masks (parser.cpp:14-48 semantics:
// int32 wrap, masked shift counts, arithmetic >>).
std::optional<int32_t> fold(const Expr& e) {
  if (e.k == EK::Int) return e.i;
  if (e.k == EK::Unary) {
    if (Un(e.i) != Un::Neg) return std::nullopt;
    if (auto v = fold(e.a[0])) return int32_t(uint32_t(0) - uint32_t(*v));
    return std::nullopt;
  }
  if (e.k != EK::Binary) return std::nullopt;
  auto l = fold(e.a[0]);
  auto r = fold(e.a[1]);
  if (!l || !r) return std::nullopt;
  uint32_t a = uint32_t(*l), b = uint32_t(*r);
  switch (Bin(e.i)) {
    case Bin::Add: return int32_t(a + b);
    case Bin::Sub: return int32_t(a - b);
    case Bin::Mul: return int32_t(a * b);
    case Bin::Div:
      if (*r == 0) return std::nullopt;
      return int32_t(uint32_t(int64_t(*l) / *r));
    case Bin::Mod:
      if (*r == 0) return std::nullopt;
      return int32_t(uint32_t(int64_t(*l) % *r));
    case Bin::Shl: return int32_t(a << (b & 31));
    case Bin::Shr: return *l >> (b & 31);
    case Bin::And: return int32_t(a & b);
    case Bin::Xor: return int32_t(a ^ b);
    case Bin::Or: return int32_t(a | b);
    default: return std::nullopt;
  }
}

class Parser {
 public:
  Parser(const std::string& src, Dialect d) : toks_(lex(src, d)), dialect_(d) {}

  Program run() {
    Program prog;
    std::vector<Tok> anns;
    while (!at(T::End)) {
      if (at(T::Ann)) {
        anns.push_back(next());
        continue;
      }
      if (at(T::Kernel)) {
        prog.kernels.push_back(kernel(anns));
        anns.clear();
      } else if (at(T::Int) || at(T::Float) || at(T::Void)) {
        if (!anns.empty())
          raise(Code::Syntax, "annotation must precede a kernel definition", anns.front().pos);
        prog.funcs.push_back(function());
      } else {
        expected("'kernel' or a function definition");
      }
    }
    if (!anns.empty())
      raise(Code::Syntax, "annotation is not followed by a kernel definition", anns.front().pos);
    return prog;
  }

 private:
  std::vector<Tok> toks_;
  size_t at_ = 0;
  Dialect dialect_;

  bool b200() const { return dialect_ == Dialect::B200; }
  const Tok& peek(size_t o = 0) const {
    size_t i = at_ + o;
    return i < toks_.size() ? toks_[i] : toks_.back();
  }
  bool at(T k, size_t o = 0) const { return peek(o).k == k; }
  bool at_ident(const char* w, size_t o = 0) const {
    return peek(o).k == T::Ident && peek(o).text == w;
  }
  Tok next() { return toks_[at_ < toks_.size() - 1 ? at_++ : at_]; }
  [[noreturn]] void expected(const std::string& what) const {
    raise(Code::Syntax, "expected " + what + ", found " + tname(peek().k), peek().pos);
  }
  Tok want(T k) {
    if (!at(k)) expected(tname(k));
    return next();
  }
  int want_int() { return want(T::IntLit).iv; }

  void annotations(const std::vector<Tok>& anns, Kernel& k) {
    for (const auto& a : anns) {
      size_t b = a.text.find_first_not_of(" \t");
      if (b200() && b != std::string::npos && a.text.compare(b, 8, "requires") == 0 &&
          (b + 8 == a.text.size() || std::isspace(static_cast<unsigned char>(a.text[b + 8])))) {
        // MK+ `//@ requires EXPR`: a launch precondition over scalar int parameters
        Parser sub(a.text.substr(b + 8), dialect_);
        Expr e = sub.expr();
        if (!sub.at(T::End)) raise(Code::Syntax, "trailing text after the requires expression", a.pos);
        std::string bad;
        walk_expr(e, [&](const Expr& x) {
          if (x.k == EK::Var) {
            bool ok = false;
            for (const auto& p : k.params) ok |= p.name == x.s && !p.array && p.ty == Ty::Int;
            if (!ok && bad.empty()) bad = "'" + x.s + "' is not a scalar int parameter";
          } else if (x.k != EK::Int && x.k != EK::Unary && x.k != EK::Binary &&
                     !(x.k == EK::Intrin && (Intr(x.i) == Intr::Min || Intr(x.i) == Intr::Max))) {
            if (bad.empty()) bad = "only scalar int arithmetic is allowed";
          }
        });
        if (!bad.empty()) raise(Code::TypeMismatch, "requires: " + bad, a.pos);
        k.reqs.push_back(std::move(e));
        continue;
      }
      std::istringstream in(a.text);
      std::string item;
      while (in >> item) {
        auto eq = item.find('=');
        if (eq == std::string::npos)
          raise(Code::Syntax, "annotation entry '" + item + "' is not key=value", a.pos);
        std::string key = item.substr(0, eq), value = item.substr(eq + 1);
        char* end = nullptr;
        long v = std::strtol(value.c_str(), &end, 10);
        if (end == value.c_str() || *end != '\0' || v <= 0)
          raise(Code::Syntax, "annotation '" + key + "' needs a positive integer", a.pos);
        if (key == "grid") k.grid = int(v);
        else if (key == "regs") k.regs = int(v);
        else if (key == "regcap") k.regcap = int(v);
        else raise(Code::Syntax, "unknown annotation key '" + key + "'", a.pos);
      }
    }
  }

  std::vector<Param> params() {
    std::vector<Param> ps;
    want(T::LParen);
    if (!at(T::RParen)) {
      while (true) {
        if (!at(T::Int) && !at(T::Float)) expected("parameter type");
        Ty t = at(T::Int) ? Ty::Int : Ty::Float;
        next();
        Tok n = want(T::Ident);
        bool arr = false;
        if (at(T::LBracket)) {
          next();
          want(T::RBracket);
          arr = true;
        }
        ps.push_back(Param{n.text, t, arr, n.pos});
        if (at(T::Comma)) {
          next();
          continue;
        }
        break;
      }
    }
    want(T::RParen);
    return ps;
  }

  Kernel kernel(const std::vector<Tok>& anns) {
    Kernel k;
    k.pos = want(T::Kernel).pos;
    k.name = want(T::Ident).text;
    k.params = params();
    want(T::Dims);
    want(T::LParen);
    k.dims.x = want_int();
    want(T::Comma);
    k.dims.y = want_int();
    want(T::Comma);
    k.dims.z = want_int();
    want(T::RParen);
    if (at(T::Fixed)) {
      next();
      k.tunable = false;
    }
    annotations(anns, k);
    k.body = block(&k.shared);
    return k;
  }

  Func function() {
    Func f;
    Tok t = next();
    f.pos = t.pos;
    if (t.k == T::Int) f.ret = Ty::Int;
    else if (t.k == T::Float) f.ret = Ty::Float;
    f.name = want(T::Ident).text;
    f.params = params();
    f.body = block(nullptr);
    return f;
  }

  Block block(std::vector<SharedArr>* shared_sink) {
    want(T::LBrace);
    Block b;
    while (!at(T::RBrace)) {
      if (at(T::End)) expected("'}'");
      if (at(T::Shared)) {
        Pos p = next().pos;
        if (!shared_sink)
          raise(Code::Syntax, "shared declarations are only allowed at kernel top level", p);
        SharedArr sh;
        sh.pos = p;
        if (!at(T::Int) && !at(T::Float)) expected("'int' or 'float'");
        sh.ty = at(T::Int) ? Ty::Int : Ty::Float;
        next();
        sh.name = want(T::Ident).text;
        want(T::LBracket);
        sh.len = want_int();
        want(T::RBracket);
        want(T::Semi);
        if (sh.len <= 0) raise(Code::Syntax, "shared array length must be positive", p);
        shared_sink->push_back(std::move(sh));
        continue;
      }
      b.push_back(stmt());
    }
    want(T::RBrace);
    return b;
  }

  Stmt for_loop(Pos p, int unroll) {
    want(T::For);
    want(T::LParen);
    Stmt s;
    s.k = SK::For;
    s.pos = p;
    s.unroll = unroll;
    s.init.push_back(simple());
    want(T::Semi);
    s.val.push_back(expr());
    want(T::Semi);
    s.step.push_back(simple());
    want(T::RParen);
    s.body = block(nullptr);
    return s;
  }

  Stmt stmt() {
    Pos p = peek().pos;
    Stmt s;
    s.pos = p;
    switch (peek().k) {
      case T::Int:
      case T::Float: {
        Stmt d = declaration();
        want(T::Semi);
        return d;
      }
      case T::If: {
        next();
        want(T::LParen);
        s.k = SK::If;
        s.val.push_back(expr());
        want(T::RParen);
        s.body = block(nullptr);
        if (at(T::Else)) {
          next();
          s.alt = block(nullptr);
          s.has_alt = true;
        }
        return s;
      }
      case T::For:
        return for_loop(p, 0);
      case T::While:
        next();
        want(T::LParen);
        s.k = SK::While;
        s.val.push_back(expr());
        want(T::RParen);
        s.body = block(nullptr);
        return s;
      case T::Syncthreads:
        next();
        want(T::LParen);
        want(T::RParen);
        want(T::Semi);
        s.k = SK::Sync;
        return s;
      case T::BarSync: {
        next();
        want(T::LParen);
        s.k = SK::BarSync;
        s.bid = want_int();
        want(T::Comma);
        s.bcount = want_int();
        want(T::RParen);
        want(T::Semi);
        if (s.bid < 0 || s.bid > 15) raise(Code::BadBarrierId, "barrier id must be in [0, 15]", p);
        if (s.bcount <= 0 || s.bcount % 32 != 0)
          raise(Code::MisalignedCount, "barrier count must be a positive multiple of 32", p);
        return s;
      }
      case T::AtomicAdd:
        next();
        want(T::LParen);
        s.k = SK::Atomic;
        lvalue(s);
        want(T::Comma);
        s.val.push_back(expr());
        want(T::RParen);
        want(T::Semi);
        return s;
      case T::Goto:
        next();
        s.k = SK::Goto;
        s.name = want(T::Ident).text;
        want(T::Semi);
        return s;
      case T::Return:
        next();
        s.k = SK::Return;
        if (!at(T::Semi)) s.val.push_back(expr());
        want(T::Semi);
        return s;
      case T::Ident: {
        if (b200()) {
          if (at_ident("unroll") && (at(T::For, 1) || (at(T::IntLit, 1) && at(T::For, 2)))) {
            next();
            int n = -1;
            if (at(T::IntLit)) {
              n = want_int();
              if (n <= 0) raise(Code::Syntax, "unroll factor must be positive", p);
            }
            return for_loop(p, n);
          }
          if ((at_ident("vload") || at_ident("vstore") || at_ident("vstore_cs")) && at(T::LParen, 1))
            return vector_access(p);
          if (at_ident("atomic_add_release") && at(T::LParen, 1)) {
            // release-ordered atomic add: earlier writes of this thread are visible to whoever
            // observes the update (load_acquire) -- the inter-block hand-off without fence()
            next();
            want(T::LParen);
            s.k = SK::Atomic;
            s.bid = 1;
            lvalue(s);
            want(T::Comma);
            s.val.push_back(expr());
            want(T::RParen);
            want(T::Semi);
            return s;
          }
          if (at_ident("async_copy") && at(T::LParen, 1)) {
            // async_copy(sarr, j, garr, i): 16-byte asynchronous global -> shared copy
            next();
            want(T::LParen);
            s.k = SK::AsyncCopy;
            Tok sa = want(T::Ident);
            s.outs.push_back(sa.text);
            want(T::Comma);
            s.val.push_back(expr());
            want(T::Comma);
            Tok ga = want(T::Ident);
            s.name = ga.text;
            s.name_pos = ga.pos;
            want(T::Comma);
            s.idx.push_back(expr());
            want(T::RParen);
            want(T::Semi);
            return s;
          }
          if ((at_ident("fence") || at_ident("warp_sync") || at_ident("async_wait")) && at(T::LParen, 1) &&
              at(T::RParen, 2)) {
            const std::string w = next().text;
            s.k = w == "fence" ? SK::Fence : w == "warp_sync" ? SK::WarpSync : SK::AsyncWait;
            next();
            next();
            want(T::Semi);
            return s;
          }
        }
        if (at(T::Colon, 1)) {
          s.k = SK::Label;
          s.name = next().text;
          next();
          return s;
        }
        if (at(T::LParen, 1)) {
          s.k = SK::Call;
          s.name = next().text;
          s.val = args();
          want(T::Semi);
          return s;
        }
        Stmt a = assignment();
        want(T::Semi);
        return a;
      }
      default:
        expected("a statement");
    }
  }

  // vload(arr, i, d0, .., dn-1) / vstore(arr, i, e0, .., en-1), n in {2, 4};
  // vstore_cs: the same store marked streaming (L2 evict-first on sm_100a: an output no later
  // access of the kernel reads); the interpreter and the lowering treat it as vstore
  Stmt vector_access(Pos p) {
    Stmt s;
    s.pos = p;
    const std::string op = next().text;
    bool load = op == "vload";
    s.k = load ? SK::VLoad : SK::VStore;
    s.bid = op == "vstore_cs" ? 1 : 0;
    want(T::LParen);
    Tok arr = want(T::Ident);
    s.name = arr.text;
    s.name_pos = arr.pos;
    want(T::Comma);
    s.idx.push_back(expr());
    while (at(T::Comma)) {
      next();
      if (load) s.outs.push_back(want(T::Ident).text);
      else s.val.push_back(expr());
    }
    want(T::RParen);
    want(T::Semi);
    size_t n = load ? s.outs.size() : s.val.size();
    if (n != 2 && n != 4)
      raise(Code::Syntax, std::string(load ? "vload" : "vstore") + " moves 2 or 4 elements", p);
    return s;
  }

  Stmt simple() {
    if (at(T::Int) || at(T::Float)) return declaration();
    if (at(T::Ident) && at(T::LParen, 1)) {
      Stmt s;
      s.pos = peek().pos;
      s.k = SK::Call;
      s.name = next().text;
      s.val = args();
      return s;
    }
    return assignment();
  }

  Stmt declaration() {
    Stmt s;
    s.pos = peek().pos;
    s.k = SK::Decl;
    s.ty = at(T::Int) ? Ty::Int : Ty::Float;
    next();
    Tok n = want(T::Ident);
    s.name = n.text;
    s.name_pos = n.pos;
    if (at(T::Assign)) {
      next();
      s.val.push_back(expr());
    }
    return s;
  }

  Stmt assignment() {
    Stmt s;
    s.pos = peek().pos;
    s.k = SK::Assign;
    lvalue(s);
    want(T::Assign);
    s.val.push_back(expr());
    return s;
  }

  void lvalue(Stmt& s) {
    Tok n = want(T::Ident);
    s.name = n.text;
    s.name_pos = n.pos;
    if (at(T::LBracket)) {
      next();
      s.idx.push_back(expr());
      want(T::RBracket);
    }
  }

  std::vector<Expr> args() {
    want(T::LParen);
    std::vector<Expr> v;
    if (!at(T::RParen)) {
      while (true) {
        v.push_back(expr());
        if (at(T::Comma)) {
          next();
          continue;
        }
        break;
      }
    }
    want(T::RParen);
    return v;
  }

  static int prec(T t) {
    switch (t) {
      case T::OrOr: return 1;
      case T::AndAnd: return 2;
      case T::Pipe: return 3;
      case T::Caret: return 4;
      case T::Amp: return 5;
      case T::EqEq:
      case T::Ne: return 6;
      case T::Lt:
      case T::Le:
      case T::Gt:
      case T::Ge: return 7;
      case T::Shl:
      case T::Shr: return 8;
      case T::Plus:
      case T::Minus: return 9;
      case T::Star:
      case T::Slash:
      case T::Percent: return 10;
      default: return -1;
    }
  }

  static Bin binop(T t) {
    switch (t) {
      case T::OrOr: return Bin::LOr;
      case T::AndAnd: return Bin::LAnd;
      case T::Pipe: return Bin::Or;
      case T::Caret: return Bin::Xor;
      case T::Amp: return Bin::And;
      case T::EqEq: return Bin::Eq;
      case T::Ne: return Bin::Ne;
      case T::Lt: return Bin::Lt;
      case T::Le: return Bin::Le;
      case T::Gt: return Bin::Gt;
      case T::Ge: return Bin::Ge;
      case T::Shl: return Bin::Shl;
      case T::Shr: return Bin::Shr;
      case T::Plus: return Bin::Add;
      case T::Minus: return Bin::Sub;
      case T::Star: return Bin::Mul;
      case T::Slash: return Bin::Div;
      default: return Bin::Mod;
    }
  }

  Expr expr() { return binary_from(1); }

  Expr binary_from(int min_prec) {
    Expr lhs = unary_expr();
    while (true) {
      int p = prec(peek().k);
      if (p < min_prec) return lhs;
      Tok op = next();
      Expr rhs = binary_from(p + 1);
      Expr e = binary(binop(op.k), std::move(lhs), std::move(rhs));
      e.pos = op.pos;
      lhs = std::move(e);
    }
  }

  Expr unary_expr() {
    if (at(T::Minus) || at(T::Bang)) {
      Tok t = next();
      Expr e = unary(t.k == T::Minus ? Un::Neg : Un::Not, unary_expr());
      e.pos = t.pos;
      return e;
    }
    return primary();
  }

  static std::optional<Builtin> member(const std::string& base, const std::string& m) {
    int axis = m == "x" ? 0 : m == "y" ? 1 : m == "z" ? 2 : -1;
    if (axis < 0) return std::nullopt;
    if (base == "threadIdx") return Builtin(int(Builtin::TidX) + axis);
    if (base == "blockIdx") return Builtin(int(Builtin::BidX) + axis);
    if (base == "blockDim") return Builtin(int(Builtin::BdimX) + axis);
    if (base == "gridDim" && axis == 0) return Builtin::GdimX;
    return std::nullopt;
  }

  Expr primary() {
    Pos p = peek().pos;
    Expr e;
    switch (peek().k) {
      case T::IntLit:
        e = lit(next().iv);
        e.pos = p;
        return e;
      case T::FloatLit:
        e = flit(next().fv);
        e.pos = p;
        return e;
      case T::LParen: {
        next();
        Expr inner = expr();
        want(T::RParen);
        return inner;
      }
      case T::Int:
      case T::Float: {
        Intr w = at(T::Int) ? Intr::CastInt : Intr::CastFloat;
        next();
        std::vector<Expr> a = args();
        if (a.size() != 1) raise(Code::Syntax, "cast takes exactly one argument", p);
        e = intrin(w, std::move(a));
        e.pos = p;
        return e;
      }
      case T::Ident: {
        Tok n = next();
        if (at(T::Dot)) {
          next();
          Tok m = want(T::Ident);
          auto b = member(n.text, m.text);
          if (!b) raise(Code::Syntax, "unknown builtin '" + n.text + "." + m.text + "'", p);
          e = builtin(*b);
          e.pos = p;
          return e;
        }
        if (at(T::LParen)) {
          if (n.text == "warp_shfl_xor") {
            std::vector<Expr> a = args();
            if (a.size() != 2) raise(Code::Syntax, "warp_shfl_xor takes (value, lane_mask)", p);
            auto mask = fold(a[1]);
            if (!mask || *mask < 1 || *mask > 31)
              raise(Code::TypeMismatch,
                    "warp_shfl_xor lane_mask must be a compile-time constant in [1, 31]", p);
            e.k = EK::Shfl;
            e.i = *mask;
            e.a.push_back(std::move(a[0]));
            e.pos = p;
            return e;
          }
          std::optional<Intr> w;
          if (n.text == "min") w = Intr::Min;
          else if (n.text == "max") w = Intr::Max;
          else if (n.text == "fmaxf") w = Intr::Fmaxf;
          else if (b200() && n.text == "shr_u") w = Intr::ShrU;
          else if (b200() && n.text == "rotr") w = Intr::Rotr;
          else if (b200() && n.text == "rotl") w = Intr::Rotl;
          else if (b200() && n.text == "ltu") w = Intr::LtU;
          else if (b200() && n.text == "fshr") w = Intr::Fshr;
          else if (b200() && n.text == "fshl") w = Intr::Fshl;
          else if (b200() && n.text == "int_rz") w = Intr::IntRz;
          else if (b200() && n.text == "load_acquire") w = Intr::Acquire;
          else if (b200() && n.text == "load_relaxed") w = Intr::Relaxed;
          else if (b200() && n.text == "warp_bcast") w = Intr::Bcast;
          else if (b200() && n.text == "addc") w = Intr::Addc;
          else if (b200() && n.text == "remu") w = Intr::RemU;
          else if (b200() && n.text == "mulhi_u") w = Intr::MulHiU;
          else if (b200() && n.text == "fma_add") w = Intr::FmaAdd;
          if (w) {
            std::vector<Expr> a = args();
            if (int(a.size()) != intr_arity(*w))
              raise(Code::Syntax, n.text + " takes exactly " +
                                      std::string(intr_arity(*w) == 4 ? "four" : intr_arity(*w) == 3 ? "three"
                                                  : intr_arity(*w) == 1 ? "one" : "two") +
                                      " argument(s)", p);
            e = intrin(*w, std::move(a));
            e.pos = p;
            return e;
          }
          e.k = EK::Call;
          e.s = n.text;
          e.a = args();
          e.pos = p;
          return e;
        }
        if (at(T::LBracket)) {
          next();
          Expr i = expr();
          want(T::RBracket);
          e = index(n.text, std::move(i));
          e.pos = p;
          return e;
        }
        e = var(n.text);
        e.pos = p;
        return e;
      }
      default:
        expected("an expression");
    }
  }
};

}  // namespace

Program parse_unchecked(const std::string& src, Dialect d) {
  if (d == Dialect::B200 && looks_like_cuda(src)) return Parser(cuda_to_mk(src), d).run();
  return Parser(src, d).run();
}

Program parse(const std::string& src, Dialect d) {
  Program p = parse_unchecked(src, d);
  validate(p);
  return p;
}

}  // namespace hf
