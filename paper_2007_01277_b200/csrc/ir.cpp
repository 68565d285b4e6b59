#include "ir.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>

namespace hf {

const char* code_name(Code c) {
  static const char* names[] = {
      "Syntax", "UnknownIdentifier", "TypeMismatch", "DuplicateName", "UnresolvedCall",
      "UnresolvedLabel", "Recursion", "BadBarrierId", "MisalignedCount", "DimensionMismatch",
      "GridMismatch", "ThreadBudgetExceeded", "SharedMemoryOverflow", "DoesNotFit",
      "OutOfBounds", "DivideByZero", "BarrierDeadlock", "BarrierOverflow", "DivergentBarrier",
      "NothingFeasible", "IncompatibleFixedDims", "InvalidArgument", "Io", "Compile", "Device"};
  int i = int(c);
  if (i < 0 || i >= int(sizeof(names) / sizeof(names[0]))) return "Unknown";
  return names[i];
}

Error::Error(Code c, std::string m, Pos p) : code(c), msg(std::move(m)), pos(p) {
  text_ = std::string("[") + code_name(c) + "] ";
  if (pos.valid()) text_ += std::to_string(pos.line) + ":" + std::to_string(pos.col) + ": ";
  text_ += msg;
}

void raise(Code c, std::string msg, Pos p) { throw Error(c, std::move(msg), p); }

const char* intr_name(Intr i) {
  switch (i) {
    case Intr::Min: return "min";
    case Intr::Max: return "max";
    case Intr::Fmaxf: return "fmaxf";
    case Intr::CastInt: return "int";
    case Intr::CastFloat: return "float";
    case Intr::ShrU: return "shr_u";
    case Intr::Rotr: return "rotr";
    case Intr::Rotl: return "rotl";
    case Intr::LtU: return "ltu";
    case Intr::Fshr: return "fshr";
    case Intr::Fshl: return "fshl";
    case Intr::IntRz: return "int_rz";
    case Intr::Acquire: return "load_acquire";
    case Intr::Relaxed: return "load_relaxed";
    case Intr::Bcast: return "warp_bcast";
    case Intr::Addc: return "addc";
    case Intr::RemU: return "remu";
    case Intr::MulHiU: return "mulhi_u";
    case Intr::FmaAdd: return "fma_add";
  }
  return "?";
}

int intr_arity(Intr i) {
  if (i == Intr::CastInt || i == Intr::CastFloat || i == Intr::IntRz || i == Intr::Acquire ||
      i == Intr::Relaxed)
    return 1;
  if (i == Intr::Fshr || i == Intr::Fshl || i == Intr::Bcast) return 3;
  if (i == Intr::Addc) return 4;
  return 2;
}

bool intr_is_extension(Intr i) { return int(i) >= int(Intr::ShrU); }

const Func* Program::func(const std::string& n) const {
  for (const auto& f : funcs)
    if (f.name == n) return &f;
  return nullptr;
}

const Kernel* Program::kernel(const std::string& n) const {
  for (const auto& k : kernels)
    if (k.name == n) return &k;
  return nullptr;
}

// ---- builders -----------------------------------------------------------------

Expr lit(int32_t v) {
  Expr e;
  e.k = EK::Int;
  e.i = v;
  return e;
}
Expr flit(float v) {
  Expr e;
  e.k = EK::Float;
  e.f = v;
  return e;
}
Expr var(std::string n) {
  Expr e;
  e.k = EK::Var;
  e.s = std::move(n);
  return e;
}
Expr builtin(Builtin b) {
  Expr e;
  e.k = EK::Builtin;
  e.i = int(b);
  return e;
}
Expr unary(Un op, Expr x) {
  Expr e;
  e.k = EK::Unary;
  e.i = int(op);
  e.a.push_back(std::move(x));
  return e;
}
Expr binary(Bin op, Expr l, Expr r) {
  Expr e;
  e.k = EK::Binary;
  e.i = int(op);
  e.a.push_back(std::move(l));
  e.a.push_back(std::move(r));
  return e;
}
Expr index(std::string arr, Expr i) {
  Expr e;
  e.k = EK::Index;
  e.s = std::move(arr);
  e.a.push_back(std::move(i));
  return e;
}
Expr intrin(Intr w, std::vector<Expr> args) {
  Expr e;
  e.k = EK::Intrin;
  e.i = int(w);
  e.a = std::move(args);
  return e;
}
Stmt decl(Ty t, std::string n) {
  Stmt s;
  s.k = SK::Decl;
  s.ty = t;
  s.name = std::move(n);
  return s;
}
Stmt decl_init(Ty t, std::string n, Expr init) {
  Stmt s = decl(t, std::move(n));
  s.val.push_back(std::move(init));
  return s;
}
Stmt assign(std::string n, Expr v) {
  Stmt s;
  s.k = SK::Assign;
  s.name = std::move(n);
  s.val.push_back(std::move(v));
  return s;
}
Stmt assign_at(std::string arr, Expr i, Expr v) {
  Stmt s = assign(std::move(arr), std::move(v));
  s.idx.push_back(std::move(i));
  return s;
}
Stmt if_(Expr c, Block then_b) {
  Stmt s;
  s.k = SK::If;
  s.val.push_back(std::move(c));
  s.body = std::move(then_b);
  return s;
}
Stmt if_else(Expr c, Block then_b, Block else_b) {
  Stmt s = if_(std::move(c), std::move(then_b));
  s.alt = std::move(else_b);
  s.has_alt = true;
  return s;
}

// ---- walkers --------------------------------------------------------------------

namespace {
template <typename B, typename F>
void walk_block(B& b, const F& fn) {
  for (auto& s : b) {
    fn(s);
    switch (s.k) {
      case SK::If:
        walk_block(s.body, fn);
        if (s.has_alt) walk_block(s.alt, fn);
        break;
      case SK::For:
        fn(s.init[0]);
        fn(s.step[0]);
        walk_block(s.body, fn);
        break;
      case SK::While:
        walk_block(s.body, fn);
        break;
      default:
        break;
    }
  }
}

// Expressions a statement evaluates itself, in reference order (ast.cpp visit order:
// target index first, then value).
template <typename S, typename F>
void stmt_exprs(S& s, const F& fn) {
  switch (s.k) {
    case SK::For:
    case SK::While:
    case SK::If:
      fn(s.val[0]);
      break;
    default:
      for (auto& e : s.idx) fn(e);
      for (auto& e : s.val) fn(e);
      break;
  }
}

template <typename E, typename F>
void expr_tree(E& e, const F& fn) {
  fn(e);
  for (auto& c : e.a) expr_tree(c, fn);
}
}  // namespace

void walk(const Block& b, const std::function<void(const Stmt&)>& fn) { walk_block(b, fn); }
void walk(Block& b, const std::function<void(Stmt&)>& fn) { walk_block(b, fn); }
void exprs_of(const Stmt& s, const std::function<void(const Expr&)>& fn) { stmt_exprs(s, fn); }
void exprs_of(Stmt& s, const std::function<void(Expr&)>& fn) { stmt_exprs(s, fn); }
void walk_expr(const Expr& e, const std::function<void(const Expr&)>& fn) { expr_tree(e, fn); }
void walk_expr(Expr& e, const std::function<void(Expr&)>& fn) { expr_tree(e, fn); }

// ---- structural equality (positions ignored; float literals bitwise) ----------

bool same(const Expr& a, const Expr& b) {
  if (a.k != b.k || a.i != b.i || a.s != b.s || a.a.size() != b.a.size()) return false;
  if (a.k == EK::Float && std::memcmp(&a.f, &b.f, sizeof(float)) != 0) return false;
  for (size_t i = 0; i < a.a.size(); ++i)
    if (!same(a.a[i], b.a[i])) return false;
  return true;
}

namespace {
bool same_exprs(const std::vector<Expr>& a, const std::vector<Expr>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (!same(a[i], b[i])) return false;
  return true;
}
bool same_stmt(const Stmt& a, const Stmt& b) {
  if (a.k != b.k || a.name != b.name || a.outs != b.outs || a.has_alt != b.has_alt) return false;
  if (a.k == SK::Decl && a.ty != b.ty) return false;
  if (a.k == SK::BarSync && (a.bid != b.bid || a.bcount != b.bcount)) return false;
  if ((a.k == SK::Atomic || a.k == SK::VStore) && a.bid != b.bid) return false;
  if (a.k == SK::For && a.unroll != b.unroll) return false;
  return same_exprs(a.idx, b.idx) && same_exprs(a.val, b.val) && same(a.body, b.body) &&
         same(a.alt, b.alt) && same(a.init, b.init) && same(a.step, b.step);
}
}  // namespace

bool same(const Block& a, const Block& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i)
    if (!same_stmt(a[i], b[i])) return false;
  return true;
}

bool same(const Kernel& a, const Kernel& b) {
  if (a.name != b.name || !(a.dims == b.dims) || a.tunable != b.tunable || a.grid != b.grid ||
      a.regs != b.regs || a.params.size() != b.params.size() ||
      a.shared.size() != b.shared.size())
    return false;
  for (size_t i = 0; i < a.params.size(); ++i)
    if (a.params[i].name != b.params[i].name || a.params[i].ty != b.params[i].ty ||
        a.params[i].array != b.params[i].array)
      return false;
  for (size_t i = 0; i < a.shared.size(); ++i)
    if (a.shared[i].name != b.shared[i].name || a.shared[i].ty != b.shared[i].ty ||
        a.shared[i].len != b.shared[i].len)
      return false;
  return same(a.body, b.body);
}

bool has_calls(const Block& b) {
  bool found = false;
  walk(b, [&](const Stmt& s) {
    if (s.k == SK::Call) found = true;
    exprs_of(s, [&](const Expr& e) {
      walk_expr(e, [&](const Expr& x) {
        if (x.k == EK::Call) found = true;
      });
    });
  });
  return found;
}

bool uses_extensions(const Kernel& k) {
  bool ext = false;
  walk(k.body, [&](const Stmt& s) {
    if (s.k == SK::VLoad || s.k == SK::VStore || s.k == SK::Fence || s.k == SK::WarpSync ||
        s.k == SK::AsyncCopy || s.k == SK::AsyncWait ||
        (s.k == SK::For && s.unroll != 0))
      ext = true;
    exprs_of(s, [&](const Expr& e) {
      walk_expr(e, [&](const Expr& x) {
        if (x.k == EK::Intrin && intr_is_extension(Intr(x.i))) ext = true;
      });
    });
  });
  return ext;
}

// ---- Mini-Kernel printer (byte-compatible with the reference's emit.cpp) --------

std::string float_text(float v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.9g", double(v));
  std::string s(buf);
  if (s.find('.') == std::string::npos && s.find('e') == std::string::npos &&
      s.find("inf") == std::string::npos && s.find("nan") == std::string::npos)
    s += ".0";
  return s;
}

namespace {

const char* bin_text(Bin op) {
  static const char* t[] = {"+", "-", "*", "/", "%", "<<", ">>", "&", "^", "|",
                            "<", "<=", ">", ">=", "==", "!=", "&&", "||"};
  return t[int(op)];
}

int bin_prec(Bin op) {
  switch (op) {
    case Bin::LOr: return 1;
    case Bin::LAnd: return 2;
    case Bin::Or: return 3;
    case Bin::Xor: return 4;
    case Bin::And: return 5;
    case Bin::Eq:
    case Bin::Ne: return 6;
    case Bin::Lt:
    case Bin::Le:
    case Bin::Gt:
    case Bin::Ge: return 7;
    case Bin::Shl:
    case Bin::Shr: return 8;
    case Bin::Add:
    case Bin::Sub: return 9;
    default: return 10;
  }
}

const char* builtin_text(int b) {
  static const char* t[] = {"threadIdx.x", "threadIdx.y", "threadIdx.z", "blockIdx.x",
                            "blockIdx.y",  "blockIdx.z",  "blockDim.x",  "blockDim.y",
                            "blockDim.z",  "gridDim.x"};
  return t[b];
}

struct MkPrinter {
  std::string o;

  void pad(int n) { o.append(size_t(n) * 2, ' '); }

  void expr(const Expr& e, int parent = 0) {
    switch (e.k) {
      case EK::Int:
        // INT_MIN has no literal form in the grammar (lexer.cpp:186-192).
        if (e.i == INT32_MIN) o += "(-2147483647 - 1)";
        else o += std::to_string(e.i);
        break;
      case EK::Float: o += float_text(e.f); break;
      case EK::Var: o += e.s; break;
      case EK::Builtin: o += builtin_text(e.i); break;
      case EK::Unary: {
        bool paren = 11 < parent;
        if (paren) o += '(';
        o += Un(e.i) == Un::Neg ? '-' : '!';
        expr(e.a[0], 11);
        if (paren) o += ')';
        break;
      }
      case EK::Binary: {
        int p = bin_prec(Bin(e.i));
        bool paren = p < parent;
        if (paren) o += '(';
        expr(e.a[0], p);
        o += ' ';
        o += bin_text(Bin(e.i));
        o += ' ';
        expr(e.a[1], p + 1);
        if (paren) o += ')';
        break;
      }
      case EK::Index:
        o += e.s;
        o += '[';
        expr(e.a[0]);
        o += ']';
        break;
      case EK::Intrin:
        o += intr_name(Intr(e.i));
        args(e.a);
        break;
      case EK::Shfl:
        o += "warp_shfl_xor(";
        expr(e.a[0]);
        o += ", " + std::to_string(e.i) + ")";
        break;
      case EK::Call:
        o += e.s;
        args(e.a);
        break;
    }
  }

  void args(const std::vector<Expr>& v) {
    o += '(';
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) o += ", ";
      expr(v[i]);
    }
    o += ')';
  }

  void lvalue(const Stmt& s) {
    o += s.name;
    if (!s.idx.empty()) {
      o += '[';
      expr(s.idx[0]);
      o += ']';
    }
  }

  void simple(const Stmt& s) {
    if (s.k == SK::Decl) {
      o += std::string(ty_name(s.ty)) + " " + s.name;
      if (!s.val.empty()) {
        o += " = ";
        expr(s.val[0]);
      }
    } else if (s.k == SK::Assign) {
      lvalue(s);
      o += " = ";
      expr(s.val[0]);
    } else if (s.k == SK::Call) {
      o += s.name;
      args(s.val);
    } else {
      raise(Code::InvalidArgument, "loop header holds a non-simple statement", s.pos);
    }
  }

  void block(const Block& b, int ind) {
    o += "{\n";
    for (const auto& s : b) stmt(s, ind + 1);
    pad(ind);
    o += "}";
  }

  void stmt(const Stmt& s, int ind) {
    switch (s.k) {
      case SK::Decl:
      case SK::Assign:
        pad(ind);
        simple(s);
        o += ";\n";
        break;
      case SK::If:
        pad(ind);
        o += "if (";
        expr(s.val[0]);
        o += ") ";
        block(s.body, ind);
        if (s.has_alt) {
          o += " else ";
          block(s.alt, ind);
        }
        o += '\n';
        break;
      case SK::For:
        pad(ind);
        if (s.unroll == -1) o += "unroll ";
        else if (s.unroll > 0) o += "unroll " + std::to_string(s.unroll) + " ";
        o += "for (";
        simple(s.init[0]);
        o += "; ";
        expr(s.val[0]);
        o += "; ";
        simple(s.step[0]);
        o += ") ";
        block(s.body, ind);
        o += '\n';
        break;
      case SK::While:
        pad(ind);
        o += "while (";
        expr(s.val[0]);
        o += ") ";
        block(s.body, ind);
        o += '\n';
        break;
      case SK::Sync:
        pad(ind);
        o += "syncthreads();\n";
        break;
      case SK::Fence:
        pad(ind);
        o += "fence();\n";
        break;
      case SK::WarpSync:
        pad(ind);
        o += "warp_sync();\n";
        break;
      case SK::AsyncWait:
        pad(ind);
        o += "async_wait();\n";
        break;
      case SK::AsyncCopy:
        pad(ind);
        o += "async_copy(" + s.outs[0] + ", ";
        expr(s.val[0]);
        o += ", " + s.name + ", ";
        expr(s.idx[0]);
        o += ");\n";
        break;
      case SK::BarSync:
        pad(ind);
        o += "bar_sync(" + std::to_string(s.bid) + ", " + std::to_string(s.bcount) + ");\n";
        break;
      case SK::Atomic:
        pad(ind);
        o += s.bid == 1 ? "atomic_add_release(" : "atomic_add(";
        lvalue(s);
        o += ", ";
        expr(s.val[0]);
        o += ");\n";
        break;
      case SK::Return:
        pad(ind);
        o += "return";
        if (!s.val.empty()) {
          o += ' ';
          expr(s.val[0]);
        }
        o += ";\n";
        break;
      case SK::Call:
        pad(ind);
        o += s.name;
        args(s.val);
        o += ";\n";
        break;
      case SK::Label:
        pad(ind);
        o += s.name + ":\n";
        break;
      case SK::Goto:
        pad(ind);
        o += "goto " + s.name + ";\n";
        break;
      case SK::VLoad:
        pad(ind);
        o += "vload(" + s.name + ", ";
        expr(s.idx[0]);
        for (const auto& d : s.outs) o += ", " + d;
        o += ");\n";
        break;
      case SK::VStore:
        pad(ind);
        o += std::string(s.bid == 1 ? "vstore_cs(" : "vstore(") + s.name + ", ";
        expr(s.idx[0]);
        for (const auto& v : s.val) {
          o += ", ";
          expr(v);
        }
        o += ");\n";
        break;
    }
  }

  void params(const std::vector<Param>& ps) {
    for (size_t i = 0; i < ps.size(); ++i) {
      if (i) o += ", ";
      o += std::string(ty_name(ps[i].ty)) + " " + ps[i].name;
      if (ps[i].array) o += "[]";
    }
  }

  void kernel(const Kernel& k) {
    std::string ann;
    if (k.grid != 1) ann += " grid=" + std::to_string(k.grid);
    if (k.regs) ann += " regs=" + std::to_string(*k.regs);
    if (k.regcap) ann += " regcap=" + std::to_string(*k.regcap);
    if (!ann.empty()) o += "//@" + ann + "\n";
    for (const auto& r : k.reqs) {
      o += "//@ requires ";
      expr(r);
      o += "\n";
    }
    o += "kernel " + k.name + "(";
    params(k.params);
    o += ") dims (" + std::to_string(k.dims.x) + ", " + std::to_string(k.dims.y) + ", " +
         std::to_string(k.dims.z) + ")";
    if (!k.tunable) o += " fixed";
    o += " {\n";
    for (const auto& sh : k.shared) {
      pad(1);
      o += std::string("shared ") + ty_name(sh.ty) + " " + sh.name + "[" +
           std::to_string(sh.len) + "];\n";
    }
    for (const auto& s : k.body) stmt(s, 1);
    o += "}\n";
  }

  void func(const Func& f) {
    o += f.ret ? ty_name(*f.ret) : "void";
    o += " " + f.name + "(";
    params(f.params);
    o += ") ";
    block(f.body, 0);
    o += '\n';
  }
};

}  // namespace

std::string print_expr(const Expr& e) {
  MkPrinter p;
  p.expr(e);
  return p.o;
}

std::string print_mk(const Kernel& k) {
  MkPrinter p;
  p.kernel(k);
  return p.o;
}

std::string print_mk(const Program& prog) {
  std::string out;
  bool first = true;
  for (const auto& f : prog.funcs) {
    if (!first) out += '\n';
    first = false;
    MkPrinter p;
    p.func(f);
    out += p.o;
  }
  for (const auto& k : prog.kernels) {
    if (!first) out += '\n';
    first = false;
    out += print_mk(k);
  }
  return out;
}

std::optional<int32_t> eval_scalar_int(const Expr& e,
                                       const std::function<std::optional<int32_t>(const std::string&)>& value) {
  auto w = [](int64_t v) { return int32_t(uint32_t(uint64_t(v))); };
  switch (e.k) {
    case EK::Int: return e.i;
    case EK::Var: return value(e.s);
    case EK::Unary: {
      auto a = eval_scalar_int(e.a[0], value);
      if (!a) return std::nullopt;
      if (Un(e.i) == Un::Not) return *a == 0 ? 1 : 0;
      return w(-int64_t(*a));
    }
    case EK::Binary: {
      auto a = eval_scalar_int(e.a[0], value), b = eval_scalar_int(e.a[1], value);
      if (!a || !b) return std::nullopt;
      int64_t x = *a, y = *b;
      switch (Bin(e.i)) {
        case Bin::Add: return w(x + y);
        case Bin::Sub: return w(x - y);
        case Bin::Mul: return w(x * y);
        case Bin::Div: return y == 0 ? std::nullopt : std::optional<int32_t>(y == -1 ? w(-x) : int32_t(x / y));
        case Bin::Mod: return y == 0 ? std::nullopt : std::optional<int32_t>(y == -1 ? 0 : int32_t(x % y));
        case Bin::Shl: return w(int64_t(uint32_t(*a) << (y & 31)));
        case Bin::Shr: return int32_t(*a >> (y & 31));
        case Bin::And: return *a & *b;
        case Bin::Or: return *a | *b;
        case Bin::Xor: return *a ^ *b;
        case Bin::Lt: return x < y;
        case Bin::Le: return x <= y;
        case Bin::Gt: return x > y;
        case Bin::Ge: return x >= y;
        case Bin::Eq: return x == y;
        case Bin::Ne: return x != y;
        case Bin::LAnd: return (x != 0) && (y != 0);
        case Bin::LOr: return (x != 0) || (y != 0);
      }
      return std::nullopt;
    }
    case EK::Intrin: {
      Intr i = Intr(e.i);
      if (i != Intr::Min && i != Intr::Max) return std::nullopt;
      auto a = eval_scalar_int(e.a[0], value), b = eval_scalar_int(e.a[1], value);
      if (!a || !b) return std::nullopt;
      return i == Intr::Min ? std::min(*a, *b) : std::max(*a, *b);
    }
    default: return std::nullopt;
  }
}

}  // namespace hf
