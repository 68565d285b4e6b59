// Semantic checks and lint for Mini-Kernel programs.
//
// Same rules and error codes as the reference validator
// (/root/reference/proj/src/validate.cpp:24-435): unique top-level names, recursion
// rejection, scoped name binding, int/float typing (mixed arithmetic promotes to float,
// float->int needs int()), label resolution, positive block dims within the 2048-thread
// SM budget; the lint flags forward gotos over declarations. MK+ statements and helpers
// are typed here as well.
#include <algorithm>
#include <map>
#include <set>

#include "ir.hpp"

namespace hf {
namespace {

constexpr int kMaxThreadsPerSm = 2048;

struct Sym {
  enum Kind { Local, ScalarParam, ArrayParam, SharedArray } kind;
  Ty ty;
  bool is_array() const { return kind == ArrayParam || kind == SharedArray; }
};

class Checker {
 public:
  explicit Checker(const Program& p) : p_(p) {}

  void run() {
    std::set<std::string> names;
    auto top = [&](const std::string& n, Pos pos) {
      if (!names.insert(n).second)
        raise(Code::DuplicateName, "top-level name '" + n + "' is not unique", pos);
    };
    for (const auto& f : p_.funcs) top(f.name, f.pos);
    for (const auto& k : p_.kernels) top(k.name, k.pos);
    recursion();
    for (const auto& f : p_.funcs) function(f);
    for (const auto& k : p_.kernels) kernel(k);
  }

 private:
  const Program& p_;
  std::vector<std::map<std::string, Sym>> scopes_;
  const Func* fn_ = nullptr;
  bool in_kernel_ = false;
  bool bcast_ok_ = false;  // the expression being typed is a whole assignment value

  static std::optional<int32_t> const_int(const Expr& e) {
    return eval_scalar_int(e, [](const std::string&) -> std::optional<int32_t> { return std::nullopt; });
  }

  static std::vector<std::string> callees(const Block& b) {
    std::vector<std::string> out;
    walk(b, [&](const Stmt& s) {
      if (s.k == SK::Call) out.push_back(s.name);
      exprs_of(s, [&](const Expr& e) {
        walk_expr(e, [&](const Expr& x) {
          if (x.k == EK::Call) out.push_back(x.s);
        });
      });
    });
    return out;
  }

  void recursion() {
    std::map<std::string, std::vector<std::string>> g;
    for (const auto& f : p_.funcs) g[f.name] = callees(f.body);
    std::map<std::string, int> state;
    std::vector<std::string> path;
    std::function<void(const std::string&)> dfs = [&](const std::string& n) {
      state[n] = 1;
      path.push_back(n);
      for (const auto& c : g[n]) {
        if (!p_.func(c)) continue;
        if (state[c] == 1) {
          std::string cyc;
          for (auto it = std::find(path.begin(), path.end(), c); it != path.end(); ++it)
            cyc += (cyc.empty() ? "" : ", ") + *it;
          raise(Code::Recursion, "recursive call cycle: [" + cyc + "]");
        }
        if (state[c] == 0) dfs(c);
      }
      path.pop_back();
      state[n] = 2;
    };
    for (const auto& f : p_.funcs)
      if (state[f.name] == 0) dfs(f.name);
  }

  void declare(const std::string& n, Sym s, Pos pos) {
    if (!scopes_.back().emplace(n, s).second)
      raise(Code::DuplicateName, "'" + n + "' is already declared in this scope", pos);
  }
  const Sym* lookup(const std::string& n) const {
    for (auto it = scopes_.rbegin(); it != scopes_.rend(); ++it) {
      auto f = it->find(n);
      if (f != it->end()) return &f->second;
    }
    return nullptr;
  }
  const Sym& need(const std::string& n, Pos pos) const {
    const Sym* s = lookup(n);
    if (!s) raise(Code::UnknownIdentifier, "unknown identifier '" + n + "'", pos);
    return *s;
  }

  void labels(const Block& b) {
    std::set<std::string> ls;
    walk(b, [&](const Stmt& s) {
      if (s.k == SK::Label && !ls.insert(s.name).second)
        raise(Code::DuplicateName, "duplicate label '" + s.name + "'", s.pos);
    });
    walk(b, [&](const Stmt& s) {
      if (s.k == SK::Goto && !ls.count(s.name))
        raise(Code::UnresolvedLabel, "goto targets unknown label '" + s.name + "'", s.pos);
    });
  }

  Ty type(const Expr& e) {
    switch (e.k) {
      case EK::Int: return Ty::Int;
      case EK::Float: return Ty::Float;
      case EK::Builtin: return Ty::Int;
      case EK::Var: {
        const Sym& s = need(e.s, e.pos);
        if (s.is_array())
          raise(Code::TypeMismatch, "array '" + e.s + "' used as a scalar", e.pos);
        return s.ty;
      }
      case EK::Unary: {
        Ty t = type(e.a[0]);
        if (Un(e.i) == Un::Not && t != Ty::Int)
          raise(Code::TypeMismatch, "'!' needs an int operand", e.pos);
        return t;
      }
      case EK::Binary: {
        Ty l = type(e.a[0]), r = type(e.a[1]);
        switch (Bin(e.i)) {
          case Bin::Add:
          case Bin::Sub:
          case Bin::Mul:
          case Bin::Div: return (l == Ty::Float || r == Ty::Float) ? Ty::Float : Ty::Int;
          case Bin::Mod:
          case Bin::Shl:
          case Bin::Shr:
          case Bin::And:
          case Bin::Xor:
          case Bin::Or:
          case Bin::LAnd:
          case Bin::LOr:
            if (l != Ty::Int || r != Ty::Int)
              raise(Code::TypeMismatch, "operator needs int operands", e.pos);
            return Ty::Int;
          default: return Ty::Int;
        }
      }
      case EK::Index: {
        const Sym& s = need(e.s, e.pos);
        if (!s.is_array()) raise(Code::TypeMismatch, "'" + e.s + "' is not an array", e.pos);
        if (type(e.a[0]) != Ty::Int)
          raise(Code::TypeMismatch, "array index must be int", e.a[0].pos);
        return s.ty;
      }
      case EK::Intrin: {
        switch (Intr(e.i)) {
          case Intr::CastInt: type(e.a[0]); return Ty::Int;
          case Intr::IntRz: type(e.a[0]); return Ty::Int;
          case Intr::Acquire:
          case Intr::Relaxed:
            if (e.a[0].k != EK::Index)
              raise(Code::TypeMismatch, std::string(intr_name(Intr(e.i))) + " takes an array element", e.a[0].pos);
            return type(e.a[0]);
          case Intr::CastFloat: type(e.a[0]); return Ty::Float;
          case Intr::Bcast: {
            if (!bcast_ok_)
              raise(Code::TypeMismatch, "warp_bcast must be the whole right-hand side of an assignment", e.pos);
            bcast_ok_ = false;
            auto w = const_int(e.a[2]);
            if (!w || *w < 2 || *w > 32 || (*w & (*w - 1)) != 0)
              raise(Code::TypeMismatch, "warp_bcast width must be a constant power of two in [2, 32]", e.a[2].pos);
            if (type(e.a[1]) != Ty::Int) raise(Code::TypeMismatch, "warp_bcast source lane must be int", e.a[1].pos);
            return type(e.a[0]);
          }
          case Intr::Fmaxf:
            type(e.a[0]);
            type(e.a[1]);
            return Ty::Float;
          case Intr::Min:
          case Intr::Max: {
            Ty a = type(e.a[0]), b = type(e.a[1]);
            return (a == Ty::Float || b == Ty::Float) ? Ty::Float : Ty::Int;
          }
          default:  // MK+ integer helpers
            for (const auto& x : e.a)
              if (type(x) != Ty::Int)
                raise(Code::TypeMismatch, std::string(intr_name(Intr(e.i))) + " needs int operands",
                      e.pos);
            return Ty::Int;
        }
      }
      case EK::Shfl: return type(e.a[0]);
      case EK::Call: {
        const Func* f = p_.func(e.s);
        if (!f) raise(Code::UnresolvedCall, "call to unknown function '" + e.s + "'", e.pos);
        call_args(*f, e.a, e.pos);
        if (!f->ret)
          raise(Code::TypeMismatch, "void function '" + e.s + "' used in an expression", e.pos);
        return *f->ret;
      }
    }
    return Ty::Int;
  }

  void call_args(const Func& f, const std::vector<Expr>& args, Pos pos) {
    if (args.size() != f.params.size())
      raise(Code::TypeMismatch,
            "'" + f.name + "' expects " + std::to_string(f.params.size()) + " arguments", pos);
    for (size_t i = 0; i < args.size(); ++i) {
      const Param& formal = f.params[i];
      if (formal.array) {
        const Sym* s = args[i].k == EK::Var ? lookup(args[i].s) : nullptr;
        if (!s || !s->is_array())
          raise(Code::TypeMismatch,
                "argument " + std::to_string(i + 1) + " of '" + f.name + "' must be an array name",
                args[i].pos);
        if (s->ty != formal.ty)
          raise(Code::TypeMismatch, "array element type mismatch in call to '" + f.name + "'",
                args[i].pos);
      } else if (type(args[i]) == Ty::Float && formal.ty == Ty::Int) {
        raise(Code::TypeMismatch,
              "cannot pass float where int is expected in call to '" + f.name + "'", args[i].pos);
      }
    }
  }

  static void assignable(Ty target, Ty value, Pos pos) {
    if (target == Ty::Int && value == Ty::Float)
      raise(Code::TypeMismatch, "cannot assign float to int without int() cast", pos);
  }

  // Type of an assignment target; `elem` reports whether it is an array element.
  Ty target(const Stmt& s, bool* elem = nullptr) {
    Pos pos = s.name_pos.valid() ? s.name_pos : s.pos;
    const Sym& sym = need(s.name, pos);
    if (elem) *elem = sym.is_array() && !s.idx.empty();
    if (sym.is_array()) {
      if (s.idx.empty()) raise(Code::TypeMismatch, "array '" + s.name + "' used as a scalar", pos);
      if (type(s.idx[0]) != Ty::Int)
        raise(Code::TypeMismatch, "array index must be int", s.idx[0].pos);
    } else if (!s.idx.empty()) {
      raise(Code::TypeMismatch, "'" + s.name + "' is not an array", pos);
    }
    return sym.ty;
  }

  void block(const Block& b) {
    scopes_.emplace_back();
    for (const auto& s : b) stmt(s);
    scopes_.pop_back();
  }

  void stmt(const Stmt& s) {
    switch (s.k) {
      case SK::Decl:
        if (!s.val.empty()) assignable(s.ty, type(s.val[0]), s.pos);
        declare(s.name, Sym{Sym::Local, s.ty}, s.pos);
        break;
      case SK::Assign: {
        Ty t = target(s);
        const Expr& v = s.val[0];
        bcast_ok_ = v.k == EK::Intrin && Intr(v.i) == Intr::Bcast && s.idx.empty();
        assignable(t, type(v), s.pos);
        bcast_ok_ = false;
        break;
      }
      case SK::If:
        if (type(s.val[0]) != Ty::Int)
          raise(Code::TypeMismatch, "condition must be int", s.val[0].pos);
        block(s.body);
        if (s.has_alt) block(s.alt);
        break;
      case SK::For:
        scopes_.emplace_back();
        stmt(s.init[0]);
        if (type(s.val[0]) != Ty::Int)
          raise(Code::TypeMismatch, "condition must be int", s.val[0].pos);
        stmt(s.step[0]);
        block(s.body);
        scopes_.pop_back();
        break;
      case SK::While:
        if (type(s.val[0]) != Ty::Int)
          raise(Code::TypeMismatch, "condition must be int", s.val[0].pos);
        block(s.body);
        break;
      case SK::Atomic: {
        bool elem = false;
        Ty t = target(s, &elem);
        if (!elem) raise(Code::TypeMismatch, "atomic_add target must be an array element", s.pos);
        assignable(t, type(s.val[0]), s.pos);
        break;
      }
      case SK::Return:
        if (in_kernel_) {
          if (!s.val.empty()) raise(Code::TypeMismatch, "kernels cannot return a value", s.pos);
        } else if (!fn_->ret) {
          if (!s.val.empty())
            raise(Code::TypeMismatch, "void function cannot return a value", s.pos);
        } else {
          if (s.val.empty())
            raise(Code::TypeMismatch, "function '" + fn_->name + "' must return a value", s.pos);
          assignable(*fn_->ret, type(s.val[0]), s.pos);
        }
        break;
      case SK::Call: {
        const Func* f = p_.func(s.name);
        if (!f) raise(Code::UnresolvedCall, "call to unknown function '" + s.name + "'", s.pos);
        call_args(*f, s.val, s.pos);
        break;
      }
      case SK::AsyncCopy: {
        Pos pos = s.name_pos.valid() ? s.name_pos : s.pos;
        const Sym& g = need(s.name, pos);
        const Sym& sh = need(s.outs[0], s.pos);
        if (g.kind != Sym::ArrayParam || sh.kind != Sym::SharedArray)
          raise(Code::TypeMismatch, "async_copy copies a global array into a shared array", s.pos);
        if (type(s.idx[0]) != Ty::Int || type(s.val[0]) != Ty::Int)
          raise(Code::TypeMismatch, "async_copy indices must be int", s.pos);
        if (g.ty != sh.ty) raise(Code::TypeMismatch, "async_copy arrays differ in element type", s.pos);
        break;
      }
      case SK::VLoad:
      case SK::VStore: {
        Pos pos = s.name_pos.valid() ? s.name_pos : s.pos;
        const Sym& arr = need(s.name, pos);
        if (!arr.is_array()) raise(Code::TypeMismatch, "'" + s.name + "' is not an array", pos);
        if (type(s.idx[0]) != Ty::Int)
          raise(Code::TypeMismatch, "vector index must be int", s.idx[0].pos);
        if (s.k == SK::VLoad) {
          for (const auto& d : s.outs) {
            const Sym& out = need(d, s.pos);
            if (out.is_array())
              raise(Code::TypeMismatch, "vload destination '" + d + "' must be a scalar", s.pos);
            assignable(out.ty, arr.ty, s.pos);
          }
        } else {
          for (const auto& v : s.val) assignable(arr.ty, type(v), s.pos);
        }
        break;
      }
      default:
        break;  // barriers, labels, gotos
    }
  }

  void declare_params(const std::vector<Param>& ps) {
    for (const auto& p : ps)
      declare(p.name, Sym{p.array ? Sym::ArrayParam : Sym::ScalarParam, p.ty}, p.pos);
  }

  void function(const Func& f) {
    fn_ = &f;
    in_kernel_ = false;
    scopes_.emplace_back();
    declare_params(f.params);
    labels(f.body);
    block(f.body);
    scopes_.pop_back();
    fn_ = nullptr;
  }

  void kernel(const Kernel& k) {
    if (k.dims.x <= 0 || k.dims.y <= 0 || k.dims.z <= 0)
      raise(Code::InvalidArgument, "block dimensions must be positive", k.pos);
    if (k.dims.count() > kMaxThreadsPerSm)
      raise(Code::ThreadBudgetExceeded,
            "block dimension product " + std::to_string(k.dims.count()) + " exceeds " +
                std::to_string(kMaxThreadsPerSm),
            k.pos);
    in_kernel_ = true;
    fn_ = nullptr;
    scopes_.emplace_back();
    declare_params(k.params);
    for (const auto& sh : k.shared) declare(sh.name, Sym{Sym::SharedArray, sh.ty}, sh.pos);
    labels(k.body);
    block(k.body);
    scopes_.pop_back();
    in_kernel_ = false;
  }
};

}  // namespace

void validate(const Program& p) { Checker(p).run(); }

std::vector<Lint> lint(const Program& p) {
  std::vector<Lint> out;
  auto body = [&](const Block& b, const std::string& owner) {
    std::vector<const Stmt*> order;
    walk(b, [&](const Stmt& s) { order.push_back(&s); });
    std::map<std::string, size_t> where;
    for (size_t i = 0; i < order.size(); ++i)
      if (order[i]->k == SK::Label) where[order[i]->name] = i;
    for (size_t i = 0; i < order.size(); ++i) {
      if (order[i]->k != SK::Goto) continue;
      auto it = where.find(order[i]->name);
      if (it == where.end() || it->second <= i) continue;
      for (size_t j = i + 1; j < it->second; ++j) {
        if (order[j]->k == SK::Decl) {
          out.push_back(Lint{order[i]->pos, "goto '" + order[i]->name + "' in " + owner +
                                                " jumps over a declaration (lift declarations first)"});
          break;
        }
      }
    }
  };
  for (const auto& f : p.funcs) body(f.body, "function '" + f.name + "'");
  for (const auto& k : p.kernels) body(k.body, "kernel '" + k.name + "'");
  return out;
}

}  // namespace hf
