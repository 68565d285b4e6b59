// Normalization passes: inline_calls, lift_declarations, rename_locals.
//
// Behaviour (including every generated name: `__inlN` suffixes, `__retN`, `__endN`,
// `__cond__inlN`, `__forinitN`, `__hN`, `_2`/`_3` de-duplication and the `k1_`/`k2_`
// prefixes) reproduces the reference passes (/root/reference/proj/src/passes.cpp:15-711)
// so fused sources are byte-identical to mkfuse's. MK+ vector statements are carried
// through every pass as ordinary reads/writes of their operands.
#include <algorithm>
#include <functional>
#include <map>
#include <set>

#include "ir.hpp"

namespace hf {
namespace {

using NameFn = std::function<std::string(const std::string&)>;

// Scope-aware identifier rewriting (declarations, free names, labels).
struct Scoped {
  NameFn on_decl, on_free, on_label;
  std::vector<std::map<std::string, std::string>> scopes;

  std::string resolve(const std::string& n) {
    for (auto it = scopes.rbegin(); it != scopes.rend(); ++it) {
      auto f = it->find(n);
      if (f != it->end()) return f->second;
    }
    return on_free ? on_free(n) : n;
  }

  void expr(Expr& e) {
    if (e.k == EK::Var || e.k == EK::Index) e.s = resolve(e.s);
    for (auto& c : e.a) expr(c);
  }

  void stmt(Stmt& s) {
    switch (s.k) {
      case SK::Decl: {
        for (auto& v : s.val) expr(v);  // the initializer sees the outer binding
        std::string fresh = on_decl ? on_decl(s.name) : s.name;
        scopes.back()[s.name] = fresh;
        s.name = fresh;
        break;
      }
      case SK::Assign:
      case SK::Atomic:
      case SK::VStore:
        s.name = resolve(s.name);
        for (auto& e : s.idx) expr(e);
        for (auto& e : s.val) expr(e);
        break;
      case SK::VLoad:
        s.name = resolve(s.name);
        expr(s.idx[0]);
        for (auto& d : s.outs) d = resolve(d);
        break;
      case SK::AsyncCopy:
        s.name = resolve(s.name);
        s.outs[0] = resolve(s.outs[0]);
        expr(s.idx[0]);
        expr(s.val[0]);
        break;
      case SK::If:
        expr(s.val[0]);
        block(s.body);
        if (s.has_alt) block(s.alt);
        break;
      case SK::For:
        scopes.emplace_back();
        stmt(s.init[0]);
        expr(s.val[0]);
        stmt(s.step[0]);
        block(s.body);
        scopes.pop_back();
        break;
      case SK::While:
        expr(s.val[0]);
        block(s.body);
        break;
      case SK::Return:
      case SK::Call:
        for (auto& e : s.val) expr(e);
        break;
      case SK::Label:
      case SK::Goto:
        if (on_label) s.name = on_label(s.name);
        break;
      default:
        break;
    }
  }

  void block(Block& b) {
    scopes.emplace_back();
    for (auto& s : b) stmt(s);
    scopes.pop_back();
  }
};

bool expr_has_call(const Expr& e) {
  bool found = false;
  walk_expr(e, [&](const Expr& x) {
    if (x.k == EK::Call) found = true;
  });
  return found;
}

std::vector<std::string> callees_of(const Block& b) {
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

// ---------------------------------------------------------------------------
// inline_calls
// ---------------------------------------------------------------------------

class Inliner {
 public:
  explicit Inliner(const std::vector<Func>& funcs) {
    for (const auto& f : funcs) fns_[f.name] = &f;
    reject_cycles(funcs);
  }

  Block block(const Block& b) {
    Block out;
    for (const auto& s : b) stmt(s, out);
    return out;
  }

 private:
  std::map<std::string, const Func*> fns_;
  int counter_ = 0;

  void reject_cycles(const std::vector<Func>& funcs) {
    std::map<std::string, std::vector<std::string>> g;
    for (const auto& f : funcs) g[f.name] = callees_of(f.body);
    std::map<std::string, int> st;
    std::vector<std::string> path;
    std::function<void(const std::string&)> dfs = [&](const std::string& n) {
      st[n] = 1;
      path.push_back(n);
      for (const auto& c : g[n]) {
        if (!fns_.count(c)) continue;
        if (st[c] == 1) {
          std::string cyc;
          for (auto it = std::find(path.begin(), path.end(), c); it != path.end(); ++it)
            cyc += (cyc.empty() ? "" : ", ") + *it;
          raise(Code::Recursion, "recursive call cycle: [" + cyc + "]");
        }
        if (st[c] == 0) dfs(c);
      }
      path.pop_back();
      st[n] = 2;
    };
    for (const auto& f : funcs)
      if (st[f.name] == 0) dfs(f.name);
  }

  const Func& fn(const std::string& n, Pos p) {
    auto it = fns_.find(n);
    if (it == fns_.end()) raise(Code::UnresolvedCall, "call to unknown function '" + n + "'", p);
    return *it->second;
  }

  // Replaces every call inside `e` (innermost first) by a result temp; the
  // inlined statements go to `pre`.
  void extract(Expr& e, Block& pre) {
    if (e.k != EK::Call) {
      for (auto& c : e.a) extract(c, pre);
      return;
    }
    for (auto& a : e.a) extract(a, pre);
    const Func& f = fn(e.s, e.pos);
    if (!f.ret) raise(Code::TypeMismatch, "void function '" + e.s + "' in expression", e.pos);
    std::string temp = expand(f, e.a, pre, true);
    Pos p = e.pos;
    e = var(temp);
    e.pos = p;
  }

  std::string expand(const Func& f, const std::vector<Expr>& args, Block& out, bool want) {
    std::string sfx = "__inl" + std::to_string(counter_++);
    std::string result;
    if (want) {
      result = "__ret" + sfx;
      out.push_back(decl(*f.ret, result));
    }
    std::map<std::string, std::string> formals;
    for (size_t i = 0; i < f.params.size(); ++i) {
      const Param& p = f.params[i];
      if (p.array) {
        if (args[i].k != EK::Var)
          raise(Code::TypeMismatch, "array argument must be an array name", args[i].pos);
        formals[p.name] = args[i].s;
      } else {
        std::string t = p.name + sfx;
        out.push_back(decl_init(p.ty, t, args[i]));
        formals[p.name] = t;
      }
    }
    Block body = f.body;
    Scoped rw;
    rw.on_decl = [&](const std::string& n) { return n + sfx; };
    rw.on_label = [&](const std::string& n) { return n + sfx; };
    rw.on_free = [&](const std::string& n) {
      auto it = formals.find(n);
      return it != formals.end() ? it->second : n;
    };
    rw.block(body);

    size_t returns = 0;
    walk(body, [&](const Stmt& s) {
      if (s.k == SK::Return) ++returns;
    });
    bool trailing = returns == 1 && !body.empty() && body.back().k == SK::Return;
    std::string end = "__end" + sfx;
    Block rewritten = returns_to_jumps(body, result, trailing ? "" : end);
    if (returns > 0 && !trailing) {
      Stmt l;
      l.k = SK::Label;
      l.name = end;
      rewritten.push_back(l);
    }
    for (auto& s : block(rewritten)) out.push_back(std::move(s));
    return result;
  }

  static Block returns_to_jumps(const Block& b, const std::string& result, const std::string& end) {
    Block out;
    for (const auto& s : b) {
      if (s.k == SK::Return) {
        if (!s.val.empty() && !result.empty()) out.push_back(assign(result, s.val[0]));
        if (!end.empty()) {
          Stmt g;
          g.k = SK::Goto;
          g.pos = s.pos;
          g.name = end;
          out.push_back(g);
        }
        continue;
      }
      Stmt c = s;
      if (c.k == SK::If) {
        c.body = returns_to_jumps(c.body, result, end);
        if (c.has_alt) c.alt = returns_to_jumps(c.alt, result, end);
      } else if (c.k == SK::For || c.k == SK::While) {
        c.body = returns_to_jumps(c.body, result, end);
      }
      out.push_back(std::move(c));
    }
    return out;
  }

  void stmt(const Stmt& s, Block& out) {
    Stmt c = s;
    switch (c.k) {
      case SK::Decl:
      case SK::Return:
        for (auto& v : c.val) extract(v, out);
        out.push_back(std::move(c));
        break;
      case SK::Assign:
      case SK::Atomic:
      case SK::VLoad:
      case SK::VStore:
      case SK::AsyncCopy:
        for (auto& e : c.idx) extract(e, out);
        for (auto& e : c.val) extract(e, out);
        out.push_back(std::move(c));
        break;
      case SK::If:
        extract(c.val[0], out);  // evaluated once on entry
        c.body = block(c.body);
        if (c.has_alt) c.alt = block(c.alt);
        out.push_back(std::move(c));
        break;
      case SK::For:
        for_loop(c, out);
        break;
      case SK::While:
        while_loop(c, out);
        break;
      case SK::Call: {
        std::vector<Expr> args = c.val;
        for (auto& a : args) extract(a, out);
        const Func& f = fn(c.name, c.pos);
        expand(f, args, out, f.ret.has_value());
        break;
      }
      default:
        out.push_back(std::move(c));
        break;
    }
  }

  // Calls in a loop condition are re-evaluated each iteration: hoist once before the
  // loop into a temp and recompute it at the end of the body.
  void while_loop(Stmt& w, Block& out) {
    Block body = block(w.body);
    if (!expr_has_call(w.val[0])) {
      Stmt n;
      n.k = SK::While;
      n.pos = w.pos;
      n.val.push_back(w.val[0]);
      n.body = std::move(body);
      out.push_back(std::move(n));
      return;
    }
    std::string temp = "__cond__inl" + std::to_string(counter_++);
    Expr first = w.val[0], again = w.val[0];
    Block tail;
    extract(again, tail);
    tail.push_back(assign(temp, std::move(again)));
    extract(first, out);
    out.push_back(decl_init(Ty::Int, temp, std::move(first)));
    for (auto& s : tail) body.push_back(s);
    Stmt n;
    n.k = SK::While;
    n.pos = w.pos;
    n.val.push_back(var(temp));
    n.body = std::move(body);
    out.push_back(std::move(n));
  }

  void for_loop(Stmt& f, Block& out) {
    bool header_calls = expr_has_call(f.val[0]);
    exprs_of(f.step[0], [&](const Expr& e) { header_calls |= expr_has_call(e); });
    Block body = block(f.body);
    if (!header_calls) {
      Block init_out;
      stmt(f.init[0], init_out);  // the init runs once; hoisting its calls is safe
      Stmt residual;
      if (!init_out.empty() && (init_out.back().k == SK::Decl || init_out.back().k == SK::Assign)) {
        residual = std::move(init_out.back());
        init_out.pop_back();
      } else {
        residual = decl_init(Ty::Int, "__forinit" + std::to_string(counter_++), lit(0));
      }
      for (auto& s : init_out) out.push_back(std::move(s));
      Stmt n;
      n.k = SK::For;
      n.pos = f.pos;
      n.unroll = f.unroll;
      n.init.push_back(std::move(residual));
      n.val.push_back(f.val[0]);
      n.step.push_back(f.step[0]);
      n.body = std::move(body);
      out.push_back(std::move(n));
      return;
    }
    // init + while over a recomputed condition; a declaring init is renamed so the
    // enclosing scope stays clean.
    Stmt init = f.init[0];
    Expr cond = f.val[0];
    Stmt step = f.step[0];
    if (init.k == SK::Decl) {
      std::string fresh = init.name + "__h" + std::to_string(counter_++);
      std::map<std::string, std::string> remap{{init.name, fresh}};
      Scoped rw;
      rw.on_free = [&](const std::string& n) {
        auto it = remap.find(n);
        return it != remap.end() ? it->second : n;
      };
      rw.scopes.emplace_back();
      rw.expr(cond);
      rw.stmt(step);
      rw.block(body);
      rw.scopes.pop_back();
      init.name = fresh;
    }
    stmt(init, out);
    Block step_out;
    stmt(step, step_out);
    for (auto& s : step_out) body.push_back(std::move(s));
    Stmt w;
    w.k = SK::While;
    w.pos = f.pos;
    w.val.push_back(std::move(cond));
    w.body = std::move(body);
    while_loop(w, out);
  }
};

// ---------------------------------------------------------------------------
// lift_declarations
// ---------------------------------------------------------------------------

class Lifter {
 public:
  explicit Lifter(const Kernel& k) {
    for (const auto& p : k.params) used_.insert(p.name);
    for (const auto& sh : k.shared) used_.insert(sh.name);
  }

  Kernel run(const Kernel& k) {
    Kernel out = k;
    scopes_.emplace_back();
    Block body = block(k.body);
    scopes_.pop_back();
    Block lifted;
    for (const auto& [t, n] : lifted_) lifted.push_back(decl(t, n));
    for (auto& s : body) lifted.push_back(std::move(s));
    out.body = std::move(lifted);
    return out;
  }

 private:
  std::set<std::string> used_;
  std::vector<std::map<std::string, std::string>> scopes_;
  std::vector<std::pair<Ty, std::string>> lifted_;

  std::string unique(const std::string& base) {
    if (used_.insert(base).second) return base;
    for (int i = 2;; ++i) {
      std::string c = base + "_" + std::to_string(i);
      if (used_.insert(c).second) return c;
    }
  }

  std::string resolve(const std::string& n) {
    for (auto it = scopes_.rbegin(); it != scopes_.rend(); ++it) {
      auto f = it->find(n);
      if (f != it->end()) return f->second;
    }
    return n;
  }

  void expr(Expr& e) {
    if (e.k == EK::Call) raise(Code::InvalidArgument, "lift_declarations needs a call-free kernel");
    if (e.k == EK::Var || e.k == EK::Index) e.s = resolve(e.s);
    for (auto& c : e.a) expr(c);
  }

  std::string bind(const Stmt& d) {
    std::string fresh = unique(d.name);
    scopes_.back()[d.name] = fresh;
    lifted_.emplace_back(d.ty, fresh);
    return fresh;
  }

  // A for-header declaration always leaves an assignment behind (an uninitialized one
  // becomes `= 0`, matching zero-initialized locals).
  Stmt header_decl(Stmt& d) {
    Expr init = d.val.empty() ? (d.ty == Ty::Int ? lit(0) : flit(0.0f)) : d.val[0];
    if (!d.val.empty()) expr(init);
    std::string fresh = bind(d);
    return assign(fresh, std::move(init));
  }

  void simple(Stmt& s) {
    if (s.k == SK::Decl) {
      s = header_decl(s);
    } else if (s.k == SK::Assign) {
      s.name = resolve(s.name);
      for (auto& e : s.idx) expr(e);
      expr(s.val[0]);
    }
  }

  Block block(const Block& b) {
    scopes_.emplace_back();
    Block out;
    for (const auto& orig : b) {
      Stmt s = orig;
      switch (s.k) {
        case SK::Decl: {
          for (auto& v : s.val) expr(v);
          std::string fresh = bind(s);
          if (!s.val.empty()) out.push_back(assign(fresh, std::move(s.val[0])));
          break;
        }
        case SK::Assign:
        case SK::Atomic:
        case SK::VStore:
          s.name = resolve(s.name);
          for (auto& e : s.idx) expr(e);
          for (auto& e : s.val) expr(e);
          out.push_back(std::move(s));
          break;
        case SK::VLoad:
          s.name = resolve(s.name);
          expr(s.idx[0]);
          for (auto& d : s.outs) d = resolve(d);
          out.push_back(std::move(s));
          break;
        case SK::AsyncCopy:
          s.name = resolve(s.name);
          s.outs[0] = resolve(s.outs[0]);
          expr(s.idx[0]);
          expr(s.val[0]);
          out.push_back(std::move(s));
          break;
        case SK::If:
          expr(s.val[0]);
          s.body = block(s.body);
          if (s.has_alt) s.alt = block(s.alt);
          out.push_back(std::move(s));
          break;
        case SK::For:
          scopes_.emplace_back();
          simple(s.init[0]);
          expr(s.val[0]);
          simple(s.step[0]);
          s.body = block(s.body);
          scopes_.pop_back();
          out.push_back(std::move(s));
          break;
        case SK::While:
          expr(s.val[0]);
          s.body = block(s.body);
          out.push_back(std::move(s));
          break;
        case SK::Return:
          for (auto& v : s.val) expr(v);
          out.push_back(std::move(s));
          break;
        case SK::Call:
          raise(Code::InvalidArgument, "lift_declarations needs a call-free kernel", s.pos);
        default:
          out.push_back(std::move(s));
          break;
      }
    }
    scopes_.pop_back();
    return out;
  }
};

}  // namespace

Kernel inline_calls(const Kernel& k, const std::vector<Func>& funcs) {
  Inliner in(funcs);
  Kernel out = k;
  out.body = in.block(k.body);
  return out;
}

Kernel lift_declarations(const Kernel& k) {
  if (has_calls(k.body))
    raise(Code::InvalidArgument, "lift_declarations needs a call-free kernel", k.pos);
  return Lifter(k).run(k);
}

bool decl_prefix_form(const Kernel& k) {
  bool seen_other = false;
  for (const auto& s : k.body) {
    if (s.k == SK::Decl) {
      if (seen_other) return false;
    } else {
      seen_other = true;
    }
  }
  for (const auto& s : k.body) {
    if (s.k != SK::If && s.k != SK::For && s.k != SK::While) continue;
    Block probe{s};
    bool nested = false;
    walk(probe, [&](const Stmt& x) {
      if (&x != &probe[0] && x.k == SK::Decl) nested = true;
    });
    if (nested) return false;
  }
  return true;
}

std::pair<Kernel, std::vector<std::pair<std::string, std::string>>> rename_locals(
    const Kernel& k, const std::string& prefix) {
  Kernel out = k;
  std::vector<std::pair<std::string, std::string>> mapping;
  std::set<std::string> taken;
  for (const auto& p : k.params) taken.insert(p.name);
  auto prefixed = [&](const std::string& n) {
    std::string c = prefix + n;
    if (taken.insert(c).second) return c;
    for (int i = 2;; ++i) {
      std::string alt = c + "_" + std::to_string(i);
      if (taken.insert(alt).second) return alt;
    }
  };
  std::map<std::string, std::string> shared_map, label_map;
  for (auto& sh : out.shared) {
    std::string fresh = prefixed(sh.name);
    mapping.emplace_back(sh.name, fresh);
    shared_map[sh.name] = fresh;
    sh.name = fresh;
  }
  Scoped rw;
  rw.on_decl = [&](const std::string& n) {
    std::string fresh = prefixed(n);
    mapping.emplace_back(n, fresh);
    return fresh;
  };
  rw.on_free = [&](const std::string& n) {
    auto it = shared_map.find(n);
    return it != shared_map.end() ? it->second : n;
  };
  rw.on_label = [&](const std::string& n) {
    auto it = label_map.find(n);
    if (it != label_map.end()) return it->second;
    std::string fresh = prefix + n;
    label_map[n] = fresh;
    mapping.emplace_back(n, fresh);
    return fresh;
  };
  rw.block(out.body);
  return {std::move(out), std::move(mapping)};
}

Kernel normalize(const Kernel& k, const std::vector<Func>& funcs, const std::string& prefix) {
  return rename_locals(lift_declarations(inline_calls(k, funcs)), prefix).first;
}

// ---------------------------------------------------------------------------
// downlower: MK+ -> plain Mini-Kernel with identical semantics
// ---------------------------------------------------------------------------

namespace {

Expr int_min() { return binary(Bin::Sub, unary(Un::Neg, lit(2147483647)), lit(1)); }

std::optional<int32_t> const_of(const Expr& e) {
  if (e.k == EK::Int) return e.i;
  if (e.k == EK::Unary && Un(e.i) == Un::Neg && e.a[0].k == EK::Int)
    return int32_t(0u - uint32_t(e.a[0].i));
  return std::nullopt;
}

// Logical right shift by a count masked to [0, 31] (exec.cpp:515-516 semantics).
Expr shr_u(const Expr& x, const Expr& n) {
  if (auto c = const_of(n)) {
    int s = *c & 31;
    if (s == 0) return x;
    return binary(Bin::And, binary(Bin::Shr, x, lit(s)), lit(int32_t((1u << (32 - s)) - 1u)));
  }
  Expr cnt = binary(Bin::And, n, lit(31));
  Expr high = binary(Bin::Shl, binary(Bin::Shl, unary(Un::Neg, lit(1)), binary(Bin::Sub, lit(31), cnt)),
                     lit(1));
  return binary(Bin::And, binary(Bin::Shr, x, n), binary(Bin::Xor, high, unary(Un::Neg, lit(1))));
}

struct Lowerer {
  int counter = 0;
  std::map<std::string, Ty> arrays;   // params + shared
  std::map<std::string, Ty> scalars;  // params + declared locals (types of warp_bcast targets)

  Expr expr(const Expr& e) {
    Expr c = e;
    for (auto& x : c.a) x = expr(x);
    if (c.k != EK::Intrin || !intr_is_extension(Intr(c.i))) return c;
    const Expr& x = c.a[0];
    const Expr& n = c.a.size() > 1 ? c.a[1] : c.a[0];
    switch (Intr(c.i)) {
      case Intr::IntRz: return intrin(Intr::CastInt, {x});
      case Intr::Acquire:
      case Intr::Relaxed: return x;  // the interpreter is sequentially consistent
      case Intr::ShrU: return shr_u(x, n);
      case Intr::Rotr: {
        Expr left = binary(Bin::Shl, x, binary(Bin::Sub, lit(32), binary(Bin::And, n, lit(31))));
        if (auto k = const_of(n)) left = binary(Bin::Shl, x, lit((32 - (*k & 31)) & 31));
        return binary(Bin::Or, shr_u(x, n), left);
      }
      case Intr::Rotl: {
        Expr cnt = binary(Bin::And, n, lit(31));
        Expr back = binary(Bin::Sub, lit(32), cnt);
        if (auto k = const_of(n)) {
          cnt = lit(*k & 31);
          back = lit((32 - (*k & 31)) & 31);
        }
        return binary(Bin::Or, binary(Bin::Shl, x, cnt), shr_u(x, back));
      }
      case Intr::LtU:
        return binary(Bin::Lt, binary(Bin::Xor, x, int_min()), binary(Bin::Xor, n, int_min()));
      case Intr::RemU: {
        // a as uint32 = 2 * shr_u(a, 1) + (a & 1); both partial values stay below 2^31 for b < 2^30
        Expr half = binary(Bin::Mod, shr_u(x, lit(1)), n);
        return binary(Bin::Mod, binary(Bin::Add, binary(Bin::Mul, half, lit(2)), binary(Bin::And, x, lit(1))), n);
      }
      case Intr::MulHiU: {
        // 16-bit limbs: a = ah:al, b = bh:bl; every partial product and sum wraps mod 2^32 like
        // the interpreter's int arithmetic, and only the bits each term contributes are kept
        Expr al = binary(Bin::And, x, lit(0xffff)), ah = shr_u(x, lit(16));
        Expr bl = binary(Bin::And, n, lit(0xffff)), bh = shr_u(n, lit(16));
        Expr ll = binary(Bin::Mul, al, bl), lh = binary(Bin::Mul, al, bh);
        Expr hl = binary(Bin::Mul, ah, bl), hh = binary(Bin::Mul, ah, bh);
        Expr mid = binary(Bin::Add, binary(Bin::Add, shr_u(ll, lit(16)), binary(Bin::And, lh, lit(0xffff))),
                          binary(Bin::And, hl, lit(0xffff)));
        return binary(Bin::Add, binary(Bin::Add, binary(Bin::Add, hh, shr_u(lh, lit(16))), shr_u(hl, lit(16))),
                      shr_u(mid, lit(16)));
      }
      case Intr::FmaAdd:
        return binary(Bin::Add, x, n);
      case Intr::Addc: {
        // ahi + bhi + ltu(alo + blo, alo), with ltu spelled out as above
        Expr lo = binary(Bin::Add, c.a[2], c.a[3]);
        Expr carry = binary(Bin::Lt, binary(Bin::Xor, lo, int_min()), binary(Bin::Xor, c.a[2], int_min()));
        return binary(Bin::Add, binary(Bin::Add, c.a[0], c.a[1]), carry);
      }
      case Intr::Fshr:
      case Intr::Fshl: {
        // fshr(lo, hi, n) = n&31 == 0 ? lo : shr_u(lo, n) | hi << (32 - n)
        // fshl(lo, hi, n) = n&31 == 0 ? hi : hi << n | shr_u(lo, 32 - n)
        bool right = Intr(c.i) == Intr::Fshr;
        const Expr& lo = c.a[0];
        const Expr& hi = c.a[1];
        const Expr& cnt = c.a[2];
        if (auto k = const_of(cnt)) {
          int s = *k & 31;
          if (s == 0) return right ? lo : hi;
          if (right) return binary(Bin::Or, shr_u(lo, lit(s)), binary(Bin::Shl, hi, lit(32 - s)));
          return binary(Bin::Or, binary(Bin::Shl, hi, lit(s)), shr_u(lo, lit(32 - s)));
        }
        Expr s = binary(Bin::And, cnt, lit(31));
        Expr back = binary(Bin::And, binary(Bin::Sub, lit(32), s), lit(31));
        Expr mix = right ? binary(Bin::Or, shr_u(lo, s), binary(Bin::Shl, hi, back))
                         : binary(Bin::Or, binary(Bin::Shl, hi, s), shr_u(lo, back));
        Expr mask = unary(Un::Neg, binary(Bin::Ne, s, lit(0)));  // 0 or -1
        Expr keep = right ? lo : hi;
        return binary(Bin::Or, binary(Bin::And, keep, binary(Bin::Xor, mask, unary(Un::Neg, lit(1)))),
                      binary(Bin::And, mix, mask));
      }
      default: return c;
    }
  }

  Block block(const Block& b) {
    Block out;
    for (const auto& s : b) stmt(s, out);
    return out;
  }

  void stmt(const Stmt& s, Block& out) {
    Stmt c = s;
    for (auto& e : c.idx) e = expr(e);
    for (auto& e : c.val) e = expr(e);
    if (c.k == SK::For) {
      c.unroll = 0;
      c.init = block(c.init);
      c.step = block(c.step);
    }
    c.body = block(c.body);
    c.alt = block(c.alt);
    if (c.k == SK::Decl) scalars[c.name] = c.ty;
    if (c.k == SK::Assign && c.idx.empty() && c.val[0].k == EK::Intrin && Intr(c.val[0].i) == Intr::Bcast) {
      // x = warp_bcast(v, src, w): the xor butterfly the interpreter executes in lock step --
      // every lane shuffles at each step, a lane whose group index differs from src in bit m
      // adopts its partner's value (exact when src is uniform within each w-lane group)
      const Expr& b = c.val[0];
      int w = 2;
      if (auto k = const_of(b.a[2])) w = *k;
      int id = counter++;
      std::string src = "__bs" + std::to_string(id);
      Ty t = scalars.count(c.name) ? scalars[c.name] : Ty::Int;
      out.push_back(assign(c.name, b.a[0]));
      out.push_back(decl_init(Ty::Int, src, b.a[1]));
      Expr tid = binary(Bin::Add, builtin(Builtin::TidX),
                        binary(Bin::Add, binary(Bin::Mul, builtin(Builtin::TidY), builtin(Builtin::BdimX)),
                               binary(Bin::Mul, builtin(Builtin::TidZ),
                                      binary(Bin::Mul, builtin(Builtin::BdimX), builtin(Builtin::BdimY)))));
      for (int m = 1; m < w; m <<= 1) {
        std::string tmp = "__bt" + std::to_string(id) + "_" + std::to_string(m);
        Expr sh;
        sh.k = EK::Shfl;
        sh.i = m;
        sh.a.push_back(var(c.name));
        sh.pos = c.pos;
        out.push_back(decl_init(t, tmp, sh));
        Expr differs = binary(Bin::Ne,
                              binary(Bin::And, binary(Bin::Xor, binary(Bin::Mod, tid, lit(32)), var(src)), lit(m)),
                              lit(0));
        out.push_back(if_(differs, Block{assign(c.name, var(tmp))}));
      }
      return;
    }
    if (c.k == SK::Fence) return;     // the interpreter is sequentially consistent
    if (c.k == SK::Atomic) c.bid = 0;  // atomic_add_release -> atomic_add (same reason)
    if (c.k == SK::WarpSync) return;  // ... and runs each warp in lock step
    if (c.k == SK::AsyncWait) return;  // the lowered copy below has already landed
    if (c.k == SK::AsyncCopy) {
      // sarr[4j + k] = garr[4i + k], k = 0..3, both indices evaluated once, copied immediately
      int id = counter++;
      std::string gb = "__ag" + std::to_string(id), sb = "__as" + std::to_string(id);
      Stmt g = decl_init(Ty::Int, gb, binary(Bin::Mul, c.idx[0], lit(4)));
      g.pos = c.pos;
      out.push_back(g);
      out.push_back(decl_init(Ty::Int, sb, binary(Bin::Mul, c.val[0], lit(4))));
      for (int k = 0; k < 4; ++k) {
        Expr gi = k == 0 ? var(gb) : binary(Bin::Add, var(gb), lit(k));
        Expr si = k == 0 ? var(sb) : binary(Bin::Add, var(sb), lit(k));
        out.push_back(assign_at(c.outs[0], si, index(c.name, gi)));
      }
      return;
    }
    if (c.k == SK::VLoad || c.k == SK::VStore) {
      int id = counter++;
      int n = int(c.k == SK::VLoad ? c.outs.size() : c.val.size());
      std::string base = "__vx" + std::to_string(id);
      Stmt bd = decl_init(Ty::Int, base, binary(Bin::Mul, c.idx[0], lit(n)));
      bd.pos = c.pos;
      out.push_back(bd);
      auto elem = [&](int k) { return k == 0 ? var(base) : binary(Bin::Add, var(base), lit(k)); };
      if (c.k == SK::VLoad) {
        for (int k = 0; k < n; ++k) out.push_back(assign(c.outs[k], index(c.name, elem(k))));
      } else {
        // all values are evaluated before any element is written
        Ty t = arrays.count(c.name) ? arrays[c.name] : Ty::Float;
        for (int k = 0; k < n; ++k)
          out.push_back(decl_init(t, base + "_" + std::to_string(k), c.val[k]));
        for (int k = 0; k < n; ++k)
          out.push_back(assign_at(c.name, elem(k), var(base + "_" + std::to_string(k))));
      }
      return;
    }
    out.push_back(std::move(c));
  }
};

}  // namespace

Kernel downlower(const Kernel& k) {
  Lowerer l;
  for (const auto& p : k.params)
    if (p.array) l.arrays[p.name] = p.ty;
    else l.scalars[p.name] = p.ty;
  for (const auto& sh : k.shared) l.arrays[sh.name] = sh.ty;
  Kernel out = k;
  out.body = l.block(k.body);
  out.reqs.clear();  // `//@ requires` is MK+ only (the reference rejects unknown annotations)
  return out;
}

Program downlower(const Program& p) {
  Program out = p;
  for (auto& k : out.kernels) k = downlower(k);
  for (auto& f : out.funcs) {
    Lowerer l;
    for (const auto& prm : f.params)
      if (prm.array) l.arrays[prm.name] = prm.ty;
      else l.scalars[prm.name] = prm.ty;
    f.body = l.block(f.body);
  }
  return out;
}

}  // namespace hf
