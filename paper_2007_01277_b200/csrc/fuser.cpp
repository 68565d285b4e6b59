// generate_fused and friends (Algorithm "Generate").
// Reference: /root/reference/proj/src/fuser.cpp:14-282 (same prologue, guard, merge and
// error contract), plus named-barrier allocation for pre-existing bar_sync statements.
#include <algorithm>
#include <map>
#include <set>

#include "fuser.hpp"

namespace hf {
namespace {

const char* const kPrologueVars[] = {"global_tid",  "tid_1",       "tid_2",      "size_1",
                                     "size_2",      "threadIdx_x", "threadIdx_y", "threadIdx_z",
                                     "blockDim_x",  "blockDim_y",  "blockDim_z"};

void require_normalized(const Kernel& k) {
  if (has_calls(k.body))
    raise(Code::InvalidArgument, "kernel '" + k.name + "' still contains calls", k.pos);
  if (!decl_prefix_form(k))
    raise(Code::InvalidArgument, "kernel '" + k.name + "' is not in lifted declaration form",
          k.pos);
}

constexpr int kMaxNamedBarrier = 15;  // ids 1..15; id 0 is the whole-block barrier

}  // namespace

Dims partition_dims(const Kernel& k, int d) {
  if (k.dims.count() == d) return k.dims;
  if (!k.tunable)
    raise(Code::DimensionMismatch, "kernel '" + k.name + "' has fixed dims " +
                                       std::to_string(k.dims.count()) +
                                       " but the partition assigns " + std::to_string(d));
  int yz = k.dims.y * k.dims.z;
  if (d % yz != 0)
    raise(Code::DimensionMismatch, "partition " + std::to_string(d) +
                                       " is not divisible by the declared y*z = " +
                                       std::to_string(yz) + " of kernel '" + k.name + "'");
  return Dims{d / yz, k.dims.y, k.dims.z};
}

void FusionConfig::check(const SM& sm) const {
  if (d1 < 32 || d2 < 32 || d1 % 32 != 0 || d2 % 32 != 0)
    raise(Code::InvalidArgument, "thread partition must be warp aligned: d1 = " +
                                     std::to_string(d1) + ", d2 = " + std::to_string(d2));
  if (d0 != d1 + d2) raise(Code::InvalidArgument, "d0 must equal d1 + d2");
  if (d0 > sm.max_threads_per_sm)
    raise(Code::ThreadBudgetExceeded,
          "fused block dimension " + std::to_string(d0) + " exceeds the SM thread budget");
  if (reg_cap && *reg_cap <= 0) raise(Code::InvalidArgument, "register cap must be positive");
}

Block build_prologue(Dims dims1, Dims dims2, int d1) {
  if (dims1.count() != d1)
    raise(Code::DimensionMismatch, "prologue dims " + std::to_string(dims1.count()) +
                                       " do not match d1 = " + std::to_string(d1));
  int d2 = int(dims2.count());
  Block out;
  for (const char* n : kPrologueVars) out.push_back(decl(Ty::Int, n));
  // global_tid = tid.x + tid.y * bdim.x + tid.z * bdim.x * bdim.y
  Expr linear = binary(
      Bin::Add,
      binary(Bin::Add, builtin(Builtin::TidX),
             binary(Bin::Mul, builtin(Builtin::TidY), builtin(Builtin::BdimX))),
      binary(Bin::Mul, binary(Bin::Mul, builtin(Builtin::TidZ), builtin(Builtin::BdimX)),
             builtin(Builtin::BdimY)));
  out.push_back(assign("global_tid", std::move(linear)));
  out.push_back(assign("tid_1", var("global_tid")));
  out.push_back(assign("tid_2", binary(Bin::Sub, var("global_tid"), lit(d1))));
  out.push_back(assign("size_1", lit(d1)));
  out.push_back(assign("size_2", lit(d2)));
  auto remap = [](Dims d, Expr base) {
    Block b;
    b.push_back(assign("blockDim_x", lit(d.x)));
    b.push_back(assign("blockDim_y", lit(d.y)));
    b.push_back(assign("blockDim_z", lit(d.z)));
    b.push_back(assign("threadIdx_x", binary(Bin::Mod, base, lit(d.x))));
    b.push_back(assign("threadIdx_y",
                       binary(Bin::Mod, binary(Bin::Div, base, lit(d.x)), lit(d.y))));
    b.push_back(assign("threadIdx_z", binary(Bin::Div, base, lit(d.x * d.y))));
    return b;
  };
  out.push_back(if_else(binary(Bin::Lt, var("global_tid"), lit(d1)),
                        remap(dims1, var("global_tid")),
                        remap(dims2, binary(Bin::Sub, var("global_tid"), lit(d1)))));
  return out;
}

Block rewrite_builtins(const Block& body) {
  Block out = body;
  walk(out, [&](Stmt& s) {
    exprs_of(s, [&](Expr& e) {
      walk_expr(e, [&](Expr& x) {
        if (x.k != EK::Builtin) return;
        static const char* names[] = {"threadIdx_x", "threadIdx_y", "threadIdx_z", nullptr,
                                      nullptr,       nullptr,       "blockDim_x",  "blockDim_y",
                                      "blockDim_z",  nullptr};
        if (const char* n = names[x.i]) {
          Pos p = x.pos;
          x = var(n);
          x.pos = p;
        }
      });
    });
  });
  return out;
}

Block replace_barriers(const Block& body, int id, int count) {
  if (id < 0 || id > 15)
    raise(Code::BadBarrierId, "barrier id " + std::to_string(id) + " outside [0, 15]");
  if (count <= 0 || count % 32 != 0)
    raise(Code::MisalignedCount,
          "barrier count " + std::to_string(count) + " is not a positive multiple of 32");
  Block out = body;
  walk(out, [&](Stmt& s) {
    if (s.k == SK::Sync) {
      s.k = SK::BarSync;
      s.bid = id;
      s.bcount = count;
    }
  });
  return out;
}

namespace {

// Gives every constituent-owned bar_sync id its own hardware barrier. A count equal to
// the constituent's declared block size means "the whole constituent" and is resized
// to the interval; smaller counts are sub-groups and must fit in the interval.
void allocate_named_barriers(Block& body, int owner, const Kernel& k, int interval,
                             int& next_id, std::vector<BarrierEntry>& table) {
  std::map<int, int> ids;
  walk(body, [&](Stmt& s) {
    if (s.k != SK::BarSync) return;
    auto it = ids.find(s.bid);
    int new_id;
    if (it == ids.end()) {
      if (next_id > kMaxNamedBarrier)
        raise(Code::BadBarrierId, "kernel '" + k.name +
                                      "' needs more named barriers than the 15 a CTA can host",
              s.pos);
      new_id = next_id++;
      ids[s.bid] = new_id;
    } else {
      new_id = it->second;
    }
    int count = s.bcount == k.dims.count() ? interval : s.bcount;
    if (count > interval)
      raise(Code::InvalidArgument,
            "bar_sync(" + std::to_string(s.bid) + ", " + std::to_string(s.bcount) +
                ") of kernel '" + k.name + "' exceeds its " + std::to_string(interval) +
                "-thread interval",
            s.pos);
    bool seen = std::any_of(table.begin(), table.end(), [&](const BarrierEntry& e) {
      return e.id == new_id && e.count == count;
    });
    if (!seen) table.push_back(BarrierEntry{new_id, count, owner, s.bid});
    s.bid = new_id;
    s.bcount = count;
  });
}

}  // namespace

Fused fuse(const Kernel& k1, const Kernel& k2, int d1, int d2, const SM& sm) {
  require_normalized(k1);
  require_normalized(k2);
  if (k1.grid != k2.grid)
    raise(Code::GridMismatch, "grid dimensions differ: '" + k1.name + "' uses " +
                                  std::to_string(k1.grid) + ", '" + k2.name + "' uses " +
                                  std::to_string(k2.grid));
  FusionConfig cfg;
  cfg.d1 = d1;
  cfg.d2 = d2;
  cfg.d0 = d1 + d2;
  cfg.check(sm);
  if (cfg.d0 > sm.max_threads_per_block)
    raise(Code::ThreadBudgetExceeded, "fused block dimension " + std::to_string(cfg.d0) +
                                          " exceeds max threads per block (" +
                                          std::to_string(sm.max_threads_per_block) + ")");
  Fused f;
  f.name = "fused_" + k1.name + "_" + k2.name;
  f.k1_name = k1.name;
  f.k2_name = k2.name;
  f.cfg = cfg;
  f.grid = k1.grid;
  f.reqs = k1.reqs;
  f.reqs.insert(f.reqs.end(), k2.reqs.begin(), k2.reqs.end());
  f.dims1 = partition_dims(k1, d1);
  f.dims2 = partition_dims(k2, d2);

  std::set<std::string> param_names;
  for (const Kernel* k : {&k1, &k2}) {
    for (const auto& p : k->params) {
      auto it = std::find_if(f.params.begin(), f.params.end(),
                             [&](const Param& q) { return q.name == p.name; });
      if (it == f.params.end()) {
        f.params.push_back(p);
        param_names.insert(p.name);
      } else if (it->ty != p.ty || it->array != p.array) {
        raise(Code::TypeMismatch,
              "parameter '" + p.name + "' has conflicting types across the two kernels");
      }
    }
  }
  for (const char* n : kPrologueVars)
    if (param_names.count(n))
      raise(Code::InvalidArgument,
            std::string("parameter '") + n + "' collides with a prologue variable");

  std::set<std::string> names;
  int64_t shared_bytes = 0;
  for (const Kernel* k : {&k1, &k2}) {
    for (const auto& sh : k->shared) {
      if (!names.insert(sh.name).second)
        raise(Code::InvalidArgument,
              "shared array '" + sh.name + "' appears in both kernels (rename first)");
      f.shared.push_back(sh);
      shared_bytes += sh.len * 4;
    }
  }
  if (shared_bytes > sm.shmem_per_sm)
    raise(Code::SharedMemoryOverflow, "fused kernel needs " + std::to_string(shared_bytes) +
                                          " bytes of shared memory; the SM has " +
                                          std::to_string(sm.shmem_per_sm));

  auto split = [&](const Kernel& k, Block& decls, Block& rest) {
    size_t i = 0;
    while (i < k.body.size() && k.body[i].k == SK::Decl) decls.push_back(k.body[i++]);
    for (; i < k.body.size(); ++i) rest.push_back(k.body[i]);
  };
  Block s1, s2;
  split(k1, f.decls, s1);
  split(k2, f.decls, s2);
  for (const auto& d : f.decls)
    if (!names.insert(d.name).second)
      raise(Code::InvalidArgument,
            "local '" + d.name + "' appears in both kernels (rename first)");

  for (auto& s : build_prologue(f.dims1, f.dims2, d1)) {
    if (s.k == SK::Decl) f.prologue_decls.push_back(std::move(s));
    else f.prologue.push_back(std::move(s));
  }

  f.body1 = replace_barriers(rewrite_builtins(s1), 1, d1);
  f.body2 = replace_barriers(rewrite_builtins(s2), 2, d2);
  f.guard1 = binary(Bin::Lt, var("global_tid"), lit(d1));
  f.guard2 = binary(Bin::Ge, var("global_tid"), lit(d1));
  f.barriers.push_back(BarrierEntry{1, d1, 1, -1});
  f.barriers.push_back(BarrierEntry{2, d2, 2, -1});
  // replace_barriers turned syncthreads into (1|2, d) BarSync; remap only the
  // constituents' own bar_sync statements, which predate the rewrite.
  auto own = [&](const Block& original, Block& rewritten, int owner, const Kernel& k, int d,
                 int& next_id) {
    // Mark original bar_sync positions: walk both trees in lock step.
    std::vector<Stmt*> dst;
    walk(rewritten, [&](Stmt& s) { dst.push_back(&s); });
    std::vector<const Stmt*> src;
    walk(original, [&](const Stmt& s) { src.push_back(&s); });
    Block holder;
    std::vector<size_t> where;
    for (size_t i = 0; i < src.size(); ++i)
      if (src[i]->k == SK::BarSync) where.push_back(i);
    if (where.empty()) return;
    for (size_t i : where) holder.push_back(*dst[i]);
    allocate_named_barriers(holder, owner, k, d, next_id, f.barriers);
    for (size_t j = 0; j < where.size(); ++j) *dst[where[j]] = holder[j];
  };
  int next_id = 3;
  own(s1, f.body1, 1, k1, d1, next_id);
  own(s2, f.body2, 2, k2, d2, next_id);
  return f;
}

// Vertical fusion (VFuse, the paper's comparison point PAPER.md:889-890; the reference keeps
// only a test-local version, test_sim.cpp:398-439): same block, every thread runs k1's body
// then k2's body. Returns of k1 jump to the end of k1's body so k2 still runs.
Kernel vertical_fuse(const Kernel& k1, const Kernel& k2) {
  require_normalized(k1);
  require_normalized(k2);
  if (!(k1.dims == k2.dims))
    raise(Code::DimensionMismatch, "vertical fusion needs equal block dims ('" + k1.name + "' vs '" +
                                       k2.name + "')");
  if (k1.grid != k2.grid)
    raise(Code::GridMismatch, "grid dimensions differ: '" + k1.name + "' uses " + std::to_string(k1.grid) +
                                  ", '" + k2.name + "' uses " + std::to_string(k2.grid));
  Kernel v;
  v.name = "vertical_" + k1.name + "_" + k2.name;
  v.dims = k1.dims;
  v.tunable = false;
  v.grid = k1.grid;
  v.params = k1.params;
  for (const auto& p : k2.params) {
    auto it = std::find_if(v.params.begin(), v.params.end(), [&](const Param& q) { return q.name == p.name; });
    if (it == v.params.end()) v.params.push_back(p);
    else if (it->ty != p.ty || it->array != p.array)
      raise(Code::TypeMismatch, "parameter '" + p.name + "' has conflicting types across the two kernels");
  }
  v.shared = k1.shared;
  for (const auto& sh : k2.shared) v.shared.push_back(sh);
  Block d1, r1, d2, r2;
  auto split = [](const Kernel& k, Block& d, Block& r) {
    size_t i = 0;
    while (i < k.body.size() && k.body[i].k == SK::Decl) d.push_back(k.body[i++]);
    for (; i < k.body.size(); ++i) r.push_back(k.body[i]);
  };
  split(k1, d1, r1);
  split(k2, d2, r2);
  bool returns = false;
  walk(r1, [&](Stmt& s) {
    if (s.k == SK::Return) {
      s.k = SK::Goto;
      s.name = "vf_k1_end";
      s.val.clear();
      returns = true;
    }
  });
  for (auto& s : d1) v.body.push_back(s);
  for (auto& s : d2) v.body.push_back(s);
  for (auto& s : r1) v.body.push_back(s);
  if (returns) {
    Stmt l;
    l.k = SK::Label;
    l.name = "vf_k1_end";
    v.body.push_back(l);
  }
  for (auto& s : r2) v.body.push_back(s);
  return v;
}

Kernel Fused::to_kernel() const {
  Kernel k;
  k.name = name;
  k.params = params;
  k.dims = Dims{cfg.d0, 1, 1};
  k.tunable = false;  // the guards bake the partition in
  k.shared = shared;
  k.grid = grid;
  k.regcap = cfg.reg_cap;
  k.reqs = reqs;
  for (const auto& s : prologue_decls) k.body.push_back(s);
  for (const auto& s : decls) k.body.push_back(s);
  for (const auto& s : prologue) k.body.push_back(s);
  k.body.push_back(if_(guard1, body1));
  k.body.push_back(if_(guard2, body2));
  return k;
}

std::string emit_structured(const Fused& f) { return print_mk(f.to_kernel()); }

// ---------------------------------------------------------------------------
// Machine model (machine.cpp:22-289 of the reference)
// ---------------------------------------------------------------------------

SM SM::pascal_like() { return SM{}; }

SM SM::volta_like() {
  SM s;
  s.lat_memory = 320;
  s.lat_atomic = 32;
  return s;
}

SM SM::b200() {
  SM s;
  s.shmem_per_sm = 233472;  // 228 KB per SM (227 KB usable per CTA)
  s.max_shmem_per_block = 232448;
  s.num_sms = 148;
  s.lat_memory = 577;
  s.lat_atomic = 318;
  return s;
}

void SM::check() const {
  auto pos = [](int64_t v, const char* n) {
    if (v <= 0) raise(Code::InvalidArgument, std::string(n) + " must be positive");
  };
  pos(regs_per_sm, "regs_per_sm");
  pos(shmem_per_sm, "shmem_per_sm");
  pos(max_threads_per_sm, "max_threads_per_sm");
  pos(max_threads_per_block, "max_threads_per_block");
  pos(warp_size, "warp_size");
  pos(max_blocks_per_sm, "max_blocks_per_sm");
  pos(num_sms, "num_sms");
  pos(issue_slots, "issue_slots");
  pos(mem_slots_per_cycle, "mem_slots_per_cycle");
  pos(lat_compute, "compute_cycles");
  pos(lat_memory, "memory_cycles");
  pos(lat_shuffle, "shuffle_cycles");
  pos(lat_atomic, "atomic_cycles");
  if (max_threads_per_block % warp_size != 0)
    raise(Code::InvalidArgument, "warp_size must divide max_threads_per_block");
}

const char* limit_name(Limit l) {
  switch (l) {
    case Limit::Registers: return "registers";
    case Limit::SharedMemory: return "shared_memory";
    case Limit::Threads: return "threads";
    case Limit::BlockSlots: return "block_slots";
  }
  return "?";
}

namespace {

// Peak number of simultaneously live declared locals over a linear statement order.
struct Liveness {
  struct Span {
    int first = -1, last = -1;
  };
  std::vector<Span> spans;
  std::vector<std::map<std::string, int>> scopes;
  int step = 0;

  int find(const std::string& n) const {
    for (auto it = scopes.rbegin(); it != scopes.rend(); ++it) {
      auto f = it->find(n);
      if (f != it->end()) return f->second;
    }
    return -1;
  }
  void touch(int id) {
    if (id < 0) return;
    if (spans[id].first < 0) spans[id].first = step;
    spans[id].last = step;
  }
  void expr(const Expr& e) {
    walk_expr(e, [&](const Expr& x) {
      if (x.k == EK::Var || x.k == EK::Index) touch(find(x.s));
    });
  }
  void stmt(const Stmt& s) {
    ++step;
    switch (s.k) {
      case SK::Decl: {
        if (!s.val.empty()) expr(s.val[0]);
        int id = int(spans.size());
        spans.emplace_back();
        scopes.back()[s.name] = id;
        if (!s.val.empty()) touch(id);
        break;
      }
      case SK::Assign:
      case SK::Atomic:
      case SK::VStore:
        touch(find(s.name));
        for (const auto& e : s.idx) expr(e);
        for (const auto& e : s.val) expr(e);
        break;
      case SK::VLoad:
        touch(find(s.name));
        expr(s.idx[0]);
        for (const auto& d : s.outs) touch(find(d));
        break;
      case SK::AsyncCopy:
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
        for (const auto& e : s.val) expr(e);
        break;
      default:
        break;
    }
  }
  void block(const Block& b) {
    scopes.emplace_back();
    for (const auto& s : b) stmt(s);
    scopes.pop_back();
  }
  int peak() const {
    std::vector<std::pair<int, int>> ev;
    for (const auto& sp : spans) {
      if (sp.first < 0) continue;
      ev.emplace_back(sp.first, 1);
      ev.emplace_back(sp.last + 1, -1);
    }
    std::sort(ev.begin(), ev.end());
    int live = 0, best = 0;
    for (const auto& [at, d] : ev) {
      (void)at;
      live += d;
      best = std::max(best, live);
    }
    return best;
  }
};

}  // namespace

int estimate_registers(const Kernel& k) {
  if (k.regs) return *k.regs;
  Liveness l;
  l.block(k.body);
  return l.peak() + 8;
}

Resources resources_of(const Kernel& k, std::optional<int> threads) {
  Resources r;
  r.regs = estimate_registers(k);
  for (const auto& sh : k.shared) r.shmem += sh.len * 4;
  r.threads = threads ? *threads : int(k.dims.count());
  return r;
}

Occupancy occupancy(const Resources& r, const SM& sm) {
  if (r.regs <= 0 || r.threads <= 0 || r.shmem < 0)
    raise(Code::InvalidArgument, "kernel resources must be positive");
  const int64_t inf = INT64_MAX;
  int64_t q[4] = {sm.regs_per_sm / (int64_t(r.regs) * r.threads),
                  r.shmem == 0 ? inf : sm.shmem_per_sm / r.shmem,
                  sm.max_threads_per_sm / r.threads, sm.max_blocks_per_sm};
  int64_t blocks = *std::min_element(q, q + 4);
  if (blocks <= 0)
    raise(Code::DoesNotFit, "kernel does not fit on one SM even once (" +
                                std::to_string(r.regs) + " regs, " + std::to_string(r.shmem) +
                                " B shared, " + std::to_string(r.threads) + " threads)");
  Occupancy o;
  o.blocks_per_sm = int(blocks);
  for (int i = 0; i < 4; ++i)
    if (q[i] == blocks) {
      o.limiting = Limit(i);
      break;
    }
  o.warps = o.blocks_per_sm * ((r.threads + sm.warp_size - 1) / sm.warp_size);
  o.fraction = double(int64_t(o.blocks_per_sm) * r.threads) / sm.max_threads_per_sm;
  return o;
}

int register_bound(const Resources& r1, const Resources& r2, int64_t fused_shmem, int d0,
                   const SM& sm) {
  if (d0 != r1.threads + r2.threads)
    raise(Code::InvalidArgument, "d0 must equal the sum of the constituent thread counts");
  int64_t b1 = sm.regs_per_sm / (int64_t(r1.threads) * r1.regs);
  int64_t b2 = sm.regs_per_sm / (int64_t(r2.threads) * r2.regs);
  int64_t bs = fused_shmem == 0 ? INT64_MAX : sm.shmem_per_sm / fused_shmem;
  int64_t bt = sm.max_threads_per_sm / d0;
  int64_t b0 = std::min(std::min(b1, b2), std::min(bs, bt));
  if (b0 <= 0) raise(Code::DoesNotFit, "no register bound can make the fused kernel resident");
  return int(sm.regs_per_sm / (b0 * d0));
}

double combined_utilization(double u1, int64_t c1, double u2, int64_t c2) {
  if (c1 <= 0 || c2 <= 0)
    raise(Code::InvalidArgument, "combined utilization needs positive cycle counts");
  return (u1 * double(c1) + u2 * double(c2)) / double(c1 + c2);
}

}  // namespace hf
