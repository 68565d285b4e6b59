// TEST INFRASTRUCTURE ONLY. Parity checker driver around the UNMODIFIED reference
// library (mkfuse, /root/reference/proj/src), built by oracle/Makefile into
// oracle/_ref/mkfuse_ref. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may execute it.
//
// The reference ships its CLI only with CLI11 (not vendored, proj/.gitignore:2), so
// this driver re-exposes the library entry points the parity tests need:
//   fuse     : normalize_kernel (passes.cpp:706) + generate_fused (fuser.cpp:158)
//              + emit_source (fuser.cpp:553); --regcap mirrors cmd_fuse (mkfuse.cpp:118-133)
//   fusereport: the exact stdout of cmd_fuse (mkfuse.cpp:136-166)
//   seq      : run_functional k1 then k2 at the partition dims (acceptance_main.cpp:147-152)
//   fused    : run_functional of the fused kernel (fuser.hpp:82-85)
//   run      : run_functional of one kernel (exec.cpp:958-965)
//   search   : search_config / fixed_partition_fuse with SimulatorBackend (search.cpp:124-175)
//   regbound / occupancy : machine.cpp:236-283
//   combine  : combined_utilization, machine.cpp:285-289
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "mkfuse/frontend.hpp"
#include "mkfuse/fuser.hpp"
#include "mkfuse/search.hpp"

using namespace mkfuse;

namespace {

struct Args {
  std::vector<std::string> pos;
  std::vector<std::string> mem;
  std::optional<uint64_t> seed;
  int d1 = 0, d2 = 0, d0 = 1024, grid = 0;
  std::string style = "goto", regcap = "off", dump, dims;
  bool time = false;
};

std::string slurp(const std::string& path) {
  std::ifstream in(path);
  if (!in) fail(ErrCode::Io, "cannot open '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

Args parse(int argc, char** argv, int first) {
  Args a;
  for (int i = first; i < argc; ++i) {
    std::string s = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) fail(ErrCode::InvalidArgument, "missing value for " + s);
      return argv[++i];
    };
    if (s == "--mem") a.mem.push_back(next());
    else if (s == "--seed") a.seed = std::stoull(next());
    else if (s == "--d1") a.d1 = std::stoi(next());
    else if (s == "--d2") a.d2 = std::stoi(next());
    else if (s == "--d0") a.d0 = std::stoi(next());
    else if (s == "--grid") a.grid = std::stoi(next());
    else if (s == "--style") a.style = next();
    else if (s == "--regcap") a.regcap = next();
    else if (s == "--dump") a.dump = next();
    else if (s == "--dims") a.dims = next();
    else if (s == "--time") a.time = true;
    else a.pos.push_back(s);
  }
  return a;
}

struct Loaded {
  Program program;
  Kernel kernel;
};

Loaded load(const std::string& path) {
  Loaded l;
  l.program = parse_program(slurp(path));
  if (l.program.kernels.empty()) fail(ErrCode::InvalidArgument, path + " defines no kernel");
  l.kernel = l.program.kernels.front();
  return l;
}

Kernel normalized(const std::string& path, const char* prefix) {
  Loaded l = load(path);
  return normalize_kernel(l.kernel, l.program.functions, prefix);
}

MemoryImage images(const Args& a) {
  MemoryImage img;
  for (const auto& p : a.mem) img.merge(MemoryImage::load(p, a.seed));
  return img;
}

void finish(const MemoryImage& out, const Args& a, double secs) {
  std::printf("digest = %s\n", out.digest_hex().c_str());
  if (a.time) std::printf("seconds = %.6f\n", secs);
  if (!a.dump.empty()) {
    std::ofstream o(a.dump);
    o << out.serialize();
  }
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Partition dims of a normalized kernel exactly as generate_fused assigns them.
Dim3 dims_for(const Kernel& k, int d) {
  if (d == 0 || k.block_dims.count() == d) return k.block_dims;
  int yz = k.block_dims.y * k.block_dims.z;
  return Dim3{d / yz, k.block_dims.y, k.block_dims.z};
}

FusedKernel make_fused(const Args& a, Kernel& n1, Kernel& n2) {
  n1 = normalized(a.pos.at(0), "k1_");
  n2 = normalized(a.pos.at(1), "k2_");
  FusedKernel f = generate_fused(n1, n2, a.d1, a.d2, SMConfig::pascal_like());
  if (a.grid > 0) f.grid_dim = a.grid;
  return f;
}

int cmd_fuse(const Args& a, bool report) {
  SMConfig sm = SMConfig::pascal_like();
  Kernel n1, n2;
  FusedKernel fused = make_fused(a, n1, n2);
  KernelResources r1 = kernel_resources(n1, a.d1);
  KernelResources r2 = kernel_resources(n2, a.d2);
  KernelResources rf = kernel_resources(fused.to_kernel(), fused.config.d0);
  int r0 = -1;
  try {
    r0 = register_bound(r1, r2, rf.shmem_per_block, fused.config.d0, sm);
  } catch (const Error&) {
  }
  if (a.regcap == "auto") {
    if (r0 > 0) fused.config.reg_cap = r0;
  } else if (a.regcap != "off") {
    fused.config.reg_cap = std::stoi(a.regcap);
  }
  EmitStyle style = a.style == "structured" ? EmitStyle::Structured : EmitStyle::Goto;
  if (!report) {
    std::fputs(emit_source(fused, style).c_str(), stdout);
    return 0;
  }
  std::printf("fused_kernel = %s\n", fused.name.c_str());
  std::printf("partition = d1 %d (%s), d2 %d (%s), d0 %d\n", fused.config.d1,
              fused.k1_name.c_str(), fused.config.d2, fused.k2_name.c_str(), fused.config.d0);
  for (const auto& e : fused.barriers.entries) {
    int uses = 0;
    const StmtBlock& body = e.owner == 1 ? fused.body1 : fused.body2;
    for_each_stmt(body, [&](const Stmt& s) {
      if (const auto* pb = std::get_if<PartialBarrierStmt>(&s.node))
        if (pb->id == e.barrier_id) ++uses;
    });
    std::printf("barrier id %d: count %d, constituent %d, uses %d\n", e.barrier_id,
                e.participant_count, e.owner, uses);
  }
  std::printf("registers = k1 %d, k2 %d, fused %d\n", r1.regs_per_thread, r2.regs_per_thread,
              rf.regs_per_thread);
  std::printf("shared_bytes = %lld\n", (long long)rf.shmem_per_block);
  if (fused.config.reg_cap)
    std::printf("reg_cap = %d\n", *fused.config.reg_cap);
  else if (r0 > 0)
    std::printf("suggested_reg_cap = %d\n", r0);
  KernelResources capped = rf;
  if (fused.config.reg_cap)
    capped.regs_per_thread = std::min(capped.regs_per_thread, *fused.config.reg_cap);
  OccupancyReport rep = occupancy(capped, sm);
  std::printf("blocks_per_sm = %d\n", rep.blocks_per_sm);
  std::printf("limiting_resource = %s\n", to_string(rep.limiting));
  std::printf("achieved_warps = %d\n", rep.achieved_warps);
  std::printf("occupancy_fraction = %.6f\n", rep.occupancy_fraction);
  return 0;
}

int cmd_seq(const Args& a) {
  Kernel n1 = normalized(a.pos.at(0), "k1_");
  Kernel n2 = normalized(a.pos.at(1), "k2_");
  MemoryImage mem = images(a);
  int g1 = a.grid > 0 ? a.grid : n1.meta.grid_dim;
  int g2 = a.grid > 0 ? a.grid : n2.meta.grid_dim;
  LaunchConfig l1{g1, dims_for(n1, a.d1), std::nullopt};
  LaunchConfig l2{g2, dims_for(n2, a.d2), std::nullopt};
  double t0 = now_s();
  MemoryImage out = run_functional(n2, l2, run_functional(n1, l1, mem));
  finish(out, a, now_s() - t0);
  return 0;
}

int cmd_fused(const Args& a) {
  Kernel n1, n2;
  FusedKernel f = make_fused(a, n1, n2);
  MemoryImage mem = images(a);
  double t0 = now_s();
  MemoryImage out = run_functional(f, launch_for(f), mem);
  finish(out, a, now_s() - t0);
  return 0;
}

int cmd_run(const Args& a) {
  Loaded l = load(a.pos.at(0));
  Kernel k = inline_calls(l.kernel, l.program.functions);
  LaunchConfig launch = launch_for(k);
  if (a.grid > 0) launch.grid_dim = a.grid;
  if (!a.dims.empty()) {
    int x = 1, y = 1, z = 1;
    std::sscanf(a.dims.c_str(), "%d,%d,%d", &x, &y, &z);
    launch.block_dims = Dim3{x, y, z};
  }
  MemoryImage mem = images(a);
  double t0 = now_s();
  MemoryImage out = run_functional(k, launch, mem);
  finish(out, a, now_s() - t0);
  return 0;
}

int cmd_search(const Args& a) {
  SMConfig sm = SMConfig::pascal_like();
  Kernel n1 = normalized(a.pos.at(0), "k1_");
  Kernel n2 = normalized(a.pos.at(1), "k2_");
  SimulatorBackend backend(sm, images(a));
  SearchResult r = (n1.tunable && n2.tunable) ? search_config(n1, n2, a.d0, backend, sm)
                                              : fixed_partition_fuse(n1, n2, backend, sm, a.d0);
  std::fputs(trace_csv(r).c_str(), stdout);
  std::printf("best = %d,%d,%s\n", r.best_config.d1, r.best_config.d2,
              r.best_config.reg_cap ? std::to_string(*r.best_config.reg_cap).c_str() : "none");
  return 0;
}

int cmd_regbound(const Args& a) {
  auto v = [&](size_t i) { return std::stoll(a.pos.at(i)); };
  KernelResources r1{int(v(0)), 0, int(v(1))}, r2{int(v(2)), 0, int(v(3))};
  std::printf("%d\n", register_bound(r1, r2, v(4), int(v(1) + v(3)), SMConfig::pascal_like()));
  return 0;
}

int cmd_occupancy(const Args& a) {
  KernelResources r{std::stoi(a.pos.at(0)), std::stoll(a.pos.at(1)), std::stoi(a.pos.at(2))};
  OccupancyReport rep = occupancy(r, SMConfig::pascal_like());
  std::printf("%d %s %d %.6f\n", rep.blocks_per_sm, to_string(rep.limiting), rep.achieved_warps,
              rep.occupancy_fraction);
  return 0;
}

// combined_utilization (machine.cpp:285-289) on "u1 c1 u2 c2" arguments; %.17g output
int cmd_combine(const Args& a) {
  double v = combined_utilization(std::stod(a.pos.at(0)), std::stoll(a.pos.at(1)), std::stod(a.pos.at(2)),
                                  std::stoll(a.pos.at(3)));
  std::printf("%.17g\n", v);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr,
                 "usage: mkfuse_ref fuse|fusereport|seq|fused|run|search|regbound|occupancy ...\n");
    return 2;
  }
  std::string cmd = argv[1];
  try {
    Args a = parse(argc, argv, 2);
    if (cmd == "fuse") return cmd_fuse(a, false);
    if (cmd == "fusereport") return cmd_fuse(a, true);
    if (cmd == "seq") return cmd_seq(a);
    if (cmd == "fused") return cmd_fused(a);
    if (cmd == "run") return cmd_run(a);
    if (cmd == "search") return cmd_search(a);
    if (cmd == "regbound") return cmd_regbound(a);
    if (cmd == "occupancy") return cmd_occupancy(a);
    if (cmd == "combine") return cmd_combine(a);
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  } catch (const Error& e) {
    std::fprintf(stderr, "error%s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
