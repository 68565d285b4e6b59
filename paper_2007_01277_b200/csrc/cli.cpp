// hfuse — the B200 drop-in for the reference CLI (/root/reference/proj/tools/mkfuse.cpp).
//
//   hfuse fuse K1 K2 --d1 N --d2 N [--style goto|structured|sm100] [--regcap n|auto|off] [-o F] [--sm S]
//              [--interval-regs R1,R2]   (sm100: per-interval setmaxnreg budgets instead of --regcap)
//   hfuse simulate K [--mem IMG]... [--seed S] [--regcap n|auto|off] [--dump-mem F] [--entry E]
//   hfuse simulate --sequential K1 K2 --mem IMG... [--dump-mem F]
//   hfuse search K1 K2 [--d0 N] --mem IMG... [--trace F] [-o F] [--style S] [--profiler-cmd CMD]
//                      [--granularity G] [--caps 32,40,...] [--reps N] [--budgets]
//                      (--budgets: also sweep per-interval setmaxnreg register budgets)
//                      [--prefilter K [--prefilter-tol F]]  (time only the K partitions the B200
//                      model ranks best, plus those predicted within F of the best; default 0.03)
//   hfuse occupancy [K] [--regs N --shmem B --threads T] [--sm S]
//   hfuse check K              hfuse lower K [-o F]           hfuse emit K [-o F]
//   hfuse profile CANDIDATE(.cu|.mk) --mem IMG... [--grid G]   (mkfuse --profiler-cmd target)
//
// Same flags, stdout keys and exit codes (0 ok; 1 + "error[Code] l:c: msg" on stderr).
// `simulate` and `search` run on the GPU: the reference's cycle simulator is replaced by
// device execution (elapsed_us from CUDA events); `--sm` defaults to pascal-like for
// `fuse`/`occupancy` (report parity) and to the live device for GPU commands.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>

#include "driver.hpp"
#include "runtime.hpp"
#include "search.hpp"

using namespace hf;

namespace {

struct Args {
  std::string cmd;
  std::vector<std::string> inputs, mem;
  std::optional<uint64_t> seed;
  std::string sm = "pascal-like", regcap = "auto", style, out, trace, entry, profiler_cmd, dump, caps, iregs;
  bool sequential = false, sm_given = false, regcap_given = false, budgets = false;
  int prefilter = 0;
  double prefilter_tol = -1.0;
  int d0 = 1024, d1 = 0, d2 = 0, regs = 0, threads = 0, granularity = 128, reps = 10, warmup = 3, grid = 0;
  int64_t shmem = 0;
};

void write_text(const std::string& path, const std::string& text) {
  std::ofstream out(path);
  if (!out) raise(Code::Io, "cannot write '" + path + "'");
  out << text;
}

Args parse_args(int argc, char** argv) {
  Args a;
  if (argc < 2) raise(Code::InvalidArgument, "usage: hfuse fuse|simulate|search|occupancy|check|lower|emit ...");
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) raise(Code::InvalidArgument, "option " + s + " needs a value");
      return argv[++i];
    };
    auto num = [&]() {
      std::string v = val();
      try {
        return std::stoi(v);
      } catch (...) {
        raise(Code::InvalidArgument, "option " + s + " needs an integer, got '" + v + "'");
      }
    };
    if (s == "--d0") a.d0 = num();
    else if (s == "--d1") a.d1 = num();
    else if (s == "--d2") a.d2 = num();
    else if (s == "--style") a.style = val();
    else if (s == "-o" || s == "--out") a.out = val();
    else if (s == "--regcap") {
      a.regcap = val();
      a.regcap_given = true;
    } else if (s == "--sm") {
      a.sm = val();
      a.sm_given = true;
    } else if (s == "--mem") a.mem.push_back(val());
    else if (s == "--seed") a.seed = std::stoull(val());
    else if (s == "--trace") a.trace = val();
    else if (s == "--profiler-cmd") a.profiler_cmd = val();
    else if (s == "--entry") a.entry = val();
    else if (s == "--dump-mem") a.dump = val();
    else if (s == "--sequential") a.sequential = true;
    else if (s == "--budgets") a.budgets = true;
    else if (s == "--regs") a.regs = num();
    else if (s == "--shmem") a.shmem = std::stoll(val());
    else if (s == "--threads") a.threads = num();
    else if (s == "--granularity") a.granularity = num();
    else if (s == "--caps") a.caps = val();
    else if (s == "--interval-regs") a.iregs = val();
    else if (s == "--prefilter") a.prefilter = num();
    else if (s == "--prefilter-tol") a.prefilter_tol = std::stod(val());
    else if (s == "--reps") a.reps = num();
    else if (s == "--warmup") a.warmup = num();
    else if (s == "--grid") a.grid = num();
    else if (!s.empty() && s[0] == '-') raise(Code::InvalidArgument, "unknown option " + s);
    else a.inputs.push_back(s);
  }
  for (const auto& p : a.inputs)
    if (!std::filesystem::exists(p)) raise(Code::Io, "input file '" + p + "' does not exist");
  for (const auto& p : a.mem)
    if (!std::filesystem::exists(p)) raise(Code::Io, "memory image '" + p + "' does not exist");
  return a;
}

Image images(const Args& a) {
  Image img;
  for (const auto& p : a.mem) img.merge(Image::parse(read_text(p), a.seed));
  return img;
}

void need_inputs(const Args& a, size_t n) {
  if (a.inputs.size() != n)
    raise(Code::InvalidArgument, a.cmd + " takes " + std::to_string(n) + " kernel file(s)");
}

int cmd_fuse(const Args& a) {
  need_inputs(a, 2);
  if (a.d1 == 0 || a.d2 == 0) raise(Code::InvalidArgument, "fuse needs --d1 and --d2");
  FuseResult r = fuse_sources(read_text(a.inputs[0]), read_text(a.inputs[1]), a.d1, a.d2, a.regcap,
                              SM::preset_or_file(a.sm));
  std::string style = a.style.empty() ? "goto" : a.style;
  Style st = style == "structured" ? Style::Structured : style == "sm100" ? Style::Sm100 : Style::Goto;
  std::string path = a.out.empty() ? (st == Style::Structured ? "fused.mk" : "fused.cu") : a.out;
  if (!a.iregs.empty()) {
    if (st != Style::Sm100) raise(Code::InvalidArgument, "--interval-regs needs --style sm100");
    if (a.regcap_given && a.regcap != "off") raise(Code::InvalidArgument, "--interval-regs and --regcap are exclusive");
    int r1 = 0, r2 = 0;
    if (std::sscanf(a.iregs.c_str(), "%d,%d", &r1, &r2) != 2)
      raise(Code::InvalidArgument, "--interval-regs needs R1,R2, got '" + a.iregs + "'");
    r.fused.cfg.reg_cap.reset();
    Sm100Options o;
    o.regs1 = r1;
    o.regs2 = r2;
    Sm100Kernel k = emit_sm100(r.fused, o);
    write_text(path, k.source);
    r.fused.cfg.reg_cap = k.launch_regs;  // the report's occupancy: the pool per thread
    std::fputs(fuse_report(r).c_str(), stdout);
    std::printf("interval_regs = %d,%d (launch %d)\n", r1, r2, k.launch_regs);
    std::printf("wrote %s\n", path.c_str());
    return 0;
  }
  write_text(path, emit(r.fused, st));
  std::fputs(fuse_report(r).c_str(), stdout);
  std::printf("wrote %s\n", path.c_str());
  return 0;
}

void print_run(double us, Image& img, const Args& a) {
  std::printf("elapsed_us = %.3f\n", us);
  std::printf("digest = %s\n", img.digest_hex().c_str());
  if (!a.dump.empty()) write_text(a.dump, img.serialize());
}

int cmd_simulate(const Args& a) {
  if (!rt::device_available()) raise(Code::Device, "simulate runs on the GPU; no CUDA device is visible");
  Image img = images(a);
  rt::upload(img);
  if (a.sequential) {
    need_inputs(a, 2);
    Loaded k1 = load_source(read_text(a.inputs[0])), k2 = load_source(read_text(a.inputs[1]));
    rt::Module m1 = rt::compile(emit_sm100(k1.kernel, k1.prog.funcs));
    rt::Module m2 = rt::compile(emit_sm100(k2.kernel, k2.prog.funcs));
    // Parity run first (the timed repetitions mutate accumulating outputs).
    rt::launch(m1, img, a.grid);
    rt::launch(m2, img, a.grid);
    rt::download(img);
    Image timing = images(a);
    rt::upload(timing);
    rt::Timing t = rt::time(rt::Mode::Sequential, m1, &m2, timing, a.grid, a.grid, a.warmup, a.reps, true);
    std::printf("k1_us = %.3f\n", rt::time(rt::Mode::Single, m1, nullptr, timing, a.grid, 0, a.warmup, a.reps, true).median_us);
    std::printf("k2_us = %.3f\n", rt::time(rt::Mode::Single, m2, nullptr, timing, a.grid, 0, a.warmup, a.reps, true).median_us);
    rt::Timing t2 = rt::time(rt::Mode::TwoStream, m1, &m2, timing, a.grid, a.grid, a.warmup, a.reps, true);
    std::printf("two_stream_us = %.3f\n", t2.median_us);
    print_run(t.median_us, img, a);
    return 0;
  }
  need_inputs(a, 1);
  Loaded k = load_source(read_text(a.inputs[0]), a.entry);
  std::optional<int> cap;
  if (a.regcap == "auto") cap = k.kernel.regcap;
  else if (a.regcap != "off") cap = std::stoi(a.regcap);
  rt::Module m = rt::compile(emit_sm100(k.kernel, k.prog.funcs), cap);
  rt::launch(m, img, a.grid);
  rt::download(img);
  Image timing = images(a);
  rt::upload(timing);
  rt::Timing t = rt::time(rt::Mode::Single, m, nullptr, timing, a.grid, 0, a.warmup, a.reps, true);
  std::printf("registers = %d\n", m.regs);
  std::printf("blocks_per_sm = %d\n", m.blocks_per_sm);
  print_run(t.median_us, img, a);
  return 0;
}

int cmd_search(const Args& a) {
  need_inputs(a, 2);
  Loaded l1 = load_source(read_text(a.inputs[0])), l2 = load_source(read_text(a.inputs[1]));
  Kernel n1 = normalize(l1.kernel, l1.prog.funcs, "k1_");
  Kernel n2 = normalize(l2.kernel, l2.prog.funcs, "k2_");
  if (a.grid > 0) n1.grid = n2.grid = a.grid;
  SearchOptions so;
  so.granularity = a.granularity;
  so.interval_regs = a.budgets;
  so.prefilter = a.prefilter;
  if (a.prefilter_tol >= 0) so.prefilter_tol = a.prefilter_tol;
  if (!a.caps.empty()) {
    std::stringstream ss(a.caps);
    std::string c;
    while (std::getline(ss, c, ',')) so.extra_caps.push_back(std::stoi(c));
  }
  std::unique_ptr<ProfilerBackend> be;
  Image img;
  SM sm = a.sm_given ? SM::preset_or_file(a.sm) : SM::b200();
  if (!a.profiler_cmd.empty()) {
    // budgets exist only in sm100 text, so a budget sweep hands the command sm100 candidates
    be = std::make_unique<ExternalCommandBackend>(a.profiler_cmd, a.budgets ? Style::Sm100 : Style::Goto);
  } else {
    if (!rt::device_available()) raise(Code::Device, "search times candidates on the GPU; no CUDA device is visible");
    if (!a.sm_given) sm = rt::sm_from_device();
    img = images(a);
    rt::upload(img);
    auto dev = std::make_unique<DeviceBackend>(img, a.grid, a.warmup, a.reps, true);
    std::map<std::string, ScalarVal> spec;
    for (const auto& [n, s] : img.scalars) spec[n] = ScalarVal{s.ty, s.i, s.f};
    dev->set_specialization(spec);  // JIT-specialize every candidate to the image's shapes
    be = std::move(dev);
  }
  SearchResult r = (n1.tunable && n2.tunable) ? search_config(n1, n2, a.d0, *be, sm, so)
                                              : fixed_partition_fuse(n1, n2, *be, sm, a.d0, so);
  std::printf("evaluated = %zu\n", r.trace.size());
  std::printf("best_d1 = %d\n", r.best_cfg.d1);
  std::printf("best_d2 = %d\n", r.best_cfg.d2);
  std::printf("best_reg_cap = %s\n", r.best_cfg.reg_cap ? std::to_string(*r.best_cfg.reg_cap).c_str() : "none");
  if (r.best_cfg.regs1 > 0) std::printf("best_interval_regs = %d/%d\n", r.best_cfg.regs1, r.best_cfg.regs2);
  std::printf("best_cycles = %lld\n", (long long)r.best_time);
  if (!a.trace.empty()) {
    write_text(a.trace, trace_csv(r));
    std::printf("wrote %s\n", a.trace.c_str());
  }
  if (!a.out.empty()) {
    std::string style = a.style.empty() ? "structured" : a.style;
    Style st = style == "goto" ? Style::Goto : style == "sm100" ? Style::Sm100 : Style::Structured;
    write_text(a.out, emit(r.best, st));
    std::printf("wrote %s\n", a.out.c_str());
  }
  return 0;
}

// `hfuse profile CANDIDATE --mem IMG...`: the B200 profiler command for the reference's
// ExternalCommandBackend (search.cpp:32-62). The candidate is the goto-style CUDA text (or
// structured .mk) mkfuse writes as <fused>_<d1>_<regcap|0>_<n>.<ext>; the register cap is
// recovered from that name. Prints the median device time in ns first (the "cycle count"
// mkfuse reads), then `us = ...`.
int cmd_profile(const Args& a) {
  need_inputs(a, 1);
  if (!rt::device_available()) raise(Code::Device, "profile runs on the GPU; no CUDA device is visible");
  std::filesystem::path path(a.inputs[0]);
  std::string text = read_text(path.string());
  Image img = images(a);
  rt::upload(img);
  std::optional<int> cap;
  {
    std::vector<std::string> parts;
    std::stringstream ss(path.stem().string());
    std::string p;
    while (std::getline(ss, p, '_')) parts.push_back(p);
    if (parts.size() >= 3) {
      char* end = nullptr;
      long v = std::strtol(parts[parts.size() - 2].c_str(), &end, 10);
      if (end && *end == '\0' && v > 0) cap = int(v);
    }
  }
  Sm100Kernel k;
  if (path.extension() == ".mk") {
    Loaded l = load_source(text, a.entry);
    if (a.grid > 0) l.kernel.grid = a.grid;
    if (!cap && l.kernel.regcap) cap = l.kernel.regcap;
    Sm100Options o;
    for (const auto& [n, s] : img.scalars) o.specialize[n] = ScalarVal{s.ty, s.i, s.f};
    k = emit_sm100(l.kernel, l.prog.funcs, o);
  } else {
    k = wrap_goto(text, a.grid);
  }
  rt::Module m = rt::compile(k, cap);
  rt::Timing t = rt::time(rt::Mode::Single, m, nullptr, img, a.grid, 0, a.warmup, a.reps, true);
  std::printf("%lld\n", (long long)(t.iqm_us * 1000.0 + 0.5));
  std::printf("us = %.3f\nregisters = %d\nblocks_per_sm = %d\n", t.iqm_us, m.regs, m.blocks_per_sm);
  rt::unload(m);
  return 0;
}

int cmd_occupancy(const Args& a) {
  SM sm = SM::preset_or_file(a.sm);
  Resources res;
  if (!a.inputs.empty()) {
    Loaded l = load_source(read_text(a.inputs[0]), a.entry);
    Kernel k = inline_calls(l.kernel, l.prog.funcs);
    res = resources_of(k);
    std::printf("kernel = %s\n", k.name.c_str());
    std::printf("regs_per_thread = %d\n", res.regs);
    std::printf("shmem_per_block = %lld\n", (long long)res.shmem);
    std::printf("threads_per_block = %d\n", res.threads);
  } else {
    if (a.regs <= 0 || a.threads <= 0)
      raise(Code::InvalidArgument, "occupancy needs a kernel file or --regs/--threads");
    res = Resources{a.regs, a.shmem, a.threads};
  }
  Occupancy o = occupancy(res, sm);
  std::printf("blocks_per_sm = %d\n", o.blocks_per_sm);
  std::printf("limiting_resource = %s\n", limit_name(o.limiting));
  std::printf("achieved_warps = %d\n", o.warps);
  std::printf("occupancy_fraction = %.6f\n", o.fraction);
  return 0;
}

int cmd_check(const Args& a) {
  need_inputs(a, 1);
  Program p = parse(read_text(a.inputs[0]));
  std::printf("ok: %zu kernel(s), %zu function(s)\n", p.kernels.size(), p.funcs.size());
  for (const auto& w : lint(p)) std::printf("lint %d:%d: %s\n", w.pos.line, w.pos.col, w.msg.c_str());
  return 0;
}

int cmd_lower(const Args& a) {
  need_inputs(a, 1);
  std::string text = print_mk(downlower(parse(read_text(a.inputs[0]))));
  parse(text, Dialect::Strict);
  if (a.out.empty()) std::fputs(text.c_str(), stdout);
  else write_text(a.out, text);
  return 0;
}

int cmd_emit(const Args& a) {
  need_inputs(a, 1);
  Loaded l = load_source(read_text(a.inputs[0]), a.entry);
  std::string text = emit_sm100(l.kernel, l.prog.funcs).source;
  if (a.out.empty()) std::fputs(text.c_str(), stdout);
  else write_text(a.out, text);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    Args a = parse_args(argc, argv);
    if (a.cmd == "fuse") return cmd_fuse(a);
    if (a.cmd == "simulate") return cmd_simulate(a);
    if (a.cmd == "search") return cmd_search(a);
    if (a.cmd == "occupancy") return cmd_occupancy(a);
    if (a.cmd == "check") return cmd_check(a);
    if (a.cmd == "lower") return cmd_lower(a);
    if (a.cmd == "emit") return cmd_emit(a);
    if (a.cmd == "profile") return cmd_profile(a);
    raise(Code::InvalidArgument, "unknown command '" + a.cmd + "'");
  } catch (const Error& e) {
    std::fprintf(stderr, "error%s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
