// hfuse — the B200 drop-in for the reference CLI (/root/reference/proj/tools/mkfuse.cpp).
//
//   hfuse fuse K1 K2 --d1 N --d2 N [--style goto|structured|sm100] [--regcap n|auto|off] [-o F] [--sm S]
//              [--interval-regs R1,R2]   (sm100: per-interval setmaxnreg budgets instead of --regcap)
//   hfuse simulate K [--mem IMG]... [--seed S] [--regcap n|auto|off] [--dump-mem F] [--entry E]
//   hfuse simulate --sequential K1 K2 --mem IMG... [--dump-mem F]
//   hfuse search K1 K2 [--d0 N] --mem IMG... [--trace F] [-o F] [--style S] [--profiler-cmd CMD]
//                      [--gpus N]  (time the sweep's candidates on N GPUs at once)
//                      [--baseline seq|2stream|both]  (time the unfused members against the winner)
//                      [--granularity G] [--caps 32,40,...] [--reps N] [--budgets]
//                      (--budgets: also sweep per-interval setmaxnreg register budgets)
//                      [--prefilter K [--prefilter-tol F]]  (time only the K partitions the B200
//                      model ranks best, plus those predicted within F of the best; default 0.03)
//   hfuse occupancy [K] [--regs N --shmem B --threads T] [--sm S]
//   hfuse check K              hfuse lower K [-o F]           hfuse emit K [-o F]
//   hfuse profile CANDIDATE(.cu|.mk) --mem IMG... [--grid G] [--reps N] [--no-flush]
//                              (mkfuse --profiler-cmd target; --no-flush: steady graph protocol)
//
// Same flags, stdout keys and exit codes (0 ok; 1 + "error[Code] l:c: msg" on stderr).
// `simulate` and `search` run on the GPU: the reference's cycle simulator is replaced by
// device execution (elapsed_us from CUDA events); `--sm` defaults to pascal-like for
// `fuse`/`occupancy` (report parity) and to the live device for GPU commands.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
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
  bool launch_only = false, counters = true, no_flush = false;
  int gpus = 1;
  std::string baseline;
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
    else if (s == "--launch-only") a.launch_only = true;  // internal: the ncu counter pass
    else if (s == "--no-counters") a.counters = false;
    else if (s == "--no-flush") a.no_flush = true;
    else if (s == "--gpus") a.gpus = num();
    else if (s == "--baseline") {
      a.baseline = val();
      if (a.baseline != "seq" && a.baseline != "2stream" && a.baseline != "both")
        raise(Code::InvalidArgument, "--baseline takes seq, 2stream or both");
    }
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
    write_text(path, sm100_text(k, std::nullopt));
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

// ---- simulate on the device --------------------------------------------------------------
// The reference prints run_timed's ProfileResult (exec.cpp:995-1007; --sequential adds
// k1_cycles / k2_cycles and combines the rest with combined_utilization, mkfuse.cpp:180-196).
// Here every key comes from a device measurement:
//   *_cycles                 graph-timed mean launch time x the SM clock (cudaDevAttrClockRate)
//   issue_slot_utilization   ncu smsp__issue_active (elapsed cycles, all schedulers)
//   achieved_occupancy       ncu sm__warps_active (of the peak warps per SM, elapsed)
//   meminst_stall_fraction   ncu (long_scoreboard + lg_throttle) / all stall reasons per issue
//   spill_loads_stores       ncu local-memory load + store instructions executed
// The ncu values come from one counter pass: the same command re-run under ncu with
// --launch-only (each kernel launched once). Without ncu (or --no-counters) they print as nan.
std::vector<std::string> g_argv;

struct Counters {
  double util = NAN, occ = NAN, mem = NAN;
  long long spills = -1;
};

std::vector<std::string> csv_fields(const std::string& line) {
  std::vector<std::string> out;
  std::string cur;
  bool q = false;
  for (char ch : line) {
    if (ch == '"') q = !q;
    else if (ch == ',' && !q) {
      out.push_back(cur);
      cur.clear();
    } else cur += ch;
  }
  out.push_back(cur);
  return out;
}

std::string ncu_path() {
  if (const char* e = std::getenv("HFUSE_NCU")) return e;
  for (const char* p : {"/usr/local/cuda/bin/ncu", "/usr/bin/ncu"})
    if (std::filesystem::exists(p)) return p;
  return "";
}

std::vector<Counters> counter_pass() {
  std::string ncu = ncu_path();
  if (ncu.empty()) return {};
  const char* metrics =
      "smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_elapsed,"
      "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,"
      "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,"
      "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio,"
      "smsp__average_warps_active_per_issue_active.ratio,"
      "smsp__sass_inst_executed_op_local_ld.sum,smsp__sass_inst_executed_op_local_st.sum";
  std::string cmd = ncu + " --csv --clock-control none --metrics " + metrics + " " + std::filesystem::read_symlink("/proc/self/exe").string();
  for (size_t i = 1; i < g_argv.size(); ++i) cmd += " '" + g_argv[i] + "'";
  cmd += " --launch-only 2>/dev/null";
  FILE* pipe = popen(cmd.c_str(), "r");
  if (!pipe) return {};
  std::vector<std::string> header;
  std::vector<std::pair<std::string, std::map<std::string, double>>> rows;  // (ID, metrics) in order
  char buf[4096];
  while (std::fgets(buf, sizeof(buf), pipe)) {
    std::string line(buf);
    while (!line.empty() && (line.back() == '\n' || line.back() == '\r')) line.pop_back();
    if (line.empty() || line[0] != '"') continue;
    std::vector<std::string> f = csv_fields(line);
    if (header.empty()) {
      header = f;
      continue;
    }
    auto col = [&](const char* name) -> std::string {
      for (size_t i = 0; i < header.size() && i < f.size(); ++i)
        if (header[i] == name) return f[i];
      return "";
    };
    std::string kname = col("Kernel Name");
    if (kname.rfind("fill_", 0) == 0 || kname.rfind("flush", 0) == 0 || kname.rfind("phase_spin", 0) == 0) continue;
    std::string id = col("ID"), v = col("Metric Value");
    v.erase(std::remove(v.begin(), v.end(), ','), v.end());
    if (rows.empty() || rows.back().first != id) rows.push_back({id, {}});
    rows.back().second[col("Metric Name")] = std::strtod(v.c_str(), nullptr);
  }
  if (pclose(pipe) != 0) return {};
  std::vector<Counters> out;
  for (auto& [id, m] : rows) {
    Counters k;
    auto get = [&](const char* n) { return m.count(n) ? m[n] : NAN; };
    k.util = get("smsp__issue_active.avg.pct_of_peak_sustained_elapsed") / 100.0;
    k.occ = get("sm__warps_active.avg.pct_of_peak_sustained_elapsed") / 100.0;
    double stalled = get("smsp__average_warps_active_per_issue_active.ratio") -
                     get("smsp__average_warps_issue_stalled_selected_per_issue_active.ratio");
    k.mem = (get("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio") +
             get("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio")) /
            stalled;
    double sp = get("smsp__sass_inst_executed_op_local_ld.sum") + get("smsp__sass_inst_executed_op_local_st.sum");
    k.spills = std::isnan(sp) ? -1 : (long long)sp;
    out.push_back(k);
  }
  return out;
}

void print_profile(long long cycles, const Counters& k) {
  // profile_report's keys and formats (exec.cpp:995-1007)
  std::printf("elapsed_cycles = %lld\n", cycles);
  std::printf("issue_slot_utilization = %.6f\n", k.util);
  std::printf("meminst_stall_fraction = %.6f\n", k.mem);
  std::printf("achieved_occupancy = %.6f\n", k.occ);
  std::printf("spill_loads_stores = %lld\n", k.spills);
}

double combined(double u1, long long c1, double u2, long long c2) {
  if (std::isnan(u1) || std::isnan(u2)) return NAN;
  return combined_utilization(u1, c1, u2, c2);  // machine.cpp:285-289
}

int cmd_simulate(const Args& a) {
  if (!rt::device_available()) raise(Code::Device, "simulate runs on the GPU; no CUDA device is visible");
  Image img = images(a);
  rt::upload(img);
  const double mhz = rt::props().clock_khz / 1000.0;
  auto cycles = [&](double us) { return (long long)std::llround(us * mhz); };
  if (a.sequential) {
    need_inputs(a, 2);
    Loaded k1 = load_source(read_text(a.inputs[0])), k2 = load_source(read_text(a.inputs[1]));
    rt::Module m1 = rt::compile(emit_sm100(k1.kernel, k1.prog.funcs));
    rt::Module m2 = rt::compile(emit_sm100(k2.kernel, k2.prog.funcs));
    // Parity run first (the timed repetitions mutate accumulating outputs).
    rt::launch(m1, img, a.grid);
    rt::launch(m2, img, a.grid);
    if (a.launch_only) {
      rt::synchronize();
      return 0;
    }
    rt::download(img);
    Image timing = images(a);
    rt::upload(timing);
    auto gt = [&](rt::Mode md, const rt::Module& x, const rt::Module* y) {
      return rt::time_graph(md, x, y, timing, a.grid, a.grid, std::max(1, a.reps), 5).mean_us;
    };
    double t1 = gt(rt::Mode::Single, m1, nullptr), t2 = gt(rt::Mode::Single, m2, nullptr);
    double tseq = gt(rt::Mode::Sequential, m1, &m2), two = gt(rt::Mode::TwoStream, m1, &m2);
    std::vector<Counters> k = a.counters ? counter_pass() : std::vector<Counters>{};
    Counters c1 = k.size() >= 2 ? k[0] : Counters{}, c2 = k.size() >= 2 ? k[1] : Counters{};
    long long y1 = cycles(t1), y2 = cycles(t2);
    Counters both;
    both.util = combined(c1.util, y1, c2.util, y2);
    both.mem = combined(c1.mem, y1, c2.mem, y2);
    both.occ = combined(c1.occ, y1, c2.occ, y2);
    both.spills = c1.spills < 0 || c2.spills < 0 ? -1 : c1.spills + c2.spills;
    std::printf("k1_cycles = %lld\n", y1);
    std::printf("k2_cycles = %lld\n", y2);
    print_profile(y1 + y2, both);
    std::printf("digest = %s\n", img.digest_hex().c_str());
    // device extras: back to back and two-stream concurrent times of the same pair
    std::printf("k1_us = %.3f\nk2_us = %.3f\nelapsed_us = %.3f\ntwo_stream_us = %.3f\n", t1, t2, tseq, two);
    if (!a.dump.empty()) write_text(a.dump, img.serialize());
    return 0;
  }
  need_inputs(a, 1);
  Loaded k = load_source(read_text(a.inputs[0]), a.entry);
  std::optional<int> cap;
  if (a.regcap == "auto") cap = k.kernel.regcap;
  else if (a.regcap != "off") cap = std::stoi(a.regcap);
  rt::Module m = rt::compile(emit_sm100(k.kernel, k.prog.funcs), cap);
  rt::launch(m, img, a.grid);
  if (a.launch_only) {
    rt::synchronize();
    return 0;
  }
  rt::download(img);
  Image timing = images(a);
  rt::upload(timing);
  double t = rt::time_graph(rt::Mode::Single, m, nullptr, timing, a.grid, 0, std::max(1, a.reps), 5).mean_us;
  std::vector<Counters> ks = a.counters ? counter_pass() : std::vector<Counters>{};
  print_profile(cycles(t), ks.empty() ? Counters{} : ks[0]);
  std::printf("digest = %s\n", img.digest_hex().c_str());
  std::printf("registers = %d\nblocks_per_sm = %d\nelapsed_us = %.3f\n", m.regs, m.blocks_per_sm, t);
  if (!a.dump.empty()) write_text(a.dump, img.serialize());
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
  std::vector<Image> imgs;  // --gpus N: one copy of the memory image per device
  SM sm = a.sm_given ? SM::preset_or_file(a.sm) : SM::b200();
  if (!a.profiler_cmd.empty()) {
    // budgets exist only in sm100 text, so a budget sweep (or --style sm100) hands the command
    // sm100 candidates (manifest + __maxnreg__ cap; `hfuse profile` builds them as they are)
    bool sm100 = a.budgets || a.style == "sm100";
    be = std::make_unique<ExternalCommandBackend>(a.profiler_cmd, sm100 ? Style::Sm100 : Style::Goto);
  } else {
    if (!rt::device_available()) raise(Code::Device, "search times candidates on the GPU; no CUDA device is visible");
    if (!a.sm_given) sm = rt::sm_from_device();
    img = images(a);
    rt::upload(img);
    std::map<std::string, ScalarVal> spec;
    for (const auto& [n, s] : img.scalars) spec[n] = ScalarVal{s.ty, s.i, s.f};
    auto dev = std::make_unique<DeviceBackend>(img, a.grid, a.warmup, a.reps, true);
    dev->set_specialization(spec);  // JIT-specialize every candidate to the image's shapes
    std::vector<int> want;  // devices of the sweep: 0 .. min(--gpus, count) - 1
    for (int d = 0; d < std::min(a.gpus, rt::device_count()); ++d) want.push_back(d);
    if (const char* e = std::getenv("HFUSE_SEARCH_DEVICES")) {  // test knob: an explicit id list
      want.clear();
      std::stringstream ss(e);
      std::string t;
      while (std::getline(ss, t, ',')) want.push_back(std::stoi(t));
    }
    int n = int(want.size());
    if (n > 1) {
      // the candidates of the sweep are timed on n GPUs at once (MultiDeviceBackend)
      std::vector<std::unique_ptr<DeviceBackend>> devs;
      std::vector<int> ids{want[0]};
      int here = 0;
      cudaGetDevice(&here);
      devs.push_back(std::move(dev));
      imgs.resize(size_t(n - 1));
      for (int i = 1; i < n; ++i) {
        int d = want[size_t(i)];
        rt::set_device(d);
        imgs[size_t(i - 1)] = images(a);
        rt::upload(imgs[size_t(i - 1)]);
        auto dd = std::make_unique<DeviceBackend>(imgs[size_t(i - 1)], a.grid, a.warmup, a.reps, true);
        dd->set_specialization(spec);
        devs.push_back(std::move(dd));
        ids.push_back(d);
      }
      rt::set_device(here);
      be = std::make_unique<MultiDeviceBackend>(std::move(devs), ids);
    } else {
      be = std::move(dev);
    }
    std::printf("devices = %d\n", std::max(1, n));
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
  if (!a.baseline.empty()) {
    // the unfused members at their declared dims against the best fused point, graph-timed on
    // the (first) device: sequential a; b and/or two-stream a || b, and the speed-up over the
    // faster of the requested baselines
    if (!a.profiler_cmd.empty()) raise(Code::InvalidArgument, "--baseline needs the device backend");
    std::map<std::string, ScalarVal> spec;
    for (const auto& [n, s] : img.scalars) spec[n] = ScalarVal{s.ty, s.i, s.f};
    Sm100Options o;
    o.specialize = spec;
    rt::Module m1 = rt::compile(emit_sm100(l1.kernel, l1.prog.funcs, o));
    rt::Module m2 = rt::compile(emit_sm100(l2.kernel, l2.prog.funcs, o));
    Sm100Options of;
    of.specialize = spec;
    rt::Module mf = rt::compile(emit_sm100(r.best, of), r.best_cfg.reg_cap);
    int grid = a.grid > 0 ? a.grid : r.best.grid;
    double tf = rt::time_graph(rt::Mode::Single, mf, nullptr, img, grid, 0, std::max(1, a.reps), 5).mean_us;
    double base = 1e300;
    std::printf("best_us = %.3f\n", tf);
    if (a.baseline != "2stream") {
      double t = rt::time_graph(rt::Mode::Sequential, m1, &m2, img, a.grid, a.grid, std::max(1, a.reps), 5).mean_us;
      std::printf("sequential_us = %.3f\n", t);
      base = std::min(base, t);
    }
    if (a.baseline != "seq") {
      double t = rt::time_graph(rt::Mode::TwoStream, m1, &m2, img, a.grid, a.grid, std::max(1, a.reps), 5).mean_us;
      std::printf("two_stream_us = %.3f\n", t);
      base = std::min(base, t);
    }
    std::printf("speedup = %.4f\n", base / tf);
    rt::unload(m1);
    rt::unload(m2);
    rt::unload(mf);
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
  } else if (is_sm100_text(text)) {
    // an sm100 candidate (search --style sm100 --profiler-cmd): the cap is already in the code
    k = parse_sm100_text(text, a.grid);
    cap.reset();
  } else {
    k = wrap_goto(text, a.grid);
  }
  rt::Module m = rt::compile(k, cap);
  // --no-flush: the steady graph protocol (back-to-back repetitions, median of 5 graph samples)
  double us = a.no_flush ? rt::time_graph(rt::Mode::Single, m, nullptr, img, a.grid, 0, std::max(1, a.reps), 5).median_us
                         : rt::time(rt::Mode::Single, m, nullptr, img, a.grid, 0, a.warmup, a.reps, true).iqm_us;
  std::printf("%lld\n", (long long)(us * 1000.0 + 0.5));
  std::printf("us = %.3f\nregisters = %d\nblocks_per_sm = %d\n", us, m.regs, m.blocks_per_sm);
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
    g_argv.assign(argv, argv + argc);
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
