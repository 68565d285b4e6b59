#include "driver.hpp"

#include <cstdio>
#include <fstream>
#include <cstring>
#include <sstream>

namespace hf {

std::string read_text(const std::string& path) {
  std::ifstream in(path);
  if (!in) raise(Code::Io, "cannot open '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

Loaded load_source(const std::string& src, const std::string& entry, Dialect dialect) {
  Loaded l;
  l.prog = parse(src, dialect);
  if (l.prog.kernels.empty()) raise(Code::InvalidArgument, "source defines no kernel");
  if (entry.empty()) {
    l.kernel = l.prog.kernels.front();
  } else {
    const Kernel* k = l.prog.kernel(entry);
    if (!k) raise(Code::InvalidArgument, "source has no kernel '" + entry + "'");
    l.kernel = *k;
  }
  return l;
}

FuseResult fuse_sources(const std::string& src1, const std::string& src2, int d1, int d2,
                        const std::string& regcap, const SM& sm, int grid) {
  FuseResult r;
  r.sm = sm;
  Loaded k1 = load_source(src1), k2 = load_source(src2);
  r.n1 = normalize(k1.kernel, k1.prog.funcs, "k1_");
  r.n2 = normalize(k2.kernel, k2.prog.funcs, "k2_");
  if (grid > 0) r.n1.grid = r.n2.grid = grid;  // members are grid-stride: any common grid works
  r.fused = fuse(r.n1, r.n2, d1, d2, sm);
  r.r1 = resources_of(r.n1, d1);
  r.r2 = resources_of(r.n2, d2);
  r.rf = resources_of(r.fused.to_kernel(), r.fused.cfg.d0);
  try {
    r.r0 = register_bound(r.r1, r.r2, r.rf.shmem, r.fused.cfg.d0, sm);
  } catch (const Error&) {
    r.r0 = -1;
  }
  if (regcap == "auto") {
    if (r.r0 > 0) r.fused.cfg.reg_cap = r.r0;
  } else if (regcap != "off") {
    int v = std::stoi(regcap);
    if (v <= 0) raise(Code::InvalidArgument, "register cap must be positive");
    r.fused.cfg.reg_cap = v;
  }
  return r;
}

std::string fuse_report(const FuseResult& r) {
  const Fused& f = r.fused;
  std::string o;
  char buf[256];
  o += "fused_kernel = " + f.name + "\n";
  std::snprintf(buf, sizeof(buf), "partition = d1 %d (%s), d2 %d (%s), d0 %d\n", f.cfg.d1, f.k1_name.c_str(),
                f.cfg.d2, f.k2_name.c_str(), f.cfg.d0);
  o += buf;
  for (const auto& e : f.barriers) {
    int uses = 0;
    walk(e.owner == 1 ? f.body1 : f.body2, [&](const Stmt& s) {
      if (s.k == SK::BarSync && s.bid == e.id) ++uses;
    });
    std::snprintf(buf, sizeof(buf), "barrier id %d: count %d, constituent %d, uses %d\n", e.id, e.count, e.owner,
                  uses);
    o += buf;
  }
  std::snprintf(buf, sizeof(buf), "registers = k1 %d, k2 %d, fused %d\n", r.r1.regs, r.r2.regs, r.rf.regs);
  o += buf;
  o += "shared_bytes = " + std::to_string(r.rf.shmem) + "\n";
  if (f.cfg.reg_cap) o += "reg_cap = " + std::to_string(*f.cfg.reg_cap) + "\n";
  else if (r.r0 > 0) o += "suggested_reg_cap = " + std::to_string(r.r0) + "\n";
  Resources capped = r.rf;
  if (f.cfg.reg_cap) capped.regs = std::min(capped.regs, *f.cfg.reg_cap);
  Occupancy occ = occupancy(capped, r.sm);
  o += "blocks_per_sm = " + std::to_string(occ.blocks_per_sm) + "\n";
  o += std::string("limiting_resource = ") + limit_name(occ.limiting) + "\n";
  o += "achieved_warps = " + std::to_string(occ.warps) + "\n";
  std::snprintf(buf, sizeof(buf), "occupancy_fraction = %.6f\n", occ.fraction);
  o += buf;
  return o;
}

// The reference's goto-style text (fuser.cpp:290-549) made launchable: `extern "C"` entry,
// parameters parsed from the signature, block size from the prologue's size_1 + size_2.
// Its semantics are the naive CUDA ones (not the interpreter's pinned ones): timing only.
Sm100Kernel wrap_goto(const std::string& text, int grid) {
  Sm100Kernel k;
  size_t g = text.find("__global__ void ");
  if (g == std::string::npos) raise(Code::InvalidArgument, "no __global__ kernel in the candidate");
  size_t name_at = g + std::string("__global__ void ").size();
  size_t lp = text.find('(', name_at), rp = text.find(')', lp);
  k.entry = text.substr(name_at, lp - name_at);
  std::stringstream ps(text.substr(lp + 1, rp - lp - 1));
  std::string item;
  while (std::getline(ps, item, ',')) {
    std::stringstream is(item);
    std::string type, name;
    is >> type >> name;
    if (type.empty()) continue;
    bool array = type.back() == '*';
    if (array) type.pop_back();
    k.params.push_back(Sm100Param{name, type == "float" ? Ty::Float : Ty::Int, array, true, false, {}, array});
  }
  auto size_of = [&](const char* key) {
    size_t at = text.find(key);
    if (at == std::string::npos) raise(Code::InvalidArgument, std::string("candidate has no ") + key);
    return std::atoi(text.c_str() + at + std::strlen(key));
  };
  k.threads = size_of("size_1 = ") + size_of("size_2 = ");
  k.grid = grid > 0 ? grid : 1;
  k.source = text.substr(0, g) + "extern \"C\" " + text.substr(g);
  return k;
}

// Exported sm_100a text: the register cap is part of the code (__maxnreg__ replaces the launch
// bounds -- nvcc ignores --maxrregcount for a kernel that carries __launch_bounds__), and a
// first-line manifest lets `hfuse profile` rebuild the launch metadata from the file alone:
//   // hfuse-sm100 entry=E threads=T smem=S launch_regs=L params=name:af,name:si,...
// (a = array, s = scalar; f = float, i = int).
std::string sm100_text(const Sm100Kernel& k, std::optional<int> cap) {
  std::string s = k.source;
  if (cap) {
    size_t at = s.find("__launch_bounds__(");
    if (at != std::string::npos) s.replace(at, s.find(')', at) - at + 1, "__maxnreg__(" + std::to_string(*cap) + ")");
  }
  std::string m = "// hfuse-sm100 entry=" + k.entry + " threads=" + std::to_string(k.threads) +
                  " smem=" + std::to_string(k.smem_bytes) + " launch_regs=" + std::to_string(k.launch_regs) +
                  " params=";
  for (size_t i = 0; i < k.params.size(); ++i) {
    const Sm100Param& p = k.params[i];
    if (p.specialized) raise(Code::InvalidArgument, "exported sm100 text cannot carry specialized scalars");
    m += (i ? "," : "") + p.name + ":" + (p.array ? "a" : "s") + (p.ty == Ty::Float ? "f" : "i");
  }
  return m + "\n" + s;
}

bool is_sm100_text(const std::string& text) { return text.rfind("// hfuse-sm100 ", 0) == 0; }

// The inverse of sm100_text's manifest (the code itself is compiled as written).
Sm100Kernel parse_sm100_text(const std::string& text, int grid) {
  if (!is_sm100_text(text)) raise(Code::InvalidArgument, "not an hfuse sm100 candidate (no manifest line)");
  std::stringstream line(text.substr(0, text.find('\n')));
  Sm100Kernel k;
  std::string tok;
  line >> tok >> tok;  // "//", "hfuse-sm100"
  while (line >> tok) {
    size_t eq = tok.find('=');
    if (eq == std::string::npos) continue;
    std::string key = tok.substr(0, eq), v = tok.substr(eq + 1);
    if (key == "entry") k.entry = v;
    else if (key == "threads") k.threads = std::stoi(v);
    else if (key == "smem") k.smem_bytes = std::stoll(v);
    else if (key == "launch_regs") k.launch_regs = std::stoi(v);
    else if (key == "params") {
      std::stringstream ps(v);
      std::string item;
      while (std::getline(ps, item, ',')) {
        size_t colon = item.find(':');
        if (colon == std::string::npos || item.size() != colon + 3)
          raise(Code::InvalidArgument, "bad parameter '" + item + "' in the sm100 manifest");
        bool array = item[colon + 1] == 'a';
        Ty ty = item[colon + 2] == 'f' ? Ty::Float : Ty::Int;
        k.params.push_back(Sm100Param{item.substr(0, colon), ty, array, array, false, {}, array});
      }
    }
  }
  if (k.entry.empty() || k.threads <= 0) raise(Code::InvalidArgument, "incomplete sm100 manifest");
  k.grid = grid > 0 ? grid : 1;
  k.source = text;
  return k;
}

std::string emit(const Fused& f, Style style) {
  switch (style) {
    case Style::Structured: return emit_structured(f);
    case Style::Goto: return emit_goto(f);
    case Style::Sm100: return sm100_text(emit_sm100(f), f.cfg.reg_cap);
  }
  return {};
}

}  // namespace hf
