// Goto-style CUDA text of a fused kernel, byte-compatible with the reference's
// CudaPrinter (/root/reference/proj/src/fuser.cpp:290-549) so `hfuse fuse --style goto`
// is a drop-in for `mkfuse fuse` (golden: proj/tests/golden/fused_batchnorm_histogram.cu).
// This is the "naive fusion" baseline text; the B200 product path is emit_sm100.cpp.
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>

#include "fuser.hpp"

namespace hf {
namespace {

int prec(Bin op) {
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

const char* op(Bin b) {
  static const char* t[] = {"+", "-", "*", "/", "%", "<<", ">>", "&", "^", "|",
                            "<", "<=", ">", ">=", "==", "!=", "&&", "||"};
  return t[int(b)];
}

struct GotoPrinter {
  std::string o;

  void pad(int n) { o.append(size_t(n) * 2, ' '); }

  std::string ex(const Expr& e, int parent = 0) {
    switch (e.k) {
      case EK::Int: return std::to_string(e.i);
      case EK::Float: {
        char buf[64];
        std::snprintf(buf, sizeof(buf), "%.9g", double(e.f));
        std::string s(buf);
        if (s.find('.') == std::string::npos && s.find('e') == std::string::npos) s += ".0";
        return s + "f";
      }
      case EK::Var: return e.s;
      case EK::Builtin: {
        static const char* t[] = {"threadIdx.x", "threadIdx.y", "threadIdx.z", "blockIdx.x",
                                  "blockIdx.y",  "blockIdx.z",  "blockDim.x",  "blockDim.y",
                                  "blockDim.z",  "gridDim.x"};
        return t[e.i];
      }
      case EK::Unary: {
        std::string t = (Un(e.i) == Un::Neg ? "-" : "!") + ex(e.a[0], 11);
        return 11 < parent ? "(" + t + ")" : t;
      }
      case EK::Binary: {
        int p = prec(Bin(e.i));
        std::string t = ex(e.a[0], p) + " " + op(Bin(e.i)) + " " + ex(e.a[1], p + 1);
        return p < parent ? "(" + t + ")" : t;
      }
      case EK::Index: return e.s + "[" + ex(e.a[0]) + "]";
      case EK::Intrin:
        switch (Intr(e.i)) {
          case Intr::CastInt:
          case Intr::IntRz: return "(int)(" + ex(e.a[0]) + ")";
          case Intr::Acquire:
          case Intr::Relaxed: return ex(e.a[0]);
          case Intr::CastFloat: return "(float)(" + ex(e.a[0]) + ")";
          default: {
            std::string t = std::string(intr_name(Intr(e.i))) + "(";
            for (size_t i = 0; i < e.a.size(); ++i) t += (i ? ", " : "") + ex(e.a[i]);
            return t + ")";
          }
        }
      case EK::Shfl:
        return "__shfl_xor_sync(0xffffffff, " + ex(e.a[0]) + ", " + std::to_string(e.i) + ")";
      case EK::Call: {
        std::string t = e.s + "(";
        for (size_t i = 0; i < e.a.size(); ++i) t += (i ? ", " : "") + ex(e.a[i]);
        return t + ")";
      }
    }
    return "?";
  }

  std::string lv(const Stmt& s) { return s.idx.empty() ? s.name : s.name + "[" + ex(s.idx[0]) + "]"; }

  std::string simple(const Stmt& s) {
    if (s.k == SK::Decl)
      return std::string(ty_name(s.ty)) + " " + s.name + (s.val.empty() ? "" : " = " + ex(s.val[0]));
    if (s.k == SK::Assign) return lv(s) + " = " + ex(s.val[0]);
    return "";
  }

  void stmt(const Stmt& s, int ind) {
    switch (s.k) {
      case SK::Decl:
        pad(ind);
        o += simple(s) + ";\n";
        break;
      case SK::Assign:
        pad(ind);
        o += lv(s) + " = " + ex(s.val[0]) + ";\n";
        break;
      case SK::If:
        pad(ind);
        o += "if (" + ex(s.val[0]) + ") {\n";
        for (const auto& x : s.body) stmt(x, ind + 1);
        pad(ind);
        o += "}";
        if (s.has_alt) {
          o += " else {\n";
          for (const auto& x : s.alt) stmt(x, ind + 1);
          pad(ind);
          o += "}";
        }
        o += "\n";
        break;
      case SK::For:
        pad(ind);
        o += "for (" + simple(s.init[0]) + "; " + ex(s.val[0]) + "; " + simple(s.step[0]) + ") {\n";
        for (const auto& x : s.body) stmt(x, ind + 1);
        pad(ind);
        o += "}\n";
        break;
      case SK::While:
        pad(ind);
        o += "while (" + ex(s.val[0]) + ") {\n";
        for (const auto& x : s.body) stmt(x, ind + 1);
        pad(ind);
        o += "}\n";
        break;
      case SK::Sync:
        pad(ind);
        o += "__syncthreads();\n";
        break;
      case SK::Fence:
        pad(ind);
        o += "__threadfence();\n";
        break;
      case SK::WarpSync:
        pad(ind);
        o += "__syncwarp();\n";
        break;
      case SK::BarSync:
        pad(ind);
        o += "asm(\"bar.sync " + std::to_string(s.bid) + ", " + std::to_string(s.bcount) + ";\");\n";
        break;
      case SK::Atomic:
        pad(ind);
        o += "atomicAdd(&" + lv(s) + ", " + ex(s.val[0]) + ");\n";
        break;
      case SK::Return:
        pad(ind);
        o += "return;\n";
        break;
      case SK::Call: {
        pad(ind);
        o += s.name + "(";
        for (size_t i = 0; i < s.val.size(); ++i) o += (i ? ", " : "") + ex(s.val[i]);
        o += ");\n";
        break;
      }
      case SK::Label:
        o += s.name + ":;\n";
        break;
      case SK::Goto:
        pad(ind);
        o += "goto " + s.name + ";\n";
        break;
      case SK::VLoad:
      case SK::VStore:
      case SK::AsyncCopy:
      case SK::AsyncWait:
        // MK+ statements have no reference spelling; expand them element-wise so the
        // naive text stays plain CUDA.
        raise(Code::InvalidArgument,
              "goto emission needs plain Mini-Kernel (downlower MK+ kernels first)", s.pos);
    }
  }

  std::string negated(const Expr& g) {
    if (g.k == EK::Binary && Bin(g.i) == Bin::Ge) return ex(g.a[0]) + " < " + ex(g.a[1]);
    return "!(" + ex(g) + ")";
  }

  void fused(const Fused& f) {
    o += "__global__ void " + f.name + "(";
    for (size_t i = 0; i < f.params.size(); ++i) {
      if (i) o += ", ";
      o += ty_name(f.params[i].ty);
      o += f.params[i].array ? "* " : " ";
      o += f.params[i].name;
    }
    o += ") {\n";
    for (const auto& s : f.prologue_decls) stmt(s, 1);
    for (const auto& s : f.prologue) stmt(s, 1);
    for (const auto& sh : f.shared) {
      pad(1);
      o += std::string("__shared__ ") + ty_name(sh.ty) + " " + sh.name + "[" + std::to_string(sh.len) +
           "];\n";
    }
    for (const auto& s : f.decls) stmt(s, 1);
    pad(1);
    o += "if (" + negated(f.guard1) + ") goto K1_end;\n";
    for (const auto& s : f.body1) stmt(s, 1);
    o += "K1_end:;\n";
    pad(1);
    o += "if (" + negated(f.guard2) + ") goto K2_end;\n";
    for (const auto& s : f.body2) stmt(s, 1);
    o += "K2_end:;\n";
    o += "}\n";
  }
};

}  // namespace

std::string emit_goto(const Fused& f) {
  GotoPrinter p;
  p.fused(f);
  return p.o;
}

// ---- machine config files (machine.cpp:55-104 format: `key = value`, '#' comments) ----

SM SM::from_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) raise(Code::Io, "cannot open machine config '" + path + "'");
  SM sm;
  std::map<std::string, int64_t*> wide = {{"regs_per_sm", &sm.regs_per_sm},
                                          {"shmem_per_sm", &sm.shmem_per_sm},
                                          {"max_shmem_per_block", &sm.max_shmem_per_block}};
  std::map<std::string, int*> narrow = {
      {"max_threads_per_sm", &sm.max_threads_per_sm},
      {"max_threads_per_block", &sm.max_threads_per_block},
      {"warp_size", &sm.warp_size},
      {"max_blocks_per_sm", &sm.max_blocks_per_sm},
      {"num_sms", &sm.num_sms},
      {"issue_slots", &sm.issue_slots},
      {"mem_slots_per_cycle", &sm.mem_slots_per_cycle},
      {"compute_cycles", &sm.lat_compute},
      {"memory_cycles", &sm.lat_memory},
      {"shuffle_cycles", &sm.lat_shuffle},
      {"atomic_cycles", &sm.lat_atomic}};
  std::string line;
  int no = 0;
  while (std::getline(in, line)) {
    ++no;
    auto h = line.find('#');
    if (h != std::string::npos) line.erase(h);
    std::istringstream row(line);
    std::string key, eq;
    int64_t v;
    if (!(row >> key)) continue;
    if (!(row >> eq >> v) || eq != "=") raise(Code::Io, "bad config line in '" + path + "'", Pos{no, 1});
    if (auto it = wide.find(key); it != wide.end()) *it->second = v;
    else if (auto it2 = narrow.find(key); it2 != narrow.end()) *it2->second = int(v);
    else raise(Code::Io, "unknown config key '" + key + "' in '" + path + "'", Pos{no, 1});
  }
  sm.check();
  return sm;
}

SM SM::preset_or_file(const std::string& spec) {
  if (spec.empty() || spec == "pascal-like") return pascal_like();
  if (spec == "volta-like") return volta_like();
  if (spec == "b200") return b200();
  return from_file(spec);
}

}  // namespace hf
