// The reference-side binding of INTEGRATION.md §3, compiled against the UNMODIFIED reference
// (/root/reference/proj/include + the library built by oracle/Makefile) and libhfuse.so: a
// mkfuse::ProfilerBackend whose evaluate() times each candidate on the B200 through the C ABI
// (include/hfuse.h: hf_profile), driven by the reference's own search_config
// (/root/reference/proj/src/search.cpp:124-143). The same program can drive the reference's
// ExternalCommandBackend (search.cpp:32-62) with `hfuse profile` as the command.
//
//   b200_backend K1.mk K2.mk IMG... [--cmd "hfuse profile --mem ... --mem ..."]
// prints the reference's cmd_search keys (mkfuse.cpp:225-231) and the trace CSV (trace_csv).
// Built by `make -C oracle binding` into oracle/_ref/ (it needs the reference headers); run by
// tests/test_binding_gpu.py on the GPU box.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "hfuse.h"
#include "mkfuse/frontend.hpp"
#include "mkfuse/fuser.hpp"
#include "mkfuse/search.hpp"

namespace {

std::string slurp(const std::string& path) {
  std::ifstream in(path);
  if (!in) mkfuse::fail(mkfuse::ErrCode::Io, "cannot open '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// ---- the binding a maintainer adds ---------------------------------
class B200Backend : public mkfuse::ProfilerBackend {
 public:
  B200Backend(std::string src1, std::string src2, const std::string& image_text)
      : s1_(std::move(src1)), s2_(std::move(src2)) {
    hf_error e;
    if (hf_image_parse(image_text.c_str(), 0, 0, &img_, &e) || hf_image_upload(img_, nullptr, &e))
      mkfuse::fail(mkfuse::ErrCode::Io, e.message);
  }
  ~B200Backend() override { hf_image_free(img_); }
  mkfuse::EvalOutcome evaluate(const mkfuse::FusedKernel& f, const mkfuse::FusionConfig& c) override {
    (void)f;
    hf_eval ev;
    hf_error e;
    int cap = c.reg_cap ? *c.reg_cap : HF_REGCAP_OFF;
    if (hf_profile(s1_.c_str(), s2_.c_str(), c.d1, c.d2, cap, img_, /*grid=*/0, /*warmup=*/3,
                   /*reps=*/10, /*flush_l2=*/0, /*specialize=*/1, &ev, &e))
      mkfuse::fail(static_cast<mkfuse::ErrCode>(e.code - 1), e.message);  // same ordinals
    return mkfuse::EvalOutcome{ev.cycles, ev.occupancy, ev.utilization};  // cycles = ns
  }

 private:
  std::string s1_, s2_;
  hf_image* img_ = nullptr;
};
// -----------------------------------------------------------------------------------------

void report(const char* tag, const mkfuse::SearchResult& r) {
  std::printf("[%s]\n", tag);
  std::printf("evaluated = %zu\n", r.trace.size());
  std::printf("best_d1 = %d\n", r.best_config.d1);
  std::printf("best_d2 = %d\n", r.best_config.d2);
  std::printf("best_reg_cap = %s\n",
              r.best_config.reg_cap ? std::to_string(*r.best_config.reg_cap).c_str() : "none");
  std::printf("best_cycles = %lld\n", static_cast<long long>(r.best_time));
  std::fputs(mkfuse::trace_csv(r).c_str(), stdout);
}

}  // namespace

int main(int argc, char** argv) {
  try {
    std::vector<std::string> pos;
    std::string cmd;
    for (int i = 1; i < argc; ++i) {
      std::string s = argv[i];
      if (s == "--cmd" && i + 1 < argc) cmd = argv[++i];
      else pos.push_back(s);
    }
    if (pos.size() < 3) {
      std::fprintf(stderr, "usage: b200_backend K1.mk K2.mk IMG... [--cmd CMD]\n");
      return 2;
    }
    std::string src1 = slurp(pos[0]), src2 = slurp(pos[1]), image;
    for (size_t i = 2; i < pos.size(); ++i) image += slurp(pos[i]) + "\n";
    mkfuse::Program p1 = mkfuse::parse_program(src1), p2 = mkfuse::parse_program(src2);
    mkfuse::Kernel n1 = mkfuse::normalize_kernel(p1.kernels.front(), p1.functions, "k1_");
    mkfuse::Kernel n2 = mkfuse::normalize_kernel(p2.kernels.front(), p2.functions, "k2_");
    mkfuse::SMConfig sm = mkfuse::SMConfig::pascal_like();
    B200Backend dev(src1, src2, image);
    report("B200Backend", mkfuse::search_config(n1, n2, 1024, dev, sm));
    if (!cmd.empty()) {
      mkfuse::ExternalCommandBackend ext(cmd);
      report("ExternalCommandBackend", mkfuse::search_config(n1, n2, 1024, ext, sm));
    }
    return 0;
  } catch (const mkfuse::Error& e) {
    std::fprintf(stderr, "error%s\n", e.what());
    return 1;
  }
}
