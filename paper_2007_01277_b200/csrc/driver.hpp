// Shared front half of the CLI and the C ABI: load sources, normalize, fuse, report.
// Mirrors cmd_fuse of the reference CLI (/root/reference/proj/tools/mkfuse.cpp:72-167).
#pragma once

#include <optional>
#include <string>

#include "fuser.hpp"

namespace hf {

struct Loaded {
  Program prog;
  Kernel kernel;
};
Loaded load_source(const std::string& src, const std::string& entry = "",
                   Dialect dialect = Dialect::B200);

struct FuseResult {
  SM sm;
  Kernel n1, n2;
  Fused fused;
  Resources r1, r2, rf;
  int r0 = -1;  // register bound, -1 when infeasible
};

// regcap: "auto" (record r0), "off", or a positive integer (mkfuse.cpp:118-133).
FuseResult fuse_sources(const std::string& src1, const std::string& src2, int d1, int d2,
                        const std::string& regcap, const SM& sm, int grid = 0);  // grid > 0: the common launch grid (overrides both //@ grid)
std::string fuse_report(const FuseResult& r);
std::string emit(const Fused& f, Style style);
std::string read_text(const std::string& path);
Sm100Kernel wrap_goto(const std::string& goto_text, int grid);
// Exported sm_100a candidate text (register cap as __maxnreg__, manifest first line) and back.
std::string sm100_text(const Sm100Kernel& k, std::optional<int> cap);
bool is_sm100_text(const std::string& text);
Sm100Kernel parse_sm100_text(const std::string& text, int grid);

}  // namespace hf
