// Horizontal fusion (Algorithm "Generate") and the machine model.
//
// Reference contract: /root/reference/proj/include/mkfuse/fuser.hpp:14-77 and
// machine.hpp:20-80. Differences on the B200 path are additive:
//  * barrier allocation: pre-existing bar_sync(id, n) statements of each constituent are
//    remapped to fresh named-barrier ids (the reference passes them through and lets the
//    two constituents collide); more than 15 ids -> BadBarrierId;
//  * an `sm100` emitter (emit_sm100.cpp) next to the byte-compatible goto / structured ones.
#pragma once

#include <map>
#include <optional>
#include <string>
#include <vector>

#include "ir.hpp"

namespace hf {

struct SM {
  int64_t regs_per_sm = 65536;
  int64_t shmem_per_sm = 98304;
  int max_threads_per_sm = 2048;
  int max_threads_per_block = 1024;
  int warp_size = 32;
  int max_blocks_per_sm = 32;
  int num_sms = 1;
  int issue_slots = 4;
  int mem_slots_per_cycle = 2;
  int lat_compute = 4, lat_memory = 400, lat_shuffle = 8, lat_atomic = 48;
  int64_t max_shmem_per_block = 49152;  // static limit; the b200 preset opts in to 227 KB

  static SM pascal_like();
  static SM volta_like();
  static SM b200();  // sm_100a constants; the runtime refreshes them
  static SM from_file(const std::string& path);
  static SM preset_or_file(const std::string& spec);
  void check() const;
};

struct Resources {
  int regs = 1;
  int64_t shmem = 0;
  int threads = 1;
};

enum class Limit { Registers, SharedMemory, Threads, BlockSlots };
const char* limit_name(Limit l);

struct Occupancy {
  int blocks_per_sm = 0;
  Limit limiting = Limit::Registers;
  int warps = 0;
  double fraction = 0.0;
};

int estimate_registers(const Kernel& k);  // peak live locals + 8 (machine.cpp:115-220)
Resources resources_of(const Kernel& k, std::optional<int> threads = std::nullopt);
Occupancy occupancy(const Resources& r, const SM& sm);
int register_bound(const Resources& r1, const Resources& r2, int64_t fused_shmem, int d0,
                   const SM& sm);
double combined_utilization(double u1, int64_t c1, double u2, int64_t c2);

struct FusionConfig {
  int d1 = 0, d2 = 0, d0 = 0;
  std::optional<int> reg_cap;
  // B200 extension: per-interval register budgets (setmaxnreg; see Sm100Options), 0 = off.
  // Exclusive with reg_cap; only the sm100 emitter honours them.
  int regs1 = 0, regs2 = 0;
  void check(const SM& sm) const;
};

struct BarrierEntry {
  int id = 0;
  int count = 0;
  int owner = 0;      // constituent 1 or 2
  int original = -1;  // -1: replaces syncthreads(); else the constituent's bar_sync id
};

struct Fused {
  std::string name, k1_name, k2_name;
  std::vector<Param> params;  // merged, deduplicated by name
  std::vector<SharedArr> shared;
  Block prologue_decls, decls, prologue;
  Expr guard1, guard2;
  Block body1, body2;
  std::vector<BarrierEntry> barriers;
  FusionConfig cfg;
  int grid = 1;
  Dims dims1, dims2;
  std::vector<Expr> reqs;  // MK+ launch preconditions of both constituents

  Kernel to_kernel() const;  // canonical structured form (valid Mini-Kernel)
};

Block build_prologue(Dims dims1, Dims dims2, int d1);
Block rewrite_builtins(const Block& body);
Block replace_barriers(const Block& body, int id, int count);
Fused fuse(const Kernel& k1, const Kernel& k2, int d1, int d2, const SM& sm);
Kernel vertical_fuse(const Kernel& k1, const Kernel& k2);  // VFuse baseline (normalized inputs)
Dims partition_dims(const Kernel& k, int d);

enum class Style { Structured, Goto, Sm100 };
std::string emit_goto(const Fused& f);        // byte-compatible with fuser.cpp:290-558
std::string emit_structured(const Fused& f);  // emit_minikernel(to_kernel())

// ---- sm_100a emission -----------------------------------------------------------
struct ScalarVal {
  Ty ty = Ty::Int;
  int32_t i = 0;
  float f = 0.0f;
};

struct Sm100Options {
  std::string entry;       // extern "C" symbol (default: the kernel name)
  int min_blocks = 0;      // __launch_bounds__(threads, min_blocks) when > 0
  bool zero_shared = true; // the interpreter zero-initializes shared memory per block
  // JIT specialization: scalar parameters (never assigned by the kernel) whose launch
  // values are folded into the code as constants; the runtime checks them at bind time.
  std::map<std::string, ScalarVal> specialize;
  // Per-interval register budgets (fused kernels only; 0 = off). B200 mechanics: the kernel
  // is compiled with __maxnreg__(launch) where launch * d0 >= regs1 * d1 + regs2 * d2, and
  // each interval re-sizes its warpgroups' allocation on entry with setmaxnreg.dec/.inc, so
  // the two constituents no longer share one register count (the reference's single
  // reg_cap, machine.cpp:269-283). Needs warpgroup-aligned intervals (d1, d2 % 128 == 0).
  int regs1 = 0, regs2 = 0;
  // Dynamic interval scheduling (fused kernels only; 0 = off, the reference's static
  // partition). Each interval runs its member as `vgridN` VIRTUAL blocks drawn one at a time
  // from its own atomic counter in the module (blockIdx.x / gridDim.x of the member become the
  // virtual block id / vgridN), so a long-running block of one member no longer strands the
  // other member's share of that CTA: the physical grid is persistent and each interval keeps
  // pulling work until its own queue is empty. Preserves the semantics of the member launched
  // with vgridN blocks (blocks are independent in CUDA); per virtual block the interval's
  // locals and shared arrays start zeroed, as in the interpreter (exec.cpp:291).
  int vgrid1 = 0, vgrid2 = 0;
  // Heterogeneous CTA partition (fused kernels only; 0 = off): blocks below split_grid run both
  // members (member 1 sees a grid of split_grid blocks), blocks above give every thread to member
  // 2 as d0/d2 sub-blocks (member 2 sees one grid of split_grid + (grid - split_grid) * d0/d2
  // blocks of d2 threads). For a member 1 with a fixed natural grid (BatchNorm's one block per
  // channel) next to a grid-stride member 2 without barriers or shared memory.
  int split_grid = 0;
};

struct Sm100Param {
  std::string name;
  Ty ty;
  bool array;
  bool written;             // array parameters only
  bool specialized = false; // scalar folded into the code (value below)
  ScalarVal value;
  bool read = false;        // array parameters: prior contents are loaded (or atomically updated)
};

struct Sm100Kernel {
  std::string source;
  std::string entry;
  int threads = 0;       // 1-D block
  int grid = 1;
  int64_t smem_bytes = 0;  // dynamic shared memory
  std::vector<Sm100Param> params;
  std::vector<BarrierEntry> barriers;
  // setmaxnreg budgets: per-thread registers at launch (the pool is launch_regs * threads)
  // and per interval; 0 = not used. The runtime refuses a module whose ptxas count differs
  // from launch_regs (an undersized pool would block setmaxnreg.inc forever).
  int launch_regs = 0;
  int interval_regs[2] = {0, 0};
  std::vector<Expr> reqs;  // `//@ requires` preconditions, checked when a launch binds scalars
};

// Launch register count for per-interval budgets; throws InvalidArgument / DoesNotFit.
int interval_launch_regs(int d1, int d2, int regs1, int regs2, int64_t regs_per_sm = 65536);

Sm100Kernel emit_sm100(const Fused& f, const Sm100Options& o = {});
// One unfused kernel (normalized internally), launched 1-D with dims.count() threads.
Sm100Kernel emit_sm100(const Kernel& k, const std::vector<Func>& funcs, const Sm100Options& o = {});

}  // namespace hf
