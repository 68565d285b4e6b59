// Device runtime: NVRTC compilation for sm_100a, module load/launch through the CUDA
// driver API (entry points resolved from the static runtime, so the library loads on
// GPU-less hosts), memory images in HBM, and CUDA-event timing (the device profiler that
// replaces the reference's cycle simulator, /root/reference/proj/src/exec.cpp:144-167).
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "fuser.hpp"
#include "image.hpp"

namespace hf::rt {

struct Module {
  std::string entry;
  std::string source;
  int threads = 0;
  int grid = 1;
  int64_t smem = 0;
  std::vector<Sm100Param> params;
  std::vector<BarrierEntry> barriers;
  std::optional<int> maxrreg;
  std::vector<Expr> reqs;           // `//@ requires` launch preconditions
  int launch_regs = 0;              // per-interval budgets (setmaxnreg), 0 = off
  int interval_regs[2] = {0, 0};
  // filled after load
  int regs = 0;
  int local_bytes = 0;  // spill / local memory per thread
  int blocks_per_sm = 0;
  std::string log;
  std::vector<char> cubin;
  void* mod = nullptr;
  void* fn = nullptr;
  int device = 0;
};

struct Props {
  int device = 0;
  int sms = 0;
  int cc_major = 0, cc_minor = 0;
  int64_t smem_per_sm = 0, smem_per_block_optin = 0;
  int regs_per_sm = 0, max_threads_per_sm = 0, max_threads_per_block = 0;
  int clock_khz = 0;
  int64_t l2_bytes = 0;
  std::string name;
};

Props props(int device = -1);
int device_count();
void set_device(int device);  // this host thread's current device (its primary context current)
SM sm_from_device(int device = -1);
bool device_available();

Module compile(const Sm100Kernel& k, std::optional<int> maxrreg = std::nullopt, bool lineinfo = true);
// NVRTC-compiles a batch into the CUBIN cache on a pool of host threads (no device work);
// a later compile() of the same (kernel, cap) only loads the module. Errors are deferred
// to that compile().
void precompile(const std::vector<std::pair<Sm100Kernel, std::optional<int>>>& ks, bool lineinfo = true);
void unload(Module& m);

void upload(Image& img, void* stream = nullptr);
void download(Image& img, void* stream = nullptr);
void release(Image& img);
void* device_ptr(Image& img, const std::string& name);

// Binds parameters by name from the image (exec.cpp:190-216) and launches.
// overlap: programmatic dependent launch (the kernel may start while the stream's previous kernel
// drains; only for kernels that do not read what that kernel writes)
void launch(const Module& m, Image& img, int grid, void* stream = nullptr, bool overlap = false);
void launch_raw(const Module& m, int grid, void** args, void* stream = nullptr, bool overlap = false);
// Throws InvalidArgument when a `//@ requires` precondition is false for these scalar values
// (args[i] points at parameter i's value; specialized parameters use their folded value).
void check_requires(const Module& m, void* const* args);

struct Timing {
  double median_us = 0, min_us = 0, mean_us = 0, max_us = 0;
  int reps = 0;
  // Interquartile mean. CUDA event timestamps on the B200 tick every 2.048 us; the start phase
  // of each repetition is random against that tick, so the mean of the middle half resolves
  // below one tick where the median cannot.
  double iqm_us = 0;
};
enum class Mode { Single, Sequential, TwoStream };
// Times `a` (Single) or the pair a;b (Sequential) / a||b on two streams (TwoStream).
// L2 is flushed before every timed repetition when `flush_l2`.
Timing time(Mode mode, const Module& a, const Module* b, Image& img, int grid_a, int grid_b, int warmup,
            int reps, bool flush_l2, void* stream = nullptr);

// Graph protocol: `reps` back-to-back repetitions of the variant (a; a then b; a || b on two
// streams) captured as ONE CUDA graph between two timing-event nodes (external event records
// inside the graph), launched `samples` times; no host synchronization inside the timed region.
// Each sample yields the mean time per repetition of the graph's own execution (no
// per-repetition front-end or event cost, no gap between graph launches, and the two-stream
// fork/join is a graph edge rather than an event wait); the summary is over samples with a
// Student-t 95 % half-width. Every repetition's working set must exceed L2 for steady-state HBM numbers
// (the caller's choice; nothing is flushed).
struct GraphTiming {
  double mean_us = 0, median_us = 0, min_us = 0, max_us = 0, ci95_us = 0;
  int samples = 0, reps = 0;
};
GraphTiming time_graph(Mode mode, const Module& a, const Module* b, Image& img, int grid_a, int grid_b,
                       int reps, int samples, void* stream = nullptr);

void synchronize();

}  // namespace hf::rt
