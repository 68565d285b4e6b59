// Profile-guided partition search (Algorithm "Main").
// Reference contract: /root/reference/proj/include/mkfuse/search.hpp:11-77 — same sweep
// (d1 = g, 2g, ..., d0 - g; uncapped then capped at r0), same strict-< fold (ties keep the
// smaller d1, then no cap), infeasible candidates skipped, NothingFeasible when none.
// The B200 backend (DeviceBackend) times each candidate on the GPU instead of simulating.
#pragma once

#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "fuser.hpp"
#include "image.hpp"

namespace hf::rt {
struct Module;
}

namespace hf {

struct EvalOutcome {
  int64_t cycles = 0;        // device backend: nanoseconds (interquartile mean)
  double occupancy = 0.0;
  double utilization = 0.0;
  double us = 0.0;           // device backend: interquartile-mean microseconds
  int regs = 0;
};

class ProfilerBackend {
 public:
  virtual ~ProfilerBackend() = default;
  virtual EvalOutcome evaluate(const Fused& fused, const FusionConfig& cfg) = 0;
  // Per-thread resources of one constituent run alone with `threads` threads; the
  // default is the reference's estimate (machine.cpp:215-230).
  virtual Resources resources(const Kernel& k, int threads) { return resources_of(k, threads); }
  // Called once with every candidate of a sweep before the first evaluate(); a backend may
  // do per-candidate work ahead of time (DeviceBackend: parallel NVRTC compilation).
  virtual void prepare(const std::vector<std::pair<Fused, FusionConfig>>& candidates) { (void)candidates; }
  // Whether evaluate() honours per-interval register budgets (only sm100 code carries them).
  virtual bool supports_budgets() const { return false; }
  // Calibration for the model pre-filter: the time of one constituent run alone with `threads`
  // threads per block (partition_dims), or nullopt when the backend cannot measure it.
  virtual std::optional<double> member_time(const Kernel& k, int threads) { return std::nullopt; }
  // Evaluates a whole sweep; entry i is candidate i's outcome or nullopt when it is infeasible
  // (does not compile or fit). The default evaluates in order; MultiDeviceBackend spreads the
  // candidates over several GPUs. The fold always consumes the results in candidate order.
  virtual std::vector<std::optional<EvalOutcome>> evaluate_many(
      const std::vector<std::pair<Fused, FusionConfig>>& candidates);
};

// Spawns `command <source-file>` and reads the first integer of its stdout (search.cpp:32-62).
class ExternalCommandBackend : public ProfilerBackend {
 public:
  explicit ExternalCommandBackend(std::string cmd, Style style = Style::Goto);
  EvalOutcome evaluate(const Fused& fused, const FusionConfig& cfg) override;
  bool supports_budgets() const override { return style_ == Style::Sm100; }

 private:
  std::string cmd_;
  Style style_;
  int counter_ = 0;
};

// Times the sm_100a emission of every candidate on the current GPU.
class DeviceBackend : public ProfilerBackend {
 public:
  DeviceBackend(Image& img, int grid, int warmup = 3, int reps = 10, bool flush_l2 = true,
                bool measured_registers = true);
  EvalOutcome evaluate(const Fused& fused, const FusionConfig& cfg) override;
  Resources resources(const Kernel& k, int threads) override;
  void prepare(const std::vector<std::pair<Fused, FusionConfig>>& candidates) override;
  bool supports_budgets() const override { return true; }
  std::optional<double> member_time(const Kernel& k, int threads) override;
  void set_specialization(std::map<std::string, ScalarVal> s) { spec_ = std::move(s); }

 private:
  std::map<std::string, ScalarVal> spec_;
  std::map<std::pair<std::string, int>, double> member_us_;  // (emitted member source, threads)
  Image& img_;
  int grid_, warmup_, reps_;
  bool flush_, measured_;
};

// One DeviceBackend per GPU (each with its own copy of the memory image): evaluate_many times
// disjoint candidates concurrently, one host thread per device pulling from a shared counter, so
// an N-GPU box searches N times faster; the fold is unchanged (candidate order, strict <).
// Every device must be the same model for the times to be comparable (checked at construction).
class MultiDeviceBackend : public ProfilerBackend {
 public:
  MultiDeviceBackend(std::vector<std::unique_ptr<DeviceBackend>> devices, std::vector<int> ids);
  EvalOutcome evaluate(const Fused& fused, const FusionConfig& cfg) override;
  Resources resources(const Kernel& k, int threads) override;
  void prepare(const std::vector<std::pair<Fused, FusionConfig>>& candidates) override;
  bool supports_budgets() const override { return true; }
  std::optional<double> member_time(const Kernel& k, int threads) override;
  std::vector<std::optional<EvalOutcome>> evaluate_many(
      const std::vector<std::pair<Fused, FusionConfig>>& candidates) override;
  size_t size() const { return devs_.size(); }

 private:
  std::vector<std::unique_ptr<DeviceBackend>> devs_;
  std::vector<int> ids_;
};

std::string cap_text(const FusionConfig& cfg);  // "none", "N" or "R1/R2" (budgets)

struct EvalPoint {
  FusionConfig cfg;
  EvalOutcome out;
};

struct SearchResult {
  Fused best;
  FusionConfig best_cfg;
  int64_t best_time = 0;
  std::vector<EvalPoint> trace;
  std::map<int, double> predicted_us;  // model pre-filter: d1 -> predicted time (all partitions)
  std::map<int, std::pair<double, double>> member_us;  // d1 -> (t1(d1), t2(d0 - d1)); key 0: (T1, T2)
};

double predict_fused(double t1, double t2, double T1, double T2);

struct SearchOptions {
  int granularity = 128;
  std::vector<int> extra_caps;  // C4: additional register caps evaluated per partition
  // B200: also evaluate per-interval register budgets (setmaxnreg) for warpgroup-aligned
  // partitions: the one-CTA-per-SM pool divided between the intervals at `budget_points`
  // shares of the constituents' register shortfall (interval_budgets()).
  bool interval_regs = false;
  int budget_points = 5;
  // B200 model pre-filter: when > 0 and the backend can time constituents
  // alone, each partition is predicted from the constituents measured alone at each interval
  // size (t1(d1), t2(d2)) and at the full block (T1, T2) -- one cheap compile + timing per
  // (kernel, size), reused across partitions -- and only the `prefilter` best-predicted
  // partitions are fused, compiled and timed. Model (predict_fused): the intervals co-run,
  // sharing the SM/HBM capacity; interval i alone uses the fraction u_i = T_i / t_i of it, so
  // while both run each is slowed by s = max(1, u1 + u2); after the shorter one (t_min) ends,
  // the other finishes at its own rate: t = t_max + t_min * (s - 1).
  int prefilter = 0;
  // ... plus every partition predicted within this fraction of the best prediction: where the
  // model cannot tell partitions apart (flat predictions) the device decides. Ten DL pairs,
  // top-3 + 3 %: 102 of 300 candidates timed, best within 0.8 % of the exhaustive sweep on
  // average, 6.5 % at worst (profiles/r01_probe_prefilter.json).
  double prefilter_tol = 0.03;
};

// Per-interval budgets for one partition: demand n1, n2 (ptxas registers of each constituent
// alone), pool = the largest multiple-of-8 count per thread that one CTA of d1 + d2 threads
// may hold on an SM. When both demands fit, the single point (ceil8 n1, ceil8 n2); else the
// shortfall D is charged to interval 1 at fractions 0, 1/(p-1), ..., 1 (interval 2 takes the
// rest of the pool), clamped to [24, 256] and deduplicated.
std::vector<std::pair<int, int>> interval_budgets(int n1, int d1, int n2, int d2, int64_t regs_per_sm,
                                                  int points);

SearchResult search_config(const Kernel& k1, const Kernel& k2, int d0, ProfilerBackend& be, const SM& sm,
                           const SearchOptions& opt = {});
SearchResult fixed_partition_fuse(const Kernel& k1, const Kernel& k2, ProfilerBackend& be, const SM& sm,
                                  int d0 = 1024, const SearchOptions& opt = {});
std::string trace_csv(const SearchResult& r);

}  // namespace hf
