/* hfuse — B200-native horizontal kernel fusion: the C ABI (drop-in boundary).
 *
 * Every entry point replaces one reference (mkfuse, /root/reference/proj) interface;
 * the citation is given per function. Conventions:
 *   - return 0 on success, otherwise 1 + the reference ErrCode ordinal
 *     (error.hpp:15-39: HF_E_SYNTAX = 1 ... HF_E_IO = 23) or HF_E_COMPILE / HF_E_DEVICE;
 *   - `err` (may be NULL) receives code, 1-based source position (0 = none) and message;
 *   - strings returned through `char**` are malloc'ed and released with hf_free();
 *   - no function throws across the ABI; device buffers passed in are caller-owned.
 * Thread safety: compiler entry points are reentrant (pure functions);
 * runtime entry points act on the calling thread's current CUDA device.
 */
#ifndef HFUSE_H
#define HFUSE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HF_OK = 0,
  HF_E_SYNTAX = 1, HF_E_UNKNOWN_IDENTIFIER, HF_E_TYPE_MISMATCH, HF_E_DUPLICATE_NAME,
  HF_E_UNRESOLVED_CALL, HF_E_UNRESOLVED_LABEL, HF_E_RECURSION, HF_E_BAD_BARRIER_ID,
  HF_E_MISALIGNED_COUNT, HF_E_DIMENSION_MISMATCH, HF_E_GRID_MISMATCH, HF_E_THREAD_BUDGET,
  HF_E_SHARED_OVERFLOW, HF_E_DOES_NOT_FIT, HF_E_OUT_OF_BOUNDS, HF_E_DIVIDE_BY_ZERO,
  HF_E_BARRIER_DEADLOCK, HF_E_BARRIER_OVERFLOW, HF_E_DIVERGENT_BARRIER, HF_E_NOTHING_FEASIBLE,
  HF_E_INCOMPATIBLE_FIXED_DIMS, HF_E_INVALID_ARGUMENT, HF_E_IO,
  HF_E_COMPILE, HF_E_DEVICE
};

enum { HF_STYLE_STRUCTURED = 0, HF_STYLE_GOTO = 1, HF_STYLE_SM100 = 2 };
enum { HF_REGCAP_OFF = -1, HF_REGCAP_AUTO = 0 };
enum { HF_TIME_SINGLE = 0, HF_TIME_SEQUENTIAL = 1, HF_TIME_TWO_STREAM = 2 };
enum { HF_BACKEND_DEVICE = 0, HF_BACKEND_COMMAND = 1 };

typedef struct hf_error {
  int code;
  int line;
  int col;
  char message[512];
} hf_error;

/* fuser.hpp:24-32 BarrierEntry, plus the constituent's original id (-1 = syncthreads). */
typedef struct hf_barrier {
  int id;
  int count;
  int owner;
  int original;
} hf_barrier;

typedef struct hf_occupancy_info {
  int blocks_per_sm;
  int limiting; /* 0 registers, 1 shared_memory, 2 threads, 3 block_slots */
  int achieved_warps;
  double occupancy_fraction;
} hf_occupancy_info;

typedef struct hf_module hf_module;
typedef struct hf_image hf_image;

typedef struct hf_module_info {
  int threads;
  int grid;
  long long smem_bytes;
  int regs;
  int local_bytes;
  int blocks_per_sm;
  int n_params;
  int n_barriers;
  int launch_regs;      /* per-interval budgets (hf_build_fused_regs): pool regs/thread, else 0 */
  int interval_regs[2]; /* setmaxnreg budget of interval 1 / 2, else 0 */
} hf_module_info;

typedef struct hf_timing {
  double median_us;
  double min_us;
  double mean_us;
  double max_us;
  int reps;
  double iqm_us; /* mean of the middle half (event timestamps tick every 2.048 us) */
} hf_timing;

/* search.hpp:11-15 EvalOutcome (device backend: cycles = interquartile-mean ns). */
typedef struct hf_eval {
  long long cycles;
  double occupancy;
  double utilization;
  double us;
  int regs;
} hf_eval;

typedef struct hf_search_opts {
  int d0;                   /* fused block size (search_config); d0 for fixed+tunable pairs */
  int granularity;          /* 128 in the reference sweep (search.cpp:137-138) */
  int backend;              /* HF_BACKEND_DEVICE or HF_BACKEND_COMMAND */
  const char* profiler_cmd; /* ExternalCommandBackend command (search.cpp:32-62) */
  int grid;                 /* 0: the kernels' //@ grid annotation */
  int warmup;
  int reps;
  int flush_l2;
  int measured_registers;   /* r0 from ptxas register counts instead of the estimate */
  int specialize;           /* fold the image's scalar values into every candidate */
  int n_extra_caps;
  const int* extra_caps;    /* additional register caps per partition (C4 sweep) */
  int out_style;            /* style of *best_src */
  int interval_regs;        /* B200: also sweep per-interval register budgets (setmaxnreg) */
  int budget_points;        /* budget shares per partition (0: 5) */
  int best_regs1;           /* out: budgets of the best point (0 when it has none) */
  int best_regs2;           /* out */
  int prefilter;            /* B200 model pre-filter: keep the k best-predicted partitions (0 off) */
  double prefilter_tol;     /* ... and all predicted within this fraction of the best (< 0: 0.03) */
  char* model_csv;          /* out: "d1,predicted_us,t1_us,t2_us" per partition (row d1 = 0: the
                               full-block times) when the pre-filter ran; release with hf_free */
} hf_search_opts;

typedef struct hf_device_props {
  int sms;
  int cc_major;
  int cc_minor;
  long long smem_per_sm;
  long long smem_per_block_optin;
  int regs_per_sm;
  int max_threads_per_sm;
  int clock_khz;
  long long l2_bytes;
  char name[128];
} hf_device_props;

void hf_free(void* p);
const char* hf_version(void);

/* ---- compiler ------------------------------------------------------------------- */

/* generate_fused + emit_source (fuser.hpp:70-77), with the normalization of cmd_fuse
 * (mkfuse.cpp:109-116: normalize_kernel(k1,"k1_") / (k2,"k2_")) and its regcap
 * handling (mkfuse.cpp:118-133). sm_spec: "pascal-like" (default when NULL),
 * "volta-like", "b200" or a key=value file. `table` receives up to table_cap entries. */
int hf_fuse(const char* src1, const char* src2, int d1, int d2, int style, int regcap,
            const char* sm_spec, char** out_src, hf_barrier* table, int table_cap,
            int* n_entries, hf_error* err);

/* The stdout report of `mkfuse fuse` (mkfuse.cpp:136-166). */
int hf_fuse_report(const char* src1, const char* src2, int d1, int d2, int regcap,
                   const char* sm_spec, char** out_report, hf_error* err);

/* normalize_kernel (frontend.hpp:53-55) of the first kernel, printed as Mini-Kernel. */
int hf_normalize(const char* src, const char* prefix, char** out_src, hf_error* err);

/* parse_program + lint_program (frontend.hpp:13-32); report as `mkfuse check`. */
int hf_check(const char* src, int strict, char** out_report, hf_error* err);

/* MK+ (B200 dialect) -> plain Mini-Kernel with identical semantics, so the reference
 * interpreter (exec.cpp:958-965) can execute B200 member kernels. */
int hf_lower(const char* src, char** out_src, hf_error* err);

/* sm_100a CUDA source of one unfused kernel (the baseline members). */
int hf_emit_kernel(const char* src, int min_blocks, char** out_src, hf_error* err);

/* machine.hpp:72-80 */
int hf_register_bound(int regs1, int threads1, int regs2, int threads2, long long fused_shmem,
                      const char* sm_spec, int* out_r0, hf_error* err);
int hf_occupancy(int regs, long long shmem, int threads, const char* sm_spec,
                 hf_occupancy_info* out, hf_error* err);

/* combined_utilization (machine.cpp:285-289): the cycle-weighted
 * utilization (u1*c1 + u2*c2) / (c1 + c2) of two kernels run back to back; `hfuse simulate
 * --sequential` combines the members' device counters with it. Returns NaN when c1 or c2 <= 0
 * (the reference throws InvalidArgument). */
double hf_combined_utilization(double u1, long long c1, double u2, long long c2);

/* ---- runtime (B200) --------------------------------------------------------------- */

int hf_device_count(void);
int hf_get_device_props(hf_device_props* out, hf_error* err);

/* Fuse, emit for sm_100a and NVRTC-compile (regcap: HF_REGCAP_OFF, HF_REGCAP_AUTO = the
 * register bound r0 of machine.cpp:269-283, or an explicit cap). grid 0 = annotation.
 * specialize (may be NULL): fold that image's scalar values into the code as constants
 * (JIT specialization; hf_run/hf_launch then require the same values). */
int hf_build_fused(const char* src1, const char* src2, int d1, int d2, int regcap, int grid,
                   int min_blocks, const hf_image* specialize, hf_module** out, hf_error* err);
/* hf_build_fused with per-interval register budgets instead of one whole-kernel cap: the
 * reference bounds both constituents by a single r0 (machine.cpp:269-283);
 * on sm_100a the fused kernel is compiled with __maxnreg__(L), L*d0 >= regs1*d1 + regs2*d2,
 * and each interval re-sizes its warpgroups with setmaxnreg.dec/.inc on entry. Requires
 * d1, d2 multiples of 128 and budgets that are multiples of 8 in [24, 256]
 * (HF_E_INVALID_ARGUMENT), a pool that fits one SM (HF_E_DOES_NOT_FIT), and ptxas to allocate
 * exactly L registers (HF_E_DEVICE otherwise: an undersized pool would block the .inc). */
int hf_build_fused_regs(const char* src1, const char* src2, int d1, int d2, int regs1, int regs2,
                        int grid, const hf_image* specialize, hf_module** out, hf_error* err);
/* hf_build_fused with every B200 option in one struct (zero-initialize, then set):
 *   regcap          HF_REGCAP_OFF (-1), HF_REGCAP_AUTO (0) or an explicit cap;
 *   regs1, regs2    per-interval register budgets as hf_build_fused_regs (regcap must be OFF);
 *   vgrid1, vgrid2  dynamic interval scheduling: each interval runs its member as vgridN
 *                   virtual blocks drawn from its own atomic queue (blockIdx.x / gridDim.x of the
 *                   member = virtual block id / vgridN), so the launch grid becomes a persistent
 *                   pool of CTAs and one member's long blocks no longer strand the other member's
 *                   threads of the same CTA. Results equal the member launched with vgridN blocks.
 *                   Needs structured members (no return/goto) and two free named barriers
 *                   (HF_E_INVALID_ARGUMENT / HF_E_BARRIER_OVERFLOW); 0 = the static partition;
 *   grid, min_blocks as hf_build_fused. B200-only; no reference analogue. */
typedef struct hf_fuse_opts {
  int regcap;
  int regs1, regs2;
  int vgrid1, vgrid2;
  int grid;
  int min_blocks;
  int split_grid; /* heterogeneous CTA partition (0 = off): blocks below it run both members
                     (member 1 sees a grid of split_grid blocks); blocks above give all d0 threads
                     to member 2 as d0/d2 sub-blocks (member 2 sees one grid of split_grid +
                     (grid - split_grid) * d0/d2 blocks of d2 threads). Needs a barrier- and
                     shared-memory-free 1-D member 2 and d0 % d2 == 0 (HF_E_INVALID_ARGUMENT). */
} hf_fuse_opts;
int hf_build_fused_opts(const char* src1, const char* src2, int d1, int d2, const hf_fuse_opts* opts,
                        const hf_image* specialize, hf_module** out, hf_error* err);
/* One unfused kernel at its declared dims (regcap: HF_REGCAP_OFF = none, HF_REGCAP_AUTO = the
 * kernel's `//@ regcap=` annotation if present (the reference's exec.cpp:954), or a cap). */
int hf_build_kernel(const char* src, int regcap, int grid, int min_blocks,
                    const hf_image* specialize, hf_module** out, hf_error* err);
/* The reference's naive goto emission (fuser.cpp:290-549) of the same pair, made launchable
 * (extern "C", parameters from its signature) — the "naive fusion" baseline; its semantics
 * are plain CUDA's, not the interpreter's, so it is timed, never parity-checked. */
int hf_build_naive(const char* src1, const char* src2, int d1, int d2, int grid, hf_module** out,
                   hf_error* err);
/* Vertical fusion (VFuse; reference test-local version test_sim.cpp:398-439):
 * both bodies run back to back by every thread of one block (equal block dims required);
 * pinned semantics like hf_build_kernel. */
int hf_build_vertical(const char* src1, const char* src2, int grid, const hf_image* specialize,
                      hf_module** out, hf_error* err);
int hf_module_get_info(const hf_module* m, hf_module_info* out);
const char* hf_module_source(const hf_module* m);  /* borrowed */
const char* hf_module_entry(const hf_module* m);   /* borrowed */
int hf_module_param(const hf_module* m, int i, const char** name, int* is_array, int* is_float,
                    int* is_written, int* is_specialized);
/* Whether array parameter i's prior contents are observed by the kernel (loads or atomic
 * read-modify-writes); a written array that is not read is pure output and needs no upload
 * (the reference binds every array by name from the image, exec.cpp:190-216). */
int hf_module_param_reads(const hf_module* m, int i, int* is_read);
int hf_module_barrier(const hf_module* m, int i, hf_barrier* out);
int hf_module_cubin(const hf_module* m, const void** data, size_t* size);
/* Raw launch: args[i] points at the i-th parameter value (device pointer or scalar);
 * specialized scalars are checked against the folded value. */
int hf_launch(const hf_module* m, int grid, void** args, void* stream, hf_error* err);
/* hf_launch / hf_run with flags. HF_LAUNCH_OVERLAP: programmatic dependent launch -- the kernel
 * may start while the previous kernel in the stream drains (every emitted kernel triggers
 * griddepcontrol.launch_dependents on entry). Only for a kernel that does not read what the
 * previous one writes (independent fused pairs in a step); B200-only, no reference analogue. */
enum { HF_LAUNCH_OVERLAP = 1 };
int hf_launch_ex(const hf_module* m, int grid, void** args, void* stream, int flags, hf_error* err);
int hf_run_ex(const hf_module* m, hf_image* img, int grid, void* stream, int flags, hf_error* err);
void hf_module_free(hf_module* m);

/* MemoryImage (memimage.hpp:36-68); seeded arrays are generated in HBM on upload. */
int hf_image_parse(const char* text, int has_seed, unsigned long long seed, hf_image** out,
                   hf_error* err);
int hf_image_merge(hf_image* dst, hf_image* src, hf_error* err); /* consumes src's entries */
int hf_image_materialize(hf_image* img, hf_error* err);         /* host-side generation */
int hf_image_upload(hf_image* img, void* stream, hf_error* err);
int hf_image_download(hf_image* img, void* stream, hf_error* err);
int hf_image_digest(const hf_image* img, unsigned long long* out, hf_error* err);
int hf_image_serialize(const hf_image* img, char** out, hf_error* err);
int hf_image_count(const hf_image* img);
int hf_image_entry(hf_image* img, int i, const char** name, void** dev_ptr, int32_t** host_ptr,
                   long long* len, int* is_float);
int hf_image_find(hf_image* img, const char* name, void** dev_ptr, int32_t** host_ptr,
                  long long* len, int* is_float);
int hf_image_set_host(hf_image* img, const char* name, const void* data, long long len,
                      hf_error* err); /* replace an array's contents with host data */
long long hf_image_bytes(const hf_image* img);
void hf_image_free(hf_image* img);

/* run_functional (sim.hpp:43-52) on the device: bind parameters by name and launch. */
int hf_run(const hf_module* m, hf_image* img, int grid, void* stream, hf_error* err);

/* Device timing with CUDA events (replaces run_timed, exec.cpp:967-982). */
int hf_time(int mode, const hf_module* a, const hf_module* b, hf_image* img, int grid_a,
            int grid_b, int warmup, int reps, int flush_l2, void* stream, hf_timing* out,
            hf_error* err);

/* Graph-timed protocol (B200-only; replaces run_timed's per-repetition measurement for
 * back-to-back comparisons): `reps` repetitions of the variant captured as one CUDA graph and
 * launched `samples` times between consecutive events, no host synchronization in the timed
 * region. Per-repetition mean / median / min / max over samples and a Student-t 95 % half-width.
 * Nothing is flushed: every repetition's working set should exceed L2. */
typedef struct hf_graph_timing {
  double mean_us;
  double median_us;
  double min_us;
  double max_us;
  double ci95_us;
  int samples;
  int reps;
} hf_graph_timing;
int hf_time_graph(int mode, const hf_module* a, const hf_module* b, hf_image* img, int grid_a,
                  int grid_b, int reps, int samples, void* stream, hf_graph_timing* out,
                  hf_error* err);

/* ProfilerBackend::evaluate (search.hpp:19-23) for one candidate on the device. */
int hf_profile(const char* src1, const char* src2, int d1, int d2, int regcap, hf_image* img,
               int grid, int warmup, int reps, int flush_l2, int specialize, hf_eval* out,
               hf_error* err);

/* search_config / fixed_partition_fuse + trace_csv (search.hpp:66-77). img may be NULL for
 * the command backend. */
int hf_search(const char* src1, const char* src2, hf_image* img, hf_search_opts* opts,
              int* best_d1, int* best_d2, int* best_regcap, long long* best_time,
              char** trace_csv, char** best_src, hf_error* err);

/* The multi-GPU step exchange on the device (B200-only; the reference is single-threaded,
 * /root/reference/SPEC.md:374). Each rank packs its step outputs into one int32 buffer
 * (hf_shard_pack: one launch for up to 32 source arrays), the buffers are all-gathered (NCCL),
 * and hf_shard_reduce reduces the [world, cells] result in one launch: hist slots -> int64 sums,
 * bn slots -> Chan's merge of (mean, biased var) in rank order in fp64 without contraction
 * (mean[C] then var[C]), crypto slots -> int64 (hit sum, winning-nonce min) pairs. `out` holds
 * 8-byte elements at each slot's out_offset; counts = per-rank elements per channel (bn). */
enum { HF_SLOT_HIST = 0, HF_SLOT_BN = 1, HF_SLOT_CRYPTO = 2 };
typedef struct hf_pack_src {
  const void* src;
  long long offset;
  long long cells;
} hf_pack_src;
typedef struct hf_reduce_slot {
  int kind;
  int channels;
  long long offset;
  long long cells;
  long long out_offset;
} hf_reduce_slot;
int hf_shard_pack(const hf_pack_src* srcs, int n, int* packed, void* stream, hf_error* err);
int hf_shard_reduce(const int* gathered, int world, long long cells, const hf_reduce_slot* slots,
                    int nslots, const double* counts, void* out, void* stream, hf_error* err);

#ifdef __cplusplus
}
#endif

#endif /* HFUSE_H */
