// The C ABI of include/hfuse.h: thin exception-to-error-code wrappers over the C++ core.
#include "hfuse.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "driver.hpp"
#include "runtime.hpp"
#include "search.hpp"
#include "shard_reduce.hpp"

struct hf_module {
  hf::rt::Module m;
};
struct hf_image {
  hf::Image img;
};

namespace {

int to_abi(hf::Code c) { return int(c) + 1; }

void clear(hf_error* err) {
  if (!err) return;
  err->code = HF_OK;
  err->line = err->col = 0;
  err->message[0] = '\0';
}

int fill(hf_error* err, hf::Code code, const std::string& msg, hf::Pos pos = {}) {
  if (err) {
    err->code = to_abi(code);
    err->line = pos.line;
    err->col = pos.col;
    std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
  }
  return to_abi(code);
}

template <typename F>
int guarded(hf_error* err, F&& body) {
  clear(err);
  try {
    body();
    return HF_OK;
  } catch (const hf::Error& e) {
    return fill(err, e.code, e.msg, e.pos);
  } catch (const std::exception& e) {
    return fill(err, hf::Code::InvalidArgument, e.what());
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

hf::SM sm_of(const char* spec) { return hf::SM::preset_or_file(spec ? spec : ""); }

std::string regcap_spec(int regcap) {
  if (regcap == HF_REGCAP_OFF) return "off";
  if (regcap == HF_REGCAP_AUTO) return "auto";
  return std::to_string(regcap);
}

hf::Style style_of(int s) {
  return s == HF_STYLE_STRUCTURED ? hf::Style::Structured : s == HF_STYLE_GOTO ? hf::Style::Goto : hf::Style::Sm100;
}

std::map<std::string, hf::ScalarVal> scalars_of(const hf_image* img) {
  std::map<std::string, hf::ScalarVal> m;
  if (!img) return m;
  for (const auto& [n, s] : img->img.scalars) m[n] = hf::ScalarVal{s.ty, s.i, s.f};
  return m;
}

// sm_100a fused module with per-interval register budgets (setmaxnreg).
hf::rt::Module build_fused_regs(const char* s1, const char* s2, int d1, int d2, int regs1, int regs2, int grid,
                                const hf_image* spec) {
  hf::SM sm = hf::rt::device_available() ? hf::rt::sm_from_device() : hf::SM::b200();
  hf::FuseResult r = hf::fuse_sources(s1, s2, d1, d2, "off", sm, grid);
  if (grid > 0) r.fused.grid = grid;
  hf::Sm100Options o;
  o.regs1 = regs1;
  o.regs2 = regs2;
  o.specialize = scalars_of(spec);
  return hf::rt::compile(hf::emit_sm100(r.fused, o), std::nullopt);
}

// sm_100a fused module with every B200 option: register cap or per-interval budgets, and
// dynamic interval scheduling (virtual grids).
hf::rt::Module build_fused_opts(const char* s1, const char* s2, int d1, int d2, const hf_fuse_opts& fo,
                                const hf_image* spec) {
  hf::SM sm = hf::rt::device_available() ? hf::rt::sm_from_device() : hf::SM::b200();
  const bool budgets = fo.regs1 > 0 || fo.regs2 > 0;
  if (budgets && fo.regcap != HF_REGCAP_OFF)
    hf::raise(hf::Code::InvalidArgument, "a register cap and per-interval register budgets are exclusive");
  hf::FuseResult r = hf::fuse_sources(s1, s2, d1, d2, regcap_spec(fo.regcap), sm, fo.grid);
  if (fo.grid > 0) r.fused.grid = fo.grid;
  hf::Sm100Options o;
  o.min_blocks = fo.min_blocks;
  o.regs1 = fo.regs1;
  o.regs2 = fo.regs2;
  o.vgrid1 = fo.vgrid1;
  o.vgrid2 = fo.vgrid2;
  o.split_grid = fo.split_grid;
  o.specialize = scalars_of(spec);
  return hf::rt::compile(hf::emit_sm100(r.fused, o), budgets ? std::nullopt : r.fused.cfg.reg_cap);
}

// sm_100a fused module; regcap AUTO means the register bound r0 with the B200 machine model.
hf::rt::Module build_fused(const char* s1, const char* s2, int d1, int d2, int regcap, int grid, int min_blocks,
                           const hf_image* spec) {
  hf::SM sm = hf::rt::device_available() ? hf::rt::sm_from_device() : hf::SM::b200();
  hf::FuseResult r = hf::fuse_sources(s1, s2, d1, d2, regcap_spec(regcap), sm, grid);
  if (grid > 0) r.fused.grid = grid;
  hf::Sm100Options o;
  o.min_blocks = min_blocks;
  o.specialize = scalars_of(spec);
  return hf::rt::compile(hf::emit_sm100(r.fused, o), r.fused.cfg.reg_cap);
}

}  // namespace

extern "C" {

void hf_free(void* p) { std::free(p); }
const char* hf_version(void) { return "hfuse-b200 0.1 (sm_100a)"; }

int hf_fuse(const char* src1, const char* src2, int d1, int d2, int style, int regcap, const char* sm_spec,
            char** out_src, hf_barrier* table, int table_cap, int* n_entries, hf_error* err) {
  return guarded(err, [&] {
    hf::FuseResult r = hf::fuse_sources(src1, src2, d1, d2, regcap_spec(regcap), sm_of(sm_spec));
    if (out_src) *out_src = dup(hf::emit(r.fused, style_of(style)));
    if (n_entries) *n_entries = int(r.fused.barriers.size());
    for (int i = 0; table && i < table_cap && i < int(r.fused.barriers.size()); ++i) {
      const auto& e = r.fused.barriers[size_t(i)];
      table[i] = hf_barrier{e.id, e.count, e.owner, e.original};
    }
  });
}

int hf_fuse_report(const char* src1, const char* src2, int d1, int d2, int regcap, const char* sm_spec,
                   char** out_report, hf_error* err) {
  return guarded(err, [&] {
    hf::FuseResult r = hf::fuse_sources(src1, src2, d1, d2, regcap_spec(regcap), sm_of(sm_spec));
    *out_report = dup(hf::fuse_report(r));
  });
}

int hf_normalize(const char* src, const char* prefix, char** out_src, hf_error* err) {
  return guarded(err, [&] {
    hf::Loaded l = hf::load_source(src);
    *out_src = dup(hf::print_mk(hf::normalize(l.kernel, l.prog.funcs, prefix ? prefix : "")));
  });
}

int hf_check(const char* src, int strict, char** out_report, hf_error* err) {
  return guarded(err, [&] {
    hf::Program p = hf::parse(src, strict ? hf::Dialect::Strict : hf::Dialect::B200);
    std::string o = "ok: " + std::to_string(p.kernels.size()) + " kernel(s), " + std::to_string(p.funcs.size()) +
                    " function(s)\n";
    for (const auto& w : hf::lint(p))
      o += "lint " + std::to_string(w.pos.line) + ":" + std::to_string(w.pos.col) + ": " + w.msg + "\n";
    if (out_report) *out_report = dup(o);
  });
}

int hf_lower(const char* src, char** out_src, hf_error* err) {
  return guarded(err, [&] {
    hf::Program p = hf::parse(src);
    hf::Program low = hf::downlower(p);
    std::string text = hf::print_mk(low);
    hf::parse(text, hf::Dialect::Strict);  // the result must be reference Mini-Kernel
    *out_src = dup(text);
  });
}

int hf_emit_kernel(const char* src, int min_blocks, char** out_src, hf_error* err) {
  return guarded(err, [&] {
    hf::Loaded l = hf::load_source(src);
    hf::Sm100Options o;
    o.min_blocks = min_blocks;
    *out_src = dup(hf::emit_sm100(l.kernel, l.prog.funcs, o).source);
  });
}

int hf_register_bound(int regs1, int threads1, int regs2, int threads2, long long fused_shmem, const char* sm_spec,
                      int* out_r0, hf_error* err) {
  return guarded(err, [&] {
    *out_r0 = hf::register_bound(hf::Resources{regs1, 0, threads1}, hf::Resources{regs2, 0, threads2}, fused_shmem,
                                 threads1 + threads2, sm_of(sm_spec));
  });
}

int hf_occupancy(int regs, long long shmem, int threads, const char* sm_spec, hf_occupancy_info* out, hf_error* err) {
  return guarded(err, [&] {
    hf::Occupancy o = hf::occupancy(hf::Resources{regs, shmem, threads}, sm_of(sm_spec));
    *out = hf_occupancy_info{o.blocks_per_sm, int(o.limiting), o.warps, o.fraction};
  });
}

double hf_combined_utilization(double u1, long long c1, double u2, long long c2) {
  if (c1 <= 0 || c2 <= 0) return std::nan("");
  return hf::combined_utilization(u1, c1, u2, c2);
}

int hf_device_count(void) {
  int n = 0;
  return hf::rt::device_available() ? (cudaGetDeviceCount(&n), n) : 0;
}

int hf_get_device_props(hf_device_props* out, hf_error* err) {
  return guarded(err, [&] {
    hf::rt::Props p = hf::rt::props();
    out->sms = p.sms;
    out->cc_major = p.cc_major;
    out->cc_minor = p.cc_minor;
    out->smem_per_sm = p.smem_per_sm;
    out->smem_per_block_optin = p.smem_per_block_optin;
    out->regs_per_sm = p.regs_per_sm;
    out->max_threads_per_sm = p.max_threads_per_sm;
    out->clock_khz = p.clock_khz;
    out->l2_bytes = p.l2_bytes;
    std::snprintf(out->name, sizeof(out->name), "%s", p.name.c_str());
  });
}

int hf_build_fused(const char* src1, const char* src2, int d1, int d2, int regcap, int grid, int min_blocks,
                   const hf_image* specialize, hf_module** out, hf_error* err) {
  return guarded(err, [&] {
    auto h = std::make_unique<hf_module>();
    h->m = build_fused(src1, src2, d1, d2, regcap, grid, min_blocks, specialize);
    *out = h.release();
  });
}

int hf_build_fused_opts(const char* src1, const char* src2, int d1, int d2, const hf_fuse_opts* opts,
                        const hf_image* specialize, hf_module** out, hf_error* err) {
  return guarded(err, [&] {
    if (!opts) hf::raise(hf::Code::InvalidArgument, "hf_build_fused_opts: opts is NULL");
    auto h = std::make_unique<hf_module>();
    h->m = build_fused_opts(src1, src2, d1, d2, *opts, specialize);
    *out = h.release();
  });
}

int hf_build_fused_regs(const char* src1, const char* src2, int d1, int d2, int regs1, int regs2, int grid,
                        const hf_image* specialize, hf_module** out, hf_error* err) {
  return guarded(err, [&] {
    auto h = std::make_unique<hf_module>();
    h->m = build_fused_regs(src1, src2, d1, d2, regs1, regs2, grid, specialize);
    *out = h.release();
  });
}

int hf_build_kernel(const char* src, int regcap, int grid, int min_blocks, const hf_image* specialize,
                    hf_module** out, hf_error* err) {
  return guarded(err, [&] {
    hf::Loaded l = hf::load_source(src);
    if (grid > 0) l.kernel.grid = grid;
    hf::Sm100Options o;
    o.min_blocks = min_blocks;
    o.specialize = scalars_of(specialize);
    std::optional<int> cap;
    if (regcap > 0) cap = regcap;
    else if (regcap != HF_REGCAP_OFF && l.kernel.regcap) cap = l.kernel.regcap;  // `//@ regcap=` (exec.cpp:954)
    auto h = std::make_unique<hf_module>();
    h->m = hf::rt::compile(hf::emit_sm100(l.kernel, l.prog.funcs, o), cap);
    *out = h.release();
  });
}

int hf_build_naive(const char* src1, const char* src2, int d1, int d2, int grid, hf_module** out, hf_error* err) {
  return guarded(err, [&] {
    hf::FuseResult r = hf::fuse_sources(src1, src2, d1, d2, "off", hf::SM::b200());
    auto h = std::make_unique<hf_module>();
    h->m = hf::rt::compile(hf::wrap_goto(hf::emit_goto(r.fused), grid > 0 ? grid : r.fused.grid));
    *out = h.release();
  });
}

int hf_build_vertical(const char* src1, const char* src2, int grid, const hf_image* specialize, hf_module** out,
                      hf_error* err) {
  return guarded(err, [&] {
    hf::Loaded l1 = hf::load_source(src1), l2 = hf::load_source(src2);
    hf::Kernel v = hf::vertical_fuse(hf::normalize(l1.kernel, l1.prog.funcs, "k1_"),
                                     hf::normalize(l2.kernel, l2.prog.funcs, "k2_"));
    if (grid > 0) v.grid = grid;
    hf::Sm100Options o;
    o.specialize = scalars_of(specialize);
    auto h = std::make_unique<hf_module>();
    h->m = hf::rt::compile(hf::emit_sm100(v, {}, o));
    *out = h.release();
  });
}

int hf_module_get_info(const hf_module* m, hf_module_info* out) {
  if (!m || !out) return to_abi(hf::Code::InvalidArgument);
  *out = hf_module_info{m->m.threads, m->m.grid, m->m.smem, m->m.regs, m->m.local_bytes, m->m.blocks_per_sm,
                        int(m->m.params.size()), int(m->m.barriers.size()), m->m.launch_regs,
                        {m->m.interval_regs[0], m->m.interval_regs[1]}};
  return HF_OK;
}

const char* hf_module_source(const hf_module* m) { return m ? m->m.source.c_str() : nullptr; }
const char* hf_module_entry(const hf_module* m) { return m ? m->m.entry.c_str() : nullptr; }

int hf_module_param(const hf_module* m, int i, const char** name, int* is_array, int* is_float, int* is_written,
                    int* is_specialized) {
  if (!m || i < 0 || i >= int(m->m.params.size())) return to_abi(hf::Code::InvalidArgument);
  const auto& p = m->m.params[size_t(i)];
  if (is_specialized) *is_specialized = p.specialized;
  if (name) *name = p.name.c_str();
  if (is_array) *is_array = p.array;
  if (is_float) *is_float = p.ty == hf::Ty::Float;
  if (is_written) *is_written = p.written;
  return HF_OK;
}

int hf_module_param_reads(const hf_module* m, int i, int* is_read) {
  if (!m || !is_read || i < 0 || i >= int(m->m.params.size())) return to_abi(hf::Code::InvalidArgument);
  *is_read = m->m.params[size_t(i)].read;
  return HF_OK;
}

int hf_module_barrier(const hf_module* m, int i, hf_barrier* out) {
  if (!m || i < 0 || i >= int(m->m.barriers.size())) return to_abi(hf::Code::InvalidArgument);
  const auto& e = m->m.barriers[size_t(i)];
  *out = hf_barrier{e.id, e.count, e.owner, e.original};
  return HF_OK;
}

int hf_module_cubin(const hf_module* m, const void** data, size_t* size) {
  if (!m) return to_abi(hf::Code::InvalidArgument);
  *data = m->m.cubin.data();
  *size = m->m.cubin.size();
  return HF_OK;
}

int hf_launch(const hf_module* m, int grid, void** args, void* stream, hf_error* err) {
  return hf_launch_ex(m, grid, args, stream, 0, err);
}

int hf_launch_ex(const hf_module* m, int grid, void** args, void* stream, int flags, hf_error* err) {
  return guarded(err, [&] {
    for (size_t i = 0; i < m->m.params.size(); ++i) {
      const auto& p = m->m.params[i];
      if (!p.specialized) continue;
      bool same = p.ty == hf::Ty::Int ? *static_cast<const int32_t*>(args[i]) == p.value.i
                                      : std::memcmp(args[i], &p.value.f, 4) == 0;
      if (!same)
        hf::raise(hf::Code::InvalidArgument, "module is specialized for a different value of scalar '" + p.name + "'");
    }
    hf::rt::check_requires(m->m, args);
    hf::rt::launch_raw(m->m, grid > 0 ? grid : m->m.grid, args, stream, (flags & HF_LAUNCH_OVERLAP) != 0);
  });
}

void hf_module_free(hf_module* m) {
  if (!m) return;
  hf::rt::unload(m->m);
  delete m;
}

int hf_image_parse(const char* text, int has_seed, unsigned long long seed, hf_image** out, hf_error* err) {
  return guarded(err, [&] {
    auto h = std::make_unique<hf_image>();
    std::optional<uint64_t> s;
    if (has_seed) s = seed;
    h->img = hf::Image::parse(text, s);
    *out = h.release();
  });
}

int hf_image_merge(hf_image* dst, hf_image* src, hf_error* err) {
  return guarded(err, [&] { dst->img.merge(std::move(src->img)); });
}

int hf_image_materialize(hf_image* img, hf_error* err) {
  return guarded(err, [&] { img->img.materialize_host(); });
}

int hf_image_upload(hf_image* img, void* stream, hf_error* err) {
  return guarded(err, [&] { hf::rt::upload(img->img, stream); });
}

int hf_image_download(hf_image* img, void* stream, hf_error* err) {
  return guarded(err, [&] { hf::rt::download(img->img, stream); });
}

int hf_image_digest(const hf_image* img, unsigned long long* out, hf_error* err) {
  return guarded(err, [&] { *out = img->img.digest(); });
}

int hf_image_serialize(const hf_image* img, char** out, hf_error* err) {
  return guarded(err, [&] { *out = dup(img->img.serialize()); });
}

int hf_image_count(const hf_image* img) { return img ? int(img->img.arrays.size()) : 0; }

namespace {
int entry_of(hf::ArrayEntry& a, void** dev_ptr, int32_t** host_ptr, long long* len, int* is_float) {
  if (dev_ptr) *dev_ptr = a.dev_valid ? a.dev : nullptr;
  if (host_ptr) *host_ptr = a.host_valid ? a.host.data() : nullptr;
  if (len) *len = a.len;
  if (is_float) *is_float = a.ty == hf::Ty::Float;
  return HF_OK;
}
}  // namespace

int hf_image_entry(hf_image* img, int i, const char** name, void** dev_ptr, int32_t** host_ptr, long long* len,
                   int* is_float) {
  if (!img || i < 0 || i >= int(img->img.arrays.size())) return to_abi(hf::Code::InvalidArgument);
  auto it = img->img.arrays.begin();
  std::advance(it, i);
  if (name) *name = it->first.c_str();
  return entry_of(it->second, dev_ptr, host_ptr, len, is_float);
}

int hf_image_find(hf_image* img, const char* name, void** dev_ptr, int32_t** host_ptr, long long* len,
                  int* is_float) {
  if (!img) return to_abi(hf::Code::InvalidArgument);
  auto it = img->img.arrays.find(name);
  if (it == img->img.arrays.end()) return to_abi(hf::Code::InvalidArgument);
  return entry_of(it->second, dev_ptr, host_ptr, len, is_float);
}

int hf_image_set_host(hf_image* img, const char* name, const void* data, long long len, hf_error* err) {
  return guarded(err, [&] {
    auto it = img->img.arrays.find(name);
    if (it == img->img.arrays.end()) hf::raise(hf::Code::InvalidArgument, std::string("no array '") + name + "'");
    if (len != it->second.len) hf::raise(hf::Code::InvalidArgument, "length mismatch");
    it->second.host.assign(static_cast<const int32_t*>(data), static_cast<const int32_t*>(data) + len);
    it->second.host_valid = true;
    it->second.mode = hf::ArrayEntry::Mode::Values;
  });
}

long long hf_image_bytes(const hf_image* img) { return img ? img->img.bytes() : 0; }

void hf_image_free(hf_image* img) {
  if (!img) return;
  if (hf::rt::device_available()) hf::rt::release(img->img);
  delete img;
}

int hf_run(const hf_module* m, hf_image* img, int grid, void* stream, hf_error* err) {
  return hf_run_ex(m, img, grid, stream, 0, err);
}

int hf_run_ex(const hf_module* m, hf_image* img, int grid, void* stream, int flags, hf_error* err) {
  return guarded(err, [&] { hf::rt::launch(m->m, img->img, grid, stream, (flags & HF_LAUNCH_OVERLAP) != 0); });
}

int hf_time(int mode, const hf_module* a, const hf_module* b, hf_image* img, int grid_a, int grid_b, int warmup,
            int reps, int flush_l2, void* stream, hf_timing* out, hf_error* err) {
  return guarded(err, [&] {
    hf::rt::Mode md = mode == HF_TIME_SEQUENTIAL ? hf::rt::Mode::Sequential
                      : mode == HF_TIME_TWO_STREAM ? hf::rt::Mode::TwoStream
                                                   : hf::rt::Mode::Single;
    hf::rt::Timing t = hf::rt::time(md, a->m, b ? &b->m : nullptr, img->img, grid_a, grid_b, warmup, reps,
                                    flush_l2 != 0, stream);
    *out = hf_timing{t.median_us, t.min_us, t.mean_us, t.max_us, t.reps, t.iqm_us};
  });
}

static_assert(sizeof(hf_pack_src) == sizeof(hf::shard::PackSrc), "hf_pack_src layout");
static_assert(sizeof(hf_reduce_slot) == sizeof(hf::shard::ReduceSlot), "hf_reduce_slot layout");

int hf_shard_pack(const hf_pack_src* srcs, int n, int* packed, void* stream, hf_error* err) {
  return guarded(err, [&] {
    hf::shard::pack(reinterpret_cast<const hf::shard::PackSrc*>(srcs), n, packed, stream);
  });
}

int hf_shard_reduce(const int* gathered, int world, long long cells, const hf_reduce_slot* slots, int nslots,
                    const double* counts, void* out, void* stream, hf_error* err) {
  return guarded(err, [&] {
    hf::shard::reduce(gathered, world, cells, reinterpret_cast<const hf::shard::ReduceSlot*>(slots), nslots, counts,
                      out, stream);
  });
}

int hf_time_graph(int mode, const hf_module* a, const hf_module* b, hf_image* img, int grid_a, int grid_b,
                  int reps, int samples, void* stream, hf_graph_timing* out, hf_error* err) {
  return guarded(err, [&] {
    hf::rt::Mode md = mode == HF_TIME_SEQUENTIAL ? hf::rt::Mode::Sequential
                      : mode == HF_TIME_TWO_STREAM ? hf::rt::Mode::TwoStream
                                                   : hf::rt::Mode::Single;
    hf::rt::GraphTiming t =
        hf::rt::time_graph(md, a->m, b ? &b->m : nullptr, img->img, grid_a, grid_b, reps, samples, stream);
    *out = hf_graph_timing{t.mean_us, t.median_us, t.min_us, t.max_us, t.ci95_us, t.samples, t.reps};
  });
}

int hf_profile(const char* src1, const char* src2, int d1, int d2, int regcap, hf_image* img, int grid, int warmup,
               int reps, int flush_l2, int specialize, hf_eval* out, hf_error* err) {
  return guarded(err, [&] {
    hf::rt::Module m = build_fused(src1, src2, d1, d2, regcap, grid, 0, specialize ? img : nullptr);
    // flushed: per-repetition events after an L2 sweep (interquartile mean); steady (flush_l2 = 0):
    // the graph protocol, `reps` back-to-back repetitions per graph, median of 5 samples
    double us = flush_l2 ? hf::rt::time(hf::rt::Mode::Single, m, nullptr, img->img, grid, 0, warmup, reps, true,
                                        nullptr).iqm_us
                         : hf::rt::time_graph(hf::rt::Mode::Single, m, nullptr, img->img, grid, 0,
                                              std::max(1, reps), 5).median_us;
    hf::rt::Props p = hf::rt::props();
    out->us = us;
    out->cycles = (long long)(us * 1000.0 + 0.5);
    out->occupancy = double(m.blocks_per_sm) * (d1 + d2) / double(p.max_threads_per_sm);
    out->utilization = 0.0;
    out->regs = m.regs;
    hf::rt::unload(m);
  });
}

int hf_search(const char* src1, const char* src2, hf_image* img, hf_search_opts* opts, int* best_d1,
              int* best_d2, int* best_regcap, long long* best_time, char** trace, char** best_src, hf_error* err) {
  return guarded(err, [&] {
    hf_search_opts o{};
    if (opts) o = *opts;
    if (o.d0 <= 0) o.d0 = 1024;
    hf::SM sm = hf::rt::device_available() ? hf::rt::sm_from_device() : hf::SM::b200();
    hf::Loaded l1 = hf::load_source(src1), l2 = hf::load_source(src2);
    hf::Kernel n1 = hf::normalize(l1.kernel, l1.prog.funcs, "k1_");
    hf::Kernel n2 = hf::normalize(l2.kernel, l2.prog.funcs, "k2_");
    if (o.grid > 0) n1.grid = n2.grid = o.grid;
    std::unique_ptr<hf::ProfilerBackend> be;
    if (o.backend == HF_BACKEND_COMMAND) {
      be = std::make_unique<hf::ExternalCommandBackend>(o.profiler_cmd ? o.profiler_cmd : "");
    } else {
      if (!img) hf::raise(hf::Code::InvalidArgument, "the device backend needs a memory image");
      auto dev = std::make_unique<hf::DeviceBackend>(img->img, o.grid, o.warmup > 0 ? o.warmup : 3,
                                                     o.reps > 0 ? o.reps : 10, o.flush_l2 != 0,
                                                     o.measured_registers != 0);
      if (o.specialize) dev->set_specialization(scalars_of(img));
      be = std::move(dev);
    }
    hf::SearchOptions so;
    so.granularity = o.granularity > 0 ? o.granularity : 128;
    for (int i = 0; i < o.n_extra_caps; ++i) so.extra_caps.push_back(o.extra_caps[i]);
    so.interval_regs = o.interval_regs != 0;
    so.prefilter = o.prefilter;
    if (o.prefilter_tol >= 0) so.prefilter_tol = o.prefilter_tol;
    if (o.budget_points > 0) so.budget_points = o.budget_points;
    hf::SearchResult r = (n1.tunable && n2.tunable) ? hf::search_config(n1, n2, o.d0, *be, sm, so)
                                                    : hf::fixed_partition_fuse(n1, n2, *be, sm, o.d0, so);
    if (best_d1) *best_d1 = r.best_cfg.d1;
    if (best_d2) *best_d2 = r.best_cfg.d2;
    if (best_regcap) *best_regcap = r.best_cfg.reg_cap ? *r.best_cfg.reg_cap : HF_REGCAP_OFF;
    if (best_time) *best_time = r.best_time;
    if (opts) {
      opts->best_regs1 = r.best_cfg.regs1;
      opts->best_regs2 = r.best_cfg.regs2;
      opts->model_csv = nullptr;
      if (!r.predicted_us.empty()) {
        // d1,predicted,t1(d1),t2(d0-d1); the d1 = 0 row holds the full-block times T1, T2
        std::string m = "d1,predicted_us,t1_us,t2_us\n";
        char buf[128];
        for (const auto& [d1, tt] : r.member_us) {
          auto p = r.predicted_us.find(d1);
          std::snprintf(buf, sizeof(buf), "%d,%.3f,%.3f,%.3f\n", d1, p == r.predicted_us.end() ? 0.0 : p->second,
                        tt.first, tt.second);
          m += buf;
        }
        opts->model_csv = dup(m);
      }
    }
    if (trace) *trace = dup(hf::trace_csv(r));
    if (best_src) *best_src = dup(hf::emit(r.best, style_of(o.out_style)));
  });
}

}  // extern "C"
