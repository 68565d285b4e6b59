// The multi-GPU step's one exchange on the device (bench.py strong scaling, shard.py): every
// rank packs its step outputs (histogram bins, BatchNorm per-channel (mean, var), crypto
// (hits, winning nonce)) into one int32 buffer, the buffers are all-gathered (NCCL), and every
// rank reduces the [world, cells] result identically. Both ends are one kernel launch each, so a
// step at 1/8 of the batch pays three launches for its exchange instead of one copy per output
// and a few hundred small tensor ops.
//
// Reduction semantics (shard.reduce_gathered is the reference, tests/test_shard_reduce_gpu.py):
//   hist   -> int64 sum over ranks;
//   bn     -> Chan's parallel merge of (count, mean, biased var) in rank order, in fp64 with no
//             contraction (__dadd_rn/__dmul_rn/__ddiv_rn: the same operation order and rounding as
//             the torch fp64 merge, so the two agree bit for bit);
//   crypto -> int64 hit counts summed, int64 winning nonces minimised.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "runtime.hpp"
#include "shard_reduce.hpp"

namespace hf::shard {
namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(Code::Device, std::string(what) + ": " + cudaGetErrorString(e));
}

struct PackArgs {
  PackSrc src[kMaxPack];
  int n;
  long long total;  // sum of cells
};

__global__ void pack_cells(PackArgs a, int* __restrict__ packed) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.total; i += stride) {
    long long base = 0;
    int s = 0;
    while (i >= base + a.src[s].cells) base += a.src[s++].cells;
    const long long j = i - base;
    packed[a.src[s].offset + j] = static_cast<const int*>(a.src[s].src)[j];
  }
}

struct ReduceArgs {
  ReduceSlot slot[kMaxSlots];
  long long items[kMaxSlots];  // work items per slot
  double counts[kMaxRanks];
  int nslots;
  int world;
  long long cells;
  long long total;
};

__global__ void reduce_cells(ReduceArgs a, const int* __restrict__ g, void* __restrict__ out) {
  long long* oi = static_cast<long long*>(out);
  double* od = static_cast<double*>(out);
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.total; i += stride) {
    long long base = 0;
    int s = 0;
    while (i >= base + a.items[s]) base += a.items[s++];
    const ReduceSlot& sl = a.slot[s];
    const long long j = i - base;
    if (sl.kind == kHist) {
      long long sum = 0;
      for (int r = 0; r < a.world; ++r) sum += g[(long long)r * a.cells + sl.offset + j];
      oi[sl.out_offset + j] = sum;
    } else if (sl.kind == kBn) {  // channel j: cells hold (mean, var) float pairs per channel
      double n = 0.0, mean = 0.0, m2 = 0.0;
      for (int r = 0; r < a.world; ++r) {
        const double c = a.counts[r];
        const double mu = __int_as_float(g[(long long)r * a.cells + sl.offset + 2 * j]);
        const double var = __int_as_float(g[(long long)r * a.cells + sl.offset + 2 * j + 1]);
        const double tot = __dadd_rn(n, c);
        const double delta = __dsub_rn(mu, mean);
        mean = __dadd_rn(mean, __dmul_rn(delta, __ddiv_rn(c, tot)));
        m2 = __dadd_rn(__dadd_rn(m2, __dmul_rn(var, c)), __dmul_rn(__dmul_rn(delta, delta), __ddiv_rn(__dmul_rn(n, c), tot)));
        n = tot;
      }
      od[sl.out_offset + j] = mean;
      od[sl.out_offset + sl.channels + j] = __ddiv_rn(m2, n);
    } else {  // crypto: int64 (hits, nonce) pairs, j = pair index
      long long hits = 0, best = 0;
      for (int r = 0; r < a.world; ++r) {  // int64 words from int32 cells (rows need not be 8-B aligned)
        const int* p = g + (long long)r * a.cells + sl.offset + 4 * j;
        const long long h = (long long)(((unsigned long long)(unsigned)p[1] << 32) | (unsigned)p[0]);
        const long long b = (long long)(((unsigned long long)(unsigned)p[3] << 32) | (unsigned)p[2]);
        hits += h;
        best = r == 0 ? b : (b < best ? b : best);
      }
      oi[sl.out_offset + 2 * j] = hits;
      oi[sl.out_offset + 2 * j + 1] = best;
    }
  }
}

}  // namespace

void pack(const PackSrc* src, int n, int* packed, void* stream) {
  if (n < 0 || n > kMaxPack) raise(Code::InvalidArgument, "pack: 0.." + std::to_string(kMaxPack) + " sources");
  PackArgs a{};
  a.n = n;
  for (int i = 0; i < n; ++i) {
    if (src[i].cells < 0 || src[i].offset < 0) raise(Code::InvalidArgument, "pack: negative offset or cells");
    a.src[i] = src[i];
    a.total += src[i].cells;
  }
  if (a.total == 0) return;
  const int threads = 256;
  const int blocks = int(std::min<long long>((a.total + threads - 1) / threads, 1184));
  pack_cells<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(a, packed);
  check(cudaGetLastError(), "pack_cells");
}

void reduce(const int* gathered, int world, long long cells, const ReduceSlot* slots, int nslots,
            const double* counts, void* out, void* stream) {
  if (nslots < 0 || nslots > kMaxSlots) raise(Code::InvalidArgument, "reduce: 0.." + std::to_string(kMaxSlots) + " slots");
  if (world < 1 || world > kMaxRanks) raise(Code::InvalidArgument, "reduce: 1.." + std::to_string(kMaxRanks) + " ranks");
  ReduceArgs a{};
  a.nslots = nslots;
  a.world = world;
  a.cells = cells;
  bool bn = false;
  for (int s = 0; s < nslots; ++s) {
    const ReduceSlot& sl = slots[s];
    if (sl.offset < 0 || sl.cells < 0 || sl.offset + sl.cells > cells)
      raise(Code::InvalidArgument, "reduce: slot " + std::to_string(s) + " outside the packed cells");
    a.slot[s] = sl;
    if (sl.kind == kHist) {
      a.items[s] = sl.cells;
    } else if (sl.kind == kBn) {
      if (sl.cells != 2LL * sl.channels) raise(Code::InvalidArgument, "reduce: a bn slot holds 2 x channels cells");
      a.items[s] = sl.channels;
      bn = true;
    } else if (sl.kind == kCrypto) {
      if (sl.cells % 4) raise(Code::InvalidArgument, "reduce: crypto slots are int64 pairs");
      a.items[s] = sl.cells / 4;
    } else {
      raise(Code::InvalidArgument, "reduce: unknown slot kind " + std::to_string(sl.kind));
    }
    a.total += a.items[s];
  }
  if (bn) {
    if (!counts) raise(Code::InvalidArgument, "reduce: bn slots need per-rank counts");
    for (int r = 0; r < world; ++r) a.counts[r] = counts[r];
  }
  if (a.total == 0) return;
  const int threads = 128;
  const int blocks = int(std::min<long long>((a.total + threads - 1) / threads, 1184));
  reduce_cells<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(a, gathered, out);
  check(cudaGetLastError(), "reduce_cells");
}

}  // namespace hf::shard
