// Device side of the multi-GPU step exchange (shard_reduce.cu): pack the step outputs into one
// int32 buffer (one launch) and reduce the all-gathered [world, cells] buffer (one launch).
#pragma once

#include "ir.hpp"

namespace hf::shard {

constexpr int kMaxPack = 32;   // source arrays per pack launch
constexpr int kMaxSlots = 32;  // reduce slots per launch
constexpr int kMaxRanks = 64;
enum SlotKind { kHist = 0, kBn = 1, kCrypto = 2 };

struct PackSrc {
  const void* src;     // device int32 cells
  long long offset;    // destination cell offset in the packed buffer
  long long cells;
};

struct ReduceSlot {
  int kind;            // SlotKind
  int channels;        // bn: C (the slot holds C (mean, var) float pairs)
  long long offset;    // first cell of the slot in each rank's row
  long long cells;
  long long out_offset;  // 8-byte element offset in `out`
};

void pack(const PackSrc* src, int n, int* packed, void* stream);
// out (8-byte elements): hist -> int64[cells]; bn -> fp64 mean[C] then var[C]; crypto ->
// int64 (hits sum, nonce min) per pair. counts: per-rank elements per channel (bn slots).
void reduce(const int* gathered, int world, long long cells, const ReduceSlot* slots, int nslots,
            const double* counts, void* out, void* stream);

}  // namespace hf::shard
