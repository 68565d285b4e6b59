// Memory images: named int32/float32 arrays and scalars bound to kernel parameters.
//
// Text format, seeded generators and digest follow the reference
// (/root/reference/proj/src/memimage.cpp:10-248):
//   array NAME (int32|float32) LEN zero | values V... | seed S range LO HI | seed S uniform LO HI
//   scalar NAME (int32|float32) VALUE
// B200 layout: entries stay *lazy* on the host (a seeded 205 MB array is one line), and
// are materialized directly in HBM by the splitmix64 fill kernels of runtime.cu, which
// reproduce memimage.cpp:10-61 bit for bit. Host copies exist only after a download.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "ir.hpp"

namespace hf {

uint64_t splitmix64(uint64_t& state);
uint64_t mix_seed(uint64_t file_seed, std::optional<uint64_t> override_seed);
float uniform_float(uint64_t bits, float lo, float hi);

struct ArrayEntry {
  enum class Mode { Zero, Values, SeedRange, SeedUniform } mode = Mode::Zero;
  Ty ty = Ty::Int;
  int64_t len = 0;
  uint64_t seed = 0;
  int32_t ilo = 0, ihi = 0;
  float flo = 0.0f, fhi = 0.0f;
  std::vector<int32_t> host;  // raw 32-bit cells (float bits for Float arrays) when materialized
  bool host_valid = false;
  void* dev = nullptr;        // device allocation (runtime.cu)
  bool dev_valid = false;
};

struct ScalarEntry {
  Ty ty = Ty::Int;
  int32_t i = 0;
  float f = 0.0f;
};

struct Image {
  std::map<std::string, ArrayEntry> arrays;
  std::map<std::string, ScalarEntry> scalars;
  int device = -1;

  static Image parse(const std::string& text, std::optional<uint64_t> seed_override = std::nullopt);
  void merge(Image&& other);
  void materialize_host();           // CPU generation (tests / oracle interop)
  std::string serialize() const;     // `values` form (needs host copies)
  uint64_t digest() const;           // FNV-1a 64 (needs host copies)
  std::string digest_hex() const;
  int64_t bytes() const;             // total array bytes
};

}  // namespace hf
