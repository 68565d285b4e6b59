// HBM write-stream ceiling on the B200: 128-bit STG (what the MK+ members' vstore emits) vs TMA
// bulk stores (st.shared into a per-CTA ring, then cp.async.bulk.global.shared::cta.bulk_group,
// stage reuse gated by cp.async.bulk.wait_group.read), pure writes and a 1:4 read:write mix (the
// Upsample / Im2Col shape). Decides whether write-heavy members should stage their outputs for TMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/tma_write_probe scripts/tma_write_probe.cu
//   gpurun_out/tma_write_probe > gpurun_out/tma_write_probe.json
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));             \
      return 1;                                                                \
    }                                                                          \
  } while (0)

// ratio = bytes written per byte read (0 = pure write); reads are LDG.128 of src, each read float4
// produces `ratio` float4 outputs
__global__ void __launch_bounds__(1024) stg_stream(const float4* __restrict__ src, float4* __restrict__ dst,
                                                   size_t nw4, int ratio) {
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nw4; i += stride) {
    float4 v;
    if (ratio) {
      v = src[i / ratio];
    } else {
      v = make_float4(float(i), 1.f, 2.f, 3.f);
    }
    dst[i] = v;
  }
}

constexpr int STAGES = 4;
constexpr int CHUNK = 16384;  // bytes per bulk store

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256) tma_stream(const float4* __restrict__ src, char* __restrict__ dst,
                                                  size_t bytes, int ratio) {
  extern __shared__ __align__(128) char buf[];
  const size_t chunks = bytes / CHUNK;
  int s = 0;
  for (size_t c = blockIdx.x, k = 0; c < chunks; c += gridDim.x, ++k) {
    if (k >= STAGES) {
      // the bulk store that last read stage s has finished reading shared memory
      if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1) : "memory");
      __syncthreads();
    }
    float4* v = reinterpret_cast<float4*>(buf + s * CHUNK);
    const size_t base4 = c * (CHUNK / 16);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) {
      size_t g = base4 + i;
      v[i] = ratio ? src[g / ratio] : make_float4(float(g), 1.f, 2.f, 3.f);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + c * CHUNK),
                   "r"(smem_addr(buf + s * CHUNK)), "r"(CHUNK)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    s = (s + 1) % STAGES;
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t wbytes = size_t(1) << 30;
  char *src, *dst;
  CK(cudaMalloc(&src, wbytes));
  CK(cudaMalloc(&dst, wbytes));
  CK(cudaMemset(src, 0, wbytes));
  CK(cudaMemset(dst, 0, wbytes));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto best = [&](auto launch) -> float {
    float bestms = 1e9f;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      if (cudaEventSynchronize(b) != cudaSuccess) return -1.f;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 2 && ms < bestms) bestms = ms;
    }
    return bestms;
  };
  const int smem = STAGES * CHUNK;
  CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  std::printf("[\n");
  bool first = true;
  for (int ratio : {0, 4}) {
    const size_t moved = wbytes + (ratio ? wbytes / ratio : 0);
    for (int per : {2, 4, 8}) {
      int grid = sms * per;
      float ms = best([&] {
        stg_stream<<<grid, 1024>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), wbytes / 16,
                                   ratio);
      });
      std::printf("%s{\"kind\": \"stg128\", \"rw\": \"%s\", \"grid\": %d, \"threads\": 1024, \"us\": %.2f, \"gbs\": %.1f}",
                  first ? "" : ",\n", ratio ? "1:4" : "write", grid, ms * 1e3, moved / (ms * 1e6));
      first = false;
    }
    for (int per : {2, 3, 4, 6, 8}) {
      int grid = sms * per;
      float ms = best([&] {
        tma_stream<<<grid, 256, smem>>>(reinterpret_cast<const float4*>(src), dst, wbytes, ratio);
      });
      std::printf(",\n{\"kind\": \"tma_bulk_store_%dx%dKB\", \"rw\": \"%s\", \"grid\": %d, \"threads\": 256, \"us\": %.2f, "
                  "\"gbs\": %.1f}",
                  STAGES, CHUNK / 1024, ratio ? "1:4" : "write", grid, ms * 1e3, moved / (ms * 1e6));
    }
  }
  std::printf("\n]\n");
  CK(cudaGetLastError());
  return 0;
}
