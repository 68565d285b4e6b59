// BatchNorm-stats read stream on the B200: register-direct LDG.128 (the MK+ member's form: 768
// threads per channel block, eight 128-bit loads in flight) vs a warp-specialized TMA pipeline (one
// producer lane issues a cp.async.bulk per 12,544-byte plane into a STAGES-deep shared ring,
// mbarrier full/empty handshakes, the consumer warps accumulate from shared memory; no block
// barrier). x = [64, 256, 3136] fp32 (205 MB, the C2 BN input); per-channel sum and sum of squares.
// Decides whether the BN member should be fed by bulk copies.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/tma_bn_probe scripts/tma_bn_probe.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      std::printf("{\"error\": \"%s\", \"line\": %d}\n", cudaGetErrorString(e), __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int N = 64, C = 256, HW = 3136;
constexpr int PLANE = HW * 4;  // bytes

__device__ __forceinline__ void block_reduce_store(float s, float q, float* out, int slot) {
  __shared__ float rs[32], rq[32];
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) { rs[w] = s; rq[w] = q; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f, b = 0.f;
    for (int i = 0; i < int(blockDim.x / 32); ++i) { a += rs[i]; b += rq[i]; }
    out[2 * slot] = a;
    out[2 * slot + 1] = b;
  }
}

// blocks = C * split; block b handles channel b / split, planes [part*N/split, (part+1)*N/split)
__global__ void __launch_bounds__(768) bn_ldg(const float4* __restrict__ x, float* out, int split) {
  const int c = blockIdx.x / split, part = blockIdx.x % split;
  const int n0 = part * (N / split), n1 = n0 + N / split;
  const int per = HW / 4;  // float4 per plane
  float s = 0.f, q = 0.f;
  const int total = (n1 - n0) * per;
  int i = threadIdx.x;
  for (; i + 7 * int(blockDim.x) < total; i += 8 * blockDim.x) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      int j = i + k * blockDim.x, n = n0 + j / per, r = j % per;
      v[k] = x[(size_t(n) * C + c) * per + r];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s += v[k].x + v[k].y + v[k].z + v[k].w;
      q += v[k].x * v[k].x + v[k].y * v[k].y + v[k].z * v[k].z + v[k].w * v[k].w;
    }
  }
  for (; i < total; i += blockDim.x) {
    int n = n0 + i / per, r = i % per;
    float4 v = x[(size_t(n) * C + c) * per + r];
    s += v.x + v.y + v.z + v.w;
    q += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  block_reduce_store(s, q, out, blockIdx.x);
}

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  long long spins = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(smem_addr(bar)), "r"(parity)
                 : "memory");
    if (++spins > (1ll << 26)) __trap();  // a probe bug must not hang the box
  }
}

template <int STAGES>
__global__ void __launch_bounds__(512) bn_tma(const char* __restrict__ x, float* out, int split) {
  extern __shared__ __align__(128) char ring[];
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  const int c = blockIdx.x / split, part = blockIdx.x % split;
  const int n0 = part * (N / split), planes = N / split;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, consumers = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&empty[s])), "r"(consumers));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  float s = 0.f, q = 0.f;
  if (warp == 0) {
    if (lane == 0) {
      for (int k = 0; k < planes; ++k) {
        const int st = k % STAGES;
        if (k >= STAGES) mbar_wait(&empty[st], ((k / STAGES) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[st])), "r"(PLANE)
                     : "memory");
        const char* src = x + (size_t(n0 + k) * C + c) * PLANE;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(ring + st * PLANE)),
            "l"(src), "r"(PLANE), "r"(smem_addr(&full[st]))
            : "memory");
      }
    }
  } else {
    const int t = threadIdx.x - 32, nt = consumers * 32;
    for (int k = 0; k < planes; ++k) {
      const int st = k % STAGES;
      mbar_wait(&full[st], (k / STAGES) & 1);
      const float4* v = reinterpret_cast<const float4*>(ring + st * PLANE);
      for (int i = t; i < HW / 4; i += nt) {
        float4 a = v[i];
        s += a.x + a.y + a.z + a.w;
        q += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&empty[st])) : "memory");
    }
  }
  block_reduce_store(s, q, out, blockIdx.x);
}

int main() {
  const size_t bytes = size_t(N) * C * HW * 4;
  float *x, *out, *ref;
  CK(cudaMalloc(&x, bytes));
  CK(cudaMalloc(&out, 2 * C * 8 * sizeof(float)));
  CK(cudaMalloc(&ref, 2 * C * 8 * sizeof(float)));
  CK(cudaMemset(x, 0x3c, bytes));  // every element 0x3c3c3c3c = 0.01149...
  float elem;
  {
    unsigned u = 0x3c3c3c3cu;
    memcpy(&elem, &u, 4);
  }
  auto check = [&](float* d, int slots) -> double {  // total of the per-block sums / expected
    static float h[2 * C * 8];
    cudaMemcpy(h, d, 2 * slots * sizeof(float), cudaMemcpyDeviceToHost);
    double t = 0;
    for (int i = 0; i < slots; ++i) t += h[2 * i];
    return t / (double(N) * C * HW * elem);
  };
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto best = [&](auto launch) -> float {
    float bestms = 1e9f;
    for (int r = 0; r < 15; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      if (cudaEventSynchronize(b) != cudaSuccess) return -1.f;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 3 && ms < bestms) bestms = ms;
    }
    return bestms;
  };
  std::printf("[\n");
  for (int split : {1, 2, 4}) {
    float ms = best([&] { bn_ldg<<<C * split, 768>>>(reinterpret_cast<const float4*>(x), ref, split); });
    CK(cudaGetLastError());
    std::printf("{\"kind\": \"ldg128x8\", \"blocks\": %d, \"threads\": 768, \"us\": %.2f, \"gbs\": %.1f, \"sum_ok\": %.6f},\n",
                C * split, ms * 1e3, bytes / (ms * 1e6), check(ref, C * split));
  }
  auto run_tma = [&](auto kern, int stages, int threads, int split, bool last) -> int {
    const int smem = stages * PLANE;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    float ms = best([&] { kern<<<C * split, threads, smem>>>(reinterpret_cast<const char*>(x), out, split); });
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::printf("{\"kind\": \"tma_ring\", \"stages\": %d, \"blocks\": %d, \"threads\": %d, \"us\": %.2f, \"gbs\": %.1f, \"sum_ok\": %.6f}%s\n",
                stages, C * split, threads, ms * 1e3, bytes / (ms * 1e6), check(out, C * split), last ? "" : ",");
    return 0;
  };
  if (run_tma(bn_tma<4>, 4, 256, 1, false)) return 1;
  if (run_tma(bn_tma<8>, 8, 256, 1, false)) return 1;
  if (run_tma(bn_tma<8>, 8, 512, 1, false)) return 1;
  if (run_tma(bn_tma<4>, 4, 256, 2, false)) return 1;
  if (run_tma(bn_tma<8>, 8, 256, 2, false)) return 1;
  if (run_tma(bn_tma<4>, 4, 256, 4, false)) return 1;
  if (run_tma(bn_tma<6>, 6, 256, 4, true)) return 1;
  std::printf("]\n");
  return 0;
}
