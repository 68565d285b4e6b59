// Does a TMA bulk-copy pipeline speed up the Hist member? 205.5 MB of fp32 binned into 64 bins
// over [-4, 4] with warp-private shared bins, fed by (a) 4 x LDG.128 in flight per thread (the
// MK+ member's scheme) or (b) cp.async.bulk 16 KB chunks into a 4-stage shared ring per block.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/tma_hist scripts/tma_hist_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void bin(int* bins, int wb, float v) {
  if (v >= -4.0f && v <= 4.0f) atomicAdd(&bins[wb + min(__float2int_rz((v + 4.0f) * 8.0f), 63)], 1);
}

__global__ void __launch_bounds__(1024) hist_ldg(const float4* __restrict__ x, int n4, int* out) {
  __shared__ int bins[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) bins[i] = 0;
  __syncthreads();
  const int wb = (threadIdx.x / 32) * 64, stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 4 * stride) {
    float4 a = x[i], b = x[min(i + stride, n4 - 1)], c = x[min(i + 2 * stride, n4 - 1)], d = x[min(i + 3 * stride, n4 - 1)];
    bin(bins, wb, a.x); bin(bins, wb, a.y); bin(bins, wb, a.z); bin(bins, wb, a.w);
    if (i + stride < n4) { bin(bins, wb, b.x); bin(bins, wb, b.y); bin(bins, wb, b.z); bin(bins, wb, b.w); }
    if (i + 2 * stride < n4) { bin(bins, wb, c.x); bin(bins, wb, c.y); bin(bins, wb, c.z); bin(bins, wb, c.w); }
    if (i + 3 * stride < n4) { bin(bins, wb, d.x); bin(bins, wb, d.y); bin(bins, wb, d.z); bin(bins, wb, d.w); }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    int s = 0;
    for (int w = 0; w < blockDim.x / 32; ++w) s += bins[w * 64 + b];
    atomicAdd(&out[b], s);
  }
}

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(1024) hist_tma(const float* __restrict__ x, int n, int* out) {
  extern __shared__ __align__(128) char buf[];
  __shared__ int bins[2048];
  __shared__ __align__(8) unsigned long long bar[STAGES];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) bins[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int per = CHUNK / 4, chunks = n / per, wb = (threadIdx.x / 32) * 64;
  auto issue = [&](int c, int s) {
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(buf + s * CHUNK)),
                 "l"(x + size_t(c) * per), "r"(CHUNK), "r"(b)
                 : "memory");
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < STAGES && blockIdx.x + s * gridDim.x < chunks; ++s) issue(blockIdx.x + s * gridDim.x, s);
  unsigned phase = 0;
  int s = 0;
  for (int c = blockIdx.x; c < chunks; c += gridDim.x) {
    unsigned done = 0, b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(b), "r"((phase >> s) & 1u));
    phase ^= 1u << s;
    const float4* v = reinterpret_cast<const float4*>(buf + s * CHUNK);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) {
      float4 q = v[i];
      bin(bins, wb, q.x); bin(bins, wb, q.y); bin(bins, wb, q.z); bin(bins, wb, q.w);
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + STAGES * gridDim.x < chunks) issue(c + STAGES * gridDim.x, s);
    s = (s + 1) % STAGES;
  }
  // tail (n not a multiple of the chunk): plain loads
  for (int i = chunks * per + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) bin(bins, wb, x[i]);
  __syncthreads();
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    int t = 0;
    for (int w = 0; w < blockDim.x / 32; ++w) t += bins[w * 64 + b];
    atomicAdd(&out[b], t);
  }
}


// (c) warp-specialized: warp 0 lane 0 produces (waits on empty[s], issues the bulk copy into
// stage s, full[s] completes on the bytes); the other warps consume (wait full[s], bin their
// share, one arrive per warp on empty[s]) -- no block barrier in the loop
template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(1024) hist_tma_ws(const float* __restrict__ x, int n, int* out) {
  extern __shared__ __align__(128) char buf[];
  __shared__ int bins[2048];
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  const int nwarps = blockDim.x / 32, cw = nwarps - 1;  // consumer warps
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) bins[i] = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&full[s])));
      asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&empty[s])), "r"(cw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int per = CHUNK / 4, chunks = n / per, wb = (threadIdx.x / 32) * 64;
  auto wait = [](unsigned long long* bar, unsigned parity) {
    unsigned done = 0, b = (unsigned)__cvta_generic_to_shared(bar);
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done) : "r"(b), "r"(parity));
  };
  if (threadIdx.x < 32) {  // producer warp
    if (threadIdx.x == 0) {
      int k = 0;
      for (int c = blockIdx.x; c < chunks; c += gridDim.x, ++k) {
        int s = k % STAGES;
        if (k >= STAGES) wait(&empty[s], ((k / STAGES) - 1) & 1);
        unsigned b = (unsigned)__cvta_generic_to_shared(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(buf + s * CHUNK)),
                     "l"(x + size_t(c) * per), "r"(CHUNK), "r"(b)
                     : "memory");
      }
    }
  } else {  // consumer warps
    const int ct = threadIdx.x - 32;
    int k = 0;
    for (int c = blockIdx.x; c < chunks; c += gridDim.x, ++k) {
      int s = k % STAGES;
      wait(&full[s], (k / STAGES) & 1);
      const float4* v = reinterpret_cast<const float4*>(buf + s * CHUNK);
      for (int i = ct; i < CHUNK / 16; i += cw * 32) {
        float4 q = v[i];
        bin(bins, wb, q.x); bin(bins, wb, q.y); bin(bins, wb, q.z); bin(bins, wb, q.w);
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0)
        asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&empty[s])));
    }
  }
  for (int i = chunks * per + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) bin(bins, wb, x[i]);
  __syncthreads();
  for (int b = threadIdx.x; b < 64; b += blockDim.x) {
    int t = 0;
    for (int w = 0; w < blockDim.x / 32; ++w) t += bins[w * 64 + b];
    atomicAdd(&out[b], t);
  }
}

__global__ void fill(float* x, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned h = i * 2654435761u;
    h ^= h >> 13;
    x[i] = (h % 10000) * 0.0009f - 4.5f;
  }
}

int main() {
  const int n = 64 * 256 * 56 * 56;
  float* x;
  int* out;
  cudaMalloc(&x, size_t(n) * 4);
  cudaMalloc(&out, 64 * 4 * 8);  // 7 result slots used
  fill<<<1184, 256>>>(x, n);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int ref[64], got[64];
  auto run = [&](const char* name, int grid, auto launch, int slot) {
    float best = 1e9f;
    for (int r = 0; r < 12; ++r) {
      cudaMemset(out + 64 * slot, 0, 256);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r >= 2 && ms < best) best = ms;
    }
    cudaMemcpy(slot == 0 ? ref : got, out + 64 * slot, 256, cudaMemcpyDeviceToHost);
    bool same = true;
    if (slot) for (int i = 0; i < 64; ++i) same &= ref[i] == got[i];
    std::printf("{\"kind\": \"%s\", \"grid\": %d, \"us\": %.2f, \"gbs\": %.1f, \"same_bins\": %s, \"err\": \"%s\"},\n",
                name, grid, best * 1e3, n * 4.0 / (best * 1e6), same ? "true" : "false",
                cudaGetErrorString(cudaGetLastError()));
  };
  std::printf("[\n");
  run("ldg128x4", 2 * sms, [&] { hist_ldg<<<2 * sms, 1024>>>(reinterpret_cast<const float4*>(x), n / 4, out); }, 0);
  constexpr int S4 = 4, C16 = 16384, S3 = 3, C32 = 32768;
  cudaFuncSetAttribute(hist_tma<S4, C16>, cudaFuncAttributeMaxDynamicSharedMemorySize, S4 * C16);
  cudaFuncSetAttribute(hist_tma<S3, C32>, cudaFuncAttributeMaxDynamicSharedMemorySize, S3 * C32);
  run("tma_4x16KB", 2 * sms, [&] { hist_tma<S4, C16><<<2 * sms, 1024, S4 * C16>>>(x, n, out + 64); }, 1);
  run("tma_3x32KB", 2 * sms, [&] { hist_tma<S3, C32><<<2 * sms, 1024, S3 * C32>>>(x, n, out + 128); }, 2);
  run("tma_4x16KB_g1", sms, [&] { hist_tma<S4, C16><<<sms, 1024, S4 * C16>>>(x, n, out + 192); }, 3);
  constexpr int S6 = 6, S8 = 8, C8 = 8192;
  cudaFuncSetAttribute(hist_tma_ws<S4, C16>, cudaFuncAttributeMaxDynamicSharedMemorySize, S4 * C16);
  cudaFuncSetAttribute(hist_tma_ws<S6, C16>, cudaFuncAttributeMaxDynamicSharedMemorySize, S6 * C16);
  cudaFuncSetAttribute(hist_tma_ws<S8, C8>, cudaFuncAttributeMaxDynamicSharedMemorySize, S8 * C8);
  run("ws_4x16KB", 2 * sms, [&] { hist_tma_ws<S4, C16><<<2 * sms, 1024, S4 * C16>>>(x, n, out + 256); }, 4);
  run("ws_6x16KB", 2 * sms, [&] { hist_tma_ws<S6, C16><<<2 * sms, 1024, S6 * C16>>>(x, n, out + 320); }, 5);
  run("ws_8x8KB", 2 * sms, [&] { hist_tma_ws<S8, C8><<<2 * sms, 1024, S8 * C8>>>(x, n, out + 384); }, 6);
  std::printf("{}]\n");
  return 0;
}
