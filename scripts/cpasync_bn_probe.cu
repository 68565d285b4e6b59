// Does a register-free load pipeline help the block-per-channel BatchNorm stream? Two hand-written
// stand-ins for the MK+ member's streaming loop (sum and sum of squares of each channel of
// x[64, 256, 3136]), timed back to back (steady protocol) on one B200:
//   regs4  : four 128-bit loads in flight per thread (the member's form, 32 registers)
//   cpasyncS: an S-stage cp.async ring per thread in shared memory (16 B per stage), the data
//            never occupies registers while in flight
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/cpasync_bn_probe scripts/cpasync_bn_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 64, C = 256, HW = 3136, HW4 = HW / 4;

__device__ __forceinline__ void reduce_store(float s1, float s2, float* out, int c) {
  for (int m = 16; m > 0; m >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, m);
    s2 += __shfl_xor_sync(0xffffffffu, s2, m);
  }
  __shared__ float a[32], b[32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { a[w] = s1; b[w] = s2; }
  __syncthreads();
  if (w == 0) {
    s1 = lane < (blockDim.x >> 5) ? a[lane] : 0.f;
    s2 = lane < (blockDim.x >> 5) ? b[lane] : 0.f;
    for (int m = 16; m > 0; m >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, m);
      s2 += __shfl_xor_sync(0xffffffffu, s2, m);
    }
    if (lane == 0) { out[2 * c] = s1; out[2 * c + 1] = s2; }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(1024, 2) regs4(const float4* __restrict__ x, float* out) {
  const int T = N * HW4, nt = blockDim.x;
  for (int c = blockIdx.x; c < C; c += gridDim.x) {
    float s1 = 0.f, s2 = 0.f;
    int j = threadIdx.x;
    for (; j + 3 * nt < T; j += 4 * nt) {
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int jj = j + k * nt, p = jj / HW4;
        v[k] = x[(p * C + c) * HW4 + jj - p * HW4];
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        s1 += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        s2 += (v[k].x * v[k].x + v[k].y * v[k].y) + (v[k].z * v[k].z + v[k].w * v[k].w);
      }
    }
    for (; j < T; j += nt) {
      int p = j / HW4;
      float4 v = x[(p * C + c) * HW4 + j - p * HW4];
      s1 += (v.x + v.y) + (v.z + v.w);
      s2 += (v.x * v.x + v.y * v.y) + (v.z * v.z + v.w * v.w);
    }
    reduce_store(s1, s2, out, c);
  }
}

template <int S>
__global__ void __launch_bounds__(1024, 2) cpasync(const float4* __restrict__ x, float* out) {
  extern __shared__ float4 ring[];  // S stages x blockDim vectors
  const int T = N * HW4, nt = blockDim.x, t = threadIdx.x;
  for (int c = blockIdx.x; c < C; c += gridDim.x) {
    float s1 = 0.f, s2 = 0.f;
    auto issue = [&](int k) {  // stage k % S <- vector j = t + k * nt (if in range)
      int jj = t + k * nt;
      if (jj < T) {
        int p = jj / HW4;
        const float4* g = x + (p * C + c) * HW4 + jj - p * HW4;
        unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&ring[(k % S) * nt + t]));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int iters = (T - t + nt - 1) / nt;
#pragma unroll
    for (int k = 0; k < S - 1; ++k) issue(k);
    for (int k = 0; k < iters; ++k) {
      issue(k + S - 1);
      asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
      float4 v = ring[(k % S) * nt + t];
      s1 += (v.x + v.y) + (v.z + v.w);
      s2 += (v.x * v.x + v.y * v.y) + (v.z * v.z + v.w * v.w);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    reduce_store(s1, s2, out, c);
  }
}

int main() {
  const size_t n4 = size_t(N) * C * HW4;
  float4* x;
  float* out;
  cudaMalloc(&x, n4 * 16);
  cudaMalloc(&out, 2 * C * 4);
  cudaMemset(x, 0, n4 * 16);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 5; ++w) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 50; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("{\"kernel\": \"%s\", \"us\": %.2f, \"gbs\": %.1f, \"err\": \"%s\"},\n", name, ms * 1e3 / 50,
           n4 * 16 / (ms * 1e6 / 50), cudaGetErrorString(e));
  };
  printf("[\n");
  for (int g : {256, 296})
    run(g == 256 ? "regs4@256" : "regs4@296", [&] { regs4<<<g, 1024>>>(x, out); });
  auto cp = [&](auto kern, int S, const char* name) {
    int smem = S * 1024 * 16;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    run(name, [&] { kern<<<256, 1024, smem>>>(x, out); });
  };
  cp(cpasync<2>, 2, "cpasync2");
  cp(cpasync<3>, 3, "cpasync3");
  cp(cpasync<4>, 4, "cpasync4");
  cp(cpasync<6>, 6, "cpasync6");
  printf("{}]\n");
  return 0;
}
