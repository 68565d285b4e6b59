// CUDA form of the reference corpus kernel proj/corpus/histogram.mk (test input of the
// restricted-CUDA frontend).
__device__ __forceinline__ int bin_of(int value, int nbins) {
  int b = value % nbins;
  return b;
}

extern "C" __global__ void __launch_bounds__(128) histogram(const int* hist_in, int* hist_out, int hist_n) {
  __shared__ int bins[64];

  // region A: clear the shared counters
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    bins[i] = 0;
  }
  __syncthreads();

  // region B: count into shared memory
  for (int i = threadIdx.x; i < hist_n; i += blockDim.x) {
    int v = hist_in[i];
    if (v >= 0) {
      int b = bin_of(v, 64);
      atomicAdd(&bins[b], 1);
    }
  }
  __syncthreads();

  // region C: merge the shared counters into the output
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    atomicAdd(&hist_out[i], bins[i]);
  }
}
