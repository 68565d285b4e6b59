// Histogram, reference (naive) form: the plain Mini-Kernel a user would write from
// torch.histc (PAPER.md:405-430). Scalar loads, one block-shared bin array, the
// division form of the bin index. This is what the naive (goto) fusion consumes.
//@ grid=256
kernel hist(float hi_x[], int hi_out[], int hi_n) dims (1024, 1, 1) {
  shared int hi_bins[64];
  for (int i = threadIdx.x; i < 64; i = i + blockDim.x) {
    hi_bins[i] = 0;
  }
  syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < hi_n; i = i + gridDim.x * blockDim.x) {
    float v = hi_x[i];
    if (v >= -4.0 && v <= 4.0) {
      int b = int((v - -4.0) * 64 / (4.0 - -4.0));
      if (b == 64) {
        b = 63;
      }
      atomic_add(hi_bins[b], 1);
    }
  }
  syncthreads();
  for (int i = threadIdx.x; i < 64; i = i + blockDim.x) {
    atomic_add(hi_out[i], hi_bins[i]);
  }
}
