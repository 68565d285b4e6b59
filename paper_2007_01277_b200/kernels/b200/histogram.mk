// Histogram (torch.histc analogue, PAPER.md:405-430), B200 form (MK+).
// 64 bins over [-4, 4]: bin = int((v - lo) * nbins / (hi - lo)), v == hi -> last bin,
// values outside [lo, hi] are ignored. Because nbins / (hi - lo) = 8 is a power of two,
// int((v + 4) * 8) is bit-identical to the division form (both scalings are exact).
// B200 mechanics: 128-bit coalesced loads (n % 4 == 0), warp-private shared-memory bins
// (32 x 64 counters: intra-warp contention only), one global atomic per bin per block.
//@ grid=256
kernel hist(float hi_x[], int hi_out[], int hi_n) dims (1024, 1, 1) {
  shared int hi_bins[2048];
  int tid = threadIdx.x;
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int wb = (tid / 32) * 64;
  int n4 = hi_n / 4;
  float v0; float v1; float v2; float v3;
  for (int i = blockIdx.x * nthr + tid; i < n4; i = i + gridDim.x * nthr) {
    vload(hi_x, i, v0, v1, v2, v3);
    if (v0 >= -4.0 && v0 <= 4.0) {
      atomic_add(hi_bins[wb + min(int((v0 + 4.0) * 8.0), 63)], 1);
    }
    if (v1 >= -4.0 && v1 <= 4.0) {
      atomic_add(hi_bins[wb + min(int((v1 + 4.0) * 8.0), 63)], 1);
    }
    if (v2 >= -4.0 && v2 <= 4.0) {
      atomic_add(hi_bins[wb + min(int((v2 + 4.0) * 8.0), 63)], 1);
    }
    if (v3 >= -4.0 && v3 <= 4.0) {
      atomic_add(hi_bins[wb + min(int((v3 + 4.0) * 8.0), 63)], 1);
    }
  }
  syncthreads();
  for (int b = tid; b < 64; b = b + nthr) {
    int s = 0;
    for (int w = 0; w < nthr / 32; w = w + 1) {
      s = s + hi_bins[w * 64 + b];
    }
    atomic_add(hi_out[b], s);
  }
}
