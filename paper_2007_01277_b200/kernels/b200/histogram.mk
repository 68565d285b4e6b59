// Histogram (torch.histc analogue, PAPER.md:405-430), B200 form (MK+).
// 64 bins over [-4, 4]: bin = int((v - lo) * nbins / (hi - lo)), v == hi -> last bin,
// values outside [lo, hi] are ignored. Because nbins / (hi - lo) = 8 is a power of two,
// int((v + 4) * 8) is bit-identical to the division form (both scalings are exact); inside the
// range guard (v + 4) * 8 is in [0, 64], so the conversion is int_rz (one cvt.rzi.s32 instead
// of the general int() lowering, which goes through int64 for |x| >= 2^31).
// B200 mechanics: four 128-bit coalesced loads in flight per thread per iteration over the
// first 4 * (n / 4) values (tail loads clamped in bounds and masked; the n % 4 trailing
// values are binned by block 0 with scalar loads, so any n works), warp-private shared-memory bins
// (32 x 64 counters: contention only inside a warp), one global atomic per bin per block.
//@ grid=256
kernel hist(float hi_x[], int hi_out[], int hi_n) dims (1024, 1, 1) {
  shared int hi_bins[2048];
  int tid = threadIdx.x;
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int wb = (tid / 32) * 64;
  int n4 = hi_n / 4;
  int last = n4 - 1;
  int stride = gridDim.x * nthr;
  float v0; float v1; float v2; float v3; float v4; float v5; float v6; float v7;
  float v8; float v9; float v10; float v11; float v12; float v13; float v14; float v15;
  for (int i = blockIdx.x * nthr + tid; i < n4; i = i + 4 * stride) {
    int j1 = i + stride;
    int j2 = j1 + stride;
    int j3 = j2 + stride;
    vload(hi_x, i, v0, v1, v2, v3);
    vload(hi_x, min(j1, last), v4, v5, v6, v7);
    vload(hi_x, min(j2, last), v8, v9, v10, v11);
    vload(hi_x, min(j3, last), v12, v13, v14, v15);
    if (v0 >= -4.0 && v0 <= 4.0) {
      atomic_add(hi_bins[wb + min(int_rz((v0 + 4.0) * 8.0), 63)], 1);
    }
    if (v1 >= -4.0 && v1 <= 4.0) {
      atomic_add(hi_bins[wb + min(int_rz((v1 + 4.0) * 8.0), 63)], 1);
    }
    if (v2 >= -4.0 && v2 <= 4.0) {
      atomic_add(hi_bins[wb + min(int_rz((v2 + 4.0) * 8.0), 63)], 1);
    }
    if (v3 >= -4.0 && v3 <= 4.0) {
      atomic_add(hi_bins[wb + min(int_rz((v3 + 4.0) * 8.0), 63)], 1);
    }
    if (j1 < n4) {
      if (v4 >= -4.0 && v4 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v4 + 4.0) * 8.0), 63)], 1);
      }
      if (v5 >= -4.0 && v5 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v5 + 4.0) * 8.0), 63)], 1);
      }
      if (v6 >= -4.0 && v6 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v6 + 4.0) * 8.0), 63)], 1);
      }
      if (v7 >= -4.0 && v7 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v7 + 4.0) * 8.0), 63)], 1);
      }
    }
    if (j2 < n4) {
      if (v8 >= -4.0 && v8 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v8 + 4.0) * 8.0), 63)], 1);
      }
      if (v9 >= -4.0 && v9 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v9 + 4.0) * 8.0), 63)], 1);
      }
      if (v10 >= -4.0 && v10 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v10 + 4.0) * 8.0), 63)], 1);
      }
      if (v11 >= -4.0 && v11 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v11 + 4.0) * 8.0), 63)], 1);
      }
    }
    if (j3 < n4) {
      if (v12 >= -4.0 && v12 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v12 + 4.0) * 8.0), 63)], 1);
      }
      if (v13 >= -4.0 && v13 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v13 + 4.0) * 8.0), 63)], 1);
      }
      if (v14 >= -4.0 && v14 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v14 + 4.0) * 8.0), 63)], 1);
      }
      if (v15 >= -4.0 && v15 <= 4.0) {
        atomic_add(hi_bins[wb + min(int_rz((v15 + 4.0) * 8.0), 63)], 1);
      }
    }
  }
  // the n % 4 trailing values the vector loop does not cover: block 0, one per thread
  if (blockIdx.x == 0 && tid < hi_n - 4 * n4) {
    v0 = hi_x[4 * n4 + tid];
    if (v0 >= -4.0 && v0 <= 4.0) {
      atomic_add(hi_bins[wb + min(int_rz((v0 + 4.0) * 8.0), 63)], 1);
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
