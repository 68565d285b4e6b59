// BatchNorm collect-statistics, reference (naive) form: per-element Welford updates
// (one division per element) over scalar loads, plane by plane, as in PyTorch's
// batch_norm_collect_statistics_kernel (PAPER.md:274-325); Chan merges across lanes.
//@ grid=256
kernel bn_stats(float bn_x[], float bn_stats[], int bn_N, int bn_C, int bn_HW) dims (1024, 1, 1) {
  shared int bn_sn[32];
  shared float bn_savg[32];
  shared float bn_sm2[32];
  int tid = threadIdx.x;
  int lane = tid % 32;
  int warp = tid / 32;
  int nwarps = blockDim.x / 32;
  float avg; float m2; int n; float o_avg; float o_m2; int o_n; int tot; float fac; float delta;
  for (int c = blockIdx.x; c < bn_C; c = c + gridDim.x) {
    avg = 0.0;
    m2 = 0.0;
    n = 0;
    for (int b = 0; b < bn_N; b = b + 1) {
      for (int i = tid; i < bn_HW; i = i + blockDim.x) {
        float v = bn_x[(b * bn_C + c) * bn_HW + i];
        n = n + 1;
        float d = v - avg;
        avg = avg + d / n;
        m2 = m2 + d * (v - avg);
      }
    }
    for (int s = 0; s < 5; s = s + 1) {
      if (s == 0) { o_n = warp_shfl_xor(n, 16); o_avg = warp_shfl_xor(avg, 16); o_m2 = warp_shfl_xor(m2, 16); }
      if (s == 1) { o_n = warp_shfl_xor(n, 8); o_avg = warp_shfl_xor(avg, 8); o_m2 = warp_shfl_xor(m2, 8); }
      if (s == 2) { o_n = warp_shfl_xor(n, 4); o_avg = warp_shfl_xor(avg, 4); o_m2 = warp_shfl_xor(m2, 4); }
      if (s == 3) { o_n = warp_shfl_xor(n, 2); o_avg = warp_shfl_xor(avg, 2); o_m2 = warp_shfl_xor(m2, 2); }
      if (s == 4) { o_n = warp_shfl_xor(n, 1); o_avg = warp_shfl_xor(avg, 1); o_m2 = warp_shfl_xor(m2, 1); }
      tot = n + o_n;
      fac = 1.0 / fmaxf(1.0, tot);
      delta = o_avg - avg;
      m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
      avg = (n * avg + o_n * o_avg) * fac;
      n = tot;
    }
    if (lane == 0) {
      bn_sn[warp] = n;
      bn_savg[warp] = avg;
      bn_sm2[warp] = m2;
    }
    syncthreads();
    if (warp == 0) {
      if (lane < nwarps) {
        n = bn_sn[lane];
        avg = bn_savg[lane];
        m2 = bn_sm2[lane];
      } else {
        n = 0;
        avg = 0.0;
        m2 = 0.0;
      }
      for (int s = 0; s < 5; s = s + 1) {
        if (s == 0) { o_n = warp_shfl_xor(n, 16); o_avg = warp_shfl_xor(avg, 16); o_m2 = warp_shfl_xor(m2, 16); }
        if (s == 1) { o_n = warp_shfl_xor(n, 8); o_avg = warp_shfl_xor(avg, 8); o_m2 = warp_shfl_xor(m2, 8); }
        if (s == 2) { o_n = warp_shfl_xor(n, 4); o_avg = warp_shfl_xor(avg, 4); o_m2 = warp_shfl_xor(m2, 4); }
        if (s == 3) { o_n = warp_shfl_xor(n, 2); o_avg = warp_shfl_xor(avg, 2); o_m2 = warp_shfl_xor(m2, 2); }
        if (s == 4) { o_n = warp_shfl_xor(n, 1); o_avg = warp_shfl_xor(avg, 1); o_m2 = warp_shfl_xor(m2, 1); }
        tot = n + o_n;
        fac = 1.0 / fmaxf(1.0, tot);
        delta = o_avg - avg;
        m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
        avg = (n * avg + o_n * o_avg) * fac;
        n = tot;
      }
      if (lane == 0) {
        bn_stats[c * 2] = avg;
        bn_stats[c * 2 + 1] = m2 / fmaxf(1.0, n);
      }
    }
    syncthreads();
  }
}
