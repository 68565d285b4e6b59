// BatchNorm collect-statistics, B200 form (MK+).
// Semantics of PyTorch's batch_norm_collect_statistics (PAPER.md:274-325, the corpus
// analogue /root/reference/proj/corpus/batchnorm.mk): per channel c of x[N, C, HW] the
// mean and the biased variance. Each thread accumulates shifted sums over its samples
// (numerically stable: the shift is one of its own samples) and the per-thread
// (count, mean, M2) triples are combined with Chan's parallel formula.
// B200 mechanics: each channel's N planes are walked as one flat float4 index space
// (128-bit coalesced loads, HW % 4 == 0) with four loads in flight per thread (36.9 vs 37.6 us
// alone with two, and 2 us off every fused BN pair on B200; same summation order), ~4 FP ops
// per element (no per-element division as in the naive Welford form), a 5-step
// warp-shuffle Chan tree and a shared-memory stage per warp.
// Grid-stride over channels, so any common grid works.
//@ grid=256
//@ requires bn_HW % 4 == 0
kernel bn_stats(float bn_x[], float bn_stats[], int bn_N, int bn_C, int bn_HW) dims (1024, 1, 1) {
  shared int bn_sn[32];
  shared float bn_savg[32];
  shared float bn_sm2[32];
  int tid = threadIdx.x;
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int hw4 = bn_HW / 4;
  int lane = tid % 32;
  int warp = tid / 32;
  int nwarps = nthr / 32;
  float v0; float v1; float v2; float v3; float v4; float v5; float v6; float v7;
  float v8; float v9; float v10; float v11; float v12; float v13; float v14; float v15;
  float e0; float e1; float e2; float e3;
  float avg; float m2; int n; float o_avg; float o_m2; int o_n; int tot; float fac; float delta;
  for (int c = blockIdx.x; c < bn_C; c = c + gridDim.x) {
    // Per-thread shifted sums (shift = the thread's first sample): s1 = sum(x - K),
    // s2 = sum((x - K)^2), pairwise within each float4. Four float4 positions per iteration
    // (j .. j + 3 nthr of the flat N * HW/4 space of channel c) keep four 128-bit loads in
    // flight, then single vectors; plane/offset come from j / (HW/4) (a constant divisor once
    // specialized). The accumulation order is the two-load form's (j, j + nthr, j + 2 nthr, ..).
    n = 0;
    float K = 0.0;
    float s1 = 0.0;
    float s2 = 0.0;
    int total4 = bn_N * hw4;
    if (tid < total4) {
      int b0 = tid / hw4;
      K = bn_x[((b0 * bn_C + c) * hw4 + tid - b0 * hw4) * 4];
    }
    int j = tid;
    while (j + 3 * nthr < total4) {
      int p0 = j / hw4;
      int p1 = (j + nthr) / hw4;
      int p2 = (j + 2 * nthr) / hw4;
      int p3 = (j + 3 * nthr) / hw4;
      vload(bn_x, (p0 * bn_C + c) * hw4 + j - p0 * hw4, v0, v1, v2, v3);
      vload(bn_x, (p1 * bn_C + c) * hw4 + j + nthr - p1 * hw4, v4, v5, v6, v7);
      vload(bn_x, (p2 * bn_C + c) * hw4 + j + 2 * nthr - p2 * hw4, v8, v9, v10, v11);
      vload(bn_x, (p3 * bn_C + c) * hw4 + j + 3 * nthr - p3 * hw4, v12, v13, v14, v15);
      e0 = v0 - K;
      e1 = v1 - K;
      e2 = v2 - K;
      e3 = v3 - K;
      s1 = s1 + ((e0 + e1) + (e2 + e3));
      s2 = s2 + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      e0 = v4 - K;
      e1 = v5 - K;
      e2 = v6 - K;
      e3 = v7 - K;
      s1 = s1 + ((e0 + e1) + (e2 + e3));
      s2 = s2 + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      e0 = v8 - K;
      e1 = v9 - K;
      e2 = v10 - K;
      e3 = v11 - K;
      s1 = s1 + ((e0 + e1) + (e2 + e3));
      s2 = s2 + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      e0 = v12 - K;
      e1 = v13 - K;
      e2 = v14 - K;
      e3 = v15 - K;
      s1 = s1 + ((e0 + e1) + (e2 + e3));
      s2 = s2 + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      n = n + 16;
      j = j + 4 * nthr;
    }
    while (j < total4) {
      int p0 = j / hw4;
      vload(bn_x, (p0 * bn_C + c) * hw4 + j - p0 * hw4, v0, v1, v2, v3);
      e0 = v0 - K;
      e1 = v1 - K;
      e2 = v2 - K;
      e3 = v3 - K;
      s1 = s1 + ((e0 + e1) + (e2 + e3));
      s2 = s2 + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      n = n + 4;
      j = j + nthr;
    }
    fac = 1.0 / fmaxf(1.0, n);
    avg = K + s1 * fac;
    m2 = fmaxf(0.0, s2 - s1 * s1 * fac);
    o_n = warp_shfl_xor(n, 16);
    o_avg = warp_shfl_xor(avg, 16);
    o_m2 = warp_shfl_xor(m2, 16);
    tot = n + o_n;
    fac = 1.0 / fmaxf(1.0, tot);
    delta = o_avg - avg;
    m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
    avg = (n * avg + o_n * o_avg) * fac;
    n = tot;
    o_n = warp_shfl_xor(n, 8);
    o_avg = warp_shfl_xor(avg, 8);
    o_m2 = warp_shfl_xor(m2, 8);
    tot = n + o_n;
    fac = 1.0 / fmaxf(1.0, tot);
    delta = o_avg - avg;
    m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
    avg = (n * avg + o_n * o_avg) * fac;
    n = tot;
    o_n = warp_shfl_xor(n, 4);
    o_avg = warp_shfl_xor(avg, 4);
    o_m2 = warp_shfl_xor(m2, 4);
    tot = n + o_n;
    fac = 1.0 / fmaxf(1.0, tot);
    delta = o_avg - avg;
    m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
    avg = (n * avg + o_n * o_avg) * fac;
    n = tot;
    o_n = warp_shfl_xor(n, 2);
    o_avg = warp_shfl_xor(avg, 2);
    o_m2 = warp_shfl_xor(m2, 2);
    tot = n + o_n;
    fac = 1.0 / fmaxf(1.0, tot);
    delta = o_avg - avg;
    m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
    avg = (n * avg + o_n * o_avg) * fac;
    n = tot;
    o_n = warp_shfl_xor(n, 1);
    o_avg = warp_shfl_xor(avg, 1);
    o_m2 = warp_shfl_xor(m2, 1);
    tot = n + o_n;
    fac = 1.0 / fmaxf(1.0, tot);
    delta = o_avg - avg;
    m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
    avg = (n * avg + o_n * o_avg) * fac;
    n = tot;
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
      o_n = warp_shfl_xor(n, 16);
      o_avg = warp_shfl_xor(avg, 16);
      o_m2 = warp_shfl_xor(m2, 16);
      tot = n + o_n;
      fac = 1.0 / fmaxf(1.0, tot);
      delta = o_avg - avg;
      m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
      avg = (n * avg + o_n * o_avg) * fac;
      n = tot;
      o_n = warp_shfl_xor(n, 8);
      o_avg = warp_shfl_xor(avg, 8);
      o_m2 = warp_shfl_xor(m2, 8);
      tot = n + o_n;
      fac = 1.0 / fmaxf(1.0, tot);
      delta = o_avg - avg;
      m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
      avg = (n * avg + o_n * o_avg) * fac;
      n = tot;
      o_n = warp_shfl_xor(n, 4);
      o_avg = warp_shfl_xor(avg, 4);
      o_m2 = warp_shfl_xor(m2, 4);
      tot = n + o_n;
      fac = 1.0 / fmaxf(1.0, tot);
      delta = o_avg - avg;
      m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
      avg = (n * avg + o_n * o_avg) * fac;
      n = tot;
      o_n = warp_shfl_xor(n, 2);
      o_avg = warp_shfl_xor(avg, 2);
      o_m2 = warp_shfl_xor(m2, 2);
      tot = n + o_n;
      fac = 1.0 / fmaxf(1.0, tot);
      delta = o_avg - avg;
      m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
      avg = (n * avg + o_n * o_avg) * fac;
      n = tot;
      o_n = warp_shfl_xor(n, 1);
      o_avg = warp_shfl_xor(avg, 1);
      o_m2 = warp_shfl_xor(m2, 1);
      tot = n + o_n;
      fac = 1.0 / fmaxf(1.0, tot);
      delta = o_avg - avg;
      m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
      avg = (n * avg + o_n * o_avg) * fac;
      n = tot;
      if (lane == 0) {
        bn_stats[c * 2] = avg;
        bn_stats[c * 2 + 1] = m2 / fmaxf(1.0, n);
      }
    }
    syncthreads();
  }
}
