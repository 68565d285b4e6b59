// BatchNorm collect-statistics, grid-balanced B200 variant (MK+).
// Measured on B200 (C2 sizes, scripts/probe_bn.py): 45.1 us at grid 296 vs 37.6 us for the
// block-per-channel form (batchnorm.mk) -- equal work per block buys nothing there (that form
// is not limited by its 40 idle blocks) and the cross-block hand-off costs ~6 us. Kept as the
// test vehicle of fence() and the deterministic inter-block merge; not used by the bench.
// Semantics of PyTorch's batch_norm_collect_statistics (PAPER.md:274-325, the corpus
// analogue /root/reference/proj/corpus/batchnorm.mk): per channel c of x[N, C, HW] the
// mean and the biased variance. Each thread accumulates shifted sums over its samples
// (numerically stable: the shift is one of its own samples) and the per-thread
// (count, mean, M2) triples are combined with Chan's parallel formula.
// B200 mechanics:
//  * Grid-balanced: the C channels are one flat float4 index space of T = C * N * HW/4
//    vectors split into gridDim.x equal contiguous ranges, so every block streams the same
//    number of bytes whatever C and the grid are (one block per channel would leave
//    gridDim.x - C blocks idle, e.g. 40 of 296 at C = 256). A block's range covers one or more
//    channel segments; each segment is reduced in the block (5-step warp-shuffle Chan tree +
//    shared-memory stage) into a partial (count, mean, M2) stored in slot (c, block - first
//    block of c) of the bn_pn/bn_pa/bn_pm workspace (bn_P slots per channel).
//  * Deterministic hand-off: after its partial, a block fences and bumps bn_cnt[c]; whoever
//    then reads the full count merges the channel's partials in block order (Chan), writes
//    bn_stats and clears bn_cnt[c] for the next launch. The merge order does not depend on
//    which block arrives last, so the result is bit-identical to the sequential interpreter.
//  * 128-bit coalesced loads, two in flight per thread, ~4 FP ops per element.
// Requires HW % 4 == 0, C * N * HW / 4 >= gridDim.x and bn_P >= gridDim.x / C + 2.
// regcap 32 keeps two 1024-thread blocks per SM (the rare merge path may spill).
//@ grid=256 regcap=32
//@ requires bn_HW % 4 == 0
kernel bn_stats_balanced(float bn_x[], float bn_stats[], int bn_pn[], float bn_pa[], float bn_pm[], int bn_cnt[],
                int bn_N, int bn_C, int bn_HW, int bn_P) dims (1024, 1, 1) {
  shared int bn_sn[32];
  shared float bn_savg[32];
  shared float bn_sm2[32];
  shared int bn_last[1];
  int tid = threadIdx.x;
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int hw4 = bn_HW / 4;
  int lane = tid % 32;
  int warp = tid / 32;
  int nwarps = nthr / 32;
  int L = bn_N * hw4;
  int G = gridDim.x;
  int q = (bn_C * L) / G;
  int r = (bn_C * L) % G;
  int b = blockIdx.x;
  int lo = b * q + (b * r) / G;
  int hi = (b + 1) * q + ((b + 1) * r) / G;
  float v0; float v1; float v2; float v3; float v4; float v5; float v6; float v7;
  float avg; float m2; int n; float o_avg; float o_m2; int o_n; int tot; float fac; float delta;
  int bf; int bl; int e; int slot; int k;
  for (int c = lo / L; c * L < hi; c = c + 1) {
    int s0 = max(lo, c * L) - c * L;
    int s1 = min(hi, c * L + L) - c * L;
    // Per-thread shifted sums (shift K = the thread's first sample): s1 = sum(x - K),
    // s2 = sum((x - K)^2), pairwise within each float4; j and j + nthr in flight.
    n = 0;
    float K = 0.0;
    float sa = 0.0;
    float sb = 0.0;
    if (s0 + tid < s1) {
      int b0 = (s0 + tid) / hw4;
      K = bn_x[((b0 * bn_C + c) * hw4 + s0 + tid - b0 * hw4) * 4];
    }
    // main loop: both vectors in range, two independent 128-bit loads issued back to back
    int j = s0 + tid;
    while (j + nthr < s1) {
      int p1 = j / hw4;
      int p2 = (j + nthr) / hw4;
      vload(bn_x, (p1 * bn_C + c) * hw4 + j - p1 * hw4, v0, v1, v2, v3);
      vload(bn_x, (p2 * bn_C + c) * hw4 + j + nthr - p2 * hw4, v4, v5, v6, v7);
      float e0 = v0 - K;
      float e1 = v1 - K;
      float e2 = v2 - K;
      float e3 = v3 - K;
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      e0 = v4 - K;
      e1 = v5 - K;
      e2 = v6 - K;
      e3 = v7 - K;
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      n = n + 8;
      j = j + 2 * nthr;
    }
    // tail: at most one vector left
    if (j < s1) {
      int p1 = j / hw4;
      vload(bn_x, (p1 * bn_C + c) * hw4 + j - p1 * hw4, v0, v1, v2, v3);
      float e0 = v0 - K;
      float e1 = v1 - K;
      float e2 = v2 - K;
      float e3 = v3 - K;
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      n = n + 4;
    }
    fac = 1.0 / fmaxf(1.0, n);
    avg = K + sa * fac;
    m2 = fmaxf(0.0, sb - sa * sa * fac);
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
        // blocks bf..bl cover channel c: the blocks holding its first and last vector
        e = c * L;
        bf = e / (q + 1);
        while ((bf + 1) * q + ((bf + 1) * r) / G <= e) {
          bf = bf + 1;
        }
        e = c * L + L - 1;
        bl = e / (q + 1);
        while ((bl + 1) * q + ((bl + 1) * r) / G <= e) {
          bl = bl + 1;
        }
        slot = c * bn_P + b - bf;
        bn_pn[slot] = n;
        bn_pa[slot] = avg;
        bn_pm[slot] = m2;
        fence();
        atomic_add(bn_cnt[c], 1);
        bn_last[0] = 0;
        if (bn_cnt[c] == bl - bf + 1) {
          bn_last[0] = 1;
          fence();
          n = bn_pn[c * bn_P];
          avg = bn_pa[c * bn_P];
          m2 = bn_pm[c * bn_P];
          for (k = 1; k <= bl - bf; k = k + 1) {
            o_n = bn_pn[c * bn_P + k];
            o_avg = bn_pa[c * bn_P + k];
            o_m2 = bn_pm[c * bn_P + k];
            tot = n + o_n;
            fac = 1.0 / fmaxf(1.0, tot);
            delta = o_avg - avg;
            m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
            avg = (n * avg + o_n * o_avg) * fac;
            n = tot;
          }
          bn_stats[c * 2] = avg;
          bn_stats[c * 2 + 1] = m2 / fmaxf(1.0, n);
          bn_cnt[c] = 0;
        }
      }
    }
    syncthreads();
  }
}
