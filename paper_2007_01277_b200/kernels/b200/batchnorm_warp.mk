// BatchNorm collect-statistics, grid-balanced B200 form without block barriers (MK+).
// Measured on B200 (C2 sizes, scripts/probe_bn_warp.py -> profiles/r01_probe_bn_warp.json):
// 49.1 us alone at grid 296 (41.0 without the hand-off) vs 37.6 us for the block-per-channel
// form, and no fused pair got faster with it (e.g. + Hist 69.6 vs 67.7 us): the per-warp
// hand-off (release, counter read, last-warp merge) is ~8 us of serial latency per warp, and
// the block-per-channel form was not limited by its idle blocks. Kept as the hardware test
// vehicle of atomic_add_release / load_relaxed; the bench uses batchnorm.mk.
// Semantics of PyTorch's batch_norm_collect_statistics (PAPER.md:274-325, the corpus analogue
// /root/reference/proj/corpus/batchnorm.mk): per channel c of x[N, C, HW] the mean and the
// biased variance, from per-thread shifted sums (shift = one of the thread's own samples)
// combined with Chan's parallel formula.
// B200 mechanics -- built for horizontal fusion:
//  * Grid-balanced: the channels form one flat float4 index space of T = C * N * HW/4 vectors
//    split into gridDim.x equal contiguous block ranges, so every block streams the same bytes
//    whatever C and the grid are. (One block per channel, batchnorm.mk, leaves the blocks past
//    C without BN work; fused with a grid-stride partner, those blocks run the partner alone on
//    a fraction of their threads.) Inside its range a block sweeps thread-interleaved (thread t
//    takes vectors t, t + blockDim, ...: the whole grid reads one advancing window, like the
//    grid-stride members), four 128-bit loads in flight per thread.
//  * No block barrier: every warp reduces each channel segment of its block with a 5-step
//    shuffle Chan tree; lane 0 stores the partial (count, mean, M2) in slot
//    (c, (block - first block of c) * warps + warp), bumps bn_cnt[c] with a release-ordered
//    atomic (red.release.gpu: no full fence, no L1 invalidate on this hot path) and re-reads
//    it (load_relaxed). The warp whose lane 0 reads the full count fences (the acquire side)
//    and merges the channel's partials with all 32 lanes -- lane l folds slots l, l + 32, ...
//    in order, then the shuffle tree: a fixed order whoever arrives last -- writes bn_stats
//    and clears bn_cnt[c] for the next launch.
// Requires HW % 4 == 0, T >= gridDim.x and bn_P >= (gridDim.x / C + 2) * blockDim / 32.
//@ grid=296 regcap=32
//@ requires bn_HW % 4 == 0
kernel bn_stats(float bn_x[], float bn_stats[], int bn_pn[], float bn_pa[], float bn_pm[], int bn_cnt[],
                int bn_N, int bn_C, int bn_HW, int bn_P) dims (1024, 1, 1) {
  int tid = threadIdx.x;
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int hw4 = bn_HW / 4;
  int lane = tid % 32;
  int nw = nthr / 32;
  int wid = tid / 32;
  int L = bn_N * hw4;
  int G = gridDim.x;
  int b = blockIdx.x;
  int T = bn_C * L;
  int q = T / G;
  int r = T % G;
  int lo = b * q + min(b, r);
  int hi = lo + q;
  if (b < r) {
    hi = hi + 1;
  }
  float v0; float v1; float v2; float v3; float v4; float v5; float v6; float v7;
  float v8; float v9; float v10; float v11; float v12; float v13; float v14; float v15;
  float e0; float e1; float e2; float e3;
  float avg; float m2; int n; float o_avg; float o_m2; int o_n; int tot; float fac; float delta;
  int bf; int bl; int e; int k; int base; int last; int parts;
  for (int c = lo / L; c * L < hi; c = c + 1) {
    int s0 = max(lo, c * L) - c * L;
    int s1 = min(hi, c * L + L) - c * L;
    n = 0;
    float K = 0.0;
    float sa = 0.0;
    float sb = 0.0;
    int j = s0 + tid;
    if (j < s1) {
      int b0 = j / hw4;
      K = bn_x[((b0 * bn_C + c) * hw4 + j - b0 * hw4) * 4];
    }
    while (j + 3 * nthr < s1) {
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
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      e0 = v4 - K;
      e1 = v5 - K;
      e2 = v6 - K;
      e3 = v7 - K;
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      e0 = v8 - K;
      e1 = v9 - K;
      e2 = v10 - K;
      e3 = v11 - K;
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      e0 = v12 - K;
      e1 = v13 - K;
      e2 = v14 - K;
      e3 = v15 - K;
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      n = n + 16;
      j = j + 4 * nthr;
    }
    while (j < s1) {
      int p0 = j / hw4;
      vload(bn_x, (p0 * bn_C + c) * hw4 + j - p0 * hw4, v0, v1, v2, v3);
      e0 = v0 - K;
      e1 = v1 - K;
      e2 = v2 - K;
      e3 = v3 - K;
      sa = sa + ((e0 + e1) + (e2 + e3));
      sb = sb + ((e0 * e0 + e1 * e1) + (e2 * e2 + e3 * e3));
      n = n + 4;
      j = j + nthr;
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
    // blocks bf..bl cover channel c: the blocks holding its first and last vector
    e = c * L;
    if (e < r * (q + 1)) {
      bf = e / (q + 1);
    } else {
      bf = (e - r) / q;
    }
    e = c * L + L - 1;
    if (e < r * (q + 1)) {
      bl = e / (q + 1);
    } else {
      bl = (e - r) / q;
    }
    parts = (bl - bf + 1) * nw;
    base = c * bn_P;
    last = 0;
    if (lane == 0) {
      bn_pn[base + (b - bf) * nw + wid] = n;
      bn_pa[base + (b - bf) * nw + wid] = avg;
      bn_pm[base + (b - bf) * nw + wid] = m2;
      atomic_add_release(bn_cnt[c], 1);
      if (load_relaxed(bn_cnt[c]) == parts) {
        last = 1;
      }
    }
    last = last | warp_shfl_xor(last, 16);
    last = last | warp_shfl_xor(last, 8);
    last = last | warp_shfl_xor(last, 4);
    last = last | warp_shfl_xor(last, 2);
    last = last | warp_shfl_xor(last, 1);
    if (last == 1) {
      fence();
      n = 0;
      avg = 0.0;
      m2 = 0.0;
      for (k = lane; k < parts; k = k + 32) {
        o_n = bn_pn[base + k];
        o_avg = bn_pa[base + k];
        o_m2 = bn_pm[base + k];
        tot = n + o_n;
        fac = 1.0 / fmaxf(1.0, tot);
        delta = o_avg - avg;
        m2 = m2 + o_m2 + delta * delta * n * o_n * fac;
        avg = (n * avg + o_n * o_avg) * fac;
        n = tot;
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
        bn_cnt[c] = 0;
      }
    }
  }
}
