// Streaming ceiling kernel (measurement only, not a member): as stream.mk with four 128-bit
// loads in flight per thread (the BN / Hist member pattern), then the stores.
kernel stream4(float s_src[], float s_dst[], int s_nr4, int s_nw4) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int n = max(s_nr4, s_nw4);
  int st = gridDim.x * nthr;
  float acc = 0.0;
  float a0; float b0; float c0; float d0; float a1; float b1; float c1; float d1;
  float a2; float b2; float c2; float d2; float a3; float b3; float c3; float d3;
  for (int i = blockIdx.x * nthr + threadIdx.x; i < n; i = i + 4 * st) {
    a0 = 0.0; b0 = 0.0; c0 = 0.0; d0 = 0.0; a1 = 0.0; b1 = 0.0; c1 = 0.0; d1 = 0.0;
    a2 = 0.0; b2 = 0.0; c2 = 0.0; d2 = 0.0; a3 = 0.0; b3 = 0.0; c3 = 0.0; d3 = 0.0;
    if (i < s_nr4) { vload(s_src, i, a0, b0, c0, d0); }
    if (i + st < s_nr4) { vload(s_src, i + st, a1, b1, c1, d1); }
    if (i + 2 * st < s_nr4) { vload(s_src, i + 2 * st, a2, b2, c2, d2); }
    if (i + 3 * st < s_nr4) { vload(s_src, i + 3 * st, a3, b3, c3, d3); }
    acc = acc + a0 + b1 + c2 + d3;
    if (i < s_nw4) { vstore(s_dst, i, acc, a0, b0, c0); }
    if (i + st < s_nw4) { vstore(s_dst, i + st, a1, b1, c1, d1); }
    if (i + 2 * st < s_nw4) { vstore(s_dst, i + 2 * st, a2, b2, c2, d2); }
    if (i + 3 * st < s_nw4) { vstore(s_dst, i + 3 * st, a3, b3, c3, d3); }
  }
  if (acc == 12345.0) {
    s_dst[0] = acc;
  }
}
