// Streaming ceiling kernel (measurement only, not a member): grid-stride 128-bit copy-like stream
// reading s_nr4 and writing s_nw4 float4s, one load in flight per thread. bench.py times it at
// each DL pair's algorithmic read / write bytes: the mix-matched HBM ceiling of that pair.
kernel stream(float s_src[], float s_dst[], int s_nr4, int s_nw4) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int n = max(s_nr4, s_nw4);
  float acc = 0.0;
  float a; float b; float c; float d;
  for (int i = blockIdx.x * nthr + threadIdx.x; i < n; i = i + gridDim.x * nthr) {
    if (i < s_nr4) {
      vload(s_src, i, a, b, c, d);
      acc = acc + a + b + c + d;
    }
    if (i < s_nw4) {
      vstore(s_dst, i, acc, a, b, c);
    }
  }
  if (acc == 12345.0) {
    s_dst[0] = acc;
  }
}
