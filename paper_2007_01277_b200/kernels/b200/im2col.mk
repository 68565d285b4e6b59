// Im2Col 3x3, padding 1, stride 1, B200 form (MK+): each thread fills 4 consecutive
// columns of one output row and writes them with one 128-bit store (W % 4 == 0); the four
// shifted input reads are scalar and L1/L2-resident (each input element feeds 9 rows).
//@ grid=256
kernel im2col(float ic_x[], float ic_col[], int ic_NC, int ic_H, int ic_W) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int w4 = ic_W / 4;
  int total = ic_NC * 9 * ic_H * w4;
  float a0; float a1; float a2; float a3;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % w4;
    int r = t / w4;
    int h = r % ic_H;
    int k = r / ic_H % 9;
    int nc = r / (ic_H * 9);
    int ih = h + k / 3 - 1;
    int iw = q * 4 + k % 3 - 1;
    a0 = 0.0;
    a1 = 0.0;
    a2 = 0.0;
    a3 = 0.0;
    if (ih >= 0 && ih < ic_H) {
      int base = (nc * ic_H + ih) * ic_W;
      if (iw >= 0) {
        a0 = ic_x[base + iw];
      }
      a1 = ic_x[base + iw + 1];
      a2 = ic_x[base + iw + 2];
      if (iw + 3 < ic_W) {
        a3 = ic_x[base + iw + 3];
      }
    }
    vstore(ic_col, t, a0, a1, a2, a3);
  }
}
