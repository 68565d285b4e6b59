// Im2Col 3x3, padding 1, stride 1, B200 form (MK+). Requires W % 4 == 0.
// Each thread owns 4 consecutive columns (w = 4q .. 4q+3) of one output position row h of
// one (n, c) plane and writes all 9 kernel-offset rows for them: per input row it reads
// one 128-bit vector plus the two neighbouring scalars (6 columns, zero padded), and emits
// three 128-bit stores (kw = 0, 1, 2). 9 loads feed 36 outputs; the stores of each
// (c, kh, kw) row are contiguous across consecutive threads. Same values as the reference
// form (pure data movement).
//@ grid=256
//@ requires ic_W % 4 == 0
kernel im2col(float ic_x[], float ic_col[], int ic_NC, int ic_H, int ic_W) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int w4 = ic_W / 4;
  int total = ic_NC * ic_H * w4;
  float m; float p0; float p1; float p2; float p3; float e;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % w4;
    int r = t / w4;
    int h = r % ic_H;
    int nc = r / ic_H;
    int col = q * 4;
    unroll for (int kh = 0; kh < 3; kh = kh + 1) {
      int ih = h + kh - 1;
      m = 0.0;
      p0 = 0.0;
      p1 = 0.0;
      p2 = 0.0;
      p3 = 0.0;
      e = 0.0;
      if (ih >= 0 && ih < ic_H) {
        int row = (nc * ic_H + ih) * ic_W;
        vload(ic_x, (row + col) / 4, p0, p1, p2, p3);
        if (col > 0) {
          m = ic_x[row + col - 1];
        }
        if (col + 4 < ic_W) {
          e = ic_x[row + col + 4];
        }
      }
      int out = ((nc * 9 + kh * 3) * ic_H + h) * w4 + q;
      vstore(ic_col, out, m, p0, p1, p2);
      vstore(ic_col, out + ic_H * w4, p0, p1, p2, p3);
      vstore(ic_col, out + 2 * ic_H * w4, p1, p2, p3, e);
    }
  }
}
