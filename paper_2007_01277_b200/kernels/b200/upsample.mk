// Upsample bilinear 2x (align_corners=False), B200 form (MK+).
// Precondition: OH == 2 * IH, OW == 2 * IW, IW even. Then rw = IW / OW = 0.5 exactly and the
// generic source-index arithmetic of the reference form (w1r = rw * (ow + 0.5) - 0.5, clamped,
// w1 = int(w1r), w1l = w1r - w1) takes exact values: for the 4 outputs ow = 4q .. 4q+3 the
// left columns are 2q-1, 2q, 2q, 2q+1 with right weights 0.75, 0.25, 0.75, 0.25 (ow = 0:
// column 0 with weight 0), so each output is computed with the same float operations, in
// the same order, on the same operands as the reference form: bit-identical results.
// B200 mechanics: 4 outputs per thread from one 64-bit load + 2 scalar loads per input row,
// constant weights (no per-output index/float conversion), one 128-bit store.
//@ grid=256
kernel upsample(float us_x[], float us_y[], int us_NC, int us_IH, int us_IW, int us_OH, int us_OW) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int ow4 = us_OW / 4;
  int total = us_NC * us_OH * ow4;
  float rh = float(us_IH) / us_OH;
  float a0; float b0; float c0; float d0; float a1; float b1; float c1; float d1;
  float t0; float t1; float y0; float y1; float y2; float y3;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % ow4;
    int r = t / ow4;
    int oh = r % us_OH;
    int nc = r / us_OH;
    float h1r = rh * (oh + 0.5) - 0.5;
    if (h1r < 0.0) {
      h1r = 0.0;
    }
    int h1 = int(h1r);
    int h1p = 0;
    if (h1 < us_IH - 1) {
      h1p = 1;
    }
    float h1l = h1r - h1;
    float h0l = 1.0 - h1l;
    int r0 = (nc * us_IH + h1) * us_IW;
    int r1 = (nc * us_IH + h1 + h1p) * us_IW;
    int c = q * 2;
    vload(us_x, (r0 + c) / 2, b0, c0);
    vload(us_x, (r1 + c) / 2, b1, c1);
    a0 = b0;
    a1 = b1;
    if (q > 0) {
      a0 = us_x[r0 + c - 1];
      a1 = us_x[r1 + c - 1];
    }
    d0 = c0;
    d1 = c1;
    if (c + 2 < us_IW) {
      d0 = us_x[r0 + c + 2];
      d1 = us_x[r1 + c + 2];
    }
    if (q == 0) {
      t0 = 1.0 * b0 + 0.0 * c0;
      t1 = 1.0 * b1 + 0.0 * c1;
    } else {
      t0 = 0.25 * a0 + 0.75 * b0;
      t1 = 0.25 * a1 + 0.75 * b1;
    }
    y0 = h0l * t0 + h1l * t1;
    y1 = h0l * (0.75 * b0 + 0.25 * c0) + h1l * (0.75 * b1 + 0.25 * c1);
    y2 = h0l * (0.25 * b0 + 0.75 * c0) + h1l * (0.25 * b1 + 0.75 * c1);
    y3 = h0l * (0.75 * c0 + 0.25 * d0) + h1l * (0.75 * c1 + 0.25 * d1);
    vstore(us_y, t, y0, y1, y2, y3);
  }
}
