// Upsample bilinear 2x (align_corners=False), B200 form (MK+). Per-output arithmetic is
// identical to the reference form (bit-exact); each thread produces 4 consecutive outputs
// of one row, shares the row setup, and writes them with one 128-bit store (OW % 4 == 0).
// Input reads are scalar and L1-resident (each input element feeds 4 outputs).
//@ grid=256
kernel upsample(float us_x[], float us_y[], int us_NC, int us_IH, int us_IW, int us_OH, int us_OW) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int ow4 = us_OW / 4;
  int total = us_NC * us_OH * ow4;
  float w1r; int w1; int w1p; float w1l; float w0l;
  float y0; float y1; float y2; float y3;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % ow4;
    int oh = t / ow4 % us_OH;
    int nc = t / (ow4 * us_OH);
    int ow = q * 4;
    if (1) {
      float rh = float(us_IH) / us_OH;
      float rw = float(us_IW) / us_OW;
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
      w1r = rw * (ow + 0.5) - 0.5;
      if (w1r < 0.0) {
        w1r = 0.0;
      }
      w1 = int(w1r);
      w1p = 0;
      if (w1 < us_IW - 1) {
        w1p = 1;
      }
      w1l = w1r - w1;
      w0l = 1.0 - w1l;
      y0 = h0l * (w0l * us_x[r0 + w1] + w1l * us_x[r0 + w1 + w1p]) + h1l * (w0l * us_x[r1 + w1] + w1l * us_x[r1 + w1 + w1p]);
      w1r = rw * (ow + 1 + 0.5) - 0.5;
      if (w1r < 0.0) {
        w1r = 0.0;
      }
      w1 = int(w1r);
      w1p = 0;
      if (w1 < us_IW - 1) {
        w1p = 1;
      }
      w1l = w1r - w1;
      w0l = 1.0 - w1l;
      y1 = h0l * (w0l * us_x[r0 + w1] + w1l * us_x[r0 + w1 + w1p]) + h1l * (w0l * us_x[r1 + w1] + w1l * us_x[r1 + w1 + w1p]);
      w1r = rw * (ow + 2 + 0.5) - 0.5;
      if (w1r < 0.0) {
        w1r = 0.0;
      }
      w1 = int(w1r);
      w1p = 0;
      if (w1 < us_IW - 1) {
        w1p = 1;
      }
      w1l = w1r - w1;
      w0l = 1.0 - w1l;
      y2 = h0l * (w0l * us_x[r0 + w1] + w1l * us_x[r0 + w1 + w1p]) + h1l * (w0l * us_x[r1 + w1] + w1l * us_x[r1 + w1 + w1p]);
      w1r = rw * (ow + 3 + 0.5) - 0.5;
      if (w1r < 0.0) {
        w1r = 0.0;
      }
      w1 = int(w1r);
      w1p = 0;
      if (w1 < us_IW - 1) {
        w1p = 1;
      }
      w1l = w1r - w1;
      w0l = 1.0 - w1l;
      y3 = h0l * (w0l * us_x[r0 + w1] + w1l * us_x[r0 + w1 + w1p]) + h1l * (w0l * us_x[r1 + w1] + w1l * us_x[r1 + w1 + w1p]);
      vstore(us_y, t, y0, y1, y2, y3);
    }
  }
}
