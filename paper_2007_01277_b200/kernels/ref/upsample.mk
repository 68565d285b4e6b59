// Upsample bilinear 2x (align_corners=False), reference (naive) form: PyTorch's
// upsample_bilinear2d_out_frame arithmetic (area_pixel_compute_source_index with the
// negative-source clamp, h1p/w1p edge steps, lambda weights), one output per thread.
//@ grid=256
kernel upsample(float us_x[], float us_y[], int us_NC, int us_IH, int us_IW, int us_OH, int us_OW) dims (1024, 1, 1) {
  int total = us_NC * us_OH * us_OW;
  float w1r; int w1; int w1p; float w1l; float w0l; float val;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t = t + gridDim.x * blockDim.x) {
    int ow = t % us_OW;
    int oh = t / us_OW % us_OH;
    int nc = t / (us_OW * us_OH);
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
      val = h0l * (w0l * us_x[r0 + w1] + w1l * us_x[r0 + w1 + w1p]) + h1l * (w0l * us_x[r1 + w1] + w1l * us_x[r1 + w1 + w1p]);
      us_y[t] = val;
    }
  }
}
