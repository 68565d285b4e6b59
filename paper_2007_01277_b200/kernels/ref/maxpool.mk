// MaxPool2d 3x3, stride 2, padding 1, with indices; reference (naive) form: one output
// per thread, scalar loads, PyTorch's scan order and NaN rule
// (max_pool2d_with_indices: `if ((val > maxval) || isnan(val))`, PAPER.md:861-868).
// Index = ih * W + iw inside the (n, c) plane (int32 here; PyTorch stores int64).
//@ grid=256
kernel maxpool(float mp_x[], float mp_y[], int mp_idx[], int mp_NC, int mp_H, int mp_W, int mp_OH, int mp_OW) dims (1024, 1, 1) {
  int total = mp_NC * mp_OH * mp_OW;
  float ninf = -1.0 / 0.0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t = t + gridDim.x * blockDim.x) {
    int ow = t % mp_OW;
    int oh = t / mp_OW % mp_OH;
    int nc = t / (mp_OW * mp_OH);
    int hstart = oh * 2 - 1;
    int wstart = ow * 2 - 1;
    int hend = min(hstart + 3, mp_H);
    int wend = min(wstart + 3, mp_W);
    hstart = max(hstart, 0);
    wstart = max(wstart, 0);
    float best = ninf;
    int bidx = hstart * mp_W + wstart;
    for (int h = hstart; h < hend; h = h + 1) {
      for (int w = wstart; w < wend; w = w + 1) {
        float v = mp_x[(nc * mp_H + h) * mp_W + w];
        if (v > best || v != v) {
          best = v;
          bidx = h * mp_W + w;
        }
      }
    }
    mp_y[t] = best;
    mp_idx[t] = bidx;
  }
}
