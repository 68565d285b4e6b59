// Im2Col 3x3, padding 1, stride 1 (PyTorch im2col_kernel semantics), reference (naive)
// form: one output element per thread, scalar load with zero padding.
// col[n][c * 9 + kh * 3 + kw][h * W + w] = x[n][c][h + kh - 1][w + kw - 1] (0 outside).
//@ grid=256
kernel im2col(float ic_x[], float ic_col[], int ic_NC, int ic_H, int ic_W) dims (1024, 1, 1) {
  int hw = ic_H * ic_W;
  int total = ic_NC * 9 * hw;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t = t + gridDim.x * blockDim.x) {
    int w = t % ic_W;
    int h = t / ic_W % ic_H;
    int k = t / hw % 9;
    int nc = t / (hw * 9);
    int ih = h + k / 3 - 1;
    int iw = w + k % 3 - 1;
    float v = 0.0;
    if (ih >= 0 && ih < ic_H && iw >= 0 && iw < ic_W) {
      v = ic_x[(nc * ic_H + ih) * ic_W + iw];
    }
    ic_col[t] = v;
  }
}
