// MaxPool2d 3x3, stride 2, padding 1, with indices; B200 form (MK+).
// Same scan order and NaN rule as the reference form (PyTorch max_pool2d_with_indices),
// so values and indices are bit-identical. Requires H == 2 * OH, W == 2 * OW, W % 8 == 0.
// B200 mechanics: each thread produces 4 consecutive outputs; per input row it issues two
// 128-bit loads (columns 8q .. 8q+7) plus one scalar load (column 8q-1), so the 3 x 9
// input window is read with 9 loads instead of 36, and stores 4 values + 4 indices with
// two 128-bit stores.
//@ grid=256
//@ requires mp_H == 2 * mp_OH && mp_W == 2 * mp_OW && mp_W % 8 == 0
kernel maxpool(float mp_x[], float mp_y[], int mp_idx[], int mp_NC, int mp_H, int mp_W, int mp_OH, int mp_OW) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int ow4 = mp_OW / 4;
  int w4 = mp_W / 4;
  int total = mp_NC * mp_OH * ow4;
  float ninf = -1.0 / 0.0;
  float cm; float c0; float c1; float c2; float c3; float c4; float c5; float c6; float c7;
  float y0; float y1; float y2; float y3;
  int i0; int i1; int i2; int i3;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % ow4;
    int r = t / ow4;
    int oh = r % mp_OH;
    int nc = r / mp_OH;
    int col = q * 8;
    int hs = max(oh * 2 - 1, 0);
    y0 = ninf;
    y1 = ninf;
    y2 = ninf;
    y3 = ninf;
    i0 = hs * mp_W + max(col - 1, 0);
    i1 = hs * mp_W + col + 1;
    i2 = hs * mp_W + col + 3;
    i3 = hs * mp_W + col + 5;
    for (int kh = 0; kh < 3; kh = kh + 1) {
      int h = oh * 2 - 1 + kh;
      if (h >= 0 && h < mp_H) {
        int row = (nc * mp_H + h) * w4;
        int hw = h * mp_W;
        vload(mp_x, row + q * 2, c0, c1, c2, c3);
        vload(mp_x, row + q * 2 + 1, c4, c5, c6, c7);
        if (col > 0) {
          cm = mp_x[row * 4 + col - 1];
          if (cm > y0 || cm != cm) {
            y0 = cm;
            i0 = hw + col - 1;
          }
        }
        if (c0 > y0 || c0 != c0) {
          y0 = c0;
          i0 = hw + col;
        }
        if (c1 > y0 || c1 != c1) {
          y0 = c1;
          i0 = hw + col + 1;
        }
        if (c1 > y1 || c1 != c1) {
          y1 = c1;
          i1 = hw + col + 1;
        }
        if (c2 > y1 || c2 != c2) {
          y1 = c2;
          i1 = hw + col + 2;
        }
        if (c3 > y1 || c3 != c3) {
          y1 = c3;
          i1 = hw + col + 3;
        }
        if (c3 > y2 || c3 != c3) {
          y2 = c3;
          i2 = hw + col + 3;
        }
        if (c4 > y2 || c4 != c4) {
          y2 = c4;
          i2 = hw + col + 4;
        }
        if (c5 > y2 || c5 != c5) {
          y2 = c5;
          i2 = hw + col + 5;
        }
        if (c5 > y3 || c5 != c5) {
          y3 = c5;
          i3 = hw + col + 5;
        }
        if (c6 > y3 || c6 != c6) {
          y3 = c6;
          i3 = hw + col + 6;
        }
        if (c7 > y3 || c7 != c7) {
          y3 = c7;
          i3 = hw + col + 7;
        }
      }
    }
    vstore(mp_y, t, y0, y1, y2, y3);
    vstore(mp_idx, t, i0, i1, i2, i3);
  }
}
