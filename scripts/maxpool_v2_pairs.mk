// MaxPool2d 3x3/s2/p1 with indices; variant A: 2 outputs per thread, per input row one
// warp-contiguous 128-bit load (columns 4q .. 4q+3) + one scalar (column 4q-1), float2 stores.
//@ grid=256
//@ requires mp_H == 2 * mp_OH && mp_W == 2 * mp_OW && mp_W % 4 == 0
kernel maxpool(float mp_x[], float mp_y[], int mp_idx[], int mp_NC, int mp_H, int mp_W, int mp_OH, int mp_OW) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int ow2 = mp_OW / 2;
  int w4 = mp_W / 4;
  int total = mp_NC * mp_OH * ow2;
  float ninf = -1.0 / 0.0;
  float cm; float c0; float c1; float c2; float c3;
  float y0; float y1;
  int i0; int i1;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % ow2;
    int r = t / ow2;
    int oh = r % mp_OH;
    int nc = r / mp_OH;
    int col = q * 4;
    int hs = max(oh * 2 - 1, 0);
    y0 = ninf;
    y1 = ninf;
    i0 = hs * mp_W + max(col - 1, 0);
    i1 = hs * mp_W + col + 1;
    for (int kh = 0; kh < 3; kh = kh + 1) {
      int h = oh * 2 - 1 + kh;
      if (h >= 0 && h < mp_H) {
        int row = (nc * mp_H + h) * w4;
        int hw = h * mp_W;
        vload(mp_x, row + q, c0, c1, c2, c3);
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
      }
    }
    vstore(mp_y, t, y0, y1);
    vstore(mp_idx, t, i0, i1);
  }
}
