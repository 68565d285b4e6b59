// MaxPool2d 3x3/s2/p1 with indices; variant B: 2 x 2 outputs per thread (output rows oh, oh+1
// from input rows 2oh-1 .. 2oh+3: the shared row is read once), per input row one
// warp-contiguous 128-bit load + one scalar, float2 stores.
//@ grid=256
//@ requires mp_H == 2 * mp_OH && mp_W == 2 * mp_OW && mp_W % 4 == 0 && mp_OH % 2 == 0
kernel maxpool(float mp_x[], float mp_y[], int mp_idx[], int mp_NC, int mp_H, int mp_W, int mp_OH, int mp_OW) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int ow2 = mp_OW / 2;
  int oh2 = mp_OH / 2;
  int w4 = mp_W / 4;
  int total = mp_NC * oh2 * ow2;
  float ninf = -1.0 / 0.0;
  float cm; float c0; float c1; float c2; float c3;
  float y0; float y1; float z0; float z1;
  int i0; int i1; int j0; int j1;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % ow2;
    int r = t / ow2;
    int oh = (r % oh2) * 2;
    int nc = r / oh2;
    int col = q * 4;
    int hs = max(oh * 2 - 1, 0);
    y0 = ninf;
    y1 = ninf;
    z0 = ninf;
    z1 = ninf;
    i0 = hs * mp_W + max(col - 1, 0);
    i1 = hs * mp_W + col + 1;
    j0 = (oh * 2 + 1) * mp_W + max(col - 1, 0);
    j1 = (oh * 2 + 1) * mp_W + col + 1;
    for (int kh = 0; kh < 5; kh = kh + 1) {
      int h = oh * 2 - 1 + kh;
      if (h >= 0 && h < mp_H) {
        int row = (nc * mp_H + h) * w4;
        int hw = h * mp_W;
        vload(mp_x, row + q, c0, c1, c2, c3);
        cm = ninf;
        if (col > 0) {
          cm = mp_x[row * 4 + col - 1];
        }
        if (kh < 3) {
          if (col > 0) {
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
        if (kh >= 2) {
          if (col > 0) {
            if (cm > z0 || cm != cm) {
              z0 = cm;
              j0 = hw + col - 1;
            }
          }
          if (c0 > z0 || c0 != c0) {
            z0 = c0;
            j0 = hw + col;
          }
          if (c1 > z0 || c1 != c1) {
            z0 = c1;
            j0 = hw + col + 1;
          }
          if (c1 > z1 || c1 != c1) {
            z1 = c1;
            j1 = hw + col + 1;
          }
          if (c2 > z1 || c2 != c2) {
            z1 = c2;
            j1 = hw + col + 2;
          }
          if (c3 > z1 || c3 != c3) {
            z1 = c3;
            j1 = hw + col + 3;
          }
        }
      }
    }
    int o = (nc * mp_OH + oh) * ow2 + q;
    vstore(mp_y, o, y0, y1);
    vstore(mp_idx, o, i0, i1);
    vstore(mp_y, o + ow2, z0, z1);
    vstore(mp_idx, o + ow2, j0, j1);
  }
}
