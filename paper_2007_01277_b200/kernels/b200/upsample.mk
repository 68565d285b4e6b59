// Upsample bilinear 2x (align_corners=False), B200 form (MK+).
// Precondition: OH == 2 * IH, OW == 2 * IW, IW and IH even. Then rh = rw = 0.5 exactly and the
// reference form's source-index arithmetic (h1r = rh * (oh + 0.5) - 0.5 clamped, h1 = int(h1r),
// h1l = h1r - h1, likewise for w) takes exact values: output row oh = 2k + 1 blends input rows
// k and k + h1p with weights 0.75 / 0.25, oh = 2k + 2 blends rows k and k + 1 with 0.25 / 0.75,
// oh = 0 is 1.0 * row 0 + 0.0 * row 1; columns follow the same rule (ow = 4q + j from input
// columns 2q - 1 .. 2q + 2, the last column clamps). Every output is computed with the same
// float operations, in the same order, on the same operands as the reference form:
// bit-identical results.
// B200 mechanics: a thread owns one output float4 column q of the four output rows 2k+1 ..
// 2k+4 that input rows k, k+1, k+2 (k even) feed: each input row is loaded once (one 64-bit
// vector plus two neighbour scalars) and interpolated horizontally once for the two output rows
// on each side of it, and the index arithmetic is shared by 16 outputs. Consecutive threads store
// consecutive 128-bit vectors of a row (full 32-B sectors per thread pair).
//@ grid=256
//@ requires us_OH == 2 * us_IH && us_OW == 2 * us_IW && us_IW % 2 == 0 && us_IH % 2 == 0
kernel upsample(float us_x[], float us_y[], int us_NC, int us_IH, int us_IW, int us_OH, int us_OW) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int ow4 = us_OW / 4;
  int ih2 = us_IH / 2;
  int total = us_NC * ih2 * ow4;
  float xa; float xb; float xc; float xd;
  float p0; float p1; float p2; float p3; float u0; float u1; float u2; float u3; float w0; float w1; float w2; float w3;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % ow4;
    int r = t / ow4;
    int k = (r % ih2) * 2;
    int nc = r / ih2;
    int k2 = min(k + 2, us_IH - 1);
    int c = q * 2;
    int base = nc * us_IH;
    // input row k -> p, k + 1 -> u, min(k + 2, IH - 1) -> w (horizontal interpolation, ow = 4q .. 4q+3)
    int row = (base + k) * us_IW;
    vload(us_x, (row + c) / 2, xb, xc);
    xa = xb;
    if (q > 0) {
      xa = us_x[row + c - 1];
    }
    xd = xc;
    if (c + 2 < us_IW) {
      xd = us_x[row + c + 2];
    }
    if (q == 0) {
      p0 = 1.0 * xb + 0.0 * xc;
    } else {
      p0 = 0.25 * xa + 0.75 * xb;
    }
    p1 = 0.75 * xb + 0.25 * xc;
    p2 = 0.25 * xb + 0.75 * xc;
    p3 = 0.75 * xc + 0.25 * xd;
    row = (base + k + 1) * us_IW;
    vload(us_x, (row + c) / 2, xb, xc);
    xa = xb;
    if (q > 0) {
      xa = us_x[row + c - 1];
    }
    xd = xc;
    if (c + 2 < us_IW) {
      xd = us_x[row + c + 2];
    }
    if (q == 0) {
      u0 = 1.0 * xb + 0.0 * xc;
    } else {
      u0 = 0.25 * xa + 0.75 * xb;
    }
    u1 = 0.75 * xb + 0.25 * xc;
    u2 = 0.25 * xb + 0.75 * xc;
    u3 = 0.75 * xc + 0.25 * xd;
    row = (base + k2) * us_IW;
    vload(us_x, (row + c) / 2, xb, xc);
    xa = xb;
    if (q > 0) {
      xa = us_x[row + c - 1];
    }
    xd = xc;
    if (c + 2 < us_IW) {
      xd = us_x[row + c + 2];
    }
    if (q == 0) {
      w0 = 1.0 * xb + 0.0 * xc;
    } else {
      w0 = 0.25 * xa + 0.75 * xb;
    }
    w1 = 0.75 * xb + 0.25 * xc;
    w2 = 0.25 * xb + 0.75 * xc;
    w3 = 0.75 * xc + 0.25 * xd;
    int o = ((nc * us_OH + 2 * k + 1) * ow4) + q;
    if (k == 0) {
      vstore(us_y, o - ow4, 1.0 * p0 + 0.0 * u0, 1.0 * p1 + 0.0 * u1, 1.0 * p2 + 0.0 * u2, 1.0 * p3 + 0.0 * u3);
    }
    vstore(us_y, o, 0.75 * p0 + 0.25 * u0, 0.75 * p1 + 0.25 * u1, 0.75 * p2 + 0.25 * u2, 0.75 * p3 + 0.25 * u3);
    vstore(us_y, o + ow4, 0.25 * p0 + 0.75 * u0, 0.25 * p1 + 0.75 * u1, 0.25 * p2 + 0.75 * u2, 0.25 * p3 + 0.75 * u3);
    vstore(us_y, o + 2 * ow4, 0.75 * u0 + 0.25 * w0, 0.75 * u1 + 0.25 * w1, 0.75 * u2 + 0.25 * w2, 0.75 * u3 + 0.25 * w3);
    if (k + 2 < us_IH) {
      vstore(us_y, o + 3 * ow4, 0.25 * u0 + 0.75 * w0, 0.25 * u1 + 0.75 * w1, 0.25 * u2 + 0.75 * w2, 0.25 * u3 + 0.75 * w3);
    }
  }
}
