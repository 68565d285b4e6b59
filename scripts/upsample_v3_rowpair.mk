// Upsample bilinear 2x (align_corners=False), B200 form (MK+).
// Precondition: OH == 2 * IH, OW == 2 * IW, IW % 2 == 0. Then rh = rw = 0.5 exactly and the
// reference form's source-index arithmetic (h1r = rh * (oh + 0.5) - 0.5 clamped, h1 = int(h1r),
// h1l = h1r - h1, likewise for w) takes exact values: output row oh = 2k + 1 blends input rows
// k and k + h1p with weights 0.75 / 0.25, oh = 2k + 2 blends rows k and k + 1 with 0.25 / 0.75,
// oh = 0 is 1.0 * row 0 + 0.0 * row 1; columns follow the same rule (ow = 4q + j from input
// columns 2q - 1 .. 2q + 2, the last column clamps). Every output is computed with the same
// float operations, in the same order, on the same operands as the reference form:
// bit-identical results.
// B200 mechanics: a thread owns one output float4 column q of the two output rows 2k + 1 and
// 2k + 2 that input rows k and k + 1 feed -- each input row's horizontal interpolation is
// computed once for both rows (48 instead of 72 FP ops per 8 outputs), loaded as one 64-bit
// vector plus two neighbour scalars, and consecutive threads store consecutive 128-bit vectors
// of a row (full 32-B sectors per thread pair, no shared-memory staging; the previous form
// staged through shared memory and was L1-throughput bound, ncu 91.5 %).
//@ grid=256
//@ requires us_OH == 2 * us_IH && us_OW == 2 * us_IW && us_IW % 2 == 0
kernel upsample(float us_x[], float us_y[], int us_NC, int us_IH, int us_IW, int us_OH, int us_OW) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int ow4 = us_OW / 4;
  int total = us_NC * us_IH * ow4;
  float xa; float xb; float xc; float xd; float ya; float yb; float yc; float yd;
  float p0; float p1; float p2; float p3; float u0; float u1; float u2; float u3;
  for (int t = blockIdx.x * nthr + threadIdx.x; t < total; t = t + gridDim.x * nthr) {
    int q = t % ow4;
    int r = t / ow4;
    int k = r % us_IH;
    int nc = r / us_IH;
    int kp = 0;
    if (k < us_IH - 1) {
      kp = 1;
    }
    int r0 = (nc * us_IH + k) * us_IW;
    int r1 = (nc * us_IH + k + kp) * us_IW;
    int c = q * 2;
    // columns c - 1 (a), c (b), c + 1 (c), c + 2 (d) of rows k (x*) and k + kp (y*)
    vload(us_x, (r0 + c) / 2, xb, xc);
    vload(us_x, (r1 + c) / 2, yb, yc);
    xa = xb;
    ya = yb;
    if (q > 0) {
      xa = us_x[r0 + c - 1];
      ya = us_x[r1 + c - 1];
    }
    xd = xc;
    yd = yc;
    if (c + 2 < us_IW) {
      xd = us_x[r0 + c + 2];
      yd = us_x[r1 + c + 2];
    }
    // horizontal interpolation of both rows (ow = 4q .. 4q + 3)
    if (q == 0) {
      p0 = 1.0 * xb + 0.0 * xc;
      u0 = 1.0 * yb + 0.0 * yc;
    } else {
      p0 = 0.25 * xa + 0.75 * xb;
      u0 = 0.25 * ya + 0.75 * yb;
    }
    p1 = 0.75 * xb + 0.25 * xc;
    u1 = 0.75 * yb + 0.25 * yc;
    p2 = 0.25 * xb + 0.75 * xc;
    u2 = 0.25 * yb + 0.75 * yc;
    p3 = 0.75 * xc + 0.25 * xd;
    u3 = 0.75 * yc + 0.25 * yd;
    int o = ((nc * us_OH + 2 * k + 1) * ow4) + q;
    if (k == 0) {
      vstore(us_y, o - ow4, 1.0 * p0 + 0.0 * u0, 1.0 * p1 + 0.0 * u1, 1.0 * p2 + 0.0 * u2, 1.0 * p3 + 0.0 * u3);
    }
    vstore(us_y, o, 0.75 * p0 + 0.25 * u0, 0.75 * p1 + 0.25 * u1, 0.75 * p2 + 0.25 * u2, 0.75 * p3 + 0.25 * u3);
    if (kp == 1) {
      vstore(us_y, o + ow4, 0.25 * p0 + 0.75 * u0, 0.25 * p1 + 0.75 * u1, 0.25 * p2 + 0.75 * u2, 0.25 * p3 + 0.75 * u3);
    }
  }
}
