// Upsample bilinear 2x (align_corners=False), B200 form (MK+).
// Precondition: OH == 2 * IH, OW == 2 * IW, IW % 4 == 0. Then rw = IW / OW = 0.5 exactly and the
// generic source-index arithmetic of the reference form (w1r = rw * (ow + 0.5) - 0.5, clamped,
// w1 = int(w1r), w1l = w1r - w1) takes exact values: output ow = 8s + k (k >= 1) blends input
// columns 4s + (k - 1) / 2 and the next one with right weight 0.25 (k odd) or 0.75 (k even);
// ow = 8s (s > 0) blends 4s - 1 and 4s with weight 0.75; ow = 0 takes column 0 with weight 0;
// the last column clamps (w1p = 0). Each output is computed with the same float operations, in
// the same order, on the same operands as the reference form: bit-identical results.
// B200 mechanics: 8 outputs per thread (the per-row source setup is amortized 8x), one 128-bit
// load + 2 scalar loads per input row, constant weights. A warp's 32 threads own 256
// consecutive outputs; they are staged in shared memory (warp_sync, no block barrier) and
// written as two warp-contiguous 128-bit stores per thread -- storing each thread's own 32 B
// directly would make every store instruction cover only half of each 32-B sector (measured
// 8% slower on B200, scripts/probe_upsample.py). The loop is warp-uniform (tw = the warp's
// first item) so warp_sync always sees the full warp.
//@ grid=256
kernel upsample(float us_x[], float us_y[], int us_NC, int us_IH, int us_IW, int us_OH, int us_OW) dims (1024, 1, 1) {
  shared float us_buf[8192];
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int lane = threadIdx.x % 32;
  int wb = (threadIdx.x / 32) * 64;
  int ow8 = us_OW / 8;
  int total = us_NC * us_OH * ow8;
  float rh = float(us_IH) / us_OH;
  float a0; float b0; float c0; float d0; float e0; float f0;
  float a1; float b1; float c1; float d1; float e1; float f1;
  float t0; float t1; float y0; float y1; float y2; float y3; float y4; float y5; float y6; float y7;
  for (int tw = blockIdx.x * nthr + threadIdx.x - lane; tw < total; tw = tw + gridDim.x * nthr) {
    int t = tw + lane;
    if (t < total) {
      int s = t % ow8;
      int r = t / ow8;
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
      int c = s * 4;
      vload(us_x, (r0 + c) / 4, b0, c0, d0, e0);
      vload(us_x, (r1 + c) / 4, b1, c1, d1, e1);
      a0 = b0;
      a1 = b1;
      if (s > 0) {
        a0 = us_x[r0 + c - 1];
        a1 = us_x[r1 + c - 1];
      }
      f0 = e0;
      f1 = e1;
      if (c + 4 < us_IW) {
        f0 = us_x[r0 + c + 4];
        f1 = us_x[r1 + c + 4];
      }
      if (s == 0) {
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
      y4 = h0l * (0.25 * c0 + 0.75 * d0) + h1l * (0.25 * c1 + 0.75 * d1);
      y5 = h0l * (0.75 * d0 + 0.25 * e0) + h1l * (0.75 * d1 + 0.25 * e1);
      y6 = h0l * (0.25 * d0 + 0.75 * e0) + h1l * (0.25 * d1 + 0.75 * e1);
      y7 = h0l * (0.75 * e0 + 0.25 * f0) + h1l * (0.75 * e1 + 0.25 * f1);
      vstore(us_buf, wb + 2 * lane, y0, y1, y2, y3);
      vstore(us_buf, wb + 2 * lane + 1, y4, y5, y6, y7);
    }
    warp_sync();
    // float4 m of the warp's 64 belongs to item tw + m / 2
    if (tw + lane / 2 < total) {
      vload(us_buf, wb + lane, y0, y1, y2, y3);
      vstore(us_y, 2 * tw + lane, y0, y1, y2, y3);
    }
    if (tw + 16 + lane / 2 < total) {
      vload(us_buf, wb + 32 + lane, y4, y5, y6, y7);
      vstore(us_y, 2 * tw + 32 + lane, y4, y5, y6, y7);
    }
    warp_sync();
  }
}
