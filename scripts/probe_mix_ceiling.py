"""Mix-matched streaming ceiling per DL pair: a plain 128-bit grid-stride kernel (MK+, run through
the same runtime) that reads R and writes W bytes -- the pair's algorithmic read and write bytes
-- timed under the bench's steady protocol at the bench's grids. The fused kernel's time over
this is its distance from what HBM delivers for that read:write mix at that size.
python scripts/probe_mix_ceiling.py > gpurun_out/probe_mix_ceiling.json"""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

STREAM = """
kernel stream(float s_src[], float s_dst[], int s_nr4, int s_nw4) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int n = max(s_nr4, s_nw4);
  float acc = 0.0;
  float a; float b; float c; float d;
  for (int i = blockIdx.x * nthr + threadIdx.x; i < n; i = i + gridDim.x * nthr) {
    if (i < s_nr4) {
      vload(s_src, i, a, b, c, d);
      acc = acc + a + b + c + d;
    }
    if (i < s_nw4) {
      vstore(s_dst, i, acc, a, b, c);
    }
  }
  if (acc == 12345.0) {
    s_dst[0] = acc;
  }
}
"""
# four 128-bit loads in flight per thread (the BN / Hist member pattern), then the stores
STREAM4 = """
kernel stream4(float s_src[], float s_dst[], int s_nr4, int s_nw4) dims (1024, 1, 1) {
  int nthr = blockDim.x * blockDim.y * blockDim.z;
  int n = max(s_nr4, s_nw4);
  int st = gridDim.x * nthr;
  float acc = 0.0;
  float a0; float b0; float c0; float d0; float a1; float b1; float c1; float d1;
  float a2; float b2; float c2; float d2; float a3; float b3; float c3; float d3;
  for (int i = blockIdx.x * nthr + threadIdx.x; i < n; i = i + 4 * st) {
    a0 = 0.0; b0 = 0.0; c0 = 0.0; d0 = 0.0; a1 = 0.0; b1 = 0.0; c1 = 0.0; d1 = 0.0;
    a2 = 0.0; b2 = 0.0; c2 = 0.0; d2 = 0.0; a3 = 0.0; b3 = 0.0; c3 = 0.0; d3 = 0.0;
    if (i < s_nr4) { vload(s_src, i, a0, b0, c0, d0); }
    if (i + st < s_nr4) { vload(s_src, i + st, a1, b1, c1, d1); }
    if (i + 2 * st < s_nr4) { vload(s_src, i + 2 * st, a2, b2, c2, d2); }
    if (i + 3 * st < s_nr4) { vload(s_src, i + 3 * st, a3, b3, c3, d3); }
    acc = acc + a0 + b1 + c2 + d3;
    if (i < s_nw4) { vstore(s_dst, i, acc, a0, b0, c0); }
    if (i + st < s_nw4) { vstore(s_dst, i + st, a1, b1, c1, d1); }
    if (i + 2 * st < s_nw4) { vstore(s_dst, i + 2 * st, a2, b2, c2, d2); }
    if (i + 3 * st < s_nw4) { vstore(s_dst, i + 3 * st, a3, b3, c3, d3); }
  }
  if (acc == 12345.0) {
    s_dst[0] = acc;
  }
}
"""
# algorithmic (read, write) bytes of each member at the C2 shapes
RW = {"bn": (205520896, 2048), "hist": (205520896, 256), "im2col": (25690112, 231211008),
      "maxpool": (205520896, 102760448), "upsample": (51380224, 205520896)}
GRIDS = [296, 592, 1184, 2368, 4736]
bench = json.loads(open(os.path.join(os.path.dirname(__file__), "..", "profiles", "r01_bench_full.json"))
                   .read().strip().splitlines()[-1])
out = {"how": __doc__.strip().splitlines()[0], "pairs": {}}
for p in bench["pairs"]:
    a, b = p["pair"].split("+")
    r, w = RW[a][0] + RW[b][0], RW[a][1] + RW[b][1]
    img = hf.Image(f"array s_src float32 {r // 4} zero\narray s_dst float32 {max(w, 16) // 4} zero\n"
                   f"scalar s_nr4 int32 {r // 16}\nscalar s_nw4 int32 {w // 16}\n").upload()
    ts = {}
    for name, text in (("stream", STREAM), ("stream4", STREAM4)):
        m = hf.Module.kernel(text, grid=GRIDS[0], specialize=img)
        for g in GRIDS:
            ts[(name, g)] = hf.time("single", m, None, img, g, warmup=5, reps=40, flush_l2=False)["iqm_us"]
        del m
    kind, g = min(ts, key=ts.get)
    out["pairs"][p["pair"]] = {"read": r, "write": w, "ceiling_us": round(ts[(kind, g)], 2), "kernel": kind, "grid": g,
                               "all_us": {f"{k}@{x}": round(v, 2) for (k, x), v in ts.items()},
                               "ceiling_gbs": round((r + w) / (ts[(kind, g)] * 1e3), 1), "fused_us": p["fused_us"],
                               "fused_over_ceiling": round(ts[(kind, g)] / p["fused_us"], 3)}
    print(p["pair"], out["pairs"][p["pair"]], file=sys.stderr, flush=True)
    del img
print(json.dumps(out, indent=1))
