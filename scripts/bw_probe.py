"""HBM bandwidth ceilings by read:write mix on this B200, measured through libhfuse itself.

The DL members span read-only (BN, Hist), 1:1-ish (MaxPool), 1:4 (Upsample) and 1:9 (Im2Col)
traffic mixes; the copy figure in MEASURED_PEAKS.json is one point of that curve. Each probe is
an MK+ streaming kernel (128-bit loads/stores, grid-stride) timed with the bench protocol
(L2 flushed before every repetition, median). Output: one JSON object per (mix, grid).

    python scripts/bw_probe.py > gpurun_out/bw_probe.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2007_01277_b200 import hfuse as hf  # noqa: E402

TOTAL = 1 << 28  # ~1 GiB of traffic per launch (>> 126 MB L2)


def source(writes: int, reads: bool, threads: int) -> str:
    outs = "".join(f", float o{j}[]" for j in range(writes))
    body = []
    if reads:
        body.append("vload(x, i, a, b, c, d);")
    else:
        body.append("a = i; b = a + 1.0; c = a + 2.0; d = a + 3.0;")
    for j in range(writes):
        body.append(f"vstore(o{j}, i, a, b, c, d);")
    if reads and writes == 0:
        body.append("s = s + a + b + c + d;")
    tail = "  if (s == 1234.5) {\n    sink[0] = s;\n  }\n" if reads and writes == 0 else ""
    return (f"kernel bw(float x[], float sink[]{outs}, int n4) dims ({threads}, 1, 1) {{\n"
            "  int nthr = blockDim.x * blockDim.y * blockDim.z;\n"
            "  float a; float b; float c; float d; float s;\n"
            "  for (int i = blockIdx.x * nthr + threadIdx.x; i < n4; i = i + gridDim.x * nthr) {\n    "
            + "\n    ".join(body) + "\n  }\n" + tail + "}\n")


def main():
    rows = []
    for name, reads, writes in (("read", True, 0), ("write", False, 1), ("copy 1:1", True, 1),
                                ("1:2", True, 2), ("1:4", True, 4), ("1:9", True, 9)):
        per = (1 if reads else 0) + writes
        n = (TOTAL // per) // 4096 * 4096
        img_text = f"array x float32 {n} seed 1 uniform -1 1\narray sink float32 4 zero\nscalar n4 int32 {n // 4}\n"
        img_text += "".join(f"array o{j} float32 {n} zero\n" for j in range(writes))
        img = hf.Image(img_text).upload()
        nbytes = 4 * n * per
        for threads, grid in ((1024, 296), (512, 592), (256, 1184), (1024, 148 * 8)):
            m = hf.Module.kernel(source(writes, reads, threads), grid=grid, specialize=img)
            t = hf.time("single", m, None, img, grid, warmup=3, reps=20)["median_us"]
            rows.append({"mix": name, "threads": threads, "grid": grid, "bytes": nbytes, "us": round(t, 2),
                         "gbs": round(nbytes / (t * 1e3), 1)})
            print(json.dumps(rows[-1]), flush=True)
        del img
    best = {}
    for r in rows:
        if r["mix"] not in best or r["gbs"] > best[r["mix"]]["gbs"]:
            best[r["mix"]] = r
    print(json.dumps({"best": {k: v["gbs"] for k, v in best.items()}}), flush=True)


if __name__ == "__main__":
    main()
