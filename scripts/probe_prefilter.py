"""Model pre-filter of the partition search vs the exhaustive device sweep,
on the ten DL pairs at grid 296, 64-thread granularity: best time found, candidates compiled and
timed, wall time, and how the model's ranking (max of the two constituents timed alone at each
interval size) tracks the measured fused times."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

G = int(os.environ.get("GRID", "296"))
K = int(os.environ.get("PREFILTER", "3"))
img = hf.Image(P.MEMBERS[P.ORDER[0]].sizes["full"](0).image)
for k in P.ORDER[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
src = {k: P.source("b200", P.MEMBERS[k].stem) for k in P.ORDER}
out = {"grid": G, "prefilter": K, "pairs": {}}
for a, b in P.PAIRS:
    t0 = time.perf_counter()
    ex = hf.search(src[a], src[b], img, d0=1024, grid=G, reps=5, warmup=2, specialize=True, granularity=64)
    t_ex = time.perf_counter() - t0
    t0 = time.perf_counter()
    pf = hf.search(src[a], src[b], img, d0=1024, grid=G, reps=5, warmup=2, specialize=True, granularity=64,
                   prefilter=K)
    t_pf = time.perf_counter() - t0
    measured = {}
    for row in ex["trace"]:
        measured[row["d1"]] = min(measured.get(row["d1"], 1e30), row["us"])
    model = pf["model"]
    mem = pf["member_us"]
    common = sorted(set(measured) & set(model))
    rank_m = sorted(common, key=lambda d: measured[d])
    rank_p = sorted(common, key=lambda d: model[d])
    out["pairs"][f"{a}+{b}"] = {
        "exhaustive": {"best_us": ex["best_time"] / 1000.0, "d1": ex["d1"], "points": len(ex["trace"]),
                       "wall_s": round(t_ex, 2)},
        "prefilter": {"best_us": pf["best_time"] / 1000.0, "d1": pf["d1"], "points": len(pf["trace"]),
                      "wall_s": round(t_pf, 2)},
        "ratio": round(pf["best_time"] / ex["best_time"], 4),
        "best_measured_rank_in_model": rank_p.index(rank_m[0]) + 1 if common else None,
        "model_us": {str(d): round(model[d], 2) for d in common},
        "measured_us": {str(d): round(measured[d], 2) for d in common},
        "member_us": {str(d): [round(x, 2) for x in v] for d, v in mem.items()},
    }
    print(a, b, json.dumps({k: v for k, v in out["pairs"][f"{a}+{b}"].items() if k in ("exhaustive", "prefilter", "ratio", "best_measured_rank_in_model")}), flush=True)
r = [p["ratio"] for p in out["pairs"].values()]
out["summary"] = {"max_ratio": max(r), "mean_ratio": sum(r) / len(r),
                  "points_exhaustive": sum(p["exhaustive"]["points"] for p in out["pairs"].values()),
                  "points_prefilter": sum(p["prefilter"]["points"] for p in out["pairs"].values())}
print(json.dumps(out["summary"]))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_prefilter.json", "w"), indent=1)
