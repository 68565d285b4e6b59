"""Summaries committed under profiles/ from the ncu runs of scripts/gpu_ncu_dl.sh and
scripts/gpu_launch_list.sh (gpurun_out/ncu_dl.csv, gpurun_out/launches_step.csv):
  profiles/r01_ncu_dl_summary.json    every DL member and fused pair: the metric pass, one row each
  profiles/traffic.json               per fused pair: DRAM bytes read + written per launch (the
                                      bench's roofline `traffic`)
  profiles/r01_launches_step_summary.json  per fused kernel: mean serialized time and share of the
                                      timed step (the dominant kernel of the `roofline` object)
python scripts/ncu_profiles.py"""
import csv
import json
import os
from collections import OrderedDict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    out = OrderedDict()
    for r in csv.DictReader(lines):
        name = r["Kernel Name"].split("(")[0].strip()
        if name.startswith(("fill_", "hf_fill", "flush", "hf_flush")):
            continue
        out.setdefault((r["ID"], name), {})[r["Metric Name"]] = (r["Metric Value"].replace(",", ""), r["Metric Unit"])
    return out


def scaled(v, unit):
    return float(v) * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)


bench = json.loads(open(os.path.join(PROF, "r01_bench_full.json")).read().strip().splitlines()[-1])
cfg = {p["pair"]: p for p in bench["pairs"]}
name_of = {"bn": "bn_stats"}
kernel_pair = {f"fused_{name_of.get(a, a)}_{name_of.get(b, b)}": f"{a}+{b}"
               for a, b in (p.split("+") for p in cfg)}

dl = rows(os.path.join(OUT, "ncu_dl.csv"))
summary = {"how": "scripts/gpu_ncu_dl.sh (ncu --metrics ... --clock-control none over scripts/ncu_members.py "
                  "--from-bench profiles/r01_bench_full.json: every member at its bench grid, every fused pair at "
                  "the bench's d0/grid/split/cap, JIT-specialized); one cold-cache launch each",
           "launches": [dict(kernel=n, **{k: v for k, (v, _) in m.items()}) for (_, n), m in dl.items()]}
json.dump(summary, open(os.path.join(PROF, "r01_ncu_dl_summary.json"), "w"), indent=1)
traffic = {}
for (_, n), m in dl.items():
    if n in kernel_pair:
        rd = scaled(*m["dram__bytes_read.sum"])
        wr = scaled(*m["dram__bytes_write.sum"])
        p = cfg[kernel_pair[n]]
        traffic[kernel_pair[n]] = {"kernel": n, "grid": p["grid"], "block": p["d0"], "dram_bytes": rd + wr,
                                   "read": rd, "write": wr, "algorithmic_bytes": p["bytes"],
                                   "ncu_ns": scaled(*m["gpu__time_duration.sum"])}
json.dump(traffic, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)

path = os.path.join(OUT, "launches_step.csv")
if os.path.exists(path):
    per = OrderedDict()
    for (_, n), m in rows(path).items():
        per.setdefault(n, []).append(scaled(*m["gpu__time_duration.sum"]) / 1e3)
    total = sum(sum(v) for v in per.values())
    steps = max(len(v) for v in per.values())
    kern = {n: {"mean_us": sum(v) / len(v), "share_of_step": sum(v) / total} for n, v in per.items()}
    dom = max(kern, key=lambda n: kern[n]["share_of_step"])
    json.dump({"how": "scripts/gpu_launch_list.sh: ncu --metrics gpu__time_duration.sum --clock-control none --nvtx "
                      "--nvtx-include step/ python bench.py --steps 3 --warmup 3 (serialized, cold-cache launches of "
                      "the timed step)",
               "launches": sum(len(v) for v in per.values()), "ncu_us_per_step": total / steps, "kernels": kern,
               "dominant": dom, "bench_roofline_kernel": bench["roofline"]["kernel"]},
              open(os.path.join(PROF, "r01_launches_step_summary.json"), "w"), indent=1)
print("ok", len(summary["launches"]), "launches;", len(traffic), "pairs")
