"""Summaries committed under profiles/ from scripts/gpu_ncu_r02.sh (gpurun_out/):
  r02_ncu_summary.json        every benched member and fused kernel (DL + crypto), one cold launch each
  r02_traffic.json            per fused DL pair: ncu dram bytes read + written per launch (bench roofline
                              `traffic`; keyed by pair with the configuration it was measured at)
  r02_issue_table.json        per pair: issue-slot utilization of the fused kernel vs each member alone
                              and vs their time-weighted combination (combined_utilization,
                              machine.cpp:285-289 / PAPER.md:970-972) -- the north star's ncu criterion
  r02_launches_step_summary.json  per fused kernel: serialized time and share of the bench's timed step
  r02_ncu_full_dominant.txt   the --set full capture of the dominant fused kernel (details page)"""
import csv
import json
import os
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, ROOT)


def rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    out = OrderedDict()
    for r in csv.DictReader(lines):
        name = r["Kernel Name"].split("(")[0].strip()
        if name.startswith(("fill_", "flush", "phase_spin")):
            continue
        v, unit = r["Metric Value"].replace(",", ""), r["Metric Unit"]
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
        try:
            val = float(v) * scale
        except ValueError:
            val = v
        out.setdefault((r["ID"], name), {})[r["Metric Name"]] = val
    return list(out.items())


def main():
    order = json.loads(open(os.path.join(OUT, "ncu_r02.order")).read().strip().splitlines()[-1])
    launches = rows(os.path.join(OUT, "ncu_r02.csv"))
    assert len(order) == len(launches), (len(order), len(launches))
    detail = json.load(open(os.path.join(PROF, "r02_bench_detail.json")))
    cfg = {r["pair"]: r for r in detail["results"]}
    cfg.update({c["pair"]: c for c in detail["crypto"]["pairs"]})
    table = OrderedDict()
    finals = OrderedDict()  # pair -> [(config, metrics)] of the search's other finalists
    for label, ((_, name), m) in zip(order, launches):
        pair, role = label.split(":", 1)
        if role.startswith("final:"):
            finals.setdefault(pair, []).append((json.loads(role[len("final:"):]), dict(kernel=name, **m)))
            continue
        table.setdefault(pair, {})[role] = dict(kernel=name, **m)
    json.dump({"how": "scripts/gpu_ncu_r02.sh: ncu --metrics ... --clock-control none over scripts/ncu_launch_r02.py "
                      "(benched configurations of profiles/r02_bench_detail.json, each pair on its own tensors)",
               "pairs": table}, open(os.path.join(PROF, "r02_ncu_summary.json"), "w"), indent=1)
    traffic, issue = {}, {}
    from paper_2007_01277_b200 import hfuse as hf
    for pair, t in table.items():
        f = t["fused"]
        c = cfg[pair]
        if pair in {r["pair"] for r in detail["results"]}:
            keep = {k: c.get(k) for k in ("d1", "d2", "reg_cap", "interval_regs", "grid", "split_grid")}
            measured = [(keep, f)] + finals.get(pair, [])
            traffic[pair] = [{"config": cf, "dram_bytes": mm["dram__bytes_read.sum"] + mm["dram__bytes_write.sum"],
                              "read": mm["dram__bytes_read.sum"], "write": mm["dram__bytes_write.sum"],
                              "algorithmic_bytes": c["bytes"], "ncu_ns": mm["gpu__time_duration.sum"]}
                             for cf, mm in measured]
        a, b = pair.split("+")
        ia, ib = t[a], t[b]
        key = "smsp__issue_active.avg.pct_of_peak_sustained_elapsed"
        comb = hf.combined_utilization(ia[key], int(ia["gpu__time_duration.sum"]), ib[key],
                                       int(ib["gpu__time_duration.sum"]))
        issue[pair] = {"fused": round(f[key], 2), a: round(ia[key], 2), b: round(ib[key], 2),
                       "combined": round(comb, 2), "above_both": f[key] > max(ia[key], ib[key]),
                       "above_combined": f[key] > comb,
                       "fused_ns": f["gpu__time_duration.sum"],
                       "members_ns": [ia["gpu__time_duration.sum"], ib["gpu__time_duration.sum"]]}
    json.dump(traffic, open(os.path.join(PROF, "r02_traffic.json"), "w"), indent=1)
    json.dump({"metric": "smsp__issue_active.avg.pct_of_peak_sustained_elapsed (%), one cold launch each; "
                         "combined = time-weighted member utilization (hf_combined_utilization)",
               "pairs": issue}, open(os.path.join(PROF, "r02_issue_table.json"), "w"), indent=1)
    # launch list of the timed step
    path = os.path.join(OUT, "launches_r02.csv")
    per = OrderedDict()
    for (_, name), m in rows(path):
        per.setdefault(name, []).append(m["gpu__time_duration.sum"])
    tot = sum(sum(v) for v in per.values())
    json.dump({"how": "ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include step/ "
                      "python bench.py --steps 3 --warmup 3 ... (serialized, cold-cache per launch)",
               "kernels": {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot}
                           for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}},
              open(os.path.join(PROF, "r02_launches_step_summary.json"), "w"), indent=1)
    rep = os.path.join(OUT, "prof_dom_r02.ncu-rep")
    if os.path.exists(rep):
        txt = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
        open(os.path.join(PROF, "r02_ncu_full_dominant.txt"), "w").write(txt)
    for p, v in issue.items():
        print(p, v["fused"], v[p.split("+")[0]], v[p.split("+")[1]], v["combined"], v["above_both"])


if __name__ == "__main__":
    main()
