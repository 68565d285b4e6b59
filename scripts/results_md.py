"""Render DESIGN.md §10 tables from a bench line + its detail file:
python scripts/results_md.py profiles/r02_bench_line.json profiles/r02_bench_detail.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
line = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
d = json.load(open(sys.argv[2]))
hbm = line["roofline"]["peak"]
ops = json.load(open(os.path.join(ROOT, "profiles", "crypto_ops.json")))
o = ["| pair | grid | d1/d2 | fused µs (±95 %) | seq µs | 2-stream µs | speed-up | copy roofline | mix ceiling µs (frac) |",
     "|---|---|---|---|---|---|---|---|---|"]
for r in d["results"]:
    sp = r["speedup"]
    cap = f" cap {r['reg_cap']}" if r["reg_cap"] else ""
    o.append(f"| {r['pair']} | {r['grid']} | {r['d1']}/{r['d2']}{cap} | {r['fused_us']:.1f} (±{r['fused_ci95']:.2f}) | "
             f"{r['seq_us']:.1f} | {r['two_stream_us']:.1f} | {'**%.3f**' % sp if sp > 1 else '%.3f' % sp} "
             f"(±{r['speedup_ci95']:.3f}) | {r['bytes'] / (hbm * 1e3) / r['fused_us']:.3f} | "
             + (f"{r['ceiling_us']:.1f} ({r['ceiling_frac']:.3f}) |" if "ceiling_us" in r else "— |"))
st = d["steps"]
o.append("")
o.append(f"Geomean speed-up vs min(seq, two-stream): {line['speedup_geomean']:.3f}. Step (`value`): "
         f"{st['fused_pdl_us']:.1f} µs (ten fused kernels as programmatic dependent launches); without overlap "
         f"{st['fused_serial_us']:.1f} µs; unfused {st['unfused_two_stream_us']:.1f} µs (two streams per pair) / "
         f"{st['unfused_pdl_us']:.1f} µs (twenty PDL launches) → step speed-up {line['step_speedup']:.3f}. "
         f"Sum of the ten mix ceilings: {sum(r.get('ceiling_us', 0) for r in d['results']):.1f} µs. "
         f"e2e {line['e2e']['value'] / 1000:.1f} ms per step ({line['e2e']['h2d_bytes_per_step'] / 1e9:.2f} GB up, "
         f"{line['e2e']['d2h_bytes_per_step'] / 1e9:.2f} GB down). Clocks {line['clocks']['sm_mhz']:.0f}/"
         f"{line['clocks']['sm_max_mhz']:.0f} MHz, reasons {line['clocks']['reasons']}.")
if not d.get("crypto"):
    print("\n".join(o))
    sys.exit(0)
o.append("")
o.append("| crypto pair | partition | registers | baseline forms | fused µs | seq µs | 2-stream µs | speed-up | "
         "issue bound µs | HBM bound µs (copy / random-page) | roofline frac |")
o.append("|---|---|---|---|---|---|---|---|---|---|---|")
dc = d["crypto"].get("dag_ceiling") or {}
for c in d["crypto"]["pairs"]:
    if c["pair"] == "upsample+blake256":
        continue
    rf = c["roofline"]
    regs = f"budgets {c['interval_regs'][0]}/{c['interval_regs'][1]}" if c.get("interval_regs") else \
        (f"cap {c['reg_cap']}" if c.get("reg_cap") else f"uncapped ({c['regs']})")
    forms = "/".join(v for v in (c.get("baseline_forms") or {}).values()) or "—"
    hb = "—" if not rf.get("hbm_us") else (f"{rf['hbm_us']:.0f} / {rf['hbm_random_us']:.0f}" if rf.get("hbm_random_us")
                                          else f"{rf['hbm_us']:.0f}")
    sp = c["speedup"]
    o.append(f"| {c['pair']} | {c['d1']}/{c['d2']} @ {c['grid']} | {regs} | {forms} | {c['fused_us']:.0f} | "
             f"{c['seq_us']:.0f} | {c['two_stream_us']:.0f} | {'**%.3f**' % sp if sp > 1 else '%.3f' % sp} | "
             f"{rf['issue_us']:.0f} | {hb} | {rf['frac']:.3f} |")
if dc:
    o.append("")
    o.append(f"Random-page DAG ceiling (measured in the bench, `{dc['kernel']}`): {dc['gbs']:.0f} GB/s "
             f"({dc['bytes'] / 1e9:.1f} GB of independent random 128-B pages in {dc['us']:.0f} µs, grid {dc['grid']}).")
c4 = next((c for c in d["crypto"]["pairs"] if c["pair"] == "upsample+blake256"), None)
if c4:
    o.append("")
    o.append(f"C4 Upsample + BLAKE-256: best d0 {c4['d0']} (Upsample {c4['d1']}), "
             + (f"budgets {c4['interval_regs']}" if c4.get("interval_regs") else f"reg_cap {c4['reg_cap']}")
             + f", grid {c4['grid']}: {c4['fused_us']:.1f} µs vs {c4['seq_us']:.1f} sequential / "
               f"{c4['two_stream_us']:.1f} two-stream — **{c4['speedup']:.3f}×** (winner of {len(c4['sweep'])} "
               f"sweep points re-timed with its baselines' protocol).")
print("\n".join(o))
