"""Render DESIGN.md §10 tables from a bench JSON line (profiles/r01_bench_full.json)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
o = []
ceil = all("ceiling_frac" in p for p in d["pairs"])
o.append("| pair | grid | d1/d2 | fused µs | seq µs | 2-stream µs | speedup | roofline |" + (" mix ceiling µs (frac) |" if ceil else "")
         + " naive goto fusion µs | VFuse µs |")
o.append("|---|---|---|---|---|---|---|---|---|---|" + ("---|" if ceil else ""))
for p in d["pairs"]:
    sp = p["speedup"]
    o.append(f"| {p['pair']} | {p['grid']} | {p['d1']}/{p['d2']}{' cap ' + str(p['reg_cap']) if p['reg_cap'] else ''} | "
             f"{p['fused_us']:.1f} | {p['seq_us']:.1f} | {p['two_stream_us']:.1f} | "
             f"{'**%.3f**' % sp if sp > 1.0 else '%.3f' % sp} | {p['roofline_frac']:.3f} | "
             + (f"{p['ceiling_us']:.1f} ({p['ceiling_frac']:.3f}) | " if ceil else "")
             + f"{p['naive_fused_us']:.1f} | {p['vertical_us']:.1f} |")
o.append("")
o.append(f"Geomean speedup vs min(seq, two-stream): {d['speedup_geomean']:.3f}. Step of all ten (`value`): "
         f"{d['value']:.1f} µs fused (programmatic dependent launches) vs "
         + (f"{min(d['unfused_two_stream_step_us'], d.get('unfused_overlap_step_us', 1e30)):.1f} µs for the faster unfused step "
            f"(step speed-up {d['step_speedup']:.3f}); without overlap the fused step takes "
            f"{d.get('fused_serial_step_us', float('nan')):.1f} µs. " if 'unfused_overlap_step_us' in d else
            f"{d['unfused_two_stream_step_us']:.1f} µs unfused on two streams. ") +
         f"e2e (host buffers, pipelined): {d['e2e']['value'] / 1000:.1f} ms per step "
         f"({d['e2e']['h2d_bytes_per_step'] / 1e9:.2f} GB up, {d['e2e']['d2h_bytes_per_step'] / 1e9:.2f} GB down); "
         + (f"reference CPU interpreter: {d['cpu_baseline']['value'] / 1e6:.1f} s per step "
            f"({d['cpu_baseline']['cores']} processes). " if d.get("cpu_baseline") else "") +
         f"Clocks {d['clocks']['sm_mhz']:.0f}/{d['clocks']['sm_max_mhz']:.0f} MHz, reasons {d['clocks']['reasons']}.")
if d.get("ratios"):
    rr = d["ratios"]
    rs = sorted({x["target_ratio"] for x in rr["rows"]})
    o.append("")
    o.append("Cells: measured t_b/t_a; fused µs / min(seq, two-stream) µs; speedup.")
    o.append("")
    o.append("| pair | " + " | ".join(f"t_b/t_a ≈ {r:g}" for r in rs) + " |")
    o.append("|---|" + "---|" * len(rs))
    for pair in dict.fromkeys(x["pair"] for x in rr["rows"]):
        cells = []
        for r in rs:
            x = next(x for x in rr["rows"] if x["pair"] == pair and x["target_ratio"] == r)
            sp = x["speedup"]
            cells.append(f"{x['ratio']:.2f}, {x['fused_us']:.1f} / {min(x['seq_us'], x['two_stream_us']):.1f}, "
                         + ("**%.3f**" % sp if sp > 1.0 else "%.3f" % sp))
        o.append(f"| {pair} | " + " | ".join(cells) + " |")
    o.append("")
    o.append("Geomean speedup per ratio: " + ", ".join(f"{k}: {v:.3f}" for k, v in rr["speedup_geomean"].items()) + ".")
if d.get("crypto"):
    o.append("")
    o.append("| crypto pair | partition | registers | fused µs | seq µs | 2-stream µs | speedup | roofline (bound) |")
    o.append("|---|---|---|---|---|---|---|---|")
    for p in d["crypto"]["c3"]:
        regs = ("budgets %d/%d" % tuple(p["interval_regs"])) if p.get("interval_regs") else (
            "cap %s" % p["reg_cap"] if p["reg_cap"] else "uncapped (%d)" % p["regs"])
        r = p.get("roofline") or {}
        o.append(f"| {p['pair']} | {p['d1']}/{p['d2']} | {regs} | {p['fused_us']:.0f} | {p['seq_us']:.0f} | "
                 f"{p['two_stream_us']:.0f} | {'**%.3f**' % p['speedup'] if p['speedup'] > 1.0 else '%.3f' % p['speedup']} | {r.get('frac', 0):.2f} issue, {r.get('alu_frac', 0):.2f} ALU pipe |")
    c4 = d["crypto"]["c4"]
    b = c4["best"]
    o.append("")
    grids = (f" (grids: fused {b['grid']}, members alone {c4['grid_a']}/{c4['grid_b']}, two-stream "
             f"{c4['two_stream_grids'][0]}/{c4['two_stream_grids'][1]})" if "grid" in b else "")
    o.append(f"C4 Upsample + BLAKE-256: best d0 {b['d0']} (Upsample {b['d1']}), reg_cap {b['reg_cap']}: {b['us']:.1f} µs vs "
             f"{c4['seq_us']:.1f} sequential / {c4['two_stream_us']:.1f} two-stream{grids} — **{c4['speedup']:.3f}×**.")
print("\n".join(o))
