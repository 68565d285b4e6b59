"""SASS evidence for the benched kernels, generated on CPU: every DL pair's
fused kernel and the crypto pairs at the configurations of profiles/r02_bench_detail.json are
built exactly as bench.py builds them (NVRTC -> sm_100a cubin, JIT-specialized to the bench
image), disassembled with cuobjdump -sass, and summarized: 128-bit global loads/stores
(LDG.E.128 / STG.E.128), local-memory traffic (LDL/STL: spills), named barriers (BAR.SYNC /
BAR.SYNC.DEFER_BLOCKING), register re-sizing (USETMAXREG, the per-interval budgets), registers.
Writes profiles/r02_sass_summary.json and one excerpt file per kernel family."""
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

PATTERNS = {"LDG.E.128": r"\bLDG\.E\.128\b", "LDG.E.64": r"\bLDG\.E\.64\b", "LDG.E": r"\bLDG\.E(\.CONSTANT)?\s",
            "STG.E.128": r"\bSTG\.E\.128\b", "STG.E": r"\bSTG\.E\s", "LDL": r"\bLDL\b", "STL": r"\bSTL\b",
            "BAR.SYNC": r"\bBAR\.SYNC", "USETMAXREG": r"\bUSETMAXREG\b", "ATOMS": r"\bATOMS\b",
            "SHFL": r"\bSHFL\b", "RED/ATOMG": r"\b(RED|ATOMG)\b", "SHF": r"\bSHF\b", "LOP3": r"\bLOP3\b",
            "IADD3": r"\bIADD3\b"}


def sass(m):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "k.cubin")
        with open(path, "wb") as f:
            f.write(m.cubin)
        res = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True, check=True).stdout
        return res + subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout


def summarize(text):
    body = [ln for ln in text.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,6}\*/", ln)]
    out = {k: sum(1 for ln in body if re.search(p, ln)) for k, p in PATTERNS.items()}
    out["instructions"] = len(body)
    for key, pat in (("regs", r"REG:(\d+)"), ("stack", r"STACK:(\d+)"), ("local", r"LOCAL:(\d+)")):
        v = re.search(pat, text)
        out[key] = int(v.group(1)) if v else None
    return out


def excerpt(text, keys=("LDG.E.128", "STG.E.128", "BAR.SYNC", "USETMAXREG", "ATOMS", "SHFL"), n=40):
    lines = [ln for ln in text.splitlines() if re.match(r"\s+/\*[0-9a-f]{4,6}\*/", ln)]
    pick = [ln for ln in lines if any(re.search(PATTERNS[k], ln) for k in keys)]
    return "\n".join(pick[:n])


def main():
    detail = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_detail.json")))
    out_dir = os.path.join(ROOT, "profiles")
    summary, blobs = {}, []
    for r in detail["results"]:
        a, b = r["pair"].split("+")
        wa, wb = P.MEMBERS[a].sizes["full"](), P.MEMBERS[b].sizes["full"]()
        img = hf.Image(wa.image).merge(hf.Image(wb.image))
        sa, sb = P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)
        m = hf.Module.from_config(sa, sb, r, specialize=img)
        text = sass(m)
        summary[r["pair"]] = {"config": [r["grid"], r["d1"], r["d2"], r["reg_cap"], r.get("split_grid")],
                              **summarize(text)}
        blobs.append(f"==== fused {r['pair']} (grid {r['grid']}, {r['d1']}/{r['d2']}, cap {r['reg_cap']}) "
                     f"{m.entry} ====\n" + excerpt(text))
    for c in (detail.get("crypto") or {}).get("pairs", []):
        if c["pair"] == "upsample+blake256" or "d1" not in c:
            continue
        a, b = c["pair"].split("+")
        wa = CR.workload(a, 1 << 20, c["grid"], target=1 << 12)
        wb = CR.workload(b, 1 << 20, c["grid"], target=1 << 12, npages=33554393)
        img = hf.Image(wa.image).merge(hf.Image(wb.image))
        fa, fb = c.get("forms") or (a, b)  # the member forms the bench fused
        sa = open(os.path.join(P.KERNELS, "b200", fa + ".mk")).read()
        sb = open(os.path.join(P.KERNELS, "b200", fb + ".mk")).read()
        if c.get("interval_regs"):
            m = hf.Module.fused_regs(sa, sb, c["d1"], c["d2"], *c["interval_regs"], grid=c["grid"], specialize=img)
        else:
            m = hf.Module.fused(sa, sb, c["d1"], c["d2"], regcap=c["reg_cap"] or "off", grid=c["grid"], specialize=img)
        text = sass(m)
        summary[c["pair"]] = {"config": [c["grid"], c["d1"], c["d2"], c["reg_cap"], c.get("interval_regs")],
                              **summarize(text)}
        blobs.append(f"==== fused {c['pair']} (grid {c['grid']}, {c['d1']}/{c['d2']}, cap {c['reg_cap']}, budgets "
                     f"{c.get('interval_regs')}) {m.entry} ====\n"
                     + excerpt(text, keys=("USETMAXREG", "LDG.E.128", "BAR.SYNC", "SHFL"), n=24))
    with open(os.path.join(out_dir, "r02_sass_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    with open(os.path.join(out_dir, "r02_sass_excerpts.txt"), "w") as f:
        f.write("# cuobjdump -sass of the benched sm_100a kernels (scripts/sass_excerpts.py): lines with\n"
                "# 128-bit global accesses, named barriers, setmaxnreg, shared atomics, shuffles\n\n")
        f.write("\n\n".join(blobs) + "\n")
    for k, v in summary.items():
        print(k, {x: v[x] for x in ("regs", "stack", "local", "LDG.E.128", "STG.E.128", "LDL", "STL", "USETMAXREG", "BAR.SYNC")})


if __name__ == "__main__":
    main()
