"""BLAKE2b 64-bit add carry forms (kernels/gen_crypto.py HF_ADD64): ltu (compare + select, the
select on the FMA pipe), addc (add.cc/addc: fewer instructions, all ALU), mix -- alone and fused
with SHA-256d (both ALU-pipe bound), against sequential / two-stream."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

G = 296
here = os.path.dirname(os.path.abspath(__file__))
sha = open(os.path.join(P.KERNELS, "b200", "sha256d.mk")).read()


def generated(form):
    """The BLAKE2b member regenerated with HF_ADD64=form (kernels/gen_crypto.py)."""
    import importlib
    os.environ["HF_ADD64"] = form
    from paper_2007_01277_b200.kernels import gen_crypto
    return importlib.reload(gen_crypto).gen_blake2b()


forms = {"ltu": open(os.path.join(P.KERNELS, "b200", "blake2b.mk")).read(),
         "addc": generated("addc"), "mix": generated("mix")}
wa = CR.workload("sha256d", 1 << 24, G, target=1 << 12)
wb = CR.workload("blake2b", 1 << 23, G, target=1 << 12)
img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
ks = hf.Module.kernel(sha, grid=G, specialize=img)
out = {"sha256d_us": hf.time("single", ks, None, img, G, warmup=2, reps=7)["iqm_us"]}
for name, src in forms.items():
    kb = hf.Module.kernel(src, grid=G, specialize=img)
    r = {"regs": kb.info.regs, "alone": hf.time("single", kb, None, img, G, warmup=2, reps=7)["iqm_us"],
         "seq": hf.time("sequential", ks, kb, img, G, G, warmup=2, reps=7)["iqm_us"],
         "two": hf.time("two_stream", ks, kb, img, G, G, warmup=2, reps=7)["iqm_us"], "fused": {}}
    for label, mk in (("uncapped", lambda: hf.Module.fused(sha, src, 512, 512, grid=G, specialize=img)),
                      ("budgets_40_56", lambda: hf.Module.fused_regs(sha, src, 512, 512, 40, 56, grid=G, specialize=img)),
                      ("budgets_48_64", lambda: hf.Module.fused_regs(sha, src, 512, 512, 48, 64, grid=G, specialize=img))):
        try:
            m = mk()
            r["fused"][label] = round(hf.time("single", m, None, img, G, warmup=2, reps=7)["iqm_us"], 1)
        except hf.HFuseError as e:
            r["fused"][label] = str(e)[:80]
    out[name] = r
    print(name, json.dumps(r), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_blake2b_carry.json", "w"), indent=1)
