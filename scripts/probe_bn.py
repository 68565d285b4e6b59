"""Time BatchNorm variants (hand-off pieces removed) at several grids. Diagnostic only."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

base = P.source("b200", "batchnorm_balanced")
start = base.index("        fence();\n        atomic_add")
end = base.index("          bn_cnt[c] = 0;\n        }\n") + len("          bn_cnt[c] = 0;\n        }\n")
variants = {
    "full": base,
    "no_handoff": base[:start] + base[end:],
    "fence_atomic_only": base[:start] + "        fence();\n        atomic_add(bn_cnt[c], 1);\n" + base[end:],
    "no_fence": base.replace("fence();", ""),
    "full_nocap": base.replace(" regcap=32", ""),
    "block_per_channel": P.source("b200", "batchnorm"),
}
img = P.MEMBERS["bn"].sizes["full"](0)
im = hf.Image(img.image).upload()
for name, src in variants.items():
    for g in (148, 296, 592, 1184, 2368):
        m = hf.Module.kernel(src, grid=g, specialize=im)
        t = hf.time("single", m, None, im, g, warmup=2, reps=10)["iqm_us"]
        print(json.dumps({"variant": name, "grid": g, "us": round(t, 2), "regs": m.info.regs}), flush=True)
