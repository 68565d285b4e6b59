"""Ethash member: nonces in flight per 8-lane group (HPP 4 vs 8; 8 ships),
alone and fused with BLAKE-256 (diagnostic)."""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
K = os.path.join(HERE, "..", "paper_2007_01277_b200", "kernels", "b200")
sys.path.insert(0, os.path.join(HERE, "..", "paper_2007_01277_b200", "kernels"))
import gen_crypto  # noqa: E402

srcs = {}
for hpp in (4, 8):
    gen_crypto.HPP = hpp
    srcs[f"hpp{hpp}"] = gen_crypto.gen_ethash()
bl = open(os.path.join(K, "blake256.mk")).read()
G = 296
we = CR.workload("ethash", 1 << 20, G, npages=1 << 25)
wb = CR.workload("blake256", 1 << 24, G)
img = hf.Image(we.image).merge(hf.Image(wb.image)).upload()
kb = hf.Module.kernel(bl, grid=G, specialize=img)
tb = hf.time("single", kb, None, img, G, warmup=1, reps=5)["iqm_us"]
print(json.dumps({"blake256_us": round(tb, 1)}), flush=True)
for name, src in srcs.items():
    for g in (296, 592):
        m = hf.Module.kernel(src, grid=g, specialize=img)
        t = hf.time("single", m, None, img, g, warmup=1, reps=5)["iqm_us"]
        print(json.dumps({"variant": name, "grid": g, "us": round(t, 1), "regs": m.info.regs,
                          "bps": m.info.blocks_per_sm, "dag_gbs": round((1 << 20) * 8192 / (t * 1e3), 1)}), flush=True)
    ke = hf.Module.kernel(src, grid=G, specialize=img)
    two = hf.time("two_stream", kb, ke, img, G, G, warmup=1, reps=5)["iqm_us"]
    seq = hf.time("sequential", kb, ke, img, G, G, warmup=1, reps=5)["iqm_us"]
    print(json.dumps({"variant": name, "two_stream": round(two, 1), "seq": round(seq, 1)}), flush=True)
    for d1, cap in ((512, None), (512, 64), (768, None), (256, None), (512, 128)):
        try:
            m = hf.Module.fused(bl, src, d1, 1024 - d1, regcap=cap or "off", grid=G, specialize=img)
            t = hf.time("single", m, None, img, G, warmup=1, reps=5)["iqm_us"]
            print(json.dumps({"variant": name, "fused_d1": d1, "cap": cap, "us": round(t, 1), "regs": m.info.regs,
                              "bps": m.info.blocks_per_sm}), flush=True)
        except hf.HFuseError as e:
            print(json.dumps({"variant": name, "fused_d1": d1, "cap": cap, "error": str(e)[:100]}), flush=True)
