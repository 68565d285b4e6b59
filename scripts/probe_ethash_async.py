"""Probe: Ethash DAG reads through registers (vload, LDG.128) vs 16-byte cp.async copies into a
shared ring (MK+ async_copy), at HPP pages in flight per lane; alone and fused with BLAKE-256
under per-interval budgets. Graph protocol. JSON lines on stdout."""
import importlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402


def gen(load, hpp):
    os.environ["HF_ETHASH_LOAD"], os.environ["HF_ETHASH_HPP"] = load, str(hpp)
    from paper_2007_01277_b200.kernels import gen_crypto
    return importlib.reload(gen_crypto).gen_ethash()


N = 1 << 20
wb = CR.workload("ethash", N, 1184, target=1 << 12, npages=33554393)
wa = CR.workload("blake256", 1 << 24, 1184, target=1 << 12)
img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
blake = open(os.path.join(P.KERNELS, "b200", "blake256.mk")).read()
for load, hpp in (("ldg", 8), ("async", 8), ("ldg", 4), ("async", 4)):
    src = gen(load, hpp)
    for cap in (None, 96):
        try:
            k = hf.Module.kernel(src, grid=592, regcap=cap, specialize=img)
        except hf.HFuseError as e:
            print(json.dumps({"load": load, "hpp": hpp, "cap": cap, "err": str(e)[:200]}), flush=True)
            continue
        for g in (296, 592, 1184):
            t = hf.time_graph("single", k, None, img, g, 0, reps=3, samples=3)["mean_us"]
            print(json.dumps({"load": load, "hpp": hpp, "cap": cap, "grid": g, "regs": k.info.regs,
                              "bps": k.info.blocks_per_sm, "us": round(t, 1),
                              "dag_gbs": round(N * 8192 / (t * 1e3), 1)}), flush=True)
    for d2 in (384, 512):
        for regs in ((24, 104), (32, 96), (32, 128)):
            try:
                m = hf.Module.fused_regs(blake, src, 512, d2, *regs, grid=592, specialize=img)
            except hf.HFuseError as e:
                print(json.dumps({"load": load, "hpp": hpp, "fused": [512, d2, regs], "err": str(e)[:120]}), flush=True)
                continue
            for g in (296, 592):
                t = hf.time_graph("single", m, None, img, g, 0, reps=3, samples=3)["mean_us"]
                print(json.dumps({"load": load, "hpp": hpp, "fused": [512, d2, regs], "grid": g,
                                  "us": round(t, 1)}), flush=True)
