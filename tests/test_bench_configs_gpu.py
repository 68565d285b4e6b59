"""Parity at the benched configurations (profiles/r02_bench_detail.json, written by bench.py):
every DL pair's fused kernel at exactly the (d0, split, register cap or budgets, launch grid,
JIT specialization) the bench timed, at the C2 sizes, against the C oracle (bit-exact for Hist,
MaxPool values and indices, Upsample, Im2Col; BN within 1e-5 of fp64). bench.py runs the same
check on every run before it prints its line; this test pins the committed configurations."""
import json
import os

import pytest

from conftest import ROOT
from oracle import check as CK
from paper_2007_01277_b200 import pairs as P

DETAIL = os.path.join(ROOT, "profiles", "r02_bench_detail.json")
CFGS = {r["pair"]: r for r in json.load(open(DETAIL))["results"]} if os.path.exists(DETAIL) else {}


@pytest.mark.gpu
@pytest.mark.parametrize("pair", sorted(CFGS))
def test_benched_fused_kernel_matches_oracle(gpu, pair):
    hf = gpu
    a, b = pair.split("+")
    c = CFGS[pair]
    wa, wb = P.MEMBERS[a].sizes["full"](), P.MEMBERS[b].sizes["full"]()
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    sa, sb = P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)
    m = hf.Module.from_config(sa, sb, c, specialize=img)
    m.run(img, c["grid"])
    img.download()
    for key, w in ((a, wa), (b, wb)):
        r = CK.check_member(key, img.array, CK.member_expected(key, w.image))
        assert r["ok"], (key, r)
