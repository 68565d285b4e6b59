"""Pins the oracle: the C restatement (hf_oracle.c) and libhfuse's host image code against
the reference's own outputs (tests/golden, made from oracle/_ref)."""
import numpy as np
import pytest

from conftest import STEMS, golden
from oracle import oracle

D = golden("corpus_digests.json")
M = golden("members.json")


@pytest.mark.parametrize("stem", STEMS)
def test_seeded_images_match_reference_generator(hf, corpus, stem):
    for seed, want in D["images"][stem].items():
        s = None if seed == "None" else int(seed)
        arrays, scalars = oracle.parse_image(corpus["images"][stem], s)
        assert f"{oracle.digest(arrays, scalars):016x}" == want
        assert hf.Image(corpus["images"][stem], s).materialize().digest_hex() == want


def member_inputs(key, size):
    from paper_2007_01277_b200 import pairs
    arrays, scalars = oracle.parse_image(pairs.MEMBERS[key].sizes[size](0).image)
    return arrays, {k: int(v) for k, v in scalars.items()}


@pytest.mark.parametrize("size", ["tiny", "parity"])
def test_c_restatement_matches_reference_interpreter(size):
    ref = {k: {n: np.array(v, np.uint32) for n, v in M["members"][k][size]["ref"]["outputs"].items()}
           for k in M["members"]}
    a, s = member_inputs("hist", size)
    assert np.array_equal(oracle.hist(a["hi_x"]), ref["hist"]["hi_out"].view(np.int32))
    a, s = member_inputs("maxpool", size)
    y, idx = oracle.maxpool(a["mp_x"], s["mp_NC"], s["mp_H"], s["mp_W"])
    assert np.array_equal(y.view(np.uint32), ref["maxpool"]["mp_y"])
    assert np.array_equal(idx, ref["maxpool"]["mp_idx"].view(np.int32))
    a, s = member_inputs("upsample", size)
    y = oracle.upsample(a["us_x"], s["us_NC"], s["us_IH"], s["us_IW"])
    assert np.array_equal(y.view(np.uint32), ref["upsample"]["us_y"])
    a, s = member_inputs("im2col", size)
    col = oracle.im2col(a["ic_x"], s["ic_NC"], s["ic_H"], s["ic_W"])
    assert np.array_equal(col.view(np.uint32), ref["im2col"]["ic_col"])
    a, s = member_inputs("bn", size)
    mean, var = oracle.bn_stats(a["bn_x"], s["bn_N"], s["bn_C"], s["bn_HW"])
    got = ref["bn"]["bn_stats"].view(np.float32).reshape(-1, 2).astype(np.float64)
    assert np.all(np.abs(got[:, 0] - mean) <= 1e-5 * np.maximum(1, np.abs(mean)))
    assert np.all(np.abs(got[:, 1] - var) <= 1e-5 * np.maximum(1, np.abs(var)))
