"""Device edge cases of the DL members the seeded workloads never produce (the
members follow PyTorch semantics): NaN, ±inf and signed zeros in the inputs,
Hist's range ends, and two NaNs in one MaxPool window. Each B200 member form alone and fused with a
partner must equal the C restatement (oracle/hf_oracle.c, itself pinned on torch in
tests/test_oracle_torch.py): bit-exact for MaxPool values and indices, Hist bins and Im2Col;
Upsample's interpolated NaNs compared as NaN (x86 keeps an input NaN's payload, the GPU returns
the canonical NaN), every other Upsample word bit-exact."""
import numpy as np
import pytest

from oracle import oracle
from paper_2007_01277_b200 import pairs

SPECIAL = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, -4.0, 4.0, np.nextafter(np.float32(4.0), np.float32(0)),
                    np.nextafter(np.float32(-4.0), np.float32(-5)), 1e-45, -1e-45, 3.4e38], np.float32)
INPUT = {"hist": "hi_x", "maxpool": "mp_x", "upsample": "us_x", "im2col": "ic_x"}


def special_input(key, rng):
    """The member's parity-size input with ~1/8 of its words replaced by special values; MaxPool
    also gets two NaNs in one 3x3 window (the later one in window order must win the index)."""
    arrays, scalars = oracle.parse_image(pairs.MEMBERS[key].sizes["parity"](0).image)
    x = np.asarray(arrays[INPUT[key]], np.float32).copy()
    pos = rng.choice(x.size, size=x.size // 8, replace=False)
    x[pos] = SPECIAL[rng.integers(0, SPECIAL.size, pos.size)]
    if key == "maxpool":
        W = int(scalars["mp_W"])
        x[5 * W + 6] = np.nan   # window (oh 3, ow 3) covers rows 5..7, cols 5..7
        x[7 * W + 7] = -np.nan  # a NaN with the sign bit set, later in window order
    return x, scalars


def check(key, img, x, s):
    if key == "hist":
        assert np.array_equal(img.array("hi_out"), oracle.hist(x))
    elif key == "maxpool":
        y, idx = oracle.maxpool(x, int(s["mp_NC"]), int(s["mp_H"]), int(s["mp_W"]))
        assert np.array_equal(img.array("mp_y").view(np.uint32), y.view(np.uint32))
        assert np.array_equal(img.array("mp_idx"), idx)
    elif key == "upsample":
        y = oracle.upsample(x, int(s["us_NC"]), int(s["us_IH"]), int(s["us_IW"]))
        got = img.array("us_y")
        nan = np.isnan(y)
        assert np.array_equal(np.isnan(got), nan)
        assert np.array_equal(got[~nan].view(np.uint32), y[~nan].view(np.uint32))
    elif key == "im2col":
        col = oracle.im2col(x, int(s["ic_NC"]), int(s["ic_H"]), int(s["ic_W"]))
        assert np.array_equal(img.array("ic_col").view(np.uint32), col.view(np.uint32))


def image(hf, keys, rng):
    img, inputs = None, {}
    for k in keys:
        part = hf.Image(pairs.MEMBERS[k].sizes["parity"](0).image)
        x, s = special_input(k, rng)
        part.set_array(INPUT[k], x.view(np.int32))
        inputs[k] = (x, s)
        img = part if img is None else img.merge(part)
    return img, inputs


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["ref", "b200"])
@pytest.mark.parametrize("key", list(INPUT))
def test_member_special_values(gpu, key, form):
    hf = gpu
    img, inputs = image(hf, [key], np.random.default_rng(11))
    img.upload()
    hf.Module.kernel(pairs.source(form, pairs.MEMBERS[key].stem), grid=7).run(img, 7)
    img.download()
    check(key, img, *inputs[key])


@pytest.mark.gpu
@pytest.mark.parametrize("pair", ["hist+maxpool", "maxpool+upsample", "im2col+upsample", "hist+im2col"])
@pytest.mark.parametrize("d1", [256, 768])
def test_fused_pair_special_values(gpu, pair, d1):
    hf = gpu
    a, b = pair.split("+")
    img, inputs = image(hf, [a, b], np.random.default_rng(d1))
    img.upload()
    mod = hf.Module.fused(pairs.source("b200", pairs.MEMBERS[a].stem), pairs.source("b200", pairs.MEMBERS[b].stem),
                          d1, 1024 - d1, grid=5)
    mod.run(img, 5)
    img.download()
    check(a, img, *inputs[a])
    check(b, img, *inputs[b])
