"""Workload definitions of the DL members (paper_2007_01277_b200/pairs.py): the batch-scaled
forms used by bench.py's workload-ratio study."""
import pytest

from paper_2007_01277_b200 import pairs


@pytest.mark.parametrize("shape", ["full", "conv3"])
@pytest.mark.parametrize("key", pairs.ORDER)
def test_scaled_member_is_the_batch_scaled_shape(key, shape):
    w1, n1 = pairs.scaled(key, 1.0, shape)
    assert w1.image == pairs.MEMBERS[key].sizes[shape](0).image  # factor 1 = the bench shape
    w2, n2 = pairs.scaled(key, 2.0, shape)
    assert n2 == 2 * n1
    # bytes scale with the batch, up to BN's per-channel constants
    assert abs(w2.bytes - 2 * w1.bytes) <= 2 * 4 * 4096
    wh, nh = pairs.scaled(key, 0.5, shape)
    assert nh * 2 == n1
    assert pairs.scaled(key, 1e-6, shape)[1] == 1  # never empty


def test_scaled_images_carry_the_batch():
    w, n = pairs.scaled("bn", 0.25)
    assert n == 16 and "scalar bn_N int32 16\n" in w.image
    w, n = pairs.scaled("maxpool", 0.5)
    assert f"scalar mp_NC int32 {32 * 64}\n" in w.image
    w, n = pairs.scaled("im2col", 2.0, "conv3")
    assert n == 64 and f"scalar ic_NC int32 {64 * 128}\n" in w.image
