"""Pins the C restatement (oracle/hf_oracle.c) on PyTorch's own operators — the semantics the
paper's DL members come from: max_pool2d with indices (NaN propagation
included), bilinear interpolate with align_corners=False, unfold (im2col), histc, and the
biased batch variance. Together with tests/test_oracle.py (the same functions against the
reference interpreter) this anchors the oracle on both sides."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import oracle


def _x(n, seed, lo=-1.0, hi=1.0):
    return oracle.fill_uniform(n, seed, lo, hi)


@pytest.mark.parametrize("NC,H,W", [(3, 16, 16), (2, 112, 112), (5, 10, 14)])
def test_maxpool_matches_torch_including_nan(NC, H, W):
    x = _x(NC * H * W, 11)
    x[7] = np.nan
    x[NC * H * W // 2] = np.nan
    y, idx = oracle.maxpool(x, NC, H, W)
    ty, ti = F.max_pool2d(torch.from_numpy(x).view(1, NC, H, W), 3, 2, 1, return_indices=True)
    assert np.array_equal(y, ty.reshape(-1).numpy(), equal_nan=True)
    assert np.array_equal(idx, ti.reshape(-1).numpy().astype(np.int32))


@pytest.mark.parametrize("NC,IH,IW", [(3, 8, 8), (4, 28, 28), (2, 14, 6)])
def test_upsample_matches_torch_bilinear(NC, IH, IW):
    x = _x(NC * IH * IW, 12)
    y = oracle.upsample(x, NC, IH, IW)
    ty = F.interpolate(torch.from_numpy(x).view(1, NC, IH, IW), scale_factor=2, mode="bilinear",
                       align_corners=False).reshape(-1).numpy()
    # PyTorch's CPU kernel evaluates the same weights with its own operation order: 1 ulp apart
    assert np.max(np.abs(y - ty)) <= 2.4e-7


@pytest.mark.parametrize("NC,H,W", [(3, 8, 8), (2, 56, 56)])
def test_im2col_matches_torch_unfold(NC, H, W):
    x = _x(NC * H * W, 13)
    col = oracle.im2col(x, NC, H, W)
    t = F.unfold(torch.from_numpy(x).view(1, NC, H, W), 3, padding=1).reshape(-1).numpy()
    assert np.array_equal(col, t)


@pytest.mark.parametrize("n", [64, 100003, 1 << 20])
def test_hist_matches_torch_histc(n):
    x = _x(n, 14, -5.0, 5.0)
    x[:3] = [4.0, -4.0, 0.0]  # both range ends and an interior bin edge
    got = oracle.hist(x)
    want = torch.histc(torch.from_numpy(x), bins=64, min=-4, max=4).numpy().astype(np.int32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("N,C,HW", [(2, 8, 3136), (4, 3, 17)])
def test_bn_stats_match_torch_biased_var(N, C, HW):
    x = _x(N * C * HW, 15, -1.0, 3.0)
    mean, var = oracle.bn_stats(x, N, C, HW)
    t = torch.from_numpy(x).double().view(N, C, HW)
    tm = t.mean(dim=(0, 2)).numpy()
    tv = t.var(dim=(0, 2), unbiased=False).numpy()
    assert np.allclose(mean, tm, rtol=0, atol=1e-12) and np.allclose(var, tv, rtol=0, atol=1e-12)
