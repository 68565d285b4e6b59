"""The graph-timed protocol (hf_time_graph) and dynamic interval scheduling (hf_build_fused_opts
vgrid) on the device."""
import numpy as np
import pytest

from oracle import check as CK
from paper_2007_01277_b200 import pairs as P


def _pair(hf, a, b, size="parity"):
    wa, wb = P.MEMBERS[a].sizes[size](), P.MEMBERS[b].sizes[size]()
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    return wa, wb, img, P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)


@pytest.mark.gpu
def test_time_graph_is_consistent(gpu):
    hf = gpu
    wa, wb, img, sa, sb = _pair(hf, "hist", "upsample", "full")
    ka, kb = hf.Module.kernel(sa, grid=592, specialize=img), hf.Module.kernel(sb, grid=592, specialize=img)
    one = hf.time_graph("single", ka, None, img, 592, 0, reps=10, samples=5)
    two = hf.time_graph("single", kb, None, img, 592, 0, reps=10, samples=5)
    seq = hf.time_graph("sequential", ka, kb, img, 592, 592, reps=10, samples=5)
    par = hf.time_graph("two_stream", ka, kb, img, 592, 592, reps=10, samples=5)
    for t in (one, two, seq, par):
        assert t["samples"] == 5 and t["reps"] == 10
        assert 0 < t["min_us"] <= t["median_us"] <= t["max_us"] and t["ci95_us"] >= 0
    # back to back, the pair costs about the sum of its members; concurrently, no more than that
    assert 0.9 * (one["mean_us"] + two["mean_us"]) <= seq["mean_us"] <= 1.15 * (one["mean_us"] + two["mean_us"])
    assert par["mean_us"] <= 1.05 * seq["mean_us"]


@pytest.mark.gpu
@pytest.mark.parametrize("a,b,vgrid", [("bn", "hist", (8, 37)), ("bn", "im2col", (8, 5)),
                                       ("im2col", "upsample", (7, 3)), ("maxpool", "upsample", (2, 9)),
                                       ("hist", "maxpool", (13, 4))])
def test_dynamic_interval_scheduling_matches_oracle(gpu, a, b, vgrid):
    """Block-level (BN, Hist: barriers + shared memory) and warp-level (Im2Col, MaxPool,
    Upsample) virtual-block queues give the oracle's outputs, over several launches (the queues
    reset themselves) and grids smaller and larger than the virtual grids."""
    hf = gpu
    wa, wb, img, sa, sb = _pair(hf, a, b)
    for grid in (3, 40):
        m = hf.Module.fused_opts(sa, sb, 256, 256, vgrid=vgrid, grid=grid, specialize=img)
        assert "hf_sched" in m.source
        for launch in range(3):
            # a fresh image per launch (re-uploading a downloaded image re-sends its contents,
            # which would accumulate the histogram)
            img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
            m.run(img, grid)
            img.download()
            for key, w in ((a, wa), (b, wb)):
                r = CK.check_member(key, img.array, CK.member_expected(key, w.image))
                assert r["ok"], (grid, launch, key, r)


@pytest.mark.gpu
@pytest.mark.parametrize("a,b,d1,d2,b1", [("bn", "im2col", 768, 256, 8), ("bn", "upsample", 896, 128, 8),
                                          ("hist", "maxpool", 512, 512, 5), ("im2col", "upsample", 768, 256, 3)])
def test_heterogeneous_grid_matches_oracle(gpu, a, b, d1, d2, b1):
    """split_grid: blocks below B1 fused, blocks above member 2 only (d0/d2 sub-blocks); the
    outputs equal the oracle for grids below, at and above B1."""
    hf = gpu
    wa, wb = P.MEMBERS[a].sizes["parity"](), P.MEMBERS[b].sizes["parity"]()
    sa, sb = P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem)
    img = hf.Image(wa.image).merge(hf.Image(wb.image))
    m = hf.Module.fused_opts(sa, sb, d1, d2, split_grid=b1, grid=b1, specialize=img)
    assert "hf_vg2" in m.source
    for grid in (max(1, b1 - 2), b1, b1 + 7):
        img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
        m.run(img, grid)
        img.download()
        for key, w in ((a, wa), (b, wb)):
            r = CK.check_member(key, img.array, CK.member_expected(key, w.image))
            assert r["ok"], (grid, key, r)
