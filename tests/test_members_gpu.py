"""Device parity of the DL members and the ten fused DL pairs.

Small sizes: bit-exact against the reference interpreter (tests/golden/members.json,
made by tests/golden/make_members.py from oracle/_ref). Full sizes (the bench workload):
against the C restatement oracle/hf_oracle.c — exact for Hist, MaxPool (values and
indices), Upsample and Im2Col; BatchNorm mean/var within 1e-5 * max(1, |x|) of the fp64
two-pass statistics (the tolerance form of test_fuser.cpp:459).
"""
import numpy as np
import pytest

from conftest import golden
from oracle import oracle
from paper_2007_01277_b200 import pairs

G = golden("members.json")
GRID = G["grid"]
BN_TOL = 1e-5


def from_bits(v):
    return np.array(v, np.uint32)


def outputs(img, names):
    return {n: img.array(n).view(np.uint32) for n in names}


def image(hf, *keys, size="parity"):
    img = hf.Image(pairs.MEMBERS[keys[0]].sizes[size](0).image)
    for k in keys[1:]:
        img.merge(hf.Image(pairs.MEMBERS[k].sizes[size](0).image))
    return img


@pytest.mark.gpu
@pytest.mark.parametrize("form", ["ref", "b200"])
@pytest.mark.parametrize("size", ["tiny", "parity"])
@pytest.mark.parametrize("key", list(pairs.MEMBERS))
def test_member_matches_interpreter(gpu, key, size, form):
    hf = gpu
    mod = hf.Module.kernel(pairs.source(form, pairs.MEMBERS[key].stem), grid=GRID)
    img = image(hf, key, size=size).upload()
    mod.run(img, GRID)
    img.download()
    assert img.digest_hex() == G["members"][key][size][form]["digest"]


@pytest.mark.gpu
@pytest.mark.parametrize("d1", G["splits"])
@pytest.mark.parametrize("pair", [f"{a}+{b}" for a, b in pairs.PAIRS])
def test_fused_pair_matches_sequential_interpreter(gpu, pair, d1):
    hf = gpu
    a, b = pair.split("+")
    sa = pairs.source("b200", pairs.MEMBERS[a].stem)
    sb = pairs.source("b200", pairs.MEMBERS[b].stem)
    mod = hf.Module.fused(sa, sb, d1, 1024 - d1, grid=GRID)
    img = image(hf, a, b).upload()
    mod.run(img, GRID)
    img.download()
    assert img.digest_hex() == G["pairs"][pair][str(d1)]["digest"]


def test_b200_forms_agree_with_naive_forms():
    """B200 member outputs vs the naive (reference-form) outputs, both from the reference
    interpreter: exact except BatchNorm (different summation order, tolerance)."""
    for key, sizes in G["members"].items():
        for size, row in sizes.items():
            for name, ref_bits in row["ref"]["outputs"].items():
                got = from_bits(row["b200"]["outputs"][name])
                want = from_bits(ref_bits)
                if key == "bn":
                    g, w = got.view(np.float32), want.view(np.float32)
                    assert np.all(np.abs(g - w) <= BN_TOL * np.maximum(1.0, np.abs(w))), (key, size)
                else:
                    assert np.array_equal(got, want), (key, size, name)


def check_full(key, img, oracle_inputs=None):
    """Compare one member's full-size device outputs with the C restatement."""
    w = pairs.MEMBERS[key].sizes["full"](0)
    arrays, scalars = oracle.parse_image(w.image)
    if key == "bn":
        mean, var = oracle.bn_stats(arrays["bn_x"], int(scalars["bn_N"]), int(scalars["bn_C"]), int(scalars["bn_HW"]))
        got = img.array("bn_stats").reshape(-1, 2).astype(np.float64)
        for g, want in ((got[:, 0], mean), (got[:, 1], var)):
            assert np.all(np.abs(g - want) <= BN_TOL * np.maximum(1.0, np.abs(want)))
    elif key == "hist":
        want = oracle.hist(arrays["hi_x"])
        assert np.array_equal(img.array("hi_out"), want)
        assert int(want.sum()) == int(scalars["hi_n"])  # uniform on [-4, 4]: every sample counted
    elif key == "maxpool":
        y, idx = oracle.maxpool(arrays["mp_x"], int(scalars["mp_NC"]), int(scalars["mp_H"]), int(scalars["mp_W"]))
        assert np.array_equal(img.array("mp_y").view(np.uint32), y.view(np.uint32))
        assert np.array_equal(img.array("mp_idx"), idx)
    elif key == "upsample":
        y = oracle.upsample(arrays["us_x"], int(scalars["us_NC"]), int(scalars["us_IH"]), int(scalars["us_IW"]))
        assert np.array_equal(img.array("us_y").view(np.uint32), y.view(np.uint32))
    elif key == "im2col":
        col = oracle.im2col(arrays["ic_x"], int(scalars["ic_NC"]), int(scalars["ic_H"]), int(scalars["ic_W"]))
        assert np.array_equal(img.array("ic_col").view(np.uint32), col.view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("pair", [f"{a}+{b}" for a, b in pairs.PAIRS])
def test_full_size_fused_pair_matches_c_oracle(gpu, pair):
    """The bench workload itself: fused (d1 = 512) at the C1/C2 sizes, grid 296."""
    hf = gpu
    a, b = pair.split("+")
    sa = pairs.source("b200", pairs.MEMBERS[a].stem)
    sb = pairs.source("b200", pairs.MEMBERS[b].stem)
    mod = hf.Module.fused(sa, sb, 512, 512, grid=296)
    img = image(hf, a, b, size="full").upload()
    mod.run(img, 296)
    img.download()
    check_full(a, img)
    check_full(b, img)


@pytest.mark.gpu
def test_vertical_fusion_matches_sequential_interpreter(gpu):
    """VFuse of two thread-count-independent members reproduces the sequential digest."""
    hf = gpu
    sa, sb = pairs.source("b200", "histogram"), pairs.source("b200", "maxpool")
    img = image(hf, "hist", "maxpool").upload()
    hf.Module.vertical(sa, sb, grid=GRID, specialize=img).run(img, GRID)
    img.download()
    assert img.digest_hex() == G["pairs"]["hist+maxpool"]["512"]["digest"]


@pytest.mark.gpu
def test_naive_goto_fusion_runs(gpu):
    """The reference's goto text of the naive forms compiles and runs on sm_100a (timing
    baseline); on these inputs it also computes the right histogram."""
    hf = gpu
    m = hf.Module.naive(pairs.source("ref", "batchnorm"), pairs.source("ref", "histogram"), 512, 512, grid=GRID)
    img = image(hf, "bn", "hist").upload()
    m.run(img, GRID)
    img.download()
    want = G["members"]["hist"]["parity"]["ref"]["outputs"]["hi_out"]
    assert [int(x) for x in img.array("hi_out").view(np.uint32)] == want


@pytest.mark.gpu
@pytest.mark.parametrize("grid", [3, 7, 16, 37])
@pytest.mark.parametrize("size", ["tiny", "parity"])
def test_grid_balanced_bn_matches_interpreter(gpu, size, grid):
    """The grid-balanced BatchNorm variant (cross-block partials + arrival counters) equals the
    interpreter bit for bit at grids where channels straddle blocks or blocks own nothing;
    a second launch on the same image gives the same digest (counters were cleared)."""
    hf = gpu
    mod = hf.Module.kernel(pairs.source("b200", "batchnorm_balanced"), grid=grid)
    img = image(hf, "bn", size=size).upload()
    for _ in range(2):
        mod.run(img, grid)
        img.download()
        assert img.digest_hex() == G["bn_grids"][size][str(grid)]


@pytest.mark.gpu
@pytest.mark.parametrize("grid", [296, 1184, 2368])
def test_full_size_bn_any_grid(gpu, grid):
    """Both BatchNorm forms at the bench's grids vs fp64 statistics, three launches back to back."""
    hf = gpu
    img = image(hf, "bn", size="full").upload()
    mod = hf.Module.kernel(pairs.source("b200", "batchnorm_balanced"), grid=grid, specialize=img)
    for _ in range(3):
        mod.run(img, grid)
    img.download()
    check_full("bn", img)
    assert int(np.abs(img.array("bn_cnt")).max()) == 0
    mod = hf.Module.kernel(pairs.source("b200", "batchnorm"), grid=grid, specialize=img)
    img.upload()
    for _ in range(3):
        mod.run(img, grid)
    img.download()
    check_full("bn", img)


@pytest.mark.gpu
@pytest.mark.parametrize("grid", [3, 7, 16, 37])
@pytest.mark.parametrize("size,dims", [("tiny", (1, 3, 16)), ("parity", (2, 8, 56 * 56))])
def test_warp_handoff_bn_matches_interpreter(gpu, size, dims, grid):
    """The warp-level hand-off BatchNorm (red.release.gpu counters, ld.relaxed re-read, fenced
    last-warp merge) equals the interpreter bit for bit, and twice in a row (counters cleared)."""
    hf = gpu
    mod = hf.Module.kernel(pairs.source("b200", "batchnorm_warp"), grid=grid)
    img = hf.Image(pairs._bn(*dims, slots=256)(0).image).upload()
    for _ in range(2):
        mod.run(img, grid)
        img.download()
        assert img.digest_hex() == G["bn_warp_grids"][size][str(grid)]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 3, 1001, 4099])
@pytest.mark.parametrize("grid", [4, 37])
def test_hist_ragged_lengths(gpu, n, grid):
    """n % 4 != 0 (and n < 4): the B200 Hist bins the trailing values too, equal to the
    reference form on the interpreter (fixture) and to the C restatement."""
    hf = gpu
    w = pairs._hist(n, -4.5, 4.5)(0)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(pairs.source("b200", "histogram"), grid=grid).run(img, grid)
    img.download()
    assert img.digest_hex() == G["hist_ragged"][f"{n}/{grid}"]
    arrays, _ = oracle.parse_image(w.image)
    assert (img.array("hi_out") == oracle.hist(arrays["hi_x"])).all()


@pytest.mark.gpu
def test_requires_violation_fails_loudly_on_device(gpu):
    """A BatchNorm launch with HW % 4 != 0 is refused at bind time (InvalidArgument), not run
    into wrong statistics; the same kernel launches once the precondition holds."""
    hf = gpu
    bad = hf.Image(pairs._bn(2, 3, 18)(0).image).upload()
    mod = hf.Module.kernel(pairs.source("b200", "batchnorm"), grid=4)
    with pytest.raises(hf.HFuseError) as e:
        mod.run(bad, 4)
    assert e.value.name == "InvalidArgument" and "bn_HW % 4 == 0" in str(e.value) and "bn_HW = 18" in str(e.value)
    good = hf.Image(pairs._bn(2, 3, 16)(0).image).upload()
    mod.run(good, 4)


@pytest.mark.gpu
def test_preexisting_named_barriers_synchronize_their_own_interval(gpu):
    """SURVEY App. C on the device: both constituents hand data across bar_sync(1, 64) in shared
    memory; fused, each gets its own barrier id (the reference would let them share id 1), so
    every thread reads its neighbour's value, over 64 blocks and 20 launches."""
    hf = gpu
    k1 = ("kernel a(int x[]) dims (64, 1, 1) {\n  shared int s[64];\n  int t = threadIdx.x;\n"
          "  s[t] = t * 3 + blockIdx.x;\n  bar_sync(1, 64);\n  x[blockIdx.x * 64 + t] = s[(t + 1) % 64];\n}\n")
    k2 = ("kernel b(int y[]) dims (64, 1, 1) {\n  shared int r[64];\n  int t = threadIdx.x;\n"
          "  r[t] = t * 7 - blockIdx.x;\n  bar_sync(1, 64);\n  y[blockIdx.x * 64 + t] = r[(t + 63) % 64];\n}\n")
    m = hf.Module.fused(k1, k2, 64, 64, grid=64)
    ids = {(b.owner, b.original): b.id for b in m.barriers}
    assert ids[(1, 1)] != ids[(2, 1)]
    img = hf.Image("array x int32 4096 zero\narray y int32 4096 zero\n").upload()
    t = np.arange(64)
    want_x = np.concatenate([((t + 1) % 64) * 3 + b for b in range(64)])
    want_y = np.concatenate([((t + 63) % 64) * 7 - b for b in range(64)])
    for _ in range(20):
        m.run(img, 64)
        img.download()
        assert np.array_equal(img.array("x"), want_x) and np.array_equal(img.array("y"), want_y)


@pytest.mark.gpu
def test_c1_full_size_equals_reference_interpreter(gpu):
    """BASELINE configs[0] on the device: the fused BatchNorm-stats + Hist kernel over the
    64x256x56x56 tensors (2 x 205.5 MB) reproduces the reference interpreter's sequential run of
    the same (lowered) member forms bit for bit (tests/golden/make_c1.py, ~9 s of CPU)."""
    hf = gpu
    ref = golden("c1_full.json")
    img = hf.Image(pairs.MEMBERS["bn"].sizes["full"](0).image).merge(
        hf.Image(pairs.MEMBERS["hist"].sizes["full"](0).image)).upload()
    m = hf.Module.fused(pairs.source("b200", "batchnorm"), pairs.source("b200", "histogram"), ref["d1"], ref["d2"],
                        grid=ref["grid"], specialize=img)
    m.run(img, ref["grid"])
    img.download()
    assert img.digest_hex() == ref["digest"]


FULL = golden("full_pairs.json")


@pytest.mark.gpu
@pytest.mark.parametrize("pair", list(FULL))
def test_full_size_pair_equals_reference_interpreter(gpu, pair):
    """Every DL pair at its C2 size (hundreds of MB): the fused kernel equals the reference
    interpreter's sequential run of the lowered members at the same split and grid, bit for bit."""
    hf = gpu
    ref = FULL[pair]
    a, b = pair.split("+")
    img = hf.Image(pairs.MEMBERS[a].sizes["full"](0).image).merge(
        hf.Image(pairs.MEMBERS[b].sizes["full"](0).image)).upload()
    m = hf.Module.fused(pairs.source("b200", pairs.MEMBERS[a].stem), pairs.source("b200", pairs.MEMBERS[b].stem),
                        ref["d1"], ref["d2"], grid=ref["grid"], specialize=img)
    m.run(img, ref["grid"])
    img.download()
    assert img.digest_hex() == ref["digest"]


@pytest.mark.gpu
def test_overlapped_launches_of_independent_pairs_match_serial(gpu):
    """Programmatic dependent launch (HF_LAUNCH_OVERLAP) of the ten fused pairs back to back on one
    stream -- each may start while its predecessor drains -- leaves the image exactly as ordinary
    serialized launches do (the pairs share only identical outputs and commutative atomics)."""
    hf = gpu
    mods = [hf.Module.fused(pairs.source("b200", pairs.MEMBERS[a].stem), pairs.source("b200", pairs.MEMBERS[b].stem),
                            512, 512, grid=GRID) for a, b in pairs.PAIRS]
    digests = []
    for overlap in (False, True):
        img = image(hf, *pairs.ORDER).upload()
        for _ in range(3):
            for m in mods:
                m.run(img, GRID, overlap=overlap)
        img.download()
        digests.append(img.digest_hex())
    assert digests[0] == digests[1]
