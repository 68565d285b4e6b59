"""CPU checks of bench.py's host logic: search-space helpers, the reference arm's job plan (the
whole C2 workload as exact batch shards of the naive members, no product library involved)."""
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402


def test_fused_grids_are_waves_of_resident_ctas():
    assert bench.fused_grids(1024, [1, 2, 16]) == [296, 592, 4736]
    assert bench.fused_grids(640, [1, 8]) == [444, 3552]
    assert bench.fused_grids(512, [1]) == [592]


def test_split_eligibility_and_natural_grids():
    ok = {k: bench.split_member(P.source("b200", P.MEMBERS[k].stem)) for k in P.ORDER}
    assert ok == {"bn": False, "hist": False, "im2col": True, "maxpool": True, "upsample": True}
    assert bench.natural_grid("bn", P.MEMBERS["bn"].sizes["full"]()) == 256
    assert bench.natural_grid("hist", P.MEMBERS["hist"].sizes["full"]()) == 0


def test_reference_arm_runs_the_whole_workload(tmp_path):
    """160 interpreter jobs per step (10 pairs x 16 exact batch shards); shard images are slices
    of the whole-batch tensors and the naive BatchNorm image carries only what it binds."""
    jobs = bench.ref_jobs(P.PAIRS, "full", bench.REF_SHARDS, str(tmp_path))
    assert len(jobs) == 10 * bench.REF_SHARDS
    assert all(j[1] == "seq" and "/ref/" in j[2] and "/ref/" in j[3] for j in jobs)
    img = bench.ref_member_image("bn", "full", 3, 16)
    names = [ln.split()[1] for ln in img.splitlines() if ln]
    assert names == ["bn_x", "bn_stats", "bn_N", "bn_C", "bn_HW"]
    assert "scalar bn_N int32 4" in img
    total = sum(int(bench.ref_member_image("hist", "full", s, 16).split()[3]) for s in range(16))
    assert total == 64 * 256 * 56 * 56


def test_reference_arm_does_not_load_the_product():
    """`from paper_2007_01277_b200 import pairs` must not map libhfuse.so (the package is lazy)."""
    import subprocess
    code = ("import sys; sys.path.insert(0, %r); from paper_2007_01277_b200 import pairs, shard; "
            "import bench; print(any('libhfuse' in l for l in open('/proc/self/maps')))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == "False"


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_crypto_nonce_slices_match_the_bench(world):
    from paper_2007_01277_b200 import shard
    for kind, total in bench.CRYPTO_COUNTS.items():
        sl = [shard.nonce_slice(total, r, world) for r in range(world)]
        assert sum(n for _, n in sl) == total
