"""Machine model (machine.cpp:236-289) against the reference and the C restatement."""
import pytest

from conftest import golden
from oracle import oracle

D = golden("corpus_digests.json")


@pytest.mark.parametrize("case", sorted(D["register_bound"]))
def test_register_bound_matches_reference(hf, case):
    r1, t1, r2, t2, sh = map(int, case.split(","))
    want = D["register_bound"][case]
    assert hf.register_bound(r1, t1, r2, t2, sh) == want
    assert oracle.register_bound(r1, t1, r2, t2, sh) == want


@pytest.mark.parametrize("case", sorted(D["occupancy"]))
def test_occupancy_matches_reference(hf, case):
    regs, sh, thr = map(int, case.split(","))
    blocks, limiting, warps, frac = D["occupancy"][case].split()
    o = hf.occupancy(regs, sh, thr)
    assert (o["blocks_per_sm"], o["limiting"], o["achieved_warps"]) == (int(blocks), limiting, int(warps))
    assert abs(o["occupancy_fraction"] - float(frac)) < 1e-6
    assert oracle.occupancy(regs, sh, thr) == (int(blocks), limiting)


def test_b200_preset_register_bound(hf):
    # d0 = 1024 on B200: r0 in {32, 64} (SURVEY §7 hard part 4)
    assert hf.register_bound(32, 512, 32, 512, 8192, sm="b200") == 32
    assert hf.register_bound(128, 512, 96, 512, 8192, sm="b200") == 64


def test_does_not_fit(hf):
    with pytest.raises(hf.HFuseError) as e:
        hf.occupancy(255, 0, 1024)
    assert e.value.name == "DoesNotFit"


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("case", [(0.5, 100, 0.25, 300), (0.2307, 2788, 0.1672, 8212), (1.0, 1, 0.0, 10**12),
                                  (0.123456789, 987654321, 0.987654321, 123456789)])
def test_combined_utilization_matches_reference(hf, case):
    """hf_combined_utilization (include/hfuse.h) == the reference's machine.cpp:285-289."""
    import subprocess
    out = subprocess.run([oracle.REF, "combine", *map(str, case)], capture_output=True, text=True, check=True)
    assert hf.combined_utilization(*case) == float(out.stdout)


def test_combined_utilization_rejects_empty_kernels(hf):
    import math
    assert math.isnan(hf.combined_utilization(0.5, 0, 0.5, 10))
