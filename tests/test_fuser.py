"""Fuser parity with the reference (fuser.cpp / passes.cpp / mkfuse.cpp) on its own corpus:
byte-identical goto and structured emission, identical `fuse` reports, error codes;
plus the B200 additions (named-barrier allocation, sm_100a emission through NVRTC)."""
import hashlib

import pytest

from conftest import STEMS, golden

EMIT = golden("corpus_emit.json")
PAIRS = [(a, b) for a in STEMS for b in STEMS]


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def test_golden_goto_file_byte_exact(hf, corpus):
    """test_fuser.cpp:385-399 / acceptance criterion 2."""
    text, barriers = hf.fuse(corpus["kernels"]["batchnorm"], corpus["kernels"]["histogram"], 896, 128, "goto")
    assert text == corpus["golden_goto"]
    assert [(b.id, b.count, b.owner) for b in barriers] == [(1, 896, 1), (2, 128, 2)]
    assert text.count("bar.sync 1, 896;") == 2 and text.count("bar.sync 2, 128;") == 2
    assert "if (!(global_tid < 896)) goto K1_end;" in text and "if (global_tid < 896) goto K2_end;" in text


@pytest.mark.parametrize("a,b", PAIRS, ids=[f"{a}+{b}" for a, b in PAIRS])
def test_emission_matches_reference(hf, corpus, a, b):
    rec = EMIT[f"{a}+{b}"]
    for style in ("goto", "structured"):
        for rc in ("off", "auto"):
            want = rec[f"{style}_{rc}"]
            try:
                got = sha(hf.fuse(corpus["kernels"][a], corpus["kernels"][b], rec["d1"], rec["d2"], style, rc)[0])
            except hf.HFuseError as e:
                got = {"error": f"error{e}"}
            assert got == want, (style, rc)
    report = hf.fuse_report(corpus["kernels"][a], corpus["kernels"][b], rec["d1"], rec["d2"], "auto")
    assert report == rec["report"]


def test_structured_output_reparses_in_strict_mode(hf, corpus):
    text, _ = hf.fuse(corpus["kernels"]["batchnorm"], corpus["kernels"]["histogram"], 896, 128, "structured")
    assert hf.check(text, strict=True).startswith("ok: 1 kernel(s)")


GRID2 = "//@ grid=2\nkernel g(int o[]) dims (64, 1, 1) { o[0] = 1; }\n"
K64 = "kernel k(int p[]) dims (64, 1, 1) { p[0] = 1; }\n"


@pytest.mark.parametrize("src1,src2,d1,d2,code", [
    (K64, GRID2, 64, 64, "GridMismatch"),
    (K64, K64.replace("k(int p", "j(int q").replace("p[0]", "q[0]"), 48, 80, "InvalidArgument"),
    (K64, K64.replace("k(int p", "j(int q").replace("p[0]", "q[0]"), 1024, 64, "ThreadBudgetExceeded"),
    ("kernel f(int p[]) dims (64, 1, 1) fixed { p[0] = 1; }\n", K64.replace("p", "q"), 96, 64,
     "DimensionMismatch"),
    (K64, "kernel j(float p[]) dims (64, 1, 1) { p[0] = 1.0; }\n", 64, 64, "TypeMismatch"),
])
def test_error_contract(hf, src1, src2, d1, d2, code):
    with pytest.raises(hf.HFuseError) as e:
        hf.fuse(src1, src2, d1, d2)
    assert e.value.name == code


def test_preexisting_named_barriers_get_distinct_ids(hf):
    """the reference lets two constituents share bar_sync(1, 64); hfuse
    allocates one hardware id per (constituent, original id) and resizes whole-block counts."""
    k1 = "kernel a(int x[]) dims (64, 1, 1) { x[threadIdx.x] = 1; bar_sync(1, 64); x[0] = 2; }\n"
    k2 = "kernel b(int y[]) dims (64, 1, 1) { y[threadIdx.x] = 1; bar_sync(1, 64); bar_sync(2, 32); }\n"
    text, barriers = hf.fuse(k1, k2, 128, 64, "structured", "off")
    got = sorted((b.id, b.count, b.owner, b.original) for b in barriers)
    assert got == [(1, 128, 1, -1), (2, 64, 2, -1), (3, 128, 1, 1), (4, 64, 2, 1), (5, 32, 2, 2)]
    assert "bar_sync(3, 128);" in text and "bar_sync(4, 64);" in text and "bar_sync(5, 32);" in text


def test_more_than_fifteen_named_barriers_is_rejected(hf):
    body1 = " ".join(f"bar_sync({i}, 32);" for i in range(8))
    body2 = " ".join(f"bar_sync({i}, 32);" for i in range(8, 14))
    k1 = f"kernel a(int x[]) dims (32, 1, 1) {{ {body1} }}\n"
    k2 = f"kernel b(int y[]) dims (32, 1, 1) {{ {body2} }}\n"
    with pytest.raises(hf.HFuseError) as e:
        hf.fuse(k1, k2, 32, 32, "structured", "off")
    assert e.value.name == "BadBarrierId"


def test_sm100_emission_pins_interpreter_semantics(hf, corpus):
    src, _ = hf.fuse(corpus["kernels"]["batchnorm"], corpus["kernels"]["histogram"], 896, 128, "sm100", "off")
    assert 'extern "C" __global__ void __launch_bounds__(1024)' in src
    assert 'asm volatile("bar.sync 1, 896;" ::: "memory");' in src
    assert "const int* __restrict__ bn_in" in src and "int* __restrict__ hist_out" in src
    assert "__fdiv_rn" in src and "hf_add(" in src and "hf_shfl_full(" in src
    assert "reinterpret_cast<int4*>(hf_smem)[hf_i] = make_int4(0, 0, 0, 0);" in src  # zeroed shared memory


@pytest.mark.parametrize("a,b", [(a, b) for i, a in enumerate(STEMS) for b in STEMS[i + 1:]][:28])
def test_sm100_corpus_pairs_compile_for_sm100a(hf, corpus, a, b):
    """NVRTC (--gpu-architecture=sm_100a) compiles every fused corpus pair on the CPU host."""
    rec = EMIT[f"{a}+{b}"]
    m = hf.Module.fused(corpus["kernels"][a], corpus["kernels"][b], rec["d1"], rec["d2"])
    assert len(m.cubin) > 1000 and m.info.threads == rec["d1"] + rec["d2"]


def test_heterogeneous_grid_needs_a_barrier_free_second_member(hf):
    """split_grid gives member 2 whole CTAs as sub-blocks: a member with barriers or shared memory
    (Hist's per-block bins) cannot be split that way and is rejected at build time."""
    import pytest
    from paper_2007_01277_b200 import pairs as P
    with pytest.raises(hf.HFuseError) as e:
        hf.Module.fused_opts(P.source("b200", "maxpool"), P.source("b200", "histogram"), 512, 512, split_grid=4)
    assert e.value.name == "InvalidArgument"
    with pytest.raises(hf.HFuseError):  # d0 not a multiple of d2
        hf.Module.fused_opts(P.source("b200", "batchnorm"), P.source("b200", "im2col"), 640, 384, split_grid=4)
    m = hf.Module.fused_opts(P.source("b200", "batchnorm"), P.source("b200", "im2col"), 768, 256, split_grid=4)
    assert "hf_b1 = min(4, (int)gridDim.x)" in m.source
