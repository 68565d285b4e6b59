"""Frontend, normalization and the MK+ dialect."""
import os

import pytest

from conftest import golden

from oracle import oracle


@pytest.mark.parametrize("src,code", [
    ("kernel k() dims (32, 1, 1) { int x = ; }", "Syntax"),
    ("kernel k() dims (32, 1, 1) { x = 1; }", "UnknownIdentifier"),
    ("kernel k(int a[]) dims (32, 1, 1) { int x = 1.5; }", "TypeMismatch"),
    ("kernel k() dims (32, 1, 1) { goto nowhere; }", "UnresolvedLabel"),
    ("kernel k() dims (32, 1, 1) { bar_sync(16, 32); }", "BadBarrierId"),
    ("kernel k() dims (32, 1, 1) { bar_sync(1, 48); }", "MisalignedCount"),
    ("kernel k(int a[]) dims (32, 1, 1) { a[0] = warp_shfl_xor(a[0], 32); }", "TypeMismatch"),
    ("int f(int x) { return g(x); }\nint g(int x) { return f(x); }\nkernel k() dims (32, 1, 1) { }", "Recursion"),
    ("kernel k() dims (4096, 1, 1) { }", "ThreadBudgetExceeded"),
    ("kernel k() dims (32, 1, 1) { }\nkernel k() dims (32, 1, 1) { }", "DuplicateName"),
    ("kernel k() dims (32, 1, 1) { int x = 99999999999; }", "Syntax"),
])
def test_rejections_map_to_reference_codes(hf, src, code):
    with pytest.raises(hf.HFuseError) as e:
        hf.check(src)
    assert e.value.name == code


def test_strict_mode_rejects_dialect_extensions(hf):
    src = "kernel k(int a[]) dims (32, 1, 1) { a[0] = shr_u(a[0], 3); }"
    assert hf.check(src).startswith("ok")
    with pytest.raises(hf.HFuseError) as e:
        hf.check(src, strict=True)
    assert e.value.name == "UnresolvedCall"
    with pytest.raises(hf.HFuseError):
        hf.check("kernel k(int a[]) dims (32, 1, 1) { a[0] = 0x10; }", strict=True)


def test_lint_flags_goto_over_declaration(hf):
    src = "kernel k() dims (32, 1, 1) { goto L; int x = 1; L: }"
    assert "jumps over a declaration" in hf.check(src)


def test_normalization_names_match_reference(hf, corpus):
    text = hf.normalize(corpus["kernels"]["histogram"], "k2_")
    for name in ("k2___ret__inl0", "k2_value__inl0", "k2_nbins__inl0", "k2_b__inl0", "k2_i_2", "k2_i_3"):
        assert name in text


MKPLUS = """
kernel ext(int xi[], int xo[], float fi[], float fo[]) dims (32, 1, 1) {
  int t = threadIdx.x;
  int a = xi[t];
  int b = xi[t + 32];
  xo[t * 8] = shr_u(a, b);
  xo[t * 8 + 1] = shr_u(a, 7);
  xo[t * 8 + 2] = rotr(a, b);
  xo[t * 8 + 3] = rotl(a, 13);
  xo[t * 8 + 4] = ltu(a, b);
  xo[t * 8 + 5] = rotr(a, 0) ^ 0xdeadbeef;
  float v0; float v1; float v2; float v3;
  vload(fi, t, v0, v1, v2, v3);
  vstore(fo, t, v3, v2 + v1, v1, v0 * 2.0);
  unroll 4 for (int i = 0; i < 4; i = i + 1) {
    xo[t * 8 + 6] = xo[t * 8 + 6] + i;
  }
}
"""
IMG = ("array xi int32 64 seed 9 range -2147483648 2147483647\narray xo int32 256 zero\n"
       "array fi float32 128 seed 3 uniform -2 2\narray fo float32 128 zero\n")


def ref_semantics(xi, fi):
    import numpy as np
    u = xi.astype(np.int64) & 0xFFFFFFFF
    out = np.zeros(256, np.int64)
    for t in range(32):
        a, b = int(u[t]), int(u[t + 32])
        s = b & 31
        out[t * 8] = a >> s
        out[t * 8 + 1] = a >> 7
        out[t * 8 + 2] = ((a >> s) | (a << (32 - s))) & 0xFFFFFFFF
        out[t * 8 + 3] = ((a << 13) | (a >> 19)) & 0xFFFFFFFF
        out[t * 8 + 4] = int(a < b)
        out[t * 8 + 5] = a ^ 0xDEADBEEF
        out[t * 8 + 6] = 6
    fo = np.zeros(128, np.float32)
    for t in range(32):
        v = fi[4 * t:4 * t + 4]
        fo[4 * t:4 * t + 4] = [v[3], np.float32(v[2] + v[1]), v[1], np.float32(v[0] * 2)]
    return out.astype(np.uint32).view(np.int32), fo


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_mkplus_lowering_runs_on_reference_interpreter(hf, tmp_path):
    """MK+ -> Mini-Kernel (hf_lower) executes on the reference's run_functional with the
    dialect's documented semantics (logical shifts, rotates, unsigned compare, vectors)."""
    import numpy as np
    low = hf.lower(MKPLUS)
    assert hf.check(low, strict=True).startswith("ok")
    k = tmp_path / "k.mk"
    k.write_text(low)
    im = tmp_path / "k.img"
    im.write_text(IMG)
    _, _, dump = oracle.ref_run("run", k, "--mem", im)
    arrays, _ = oracle.parse_image(dump)
    inputs, _ = oracle.parse_image(IMG)
    xo, fo = ref_semantics(inputs["xi"], inputs["fi"])
    assert np.array_equal(arrays["xo"], xo)
    assert np.array_equal(arrays["fo"].view(np.uint32), fo.view(np.uint32))


def test_member_kernels_parse_and_lower(hf):
    from paper_2007_01277_b200 import pairs
    for m in pairs.MEMBERS.values():
        for form in ("ref", "b200"):
            src = pairs.source(form, m.stem)
            assert hf.check(src).startswith("ok: 1 kernel(s)")
            assert hf.check(hf.lower(src), strict=True).startswith("ok: 1 kernel(s)")


HANDOFF = """kernel k(int part[], int cnt[], int out[]) dims (64, 1, 1) {
  shared int s[2];
  int lane = threadIdx.x % 32;
  if (lane == 0) {
    part[threadIdx.x / 32] = threadIdx.x + 5;
    atomic_add_release(cnt[0], 1);
    if (load_relaxed(cnt[0]) == 2) {
      fence();
      out[0] = part[0] + load_acquire(part[1]);
    }
  }
}
"""


def test_release_acquire_handoff_constructs(hf):
    """MK+ inter-block hand-off: atomic_add_release / load_relaxed / load_acquire print back as
    written, lower to atomic_add / plain loads for the (sequentially consistent) interpreter,
    and emit red.release / ld.relaxed / ld.acquire at gpu scope for sm_100a."""
    assert hf.check(HANDOFF).startswith("ok")
    low = hf.lower(HANDOFF)
    assert "atomic_add(cnt[0], 1);" in low and "release" not in low and "load_" not in low
    assert hf.check(low, strict=True).startswith("ok")
    cu = hf.emit_kernel(HANDOFF)
    assert "hf_red_release(&cnt[0], 1);" in cu
    assert "hf_ld_relaxed(&cnt[0])" in cu and "hf_ld_acquire(&part[1])" in cu
    assert "red.release.gpu.global.add.s32" in cu and "ld.acquire.gpu.global.s32" in cu
    for bad, code in [("a[0] = load_acquire(3);", "TypeMismatch"),
                      ("atomic_add_release(s[0], 1);", "InvalidArgument")]:
        src = "kernel k(int a[]) dims (32, 1, 1) {\n  shared int s[2];\n  " + bad + "\n}\n"
        with pytest.raises(hf.HFuseError) as e:
            hf.emit_kernel(src) if code == "InvalidArgument" else hf.check(src)
        assert e.value.name == code


BCAST = """kernel k(int xi[], int xo[], float fo[]) dims (64, 1, 1) {
  int lane = threadIdx.x % 32;
  int v = xi[threadIdx.x];
  float f = float(v) * 0.5;
  int g = lane / 8;
  v = warp_bcast(v, (g + 3) % 8, 8);
  f = warp_bcast(f, 5, 32);
  xo[threadIdx.x] = v;
  fo[threadIdx.x] = f;
}
"""


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_warp_bcast_lowering_on_reference_interpreter(hf, tmp_path):
    """MK+ warp_bcast (group-uniform source lane): its butterfly lowering runs on the reference
    interpreter and gives lane (lane & ~(w-1)) + src's value; the sm_100a emission is one
    shfl.idx when the warp is full."""
    import numpy as np
    low = hf.lower(BCAST)
    assert "warp_bcast" not in low and hf.check(low, strict=True).startswith("ok")
    img = "array xi int32 64 seed 9 range -1000 1000\narray xo int32 64 zero\narray fo float32 64 zero\n"
    (tmp_path / "k.mk").write_text(low)
    (tmp_path / "k.img").write_text(img)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    arrays, _ = oracle.parse_image(dump)
    xi = np.asarray(oracle.parse_image(img)[0]["xi"], np.int64)
    t = np.arange(64)
    src8 = (t & ~7) + (((t % 32) // 8 + 3) % 8) + (t // 32) * 0
    assert [int(v) for v in arrays["xo"]] == [int(xi[(t0 & ~31) | (src8[t0] & 31)]) for t0 in t]
    want_f = [np.float32(np.float32(xi[(t0 & ~31) + 5]) * np.float32(0.5)) for t0 in t]
    assert np.array_equal(np.asarray(arrays["fo"], np.float32), np.asarray(want_f, np.float32))
    cu = hf.emit_kernel(BCAST)
    assert "hf_bcast(" in cu and "__shfl_sync(0xffffffffu, v, src, w)" in cu
    with pytest.raises(hf.HFuseError) as e:
        hf.check(BCAST.replace("v = warp_bcast(v, (g + 3) % 8, 8);", "v = 1 + warp_bcast(v, 1, 8);"))
    assert e.value.name == "TypeMismatch" and "whole right-hand side" in e.value.message
    with pytest.raises(hf.HFuseError) as e:
        hf.check(BCAST.replace("(g + 3) % 8, 8)", "(g + 3) % 8, 6)"))
    assert "power of two" in e.value.message


ADDC = """kernel k(int al[], int ah[], int bl[], int bh[], int ol[], int oh[]) dims (64, 1, 1) {
  int t = threadIdx.x;
  oh[t] = addc(ah[t], bh[t], al[t], bl[t]);
  ol[t] = al[t] + bl[t];
}
"""


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_addc_is_the_high_word_of_a_64_bit_add(hf, tmp_path):
    """MK+ addc(ahi, bhi, alo, blo): lowered (ltu carry) on the reference interpreter it equals
    the high word of the 64-bit sum; the sm_100a emission is add.cc + addc."""
    import numpy as np
    img = "".join(f"array {n} int32 64 seed {i + 3} range -2147483648 2147483647\n"
                  for i, n in enumerate(["al", "ah", "bl", "bh"])) + "array ol int32 64 zero\narray oh int32 64 zero\n"
    (tmp_path / "k.mk").write_text(hf.lower(ADDC))
    (tmp_path / "k.img").write_text(img)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    out, _ = oracle.parse_image(dump)
    x, _ = oracle.parse_image(img)
    u = {k: np.asarray(x[k], np.int64) & 0xFFFFFFFF for k in ("al", "ah", "bl", "bh")}
    s = ((u["ah"] << 32) | u["al"]) + ((u["bh"] << 32) | u["bl"])
    assert np.array_equal(np.asarray(out["oh"], np.int64) & 0xFFFFFFFF, (s >> 32) & 0xFFFFFFFF)
    assert np.array_equal(np.asarray(out["ol"], np.int64) & 0xFFFFFFFF, s & 0xFFFFFFFF)
    assert "add.cc.u32" in hf.emit_kernel(ADDC)


MULHI = """kernel k(int a[], int b[], int o[]) dims (256, 1, 1) {
  int t = threadIdx.x;
  o[t] = mulhi_u(a[t], b[t]);
}
"""


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_mulhi_u_is_the_high_word_of_an_unsigned_product(hf, tmp_path):
    """MK+ mulhi_u(a, b): lowered (16-bit limbs) on the reference interpreter it equals the high
    word of the unsigned 64-bit product, incl. 0, 1, -1 and powers of two (x >> n as
    mulhi_u(x, 2^(32-n))); the sm_100a emission is __umulhi."""
    import numpy as np
    special = [0, 1, -1, -2147483648, 2147483647, 65535, 65536, -65536, 1 << 16, 1 << 26, 1 << 31 - 1]
    img = ("array a int32 256 seed 5 range -2147483648 2147483647\n"
           "array b int32 256 values " + " ".join(str(v) for v in special) + " " +
           " ".join(str(((i * 2654435761) & 0xFFFFFFFF) - (1 << 32) if ((i * 2654435761) & 0xFFFFFFFF) >= 1 << 31
                        else (i * 2654435761) & 0xFFFFFFFF) for i in range(256 - len(special))) +
           "\narray o int32 256 zero\n")
    (tmp_path / "k.mk").write_text(hf.lower(MULHI))
    (tmp_path / "k.img").write_text(img)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    out, _ = oracle.parse_image(dump)
    x, _ = oracle.parse_image(img)
    ua = np.asarray(x["a"], np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    ub = np.asarray(x["b"], np.int64).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    want = ((ua * ub) >> np.uint64(32)).astype(np.int64)
    assert np.array_equal(np.asarray(out["o"], np.int64) & 0xFFFFFFFF, want)
    assert "__umulhi(" in hf.emit_kernel(MULHI)


FMAADD = """kernel k(int a[], int b[], int o[]) dims (256, 1, 1) {
  int t = threadIdx.x;
  o[t] = fma_add(fma_add(a[t], b[t]), 7);
}
"""


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_fma_add_is_a_wrapping_add(hf, tmp_path):
    """MK+ fma_add(a, b): lowered to a plain + it wraps like the interpreter's int add (checked on
    the reference interpreter at the int32 extremes); the sm_100a emission is a mad.lo.u32 with the
    constant-memory one, so ptxas issues it on the FMA pipe (IMAD) instead of an IADD3."""
    import numpy as np
    special = [0, 1, -1, -2147483648, 2147483647, 2147483641, -7, 65536]
    img = ("array a int32 256 seed 9 range -2147483648 2147483647\n"
           "array b int32 256 values " + " ".join(str(v) for v in special) + " " +
           " ".join(str((i * 7919) % 100003 - 50000) for i in range(256 - len(special))) +
           "\narray o int32 256 zero\n")
    low = hf.lower(FMAADD)
    assert "fma_add" not in low
    (tmp_path / "k.mk").write_text(low)
    (tmp_path / "k.img").write_text(img)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    out, _ = oracle.parse_image(dump)
    x, _ = oracle.parse_image(img)
    want = (np.asarray(x["a"], np.int64) + np.asarray(x["b"], np.int64) + 7) & 0xFFFFFFFF
    assert np.array_equal(np.asarray(out["o"], np.int64) & 0xFFFFFFFF, want)
    src = hf.emit_kernel(FMAADD)
    assert "hf_fma_add(hf_fma_add(" in src and "mad.lo.u32" in src and "__constant__ unsigned hf_one" in src


def test_vstore_cs_is_a_streaming_vstore(hf):
    """vstore_cs: same semantics as vstore (the lowering is identical), printed back as written,
    kept through fusion, emitted as an evict-first __stcs store on sm_100a."""
    cs = MKPLUS.replace("vstore(fo", "vstore_cs(fo")
    assert hf.lower(cs) == hf.lower(MKPLUS)
    assert "vstore_cs(fo, t" in hf.normalize(cs)
    assert "__stcs(reinterpret_cast<float4*>(fo)" in hf.emit_kernel(cs)
    assert "__stcs" not in hf.emit_kernel(MKPLUS)
    other = MKPLUS.replace("kernel ext(", "kernel ext2(")
    fused, _ = hf.fuse(cs, other, 32, 32, style="structured")
    assert fused.count("vstore_cs(") == 1 and fused.count("vstore(") == 1
