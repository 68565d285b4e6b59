"""MK+ async_copy / async_wait (16-byte cp.async global -> shared, no register holds the data in
flight): parsed and type-checked, lowered to plain Mini-Kernel element copies the reference
interpreter runs, and on the B200 bit-identical to that interpreter run."""
import pytest

from oracle import oracle

SRC = """//@ grid=3
kernel stage(int g[], int out[], int n4) dims (64, 1, 1) {
  shared int s[512];
  int t = threadIdx.x;
  int a; int b; int c; int d;
  for (int v = blockIdx.x * 64 + t; v < n4; v = v + gridDim.x * 64) {
    async_copy(s, t, g, v);
    async_copy(s, t + 64, g, n4 - 1 - v);
    async_wait();
    vload(s, t, a, b, c, d);
    out[v * 2] = a * 3 + b - c ^ d;
    vload(s, t + 64, a, b, c, d);
    out[v * 2 + 1] = a + b * c - d;
  }
}
"""
IMG = "array g int32 1600 seed 9 range -100000 100000\narray out int32 800 zero\nscalar n4 int32 400\n"


def test_async_copy_parses_lowers_and_checks(hf):
    low = hf.lower(SRC)
    assert "async_copy" not in low and "async_wait" not in low
    assert "s[__as0] = g[__ag0];" in low.replace("  ", " ") or "__as0" in low
    bad = SRC.replace("async_copy(s, t, g, v);", "async_copy(g, t, s, v);")
    with pytest.raises(hf.HFuseError) as e:
        hf.lower(bad)
    assert e.value.name == "TypeMismatch"


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_lowered_async_copy_runs_on_reference_interpreter(hf, tmp_path):
    (tmp_path / "k.mk").write_text(hf.lower(SRC))
    (tmp_path / "k.img").write_text(IMG)
    digest, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    arrays, _ = oracle.parse_image(dump)
    g = arrays["g"].reshape(-1, 4).astype("int64")
    v = 7
    a, b, c, d = g[v]
    assert arrays["out"][2 * v] == ((a * 3 + b - c) ^ d)


@pytest.mark.gpu
def test_async_copy_on_device_matches_interpreter(gpu, tmp_path):
    hf = gpu
    if not oracle.have_ref():
        pytest.skip("reference build (oracle/_ref) not present")
    (tmp_path / "k.mk").write_text(hf.lower(SRC))
    (tmp_path / "k.img").write_text(IMG)
    want, _, _ = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    m = hf.Module.kernel(SRC)
    assert "cp.async.cg.shared.global" in m.source and "cp.async.wait_all" in m.source
    img = hf.Image(IMG).upload()
    m.run(img)
    img.download()
    assert img.digest_hex() == want
