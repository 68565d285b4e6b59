"""Crypto members (C3/C4): the Python restatement is pinned on standard test vectors; the
generated MK+ kernels (kernels/gen_crypto.py) run on the reference interpreter (after
`hfuse lower`) and on the B200, and must reproduce the restatement's outputs exactly."""
import os
import struct
import subprocess

import pytest

from oracle import crypto_ref as C
from oracle import oracle
from paper_2007_01277_b200 import crypto

KERNELS = os.path.join(os.path.dirname(__file__), "..", "paper_2007_01277_b200", "kernels", "b200")
KINDS = list(crypto.MEMBERS)


def src(kind):
    with open(os.path.join(KERNELS, kind + ".mk")) as f:
        return f.read()


def test_known_answer_vectors():
    assert C.blake256(b"\x00").hex() == "0ce8d4ef4dd7cd8d62dfded9d4edb0a774ae6a41929a74da23109e8f11139c87"
    assert C.blake256(b"\x00" * 72).hex() == "d419bad32d504fb7d44d460c42c5593fe544fa4c135dec31e21bd9abdcc22d41"
    assert C.keccak256(b"").hex() == "c5d2460186f7233c927e7db2dcc703c0e500b653ca82273b7bfad8045d85a470"
    assert C.keccak512(b"").hex().startswith("0eab42de4c3ceb9235fc91acffe746b29c29a8c366b7c60e4e67c466f36a4304")
    words = list(struct.unpack(">20I", crypto.GENESIS_HEADER))
    nonce = struct.unpack("<I", crypto.GENESIS_HEADER[76:80])[0]
    d = C.sha256d_header(words, nonce)
    assert b"".join(struct.pack(">I", x) for x in d)[::-1].hex() == \
        "000000000019d6689c085ae165831e934ff763ae46a2a6c172b3f1b60a8ce26f"


def test_generated_sources_are_current(tmp_path):
    from paper_2007_01277_b200.kernels import gen_crypto
    for kind, gen in (("sha256d", gen_crypto.gen_sha256d), ("blake256", gen_crypto.gen_blake256),
                      ("blake2b", gen_crypto.gen_blake2b), ("blake2b_addc", gen_crypto.gen_blake2b_addc),
                      ("ethash", gen_crypto.gen_ethash), ("ethash_reg", gen_crypto.gen_ethash_reg)):
        assert gen() == src(kind), kind


def reference_outputs(kind, count, grid, nonce0, target, words=None, threads=None, npages=1 << 10):
    words = words or crypto.header_words(2024, 20)
    dag = C.LazyDag(77, npages) if kind == "ethash" else None
    return C.search_outputs(kind, words, nonce0, count, target, grid, threads or crypto.THREADS[kind], dag=dag,
                            n_pages=npages)


PRIME_PAGES = 1021  # Ethash's modulo page walk over a non-power-of-two DAG (the bench: 33,554,393)


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_ethash_modulo_walk_on_reference_interpreter(hf, tmp_path):
    """remu (MK+ unsigned remainder) lowered to plain Mini-Kernel walks a prime page count
    exactly like crypto_ref's `fnv(...) % n_pages` (the Ethash spec's hashimoto)."""
    count, grid, nonce0, target = 6, 1, 4242, 1 << 31
    w = crypto.workload("ethash", count=count, grid=grid, nonce0=nonce0, target=target, npages=PRIME_PAGES)
    (tmp_path / "k.mk").write_text(hf.lower(src("ethash")))
    (tmp_path / "k.img").write_text(w.image)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img", "--grid", grid)
    arrays, _ = oracle.parse_image(dump)
    want = reference_outputs("ethash", count, grid, nonce0, target, npages=PRIME_PAGES)
    assert int(arrays["eh_chk"][0]) == want["chk"] and int(arrays["eh_cnt"][0]) == want["cnt"]


@pytest.mark.gpu
@pytest.mark.parametrize("form", crypto.FORMS["ethash"])
def test_ethash_modulo_walk_on_device(gpu, form):
    hf = gpu
    count, grid, nonce0, target = 2600, 4, 99, 1 << 28
    w = crypto.workload("ethash", count=count, grid=grid, nonce0=nonce0, target=target, npages=PRIME_PAGES)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src(form), grid=grid, specialize=img).run(img, grid)
    img.download()
    thr = crypto.FORM_THREADS.get(form, crypto.THREADS["ethash"])
    assert device_outputs(img, "ethash") == reference_outputs("ethash", count, grid, nonce0, target, threads=thr,
                                                              npages=PRIME_PAGES)


FORMS = [(k, f) for k in KINDS for f in crypto.FORMS[k]]


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("kind,form", FORMS)
def test_lowered_kernels_on_reference_interpreter(hf, kind, form, tmp_path):
    count, grid, nonce0, target = (6 if kind == "ethash" else 40), 1, 1000, 1 << 31
    w = crypto.workload(kind, count=count, grid=grid, nonce0=nonce0, target=target)
    (tmp_path / "k.mk").write_text(hf.lower(src(form)))
    (tmp_path / "k.img").write_text(w.image)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img", "--grid", grid)
    arrays, _ = oracle.parse_image(dump)
    p = crypto.MEMBERS[kind]
    want = reference_outputs(kind, count, grid, nonce0, target)
    assert int(arrays[f"{p}_cnt"][0]) == want["cnt"]
    assert int(arrays[f"{p}_chk"][0]) == want["chk"]
    assert [int(x) for x in arrays[f"{p}_bmin"]] == want["bmin"]


def device_outputs(img, kind):
    p = crypto.MEMBERS[kind]
    return {"cnt": int(img.array(f"{p}_cnt")[0]), "chk": int(img.array(f"{p}_chk")[0]),
            "bmin": [int(x) for x in img.array(f"{p}_bmin")]}


@pytest.mark.gpu
@pytest.mark.parametrize("kind,form", FORMS)
def test_crypto_member_on_device(gpu, kind, form):
    hf = gpu
    count, grid, nonce0, target = (2600 if kind == "ethash" else 4096), 4, 77, 1 << 27
    w = crypto.workload(kind, count=count, grid=grid, nonce0=nonce0, target=target)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src(form), grid=grid, specialize=img).run(img, grid)
    img.download()
    thr = crypto.FORM_THREADS.get(form, crypto.THREADS[kind])
    assert device_outputs(img, kind) == reference_outputs(kind, count, grid, nonce0, target, threads=thr)


@pytest.mark.gpu
def test_sha256d_genesis_block_on_device(gpu):
    hf = gpu
    words = list(struct.unpack(">20I", crypto.GENESIS_HEADER))
    nonce = struct.unpack("<I", crypto.GENESIS_HEADER[76:80])[0]  # 2083236893
    w = crypto.workload("sha256d", count=1, grid=1, nonce0=nonce, target=1, words=words)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src("sha256d"), grid=1).run(img, 1)
    img.download()
    out = device_outputs(img, "sha256d")
    assert out["cnt"] == 1 and out["bmin"] == [nonce]  # digest word 7 == 0: a valid block
    assert out["chk"] == crypto.i32(0x6FE28C0A)  # first digest word of 000000000019d6...e26f


@pytest.mark.gpu
@pytest.mark.parametrize("a,b", [("sha256d", "blake2b"), ("blake256", "ethash")])
def test_fused_crypto_pairs_on_device(gpu, a, b):
    hf = gpu
    grid = 3
    ca, cb = (2048, 2048) if b != "ethash" else (2048, 256)
    wa = crypto.workload(a, count=ca, grid=grid, nonce0=5, target=1 << 28)
    wb = crypto.workload(b, count=cb, grid=grid, nonce0=9, target=1 << 28)
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    d2 = 512 if b == "ethash" else crypto.THREADS[b]  # the lean Ethash runs in any interval <= 1024
    m = hf.Module.fused(src(a), src(b), crypto.THREADS[a], d2, grid=grid, specialize=img)
    m.run(img, grid)
    img.download()
    assert device_outputs(img, a) == reference_outputs(a, ca, grid, 5, 1 << 28)
    assert device_outputs(img, b) == reference_outputs(b, cb, grid, 9, 1 << 28, threads=d2)


@pytest.mark.gpu
@pytest.mark.parametrize("a,b,d2,regs", [("sha256d", "blake2b", 512, (40, 56)),
                                         ("blake256", "ethash", 384, (32, 120)),
                                         ("blake256", "ethash", 512, (24, 104))])
def test_fused_crypto_pairs_with_interval_budgets(gpu, a, b, d2, regs):
    """Per-interval register budgets (setmaxnreg) change register allocation only: the fused
    outputs stay bit-identical to the restatement, and ptxas allocated the promised pool."""
    hf = gpu
    grid = 3
    ca, cb = (2048, 2048) if b != "ethash" else (2048, 384)
    wa = crypto.workload(a, count=ca, grid=grid, nonce0=5, target=1 << 28)
    wb = crypto.workload(b, count=cb, grid=grid, nonce0=9, target=1 << 28)
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    m = hf.Module.fused_regs(src(a), src(b), crypto.THREADS[a], d2, *regs, grid=grid, specialize=img)
    assert m.info.interval_regs == regs
    assert "setmaxnreg" in m.source
    m.run(img, grid)
    img.download()
    assert device_outputs(img, a) == reference_outputs(a, ca, grid, 5, 1 << 28)
    assert device_outputs(img, b) == reference_outputs(b, cb, grid, 9, 1 << 28, threads=d2)


@pytest.mark.gpu
def test_sha256d_blake2b_fused_at_scale(gpu):
    """2^20 nonces of each member through the fused kernel at the bench's grid (296) equals the
    hashlib-based restatement: hit count, checksum and every block's minimum winning nonce."""
    hf = gpu
    grid, n = 296, 1 << 20
    wa = crypto.workload("sha256d", count=n, grid=grid, nonce0=123, target=1 << 20)
    wb = crypto.workload("blake2b", count=n, grid=grid, nonce0=456, target=1 << 20)
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    m = hf.Module.fused(src("sha256d"), src("blake2b"), 512, 512, grid=grid, specialize=img)
    m.run(img, grid)
    img.download()
    assert device_outputs(img, "sha256d") == reference_outputs("sha256d", n, grid, 123, 1 << 20)
    assert device_outputs(img, "blake2b") == reference_outputs("blake2b", n, grid, 456, 1 << 20)


PIPE_VARIANTS = [("sha256d", {"HF_SHA_ADDS": "fma"}), ("blake256", {"HF_B256_ADDS": "a"}),
                 ("blake256", {"HF_B256_ADDS": "ac"})]


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("kind,env", PIPE_VARIANTS)
def test_fma_add_generator_variants_on_reference_interpreter(hf, kind, env, tmp_path, monkeypatch):
    """The generator's pipe-balance variants (adds as MK+ fma_add, profiles/r02_probe_hash_adds.jsonl)
    compute the same hash: lowered, they reproduce the restatement on the reference interpreter."""
    import importlib
    from paper_2007_01277_b200.kernels import gen_crypto
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = importlib.reload(gen_crypto)
    try:
        text = {"sha256d": g.gen_sha256d, "blake256": g.gen_blake256}[kind]()
    finally:
        monkeypatch.undo()
        importlib.reload(gen_crypto)
    assert "fma_add(" in text
    count, grid, nonce0, target = 40, 1, 1000, 1 << 31
    w = crypto.workload(kind, count=count, grid=grid, nonce0=nonce0, target=target)
    (tmp_path / "k.mk").write_text(hf.lower(text))
    (tmp_path / "k.img").write_text(w.image)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img", "--grid", grid)
    arrays, _ = oracle.parse_image(dump)
    p = crypto.MEMBERS[kind]
    want = reference_outputs(kind, count, grid, nonce0, target)
    assert int(arrays[f"{p}_chk"][0]) == want["chk"] and int(arrays[f"{p}_cnt"][0]) == want["cnt"]


WRAP = [(0x7FFFFFE0, 40), (-24, 40)]  # across 2^31 (signed overflow) and across 2^32 -> 0


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
@pytest.mark.parametrize("nonce0,count", WRAP)
@pytest.mark.parametrize("kind", ["sha256d", "blake256", "blake2b"])
def test_nonce_range_wrap_on_reference_interpreter(hf, kind, nonce0, count, tmp_path):
    """Nonce ranges that cross 2^31 (the int32 nonce turns negative) and 2^32 (wraps to 0): the
    lowered member on the reference interpreter equals the restatement, per-block minimum included
    (a hit below 0x7fffffff after the wrap is a smaller signed value than one before it)."""
    grid, target = 1, 1 << 31
    w = crypto.workload(kind, count=count, grid=grid, nonce0=nonce0, target=target)
    (tmp_path / "k.mk").write_text(hf.lower(src(kind)))
    (tmp_path / "k.img").write_text(w.image)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img", "--grid", grid)
    arrays, _ = oracle.parse_image(dump)
    p = crypto.MEMBERS[kind]
    want = reference_outputs(kind, count, grid, nonce0, target)
    assert int(arrays[f"{p}_cnt"][0]) == want["cnt"] and int(arrays[f"{p}_chk"][0]) == want["chk"]
    assert [int(x) for x in arrays[f"{p}_bmin"]] == want["bmin"]


@pytest.mark.gpu
@pytest.mark.parametrize("nonce0", [0x7FFFFF00, -700])
@pytest.mark.parametrize("kind,form", FORMS)
def test_nonce_range_wrap_on_device(gpu, kind, form, nonce0):
    """The same wraps on the B200 with a ragged count (not a multiple of the block) over 3 blocks."""
    hf = gpu
    count, grid, target = (1300 if kind == "ethash" else 3001), 3, 1 << 28
    w = crypto.workload(kind, count=count, grid=grid, nonce0=nonce0, target=target)
    img = hf.Image(w.image).upload()
    hf.Module.kernel(src(form), grid=grid, specialize=img).run(img, grid)
    img.download()
    thr = crypto.FORM_THREADS.get(form, crypto.THREADS[kind])
    assert device_outputs(img, kind) == reference_outputs(kind, count, grid, nonce0, target, threads=thr)
