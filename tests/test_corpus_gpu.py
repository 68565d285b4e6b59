"""Device parity of the fused corpus pairs against the reference interpreter.

For each of the 28 acceptance pairs (acceptance_main.cpp:136-168) the sm_100a fused
kernel runs on the B200 over the seeded pair image; its FNV-1a digest must equal the
digest of the reference's sequential run_functional (k1 then k2) on the same inputs,
recorded in tests/golden/corpus_digests.json. Bit-exact: the corpus has no float atomics.
"""
import pytest

from conftest import STEMS, golden

DIGESTS = golden("corpus_digests.json")
PAIRS = [(a, b) for i, a in enumerate(STEMS) for b in STEMS[i + 1:]]
SEEDS = list(range(1, 21))  # every seed of acceptance_main.cpp:136-168


def pair_image(hf, corpus, a, b, seed):
    img = hf.Image(corpus["images"][a], seed)
    if a != b:
        img.merge(hf.Image(corpus["images"][b], seed))
    return img


@pytest.mark.gpu
@pytest.mark.parametrize("a,b", PAIRS, ids=[f"{a}+{b}" for a, b in PAIRS])
def test_fused_pair_matches_reference(gpu, corpus, a, b):
    hf = gpu
    rec = DIGESTS["pairs"][f"{a}+{b}"]
    mod = hf.Module.fused(corpus["kernels"][a], corpus["kernels"][b], rec["d1"], rec["d2"])
    for seed in SEEDS:
        img = pair_image(hf, corpus, a, b, seed).upload()
        mod.run(img)
        img.download()
        assert img.digest_hex() == rec["seeds"][str(seed)]["sequential"], f"seed {seed}"


@pytest.mark.gpu
@pytest.mark.parametrize("stem", STEMS)
def test_unfused_kernel_matches_reference(gpu, corpus, stem):
    hf = gpu
    mod = hf.Module.kernel(corpus["kernels"][stem])
    for seed, want in DIGESTS["kernels"][stem].items():
        img = hf.Image(corpus["images"][stem], int(seed)).upload()
        mod.run(img)
        img.download()
        assert img.digest_hex() == want, f"seed {seed}"


@pytest.mark.gpu
def test_device_fill_matches_reference_generator(gpu, corpus):
    """Seeded arrays generated in HBM equal the CPU splitmix64 stream (memimage.cpp:10-61)."""
    hf = gpu
    for stem in STEMS:
        for seed in (None, 5):
            dev = hf.Image(corpus["images"][stem], seed).upload().download()
            host = hf.Image(corpus["images"][stem], seed).materialize()
            assert dev.digest() == host.digest()
