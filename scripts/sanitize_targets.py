"""Small launches of every fused-kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): named-barrier rewriting must not introduce shared-memory races or barrier misuse.
  compute-sanitizer --tool racecheck python scripts/sanitize_targets.py
Covers: corpus pairs (reference Mini-Kernel), the ten DL pairs (B200 forms, parity sizes, two
splits), the crypto pairs (one register cap and per-interval budgets), the hand-off BatchNorm,
a CUDA-frontend pair, and (round 2) dynamic interval scheduling (block- and warp-level queues,
two launches each), an MK+ async_copy kernel and the multi-GPU exchange's pack and reduce kernels."""
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden  # noqa: E402
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

n = 0
if sys.argv[1:2] == ["ethash"]:  # the Ethash forms alone (their 1,024-thread / 192 KB launches)
    # optional: block size of the lean form (tunable) and nonce count
    block = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    count = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
    we = CR.workload("ethash", count, 2, nonce0=3, target=1 << 28)
    img = hf.Image(we.image).upload()
    for form in CR.FORMS["ethash"]:
        text = open(os.path.join(P.KERNELS, "b200", form + ".mk")).read()
        if block and form == "ethash":
            text = text.replace("dims (1024, 1, 1)", f"dims ({block}, 1, 1)")
        m = hf.Module.kernel(text, grid=2, specialize=img)
        print(form, m.entry, "regs", m.info.regs, flush=True)
        m.run(img, 2)
        n += 1
    print(f"sanitize targets: {n} fused launches")
    sys.exit(0)
corpus = golden("corpus_sources.json")
digests = golden("corpus_digests.json")
for a, b in [("histogram", "batchnorm"), ("batchnorm", "shuffle_reduce"), ("streamer", "hasher"),
             ("strided_sum", "histogram")]:
    rec = digests["pairs"][f"{a}+{b}"]  # the acceptance splits: the corpus kernels are sized for them
    m = hf.Module.fused(corpus["kernels"][a], corpus["kernels"][b], rec["d1"], rec["d2"])
    img = hf.Image(corpus["images"][a]).merge(hf.Image(corpus["images"][b])).upload()
    m.run(img)
    n += 1
for a, b in P.PAIRS:
    img = hf.Image(P.MEMBERS[a].sizes["parity"](0).image).merge(hf.Image(P.MEMBERS[b].sizes["parity"](0).image)).upload()
    for d1 in (256, 768):
        hf.Module.fused(P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem), d1, 1024 - d1,
                        grid=4).run(img, 4)
        n += 1
src = {k: open(os.path.join(P.KERNELS, "b200", k + ".mk")).read() for k in CR.MEMBERS}
for a, b, d2, regs in [("sha256d", "blake2b", 512, (40, 56)), ("blake256", "ethash", 384, (32, 120))]:
    wa = CR.workload(a, 1024, 2, nonce0=5, target=1 << 28)
    wb = CR.workload(b, 256 if b == "ethash" else 1024, 2, nonce0=9, target=1 << 28)
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    hf.Module.fused(src[a], src[b], 512, d2, grid=2, specialize=img).run(img, 2)
    hf.Module.fused_regs(src[a], src[b], 512, d2, *regs, grid=2, specialize=img).run(img, 2)
    n += 2
# Ethash alone in both forms (the lean member parks seeds in shared memory across warp_sync and
# stages DAG pages through cp.async; 1,024 threads at 2 blocks)
# 4,096 nonces: every warp of both blocks walks (at 64 nonces only 2 of 32 warps would; see
# profiles/r02_racecheck_ethash_shapes.log for that degenerate shape)
we = CR.workload("ethash", 4096, 2, nonce0=3, target=1 << 28)
img = hf.Image(we.image).upload()
for form in ([] if sys.argv[1:] == ["no-ethash"] else CR.FORMS["ethash"]):
    hf.Module.kernel(open(os.path.join(P.KERNELS, "b200", form + ".mk")).read(), grid=2, specialize=img).run(img, 2)
    n += 1
img = hf.Image(P._bn(2, 8, 56 * 56, slots=256)(0).image).upload()
hf.Module.kernel(P.source("b200", "batchnorm_warp"), grid=7).run(img, 7)
n += 1
cu = os.path.join(ROOT, "tests", "cuda")
m = hf.Module.fused(open(os.path.join(cu, "histogram.cu")).read(), open(os.path.join(cu, "batchnorm.cu")).read(),
                    128, 896)
img = hf.Image(corpus["images"]["histogram"]).merge(hf.Image(corpus["images"]["batchnorm"])).upload()
m.run(img)
n += 1
for a, b, vg in [("bn", "hist", (8, 37)), ("im2col", "upsample", (7, 3)), ("hist", "maxpool", (13, 4))]:
    wa, wb = P.MEMBERS[a].sizes["parity"](), P.MEMBERS[b].sizes["parity"]()
    img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
    m = hf.Module.fused_opts(P.source("b200", P.MEMBERS[a].stem), P.source("b200", P.MEMBERS[b].stem), 256, 256,
                             vgrid=vg, grid=5, specialize=img)
    for _ in range(2):
        m.run(img, 5)
        n += 1
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_async_copy as TA  # noqa: E402
img = hf.Image(TA.IMG).upload()
hf.Module.kernel(TA.SRC).run(img)
n += 1
# the multi-GPU step exchange kernels (csrc/shard_reduce.cu): pack + reduce over an odd-length
# layout at world 8 (int64 words at odd cell offsets)
import test_shard_reduce_gpu as TS  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2007_01277_b200 import shard as SH  # noqa: E402
lay, g, counts = TS.layout_and_data(torch, 8, np.random.default_rng(8))
SH.reduce_gathered_device(hf, lay, g, counts)
srcs = [torch.arange(k, dtype=torch.int32, device="cuda") for k in (64, 63, 1)]
packed = torch.zeros(200, dtype=torch.int32, device="cuda")
hf.shard_pack([(t.data_ptr(), o, t.numel()) for t, o in zip(srcs, (0, 70, 140))], packed.data_ptr())
n += 2
import ctypes  # noqa: E402
assert ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize() == 0
print(f"sanitize targets: {n} fused launches")
