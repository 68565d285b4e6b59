"""Launch the C3/C4 crypto members and their fused pairs once each (for ncu), at the
configurations the bench search picks (round-1: per-interval budgets for BLAKE-256 + Ethash)."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import crypto as CR  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

G = 296
src = {k: open(os.path.join(P.KERNELS, "b200", k + ".mk")).read() for k in CR.MEMBERS}
wb = CR.workload("blake256", 1 << 22, G)
we = CR.workload("ethash", 1 << 18, G, npages=1 << 25)
img = hf.Image(wb.image).merge(hf.Image(we.image)).upload()
hf.Module.kernel(src["blake256"], grid=G, specialize=img).run(img, G)
hf.Module.kernel(src["ethash"], grid=G, specialize=img).run(img, G)
hf.Module.fused(src["blake256"], src["ethash"], 512, 512, regcap=64, grid=G, specialize=img).run(img, G)
hf.Module.fused_regs(src["blake256"], src["ethash"], 512, 512, 24, 104, grid=G, specialize=img).run(img, G)
hf.Module.fused_regs(src["blake256"], src["ethash"], 512, 384, 32, 120, grid=G, specialize=img).run(img, G)
ws, w2 = CR.workload("sha256d", 1 << 22, G), CR.workload("blake2b", 1 << 21, G)
img2 = hf.Image(ws.image).merge(hf.Image(w2.image)).upload()
hf.Module.kernel(src["sha256d"], grid=G, specialize=img2).run(img2, G)
hf.Module.kernel(src["blake2b"], grid=G, specialize=img2).run(img2, G)
hf.Module.fused(src["sha256d"], src["blake2b"], 512, 512, grid=G, specialize=img2).run(img2, G)
wu = P.MEMBERS["upsample"].sizes["full"](0)
wb4 = CR.workload("blake256", 1 << 21, G)
img3 = hf.Image(wu.image).merge(hf.Image(wb4.image)).upload()
su = P.source("b200", "upsample")
hf.Module.kernel(su, grid=G, specialize=img3).run(img3, G)
hf.Module.kernel(src["blake256"], grid=G, specialize=img3).run(img3, G)
hf.Module.fused(su, src["blake256"], 384, 512, regcap=40, grid=G, specialize=img3).run(img3, G)
import ctypes  # noqa: E402
ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize()
print("done")
