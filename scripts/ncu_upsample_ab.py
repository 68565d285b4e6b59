"""Launch the previous (per-thread 32-B stores) and the staged Upsample once each (ncu A/B)."""
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

w = P.MEMBERS["upsample"].sizes["full"](0)
img = hf.Image(w.image).upload()
old = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "upsample_v1.mk")).read()
hf.Module.kernel(old, grid=296, specialize=img).run(img, 296)
hf.Module.kernel(P.source("b200", "upsample"), grid=296, specialize=img).run(img, 296)
import ctypes  # noqa: E402
ctypes.CDLL("libcudart.so.12").cudaDeviceSynchronize()
print("done")
