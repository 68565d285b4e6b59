import sys, json; sys.path.insert(0,'.')
from paper_2007_01277_b200 import hfuse as hf, pairs as P
wa, wb = P.MEMBERS['bn'].sizes['full'](), P.MEMBERS['im2col'].sizes['full']()
img = hf.Image(wa.image).merge(hf.Image(wb.image)).upload()
sa, sb = P.source('b200','batchnorm'), P.source('b200','im2col')
m = hf.Module.fused(sa, sb, 544, 96, regcap=32, grid=3552, specialize=img)
ka, kb = hf.Module.kernel(sa, grid=296, specialize=img), hf.Module.kernel(sb, grid=296, specialize=img)
for R in (1, 5, 20, 50):
    t = hf.time_graph('single', m, None, img, 3552, 0, reps=R, samples=5)
    s = hf.time_graph('two_stream', ka, kb, img, 296, 1184, reps=R, samples=5)
    print(json.dumps({"R": R, "fused": round(t['mean_us'],2), "ci": round(t['ci95_us'],2), "two": round(s['mean_us'],2)}))
