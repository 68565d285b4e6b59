"""Per-repetition timing (hf.time: events around each launch, the per-pair tables) vs the mean of
back-to-back launches (events around 50 launches, as the step): the difference is the per-launch
front-end gap the tables include and the step amortizes.
python scripts/probe_launch_gap.py > gpurun_out/probe_launch_gap.json"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import pairs as P  # noqa: E402

img = hf.Image(P.MEMBERS["bn"].sizes["full"](0).image)
for k in P.ORDER[1:]:
    img.merge(hf.Image(P.MEMBERS[k].sizes["full"](0).image))
img.upload()
stream = torch.cuda.current_stream()
out = {}
for k in P.ORDER:
    m = hf.Module.kernel(P.source("b200", P.MEMBERS[k].stem), grid=296, specialize=img)
    for g in (296, 2368):
        per = hf.time("single", m, None, img, g, warmup=5, reps=60, flush_l2=False, stream=stream)
        for _ in range(5):
            m.run(img, g, stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(50):
            m.run(img, g, stream)
        b.record(stream)
        torch.cuda.synchronize()
        out[f"{k}@{g}"] = {"per_rep_iqm_us": round(per["iqm_us"], 2), "per_rep_mean_us": round(per["mean_us"], 2),
                           "back_to_back_us": round(a.elapsed_time(b) * 1e3 / 50, 2)}
        print(k, g, out[f"{k}@{g}"], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
