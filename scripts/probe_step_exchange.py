"""Probe: device time of the multi-GPU step's exchange around the all-gather (which needs >1 GPU
and is left out): round 2's first form (one cudaMemcpyAsync per output into the send buffer, then
shard.reduce_gathered's torch ops) vs the one-launch pack + one-launch reduce
(csrc/shard_reduce.cu), on the bench's C2 layout (4 Hist + 4 BN outputs) for a gathered buffer of
world 2 / 4 / 8. 200 back-to-back exchanges queued behind a device spin, CUDA events. JSON lines
(profiles/r02_probe_step_exchange.jsonl)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2007_01277_b200 import hfuse as hf  # noqa: E402
from paper_2007_01277_b200 import shard as SH  # noqa: E402

cudart = ctypes.CDLL("libcudart.so.12")
lay = SH.Layout()
srcs = []
for i in range(4):
    srcs.append((torch.randint(0, 1000, (64,), dtype=torch.int32, device="cuda"), lay.add("hist", f"{i}:hist", 64)))
for i in range(4):
    st = torch.rand(512, device="cuda").view(torch.int32)
    srcs.append((st, lay.add("bn", f"{i}:bn", 512, 256)))
packed = torch.zeros(lay.cells, dtype=torch.int32, device="cuda")
stream = torch.cuda.current_stream()
ptrs = [(t.data_ptr(), off, t.numel()) for t, off in srcs]
REPS = 200


def old(g, counts):
    for p, off, n in ptrs:
        cudart.cudaMemcpyAsync(ctypes.c_void_p(packed.data_ptr() + 4 * off), ctypes.c_void_p(p),
                               ctypes.c_size_t(4 * n), 3, ctypes.c_void_p(stream.cuda_stream))
    return SH.reduce_gathered(lay, g, counts)


def new(g, counts):
    hf.shard_pack(ptrs, packed.data_ptr(), stream.cuda_stream)
    return SH.reduce_gathered_device(hf, lay, g, counts)


for world in (2, 4, 8):
    g = packed.repeat(world, 1).contiguous()
    counts = [8 * 3136] * world
    for name, fn in (("memcpy+torch", old), ("pack+kernel", new)):
        for _ in range(3):
            fn(g, counts)
        torch.cuda.synchronize()
        torch.cuda._sleep(int(60e-3 * 2e9))  # the host queues all repetitions before the GPU starts them
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(REPS):
            fn(g, counts)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"world": world, "form": name, "us_per_exchange": round(e0.elapsed_time(e1) * 1e3 / REPS, 2)}),
              flush=True)
