"""The NCCL branch of bench.py's step exchange on a real GPU: a one-rank NCCL process group runs
Dist.gather_async (async all_gather_into_tensor on NCCL's stream, waited for on the compute
stream) between hf.shard_pack and shard.reduce_gathered_device, twice with the double-buffered
send buffers, and the reduced result equals the torch restatement (tests/test_shard_reduce_gpu.py
covers world 1-8 of the reduction itself; multi-rank NCCL needs more than the one GPU here)."""
import importlib.util
import os
import socket

import numpy as np
import pytest

from conftest import ROOT
from paper_2007_01277_b200 import shard as SH


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
def test_nccl_async_exchange_one_rank(gpu):
    import torch
    import torch.distributed as dist
    hf = gpu
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        D = bench.Dist.__new__(bench.Dist)
        D.world, D.rank, D.backend, D.local, D.dist = 1, 0, "nccl", 0, dist
        rng = np.random.default_rng(5)
        lay = SH.Layout()
        outs = [torch.tensor(rng.integers(0, 999, 64), dtype=torch.int32, device="cuda")]
        lay.add("hist", "h", 64)
        st = torch.tensor(np.stack([rng.normal(0, 1, 256), rng.uniform(0.1, 2, 256)], 1).astype(np.float32),
                          device="cuda").reshape(-1).view(torch.int32)
        outs.append(st)
        lay.add("bn", "b", 512, 256)
        srcs = [(t.data_ptr(), off, t.numel()) for t, (_, _, off, _, _) in zip(outs, lay.slots)]
        bufs = [torch.zeros(lay.cells, dtype=torch.int32, device="cuda") for _ in range(2)]
        stream = torch.cuda.current_stream()
        pending, got = None, None
        for k in range(3):
            hf.shard_pack(srcs, bufs[k % 2].data_ptr(), stream.cuda_stream)
            prev, pending = pending, D.gather_async(bufs[k % 2])
            if prev is not None:
                got = SH.reduce_gathered_device(hf, lay, prev(), [4096])
        got = SH.reduce_gathered_device(hf, lay, pending(), [4096])
        torch.cuda.synchronize()
        want = SH.reduce_gathered(lay, bufs[0].view(1, -1), [4096])
        assert torch.equal(got["h"], want["h"])
        assert torch.equal(got["b"][0], want["b"][0]) and torch.equal(got["b"][1], want["b"][1])
    finally:
        dist.destroy_process_group()
