"""World-size-2 gloo test of the multi-GPU host path (paper_2007_01277_b200/shard.py):
two ranks each compute their batch shard's histogram and BatchNorm statistics (with the
C restatement standing in for the device kernels), then run the single reduction; the
merged result must equal the whole-batch result (hist exact, BN within 1e-5)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import oracle
    from paper_2007_01277_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, C, HW = 4, 3, 64
    full = oracle.fill_uniform(world * N * C * HW, 77, -1.0, 3.0).reshape(world * N, C, HW)
    mine = np.ascontiguousarray(full[rank * N:(rank + 1) * N])
    mean, var = oracle.bn_stats(mine, N, C, HW)
    stats = torch.tensor(np.stack([mean, var], 1).reshape(-1), dtype=torch.float32)
    bins = torch.tensor(oracle.hist(mine.reshape(-1) * 2.0), dtype=torch.int32)
    merged = shard.reduce_outputs(dist, hist_bins=bins, bn_stats=stats, bn_count=N * HW)
    if rank == 0:
        fm, fv = oracle.bn_stats(np.ascontiguousarray(full), world * N, C, HW)
        fh = oracle.hist(full.reshape(-1) * 2.0)
        q.put((bins.numpy().tolist(), fh.tolist(), merged[0].tolist(), fm.tolist(), merged[1].tolist(), fv.tolist()))
    dist.destroy_process_group()


def test_two_rank_reduction_matches_whole_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got_bins, want_bins, gm, fm, gv, fv = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got_bins == want_bins
    assert np.allclose(gm, fm, rtol=0, atol=1e-5) and np.allclose(gv, fv, rtol=0, atol=1e-5)


def test_chan_merge_is_exact_in_fp64():
    from paper_2007_01277_b200 import shard
    rng = np.random.default_rng(0)
    x = rng.normal(3.0, 2.0, size=(5, 1000))
    m, v = shard.merge_bn_stats([1000] * 5, [xi.mean(keepdims=True) for xi in x], [xi.var(keepdims=True) for xi in x])
    assert np.allclose(m, x.mean(), atol=1e-12) and np.allclose(v, x.var(), atol=1e-12)
