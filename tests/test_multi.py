"""Multi-rank host path of the strong-scaling bench, on CPU with gloo at world
sizes 2 and 4: every rank takes its exact batch shard (pairs.shard), computes its shard's
histogram and BatchNorm statistics (the C restatement stands in for the device kernels), and the
step's single collective (shard.all_gather_packed + reduce_gathered, the code bench.py runs)
must give the whole-batch result: histogram bit-exact, BN within 1e-5 of the fp64 whole-batch
statistics; crypto: hit counts summed and the winning nonce = MIN over ranks."""
import os
import socket

import numpy as np
import pytest
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
    from paper_2007_01277_b200 import pairs as P
    from paper_2007_01277_b200 import shard as SH
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # a small BN / Hist workload, sharded exactly like the bench shards the C2 batch
    N, C, HW = 8, 3, 64
    n_img = C * HW
    x_full = oracle.fill_uniform(N * n_img, 1, -1.0, 1.0)
    off = rank * (N // world) * n_img
    mine = oracle.fill_uniform((N // world) * n_img, P.slice_seed(1, off), -1.0, 1.0)
    assert np.array_equal(mine, x_full[off:off + mine.size])  # the shard IS the slice
    mean, var = oracle.bn_stats(mine, N // world, C, HW)
    bins = oracle.hist(mine * 4.0)
    layout = SH.Layout()
    layout.add("hist", "h", 64)
    layout.add("bn", "b", 2 * C, C)
    layout.add("crypto", "c", 8)  # two (hits, nonce) int64 pairs
    # crypto: (hits, winning nonce) of two members; rank r wins nonce 1000 - r on member 0 and
    # has no hit on member 1 unless it is the last rank
    hits = [rank + 1, 1 if rank == world - 1 else 0]
    win = [1000 - rank, 77 if rank == world - 1 else SH.NO_HIT]
    crypto = torch.tensor([hits[0], win[0], hits[1], win[1]], dtype=torch.int64).view(torch.int32)
    packed = torch.cat([torch.tensor(bins, dtype=torch.int32),
                        torch.tensor(np.stack([mean, var], 1).reshape(-1), dtype=torch.float32).view(torch.int32),
                        crypto])
    assert packed.numel() == layout.cells
    gathered = SH.all_gather_packed(dist, packed)
    red = SH.reduce_gathered(layout, gathered, [(N // world) * HW] * world)
    if rank == 0:
        fm, fv = oracle.bn_stats(x_full, N, C, HW)
        m, v = red["b"]
        q.put({"bins": red["h"].tolist(), "want_bins": oracle.hist(x_full * 4.0).tolist(),
               "mean": m.tolist(), "var": v.tolist(), "fmean": fm.tolist(), "fvar": fv.tolist(),
               "hits": red["c"][0].tolist(), "win": red["c"][1].tolist()})
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bench_reduction_equals_whole_batch(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    got = q.get(timeout=10)
    assert got["bins"] == got["want_bins"]
    tol = lambda a, b: np.all(np.abs(np.array(a) - np.array(b)) <= 1e-5 * np.maximum(1, np.abs(b)))  # noqa: E731
    assert tol(got["mean"], got["fmean"]) and tol(got["var"], got["fvar"])
    assert got["hits"] == [sum(range(1, world + 1)), 1]
    assert got["win"] == [1000 - (world - 1), 77]


def test_chan_merge_is_exact_in_fp64():
    from paper_2007_01277_b200 import shard
    rng = np.random.default_rng(0)
    x = rng.normal(3.0, 2.0, size=(5, 1000))
    m, v = shard.merge_bn_stats([1000] * 5, [xi.mean(keepdims=True) for xi in x], [xi.var(keepdims=True) for xi in x])
    assert np.allclose(m, x.mean(), atol=1e-12) and np.allclose(v, x.var(), atol=1e-12)


def test_torch_merge_matches_numpy_merge():
    import torch
    from paper_2007_01277_b200 import shard
    rng = np.random.default_rng(1)
    means, variances = rng.normal(size=(4, 7)), rng.uniform(0.5, 2, size=(4, 7))
    counts = [10, 20, 30, 40]
    m1, v1 = shard.merge_bn_stats(counts, means, variances)
    m2, v2 = shard.merge_bn_torch(counts, torch.tensor(means), torch.tensor(variances))
    assert np.array_equal(m1, m2.numpy()) and np.array_equal(v1, v2.numpy())


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_shards_tile_the_whole_batch(world):
    """pairs.shard: the g shards of every member are the contiguous slices of the whole-batch
    input (same seeds, consecutive offsets) and their bytes add up to the whole workload's."""
    from paper_2007_01277_b200 import pairs as P
    for key in P.ORDER:
        whole = P.MEMBERS[key].sizes["full"]()
        parts = [P.shard(key, "full", r, world) for r in range(world)]
        n = [int(p.image.split("\n")[0].split()[3]) for p in parts]
        assert sum(n) == int(whole.image.split("\n")[0].split()[3])
        offs = [P.shard_offset(key, "full", r, world) for r in range(world)]
        assert offs == [sum(n[:r]) for r in range(world)]
        seed0 = int(whole.image.split("\n")[0].split()[5])
        for p, o in zip(parts, offs):
            assert int(p.image.split("\n")[0].split()[5]) == P.slice_seed(seed0, o)
        if key not in ("bn", "hist"):  # per-image outputs: bytes split exactly
            assert sum(p.bytes for p in parts) == whole.bytes


def test_nonce_slices_cover_the_range():
    from paper_2007_01277_b200 import shard
    for world in (1, 2, 4, 8):
        sl = [shard.nonce_slice(1 << 20, r, world) for r in range(world)]
        assert sl[0][0] == 0 and all(a[0] + a[1] == b[0] for a, b in zip(sl, sl[1:]))
        assert sum(c for _, c in sl) == 1 << 20


def test_torch_merge_is_bit_identical_to_the_numpy_merge():
    """merge_bn_torch (the bench's reduction restated in torch, and the reference the device merge
    in csrc/shard_reduce.cu is tested against bit for bit) equals merge_bn_stats exactly."""
    import torch
    from paper_2007_01277_b200 import shard as SH
    rng = np.random.default_rng(3)
    for world in (1, 2, 5, 8):
        means = rng.normal(0, 1, (world, 256)).astype(np.float32)
        vars_ = rng.uniform(0.1, 2, (world, 256)).astype(np.float32)
        counts = [int(c) for c in rng.integers(1000, 9000, world)]
        m, v = SH.merge_bn_stats(counts, list(means), list(vars_))
        tm, tv = SH.merge_bn_torch(counts, torch.tensor(means), torch.tensor(vars_))
        assert np.array_equal(tm.numpy(), m) and np.array_equal(tv.numpy(), v)
