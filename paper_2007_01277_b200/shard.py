"""Multi-GPU plumbing for the batch-sharded DL pairs and the nonce-range-sharded crypto pairs
(SURVEY.md §8e, C3/C5). Strong scaling: rank r of g owns batch images [r*N/g, (r+1)*N/g) of
every member (pairs.shard: exact slices of the whole-batch tensors) and nonces
[r*T/g, (r+1)*T/g) of a fixed range T.

The fused kernels have no exchange step; the only collective of a step is ONE all-gather of a
small packed buffer per rank, reduced identically on every rank:
  * histogram bins: int32 sum (bit-exact, order-free);
  * BatchNorm per-channel (mean, biased var) of each rank's shard: Chan's parallel merge in
    rank order, in fp64 (deterministic; equals the whole-batch statistics within fp rounding);
  * crypto: hit counts summed, winning nonce = MIN over ranks (sentinel = no hit).
The reference is single-threaded by design and has no
counterpart. Works with any torch.distributed backend (NCCL on the B200 box, gloo in the
CPU tests); the merge runs with torch ops on whatever device the packed buffer lives on.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

NO_HIT = (1 << 63) - 1  # winning-nonce sentinel of a shard without a hit


def merge_bn_stats(counts, means, variances):
    """Chan et al. merge of per-shard (n, mean, biased var) -> (mean, biased var), in order (numpy fp64)."""
    n = np.float64(0)
    mean = np.zeros_like(np.asarray(means[0], np.float64))
    m2 = np.zeros_like(mean)
    for c, mu, var in zip(counts, means, variances):
        c = np.float64(c)
        mu = np.asarray(mu, np.float64)
        tot = n + c
        delta = mu - mean
        mean = mean + delta * (c / tot)
        m2 = m2 + np.asarray(var, np.float64) * c + delta * delta * (n * c / tot)
        n = tot
    return mean, m2 / n


def merge_bn_torch(counts, means, variances):
    """merge_bn_stats with torch ops (same order, fp64): means/variances are [world, C]."""
    import torch
    means = means.to(torch.float64)
    variances = variances.to(torch.float64)
    n = 0.0
    mean = torch.zeros_like(means[0])
    m2 = torch.zeros_like(mean)
    for r, c in enumerate(counts):
        c = float(c)
        tot = n + c
        delta = means[r] - mean
        mean = mean + delta * (c / tot)
        m2 = m2 + variances[r] * c + delta * delta * (n * c / tot)
        n = tot
    # a true division (torch turns division by a Python scalar into a reciprocal multiply, which
    # rounds differently from merge_bn_stats and the device merge)
    return mean, m2 / torch.tensor(n, dtype=torch.float64, device=m2.device)


@dataclass
class Layout:
    """Packed int32 cells of one rank's step outputs: (kind, tag, offset, cells, C)."""
    slots: List[Tuple[str, str, int, int, int]] = field(default_factory=list)
    cells: int = 0

    def add(self, kind: str, tag: str, cells: int, channels: int = 0) -> int:
        off = self.cells
        self.slots.append((kind, tag, off, cells, channels))
        self.cells += cells
        return off


def all_gather_packed(dist, packed):
    """The step's single collective: every rank's packed int32 buffer -> [world, cells]."""
    import torch
    world = dist.get_world_size()
    if dist.get_backend() == "nccl":
        out = torch.empty((world, packed.numel()), dtype=packed.dtype, device=packed.device)
        dist.all_gather_into_tensor(out, packed)
        return out
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed)
    return torch.stack(parts)


def reduce_gathered(layout: Layout, gathered, bn_counts):
    """Reduce [world, cells] gathered buffers: {tag: hist bins (int64 sum)} and
    {tag: (mean, var) fp64 Chan merge over ranks in order}; bn_counts[r] = elements per channel
    of rank r's shard."""
    import torch
    out = {}
    for kind, tag, off, cells, ch in layout.slots:
        block = gathered[:, off:off + cells]
        if kind == "hist":
            out[tag] = block.to(torch.int64).sum(0)
        elif kind == "bn":
            st = block.contiguous().view(torch.float32).reshape(block.shape[0], ch, 2)
            out[tag] = merge_bn_torch(bn_counts, st[:, :, 0], st[:, :, 1])
        elif kind == "crypto":  # (hits, winning nonce) pairs as int64 = 2 int32 cells each
            # a flat copy: offset 0 and an even length whatever the slot's offset and the row stride
            v = block.reshape(-1).clone().view(torch.int64).reshape(block.shape[0], -1, 2)
            out[tag] = (v[:, :, 0].sum(0), v[:, :, 1].min(0).values)
        else:
            raise ValueError(kind)
    return out


def reduce_gathered_device(hf, layout: Layout, gathered, bn_counts):
    """reduce_gathered in ONE kernel launch (hf.shard_reduce, csrc/shard_reduce.cu) for a CUDA
    [world, cells] int32 buffer: the same dict, bit-identical (the kernel's fp64 Chan merge keeps
    merge_bn_torch's operation order with no contraction; tests/test_shard_reduce_gpu.py)."""
    import torch
    slots, views, o = [], [], 0
    for kind, tag, off, cells, ch in layout.slots:
        n = {"hist": cells, "bn": 2 * ch, "crypto": cells // 2}[kind]
        slots.append((kind, ch, off, cells, o))
        views.append((kind, tag, o, n, ch))
        o += n
    out = torch.empty(max(1, o), dtype=torch.int64, device=gathered.device)
    g = gathered.contiguous()
    counts = [float(c) for c in bn_counts] if bn_counts is not None else None
    hf.shard_reduce(g.data_ptr(), g.shape[0], g.shape[1], slots, counts, out.data_ptr(),
                    torch.cuda.current_stream(g.device).cuda_stream)
    res = {}
    for kind, tag, o, n, ch in views:
        block = out[o:o + n]
        if kind == "hist":
            res[tag] = block
        elif kind == "bn":
            f = block.view(torch.float64)
            res[tag] = (f[:ch], f[ch:])
        else:
            p = block.reshape(-1, 2)
            res[tag] = (p[:, 0], p[:, 1])
    return res


def nonce_slice(total: int, rank: int, world: int) -> Tuple[int, int]:
    """(nonce0, count) of rank's contiguous slice of [0, total)."""
    if total % world:
        raise ValueError(f"nonce range {total} does not split over {world} ranks")
    per = total // world
    return rank * per, per
