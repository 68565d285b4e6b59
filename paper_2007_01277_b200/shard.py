"""Multi-GPU plumbing for the batch-sharded DL pairs.

Each rank runs the fused pairs on its own batch shard; the only exchange is one reduction
of the small outputs: histogram bins (int32 all-reduce sum, bit-exact) and the BatchNorm
per-channel statistics (all-gather of (mean, var) per rank, merged in rank order with
Chan's parallel formula — deterministic). Works with any torch.distributed backend
(NCCL on the B200 box, gloo in the CPU tests)."""
from __future__ import annotations

import numpy as np


def merge_bn_stats(counts, means, variances):
    """Chan et al. merge of per-shard (n, mean, biased var) -> (mean, biased var), in order."""
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


def reduce_outputs(dist, hist_bins=None, bn_stats=None, bn_count=None):
    """The path's single collective step. hist_bins: int32 tensor (summed in place);
    bn_stats: float32 tensor [2C] = (mean, var) pairs of this rank's shard. Returns the
    merged (mean, var) as float64 numpy arrays when bn_stats is given."""
    import torch
    if hist_bins is not None:
        dist.all_reduce(hist_bins)
    if bn_stats is None:
        return None
    world = dist.get_world_size()
    parts = [torch.empty_like(bn_stats) for _ in range(world)]
    dist.all_gather(parts, bn_stats)
    st = [p.cpu().numpy().astype(np.float64).reshape(-1, 2) for p in parts]
    return merge_bn_stats([bn_count] * world, [s[:, 0] for s in st], [s[:, 1] for s in st])
