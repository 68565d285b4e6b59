"""Catalog of the DL member kernels and their synthetic workloads.

Each member has two Mini-Kernel sources under kernels/: `ref/` — the naive form a user
would write (the input of the naive goto fusion and the semantic reference) — and `b200/`
— the MK+ form with the Blackwell mechanics the fused hot path uses. Images are
memory-image texts (memimage.cpp format) whose seeded arrays are generated in HBM.
`bytes` is the algorithmic HBM traffic of one launch (the roofline numerator).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Dict

KERNELS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "kernels")


def source(form: str, stem: str) -> str:
    with open(os.path.join(KERNELS, form, stem + ".mk")) as f:
        return f.read()


@dataclass
class Workload:
    image: str        # memory-image text
    bytes: int        # algorithmic bytes per launch (reads + writes)
    desc: str
    write: int = 0    # of which written

    @property
    def read(self) -> int:
        return self.bytes - self.write


@dataclass
class Member:
    key: str
    stem: str
    sizes: Dict[str, Callable[[int], Workload]]  # size name -> f(seed offset) -> Workload
    # "full": the C2 shapes (ResNet-50 conv2_x, 56 x 56); "conv3": ResNet-50 conv3_x shapes
    # (28 x 28 spatial, twice the channels; bench.py --shapes conv3); parity / tiny: test sizes


BN_SLOTS = 64  # >= grid / C + 2 for every grid the bench tries (C = 256: grids up to 15,872)
GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def slice_seed(seed: int, offset: int) -> int:
    """Seed of the stream that starts `offset` elements into the stream of `seed`.

    A seeded array's element i is mix(seed + (i + 1) * golden) (memimage.cpp:26-29, 52-61),
    so elements [offset, offset + n) of the array seeded `seed` are exactly the array of length
    n seeded seed + offset * golden (mod 2^64). Batch shards are therefore bit-exact slices of
    the whole-batch tensors with no image-format extension (the reference parser reads the
    seed as uint64, memimage.cpp:135)."""
    return (seed + offset * GOLDEN) & M64


def _bn(N: int, C: int, HW: int, slots: int = BN_SLOTS) -> Callable[..., Workload]:
    def make(seed: int = 0, offset: int = 0) -> Workload:
        n = N * C * HW
        # + the B200 form's grid-balancing workspace: BN_SLOTS partial (count, mean, M2) slots
        # per channel and one arrival counter per channel (zero between launches)
        img = (f"array bn_x float32 {n} seed {slice_seed(1 + seed, offset)} uniform -1 1\n"
               f"array bn_stats float32 {2 * C} zero\n"
               f"array bn_pn int32 {slots * C} zero\narray bn_pa float32 {slots * C} zero\n"
               f"array bn_pm float32 {slots * C} zero\narray bn_cnt int32 {C} zero\n"
               f"scalar bn_N int32 {N}\nscalar bn_C int32 {C}\nscalar bn_HW int32 {HW}\n"
               f"scalar bn_P int32 {slots}\n")
        return Workload(img, 4 * n + 8 * C, f"bn_stats x[{N},{C},{HW}] fp32", 8 * C)
    return make


def _hist(n: int, lo: float = -4.0, hi: float = 4.0) -> Callable[..., Workload]:
    def make(seed: int = 0, offset: int = 0) -> Workload:
        img = (f"array hi_x float32 {n} seed {slice_seed(2 + seed, offset)} uniform {lo:g} {hi:g}\n"
               f"array hi_out int32 64 zero\nscalar hi_n int32 {n}\n")
        return Workload(img, 4 * n + 4 * 64, f"hist 64 bins over [-4,4], {n} fp32", 4 * 64)
    return make


def _maxpool(NC: int, H: int, W: int) -> Callable[..., Workload]:
    def make(seed: int = 0, offset: int = 0) -> Workload:
        OH, OW = H // 2, W // 2
        n, m = NC * H * W, NC * OH * OW
        img = (f"array mp_x float32 {n} seed {slice_seed(3 + seed, offset)} uniform -1 1\n"
               f"array mp_y float32 {m} zero\narray mp_idx int32 {m} zero\n"
               f"scalar mp_NC int32 {NC}\nscalar mp_H int32 {H}\nscalar mp_W int32 {W}\n"
               f"scalar mp_OH int32 {OH}\nscalar mp_OW int32 {OW}\n")
        return Workload(img, 4 * n + 8 * m, f"maxpool 3x3/s2/p1 x[{NC},{H},{W}] fp32 + int32 idx", 8 * m)
    return make


def _upsample(NC: int, IH: int, IW: int) -> Callable[..., Workload]:
    def make(seed: int = 0, offset: int = 0) -> Workload:
        OH, OW = 2 * IH, 2 * IW
        n, m = NC * IH * IW, NC * OH * OW
        img = (f"array us_x float32 {n} seed {slice_seed(4 + seed, offset)} uniform -1 1\n"
               f"array us_y float32 {m} zero\n"
               f"scalar us_NC int32 {NC}\nscalar us_IH int32 {IH}\nscalar us_IW int32 {IW}\n"
               f"scalar us_OH int32 {OH}\nscalar us_OW int32 {OW}\n")
        return Workload(img, 4 * n + 4 * m, f"upsample bilinear 2x x[{NC},{IH},{IW}] fp32", 4 * m)
    return make


def _im2col(NC: int, H: int, W: int) -> Callable[..., Workload]:
    def make(seed: int = 0, offset: int = 0) -> Workload:
        n, m = NC * H * W, NC * 9 * H * W
        img = (f"array ic_x float32 {n} seed {slice_seed(5 + seed, offset)} uniform -1 1\n"
               f"array ic_col float32 {m} zero\n"
               f"scalar ic_NC int32 {NC}\nscalar ic_H int32 {H}\nscalar ic_W int32 {W}\n")
        return Workload(img, 4 * n + 4 * m, f"im2col 3x3/p1 x[{NC},{H},{W}] fp32", 4 * m)
    return make


MEMBERS: Dict[str, Member] = {
    "bn": Member("bn", "batchnorm", {
        "full": _bn(64, 256, 56 * 56),
        "conv3": _bn(64, 512, 28 * 28),
        "parity": _bn(2, 8, 56 * 56),
        "tiny": _bn(1, 3, 16),
    }),
    "hist": Member("hist", "histogram", {
        "full": _hist(64 * 256 * 56 * 56),
        "conv3": _hist(64 * 512 * 28 * 28),
        "parity": _hist(2 * 8 * 56 * 56, -4.5, 4.5),
        "tiny": _hist(64, -5.0, 5.0),
    }),

    "maxpool": Member("maxpool", "maxpool", {
        "full": _maxpool(64 * 64, 112, 112),
        "conv3": _maxpool(64 * 128, 56, 56),
        "parity": _maxpool(3, 16, 16),
        "tiny": _maxpool(1, 8, 8),
    }),
    "upsample": Member("upsample", "upsample", {
        "full": _upsample(64 * 256, 28, 28),
        "conv3": _upsample(64 * 512, 14, 14),
        "parity": _upsample(3, 8, 8),
        "tiny": _upsample(1, 4, 4),
    }),
    "im2col": Member("im2col", "im2col", {
        "full": _im2col(32 * 64, 56, 56),
        "conv3": _im2col(32 * 128, 28, 28),
        "parity": _im2col(3, 8, 8),
        "tiny": _im2col(1, 4, 4),
    }),
}

ORDER = ["bn", "hist", "im2col", "maxpool", "upsample"]
# The ten DL pairs of the paper.
PAIRS = [(a, b) for i, a in enumerate(ORDER) for b in ORDER[i + 1:]]

# Batch-scaled members for the paper's workload-ratio study (each pair is
# reported at several execution-time ratios of its two kernels): the batch dimension of a
# member's C2 / conv3_x shape, as (workload of batch n, default batch n).
BATCHED: Dict[str, Dict[str, tuple]] = {
    "full": {
        "bn": (lambda n: _bn(n, 256, 56 * 56), 64),
        "hist": (lambda n: _hist(n * 256 * 56 * 56), 64),
        "im2col": (lambda n: _im2col(n * 64, 56, 56), 32),
        "maxpool": (lambda n: _maxpool(n * 64, 112, 112), 64),
        "upsample": (lambda n: _upsample(n * 256, 28, 28), 64),
    },
    "conv3": {
        "bn": (lambda n: _bn(n, 512, 28 * 28), 64),
        "hist": (lambda n: _hist(n * 512 * 28 * 28), 64),
        "im2col": (lambda n: _im2col(n * 128, 28, 28), 32),
        "maxpool": (lambda n: _maxpool(n * 128, 56, 56), 64),
        "upsample": (lambda n: _upsample(n * 512, 14, 14), 64),
    },
}


def scaled(key: str, factor: float, shape: str = "full", seed: int = 0) -> "tuple[Workload, int]":
    """Member `key` at `factor` times its default batch (rounded, at least 1): (workload, batch)."""
    make, n0 = BATCHED[shape][key]
    n = max(1, int(round(n0 * factor)))
    return make(n)(seed), n


def shard_offset(key: str, shape: str, rank: int, world: int) -> int:
    """Element offset of rank's batch shard in member `key`'s seeded input tensor."""
    make, n0 = BATCHED[shape][key]
    if n0 % world:
        raise ValueError(f"batch {n0} of {key} does not split over {world} ranks")
    per_image = int(make(1)(0).image.split("\n")[0].split()[3])
    return rank * (n0 // world) * per_image


def shard(key: str, shape: str, rank: int, world: int) -> Workload:
    """Rank `rank`'s batch shard (batch / world images) of member `key` at `shape`: the
    contiguous slice of the whole-batch input tensor starting at shard_offset (the same values,
    slice_seed), for the strong-scaling multi-GPU path. world = 1 is the
    whole-batch workload, identical to MEMBERS[key].sizes[shape]()."""
    make, n0 = BATCHED[shape][key]
    return make(n0 // world)(0, shard_offset(key, shape, rank, world))
