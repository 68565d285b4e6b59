"""The multi-GPU step exchange on the device (csrc/shard_reduce.cu): hf.shard_pack gathers the
step outputs into one buffer in one launch, and shard.reduce_gathered_device reduces an
all-gathered [world, cells] buffer in one launch with exactly shard.reduce_gathered's results
(the torch restatement the gloo tests pin): hist sums, the fp64 Chan merge of BN statistics bit
for bit, crypto hit sums and winning-nonce minima. Rows of odd length (int64 words not 8-byte
aligned) included."""
import numpy as np
import pytest

from paper_2007_01277_b200 import shard as SH


def layout_and_data(torch, world, rng):
    lay = SH.Layout()
    lay.add("hist", "h0", 64)
    lay.add("bn", "b0", 2 * 256, 256)
    lay.add("hist", "h1", 63)          # odd cells: every later row offset is odd
    lay.add("crypto", "c", 4 * 3)      # three (hits, nonce) int64 pairs
    lay.add("bn", "b1", 2 * 512, 512)
    rows = []
    for r in range(world):
        row = np.zeros(lay.cells, np.int32)
        for kind, tag, off, cells, ch in lay.slots:
            if kind == "hist":
                row[off:off + cells] = rng.integers(0, 1 << 20, cells)
            elif kind == "bn":
                st = np.empty((ch, 2), np.float32)
                st[:, 0] = rng.normal(0, 1, ch)
                st[:, 1] = rng.uniform(0.1, 2, ch)
                row[off:off + cells] = st.reshape(-1).view(np.int32)
            else:
                pairs = np.empty((cells // 4, 2), np.int64)
                pairs[:, 0] = rng.integers(0, 50, cells // 4)
                pairs[:, 1] = rng.integers(-(1 << 40), 1 << 40, cells // 4)
                pairs[r % (cells // 4), 1] = SH.NO_HIT
                row[off:off + cells] = pairs.reshape(-1).view(np.int32)
        rows.append(row)
    g = torch.tensor(np.stack(rows), dtype=torch.int32, device="cuda")
    counts = [int(rng.integers(1000, 5000)) for _ in range(world)]
    return lay, g, counts


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_device_reduce_equals_torch_reduce(gpu, world):
    import torch
    hf = gpu
    lay, g, counts = layout_and_data(torch, world, np.random.default_rng(world))
    want = SH.reduce_gathered(lay, g, counts)
    got = SH.reduce_gathered_device(hf, lay, g, counts)
    torch.cuda.synchronize()
    for kind, tag, *_ in lay.slots:
        if kind == "hist":
            assert torch.equal(got[tag], want[tag])
        elif kind == "bn":
            assert torch.equal(got[tag][0], want[tag][0]) and torch.equal(got[tag][1], want[tag][1])
        else:
            assert torch.equal(got[tag][0], want[tag][0]), (tag, got[tag][0].tolist(), want[tag][0].tolist())
            assert torch.equal(got[tag][1], want[tag][1]), (tag, got[tag][1].tolist(), want[tag][1].tolist())


@pytest.mark.gpu
def test_pack_is_one_launch_concatenation(gpu):
    import torch
    hf = gpu
    srcs = [torch.arange(n, dtype=torch.int32, device="cuda") * (i + 1) for i, n in enumerate((64, 512, 63, 1))]
    packed = torch.full((700,), -1, dtype=torch.int32, device="cuda")
    offs, o = [], 5
    for t in srcs:
        offs.append(o)
        o += t.numel() + 3
    hf.shard_pack([(t.data_ptr(), off, t.numel()) for t, off in zip(srcs, offs)], packed.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    want = torch.full((700,), -1, dtype=torch.int32, device="cuda")
    for t, off in zip(srcs, offs):
        want[off:off + t.numel()] = t
    assert torch.equal(packed, want)


@pytest.mark.gpu
def test_reduce_rejects_bad_layouts(gpu):
    import torch
    hf = gpu
    g = torch.zeros((2, 10), dtype=torch.int32, device="cuda")
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    with pytest.raises(hf.HFuseError):
        hf.shard_reduce(g.data_ptr(), 2, 10, [("hist", 0, 8, 4, 0)], None, out.data_ptr())  # past the row
    with pytest.raises(hf.HFuseError):
        hf.shard_reduce(g.data_ptr(), 2, 10, [("bn", 4, 0, 8, 0)], None, out.data_ptr())  # bn without counts
