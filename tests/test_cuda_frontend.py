"""The restricted-CUDA frontend (csrc/cuda_frontend.cpp): `__global__` CUDA C in, the same IR the
Mini-Kernel frontend produces out. CUDA mirrors of the reference corpus kernels
(tests/cuda/*.cu) must fuse to the reference's golden goto text byte for byte, run on the
reference interpreter after lowering, and match the reference digests on the B200."""
import os

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import oracle

CUDA = os.path.join(ROOT, "tests", "cuda")
EMIT = golden("corpus_emit.json")
DIGESTS = golden("corpus_digests.json")


def cu(name):
    with open(os.path.join(CUDA, name)) as f:
        return f.read()


def test_cuda_corpus_pair_reproduces_reference_golden(hf, corpus):
    """CUDA batchnorm + histogram -> goto style at 896/128 == proj/tests/golden/
    fused_batchnorm_histogram.cu, and the same `fuse` report as the Mini-Kernel inputs."""
    src, table = hf.fuse(cu("batchnorm.cu"), cu("histogram.cu"), 896, 128, style="goto")
    assert src == corpus["golden_goto"]
    assert [(b.id, b.count, b.owner) for b in table] == [(1, 896, 1), (2, 128, 2)]
    rep_cu = hf.fuse_report(cu("batchnorm.cu"), cu("histogram.cu"), 896, 128)
    rep_mk = hf.fuse_report(corpus["kernels"]["batchnorm"], corpus["kernels"]["histogram"], 896, 128)
    assert rep_cu == rep_mk == EMIT["batchnorm+histogram"]["report"]


HEADER = r"""
// every construct of the subset in one kernel
__device__ float lerp(float a, float b, float w) { return a + w * (b - a); }

//@ grid=2
//@ requires n % 4 == 0
extern "C" __global__ void __launch_bounds__(64) features(const float* __restrict__ x, float* y,
                                                          int* __restrict__ cnt, const int n) {
"""


def features_src():
    body = r"""
  __shared__ int s[2 * 32];
  int t = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
  s[threadIdx.x] = 0;
  __syncthreads();
  #pragma unroll 4
  for (int k = 0; k < 4; ++k) {
    acc += k * 3;
    acc <<= 1;
  }
  acc ^= 0x0f;
  acc %= 1000;
  if (t < n) {
    float v = x[t];
    y[t] = lerp(v, 2.0f * v, .25f) + (float)(acc) * 1e-3f;
    int b = __float2int_rz((v + 4.0f) * 8.0f);
    if (b < 0) b = 0;
    else if (b > 63) b = 63;
    else { b = b; }
    atomicAdd(&s[b], 1);
  } else {
    acc = ~acc + (-1);
  }
  {
    int w = __shfl_xor_sync(0xffffffff, acc, 16);
    acc = min(acc, w) + max(acc, w) - (acc >> 2);
  }
  __syncwarp();
  __syncthreads();
  if (threadIdx.x < 64) atomicAdd(&cnt[threadIdx.x], s[threadIdx.x]);
  if (t == 0) cnt[64] = acc + (int)(1.9f) + int(2.5f);
}
"""
    return HEADER + body.lstrip("\n")


def reference_features(x, n, grid):
    """numpy restatement of features_src() (all threads, all blocks)."""
    acc0 = 0
    for k in range(4):
        acc0 = ((acc0 + k * 3) << 1)
    acc0 = (acc0 ^ 0x0F) % 1000
    y = np.zeros_like(x)
    bins = np.zeros(65, np.int64)
    accs = {}
    for blk in range(grid):
        s = np.zeros(64, np.int64)
        for tx in range(64):
            t = blk * 64 + tx
            acc = acc0
            if t < n:
                v = np.float32(x[t])
                lerp = np.float32(v + np.float32(np.float32(0.25) * np.float32(np.float32(2.0) * v - v)))
                y[t] = np.float32(lerp + np.float32(np.float32(acc) * np.float32(1e-3)))
                b = int(np.float32(np.float32(v + np.float32(4.0)) * np.float32(8.0)))
                b = min(max(b, 0), 63)
                s[b] += 1
            else:
                acc = (~acc) - 1
            accs[t] = acc
        bins[:64] += s
    # shuffle stage: lanes t and t ^ 16 of the same warp
    final0 = None
    for t in accs:
        w = accs[t ^ 16]
        a = accs[t]
        r = min(a, w) + max(a, w) - (a >> 2)
        if t == 0:
            final0 = r
    bins[64] = final0 + 1 + 2
    return y, bins


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_cuda_features_lower_and_run_on_reference_interpreter(hf, tmp_path):
    src = features_src()
    assert hf.check(src).startswith("ok: 1 kernel(s), 1 function(s)")
    low = hf.lower(src)
    assert hf.check(low, strict=True).startswith("ok")
    n, grid = 100, 2
    img = (f"array x float32 128 seed 3 uniform -5 5\narray y float32 128 zero\n"
           f"array cnt int32 65 zero\nscalar n int32 {n}\n")
    (tmp_path / "k.mk").write_text(low)
    (tmp_path / "k.img").write_text(img)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img", "--grid", grid)
    arrays, _ = oracle.parse_image(dump)
    inputs, _ = oracle.parse_image(img)
    y, bins = reference_features(np.asarray(inputs["x"], np.float32), n, grid)
    assert np.array_equal(np.asarray(arrays["y"], np.float32).view(np.uint32), y.view(np.uint32))
    assert [int(v) for v in arrays["cnt"]] == [int(v) for v in bins]
    # and the sm_100a emission compiles (NVRTC, compile-only without a GPU)
    m = hf.Module.kernel(src, grid=grid)
    assert len(m.cubin) > 1000 and m.info.threads == 64


@pytest.mark.parametrize("body,line,what", [
    ("  int v = t > 0 ? 1 : 2;\n", 3, "?:"),
    ("  float a[4];\n", 3, "local arrays"),
    ("  for (int i = 0; i < 4; ++i) { break; }\n", 3, "break"),
    ("  unsigned int u = 3;\n", 3, "unsigned"),
    ("  int v = atomicAdd(&c[0], 1);\n", 3, "atomicAdd"),
    ("  float v = __shfl_xor_sync(0x0000ffff, 1.0f, 1);\n", 3, "full mask"),
    ("  int* p = c;\n", 3, "pointers"),
    ("  c[0] = c[1]++;\n", 3, "++/--"),
    ("  c[0] = sqrtf(2.0f);\n", 3, "sqrtf"),
])
def test_cuda_rejections_point_at_the_cuda_line(hf, body, line, what):
    src = "__global__ void __launch_bounds__(32) k(int* c) {\n  int t = threadIdx.x;\n" + body + "}\n"
    with pytest.raises(hf.HFuseError) as e:
        hf.check(src)
    assert e.value.name == "Syntax" and e.value.line == line and what in e.value.message, e.value.message


def test_cuda_block_shape_is_required(hf):
    with pytest.raises(hf.HFuseError) as e:
        hf.check("__global__ void k(int* c) { c[0] = 1; }\n")
    assert "block shape" in e.value.message
    assert hf.check("//@ block=32,2\n__global__ void k(int* c) { c[0] = 1; }\n").startswith("ok")


@pytest.mark.gpu
def test_cuda_corpus_pair_on_device(gpu, corpus):
    """The fused CUDA batchnorm + histogram on the B200 equals the reference's sequential
    run_functional of the Mini-Kernel originals, for every recorded seed."""
    hf = gpu
    rec = DIGESTS["pairs"]["histogram+batchnorm"]
    mod = hf.Module.fused(cu("histogram.cu"), cu("batchnorm.cu"), rec["d1"], rec["d2"])
    for seed, want in rec["seeds"].items():
        img = hf.Image(corpus["images"]["histogram"], int(seed)).merge(
            hf.Image(corpus["images"]["batchnorm"], int(seed))).upload()
        mod.run(img)
        img.download()
        assert img.digest_hex() == want["sequential"], f"seed {seed}"
