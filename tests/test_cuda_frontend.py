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
    ("  float v = t > 0 ? 1.0f : 2.0f;\n", 3, "?:"),
    ("  float a[4];\n", 3, "local arrays"),
    ("  do { t = t + 1; } while (t < 4);\n", 3, "'do'"),
    ("  break;\n", 3, "outside a loop"),
    ("  double u = 3;\n", 3, "double"),
    ("  unsigned u = 3u; float f = u;\n", 3, "unsigned -> float"),
    ("  unsigned u = 3u; u = u / 3u;\n", 3, "power-of-two"),
    ("  float4 v = reinterpret_cast<const float4*>(c)[0];\n", 3, "element type"),
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


UNSIGNED = r"""
__device__ unsigned rotr(unsigned x, int n) { return (x >> n) | (x << (32 - n)); }

//@ grid=1
__global__ void __launch_bounds__(64) words(const uint32_t* __restrict__ in, uint32_t* out, int* flags) {
  int t = threadIdx.x;
  uint32_t a = in[t], b = in[(t + 1) % 64];
  unsigned int s = a + b * 2654435761u;
  s ^= rotr(s, 13);
  s += 0x9e3779b9;
  out[t] = s;
  out[64 + t] = a >> 7;
  out[128 + t] = a / 16u + a % 8u;
  out[192 + t] = min(a, b) ^ max(a, b);
  out[256 + t] = __funnelshift_r(a, b, 5);
  flags[t] = (a < b) + 2 * (a >= 0x80000000u) + 4 * (b <= a) + 8 * (a > 7u);
}
"""


def unsigned_reference(x):
    x = np.asarray(x, np.uint64)
    b = np.roll(x, -1)
    M = 0xFFFFFFFF
    s = (x + b * 2654435761) & M
    s ^= ((s >> 13) | (s << 19)) & M
    s = (s + 0x9E3779B9) & M
    out = np.concatenate([s, x >> 7, (x // 16 + x % 8) & M, np.minimum(x, b) ^ np.maximum(x, b),
                          ((x | (b << 32)) >> 5) & M])
    flags = (x < b).astype(np.int64) + 2 * (x >= 0x80000000) + 4 * (b <= x) + 8 * (x > 7)
    return out.astype(np.uint32), flags


VECTORS = r"""
//@ grid=2
__global__ void __launch_bounds__(32) vec(const float* __restrict__ x, float* y, const int* __restrict__ k,
                                          int* m) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  float4 v = reinterpret_cast<const float4*>(x)[t];
  float4 w;
  w = make_float4(v.w, v.z + 1.0f, v.y * 2.0f, v.x);
  w.x += __ldg(&x[0]);
  reinterpret_cast<float4*>(y)[t] = w;
  int2 q = ((const int2*)k)[t];
  reinterpret_cast<int2*>(m)[t] = make_int2(q.y, q.x - q.y);
}
"""


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_cuda_unsigned_and_vectors_on_reference_interpreter(hf, tmp_path):
    """uint32_t arithmetic (shr_u, ltu, power-of-two / and %, unsigned min/max, wide literals,
    funnel shifts) and float4/int2 loads, stores, components: lowered to Mini-Kernel, run on the
    reference interpreter, equal to numpy's uint32 / float32 semantics."""
    for src, img, check in [
        (UNSIGNED, "array in int32 64 seed 11 range -2147483648 2147483647\narray out int32 320 zero\n"
                   "array flags int32 64 zero\n", "u"),
        (VECTORS, "array x float32 256 seed 5 uniform -1 1\narray y float32 256 zero\n"
                  "array k int32 128 seed 6 range -1000 1000\narray m int32 128 zero\n", "v")]:
        assert hf.check(src).startswith("ok")
        (tmp_path / "k.mk").write_text(hf.lower(src))
        (tmp_path / "k.img").write_text(img)
        grid = 1 if check == "u" else 2
        _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img", "--grid", grid)
        arrays, _ = oracle.parse_image(dump)
        inputs, _ = oracle.parse_image(img)
        if check == "u":
            want, flags = unsigned_reference(np.asarray(inputs["in"], np.int64) & 0xFFFFFFFF)
            assert np.array_equal(np.asarray(arrays["out"]).astype(np.int64) & 0xFFFFFFFF, want.astype(np.int64))
            assert [int(v) for v in arrays["flags"]] == [int(v) for v in flags]
        else:
            x = np.asarray(inputs["x"], np.float32).reshape(-1, 4)[:64]
            y = np.stack([x[:, 3], x[:, 2] + np.float32(1), x[:, 1] * np.float32(2), x[:, 0]], 1)
            y[:, 0] = y[:, 0] + np.float32(inputs["x"][0])
            got = np.asarray(arrays["y"], np.float32).reshape(-1, 4)[:64]
            assert np.array_equal(got.view(np.uint32), y.astype(np.float32).view(np.uint32))
            q = np.asarray(inputs["k"], np.int64).reshape(-1, 2)[:64]
            assert [int(v) for v in np.asarray(arrays["m"]).reshape(-1, 2)[:64].ravel()] == \
                [int(v) for v in np.stack([q[:, 1], q[:, 0] - q[:, 1]], 1).ravel()]
        m = hf.Module.kernel(src, grid=grid)  # and the sm_100a emission compiles (NVRTC)
        assert len(m.cubin) > 1000


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_cuda_b200_hist_member_equals_the_mkplus_member(hf, tmp_path):
    """The bench's vectorized Hist member written in CUDA (float4 loads, __float2int_rz, shared
    atomics) gives the MK+ member's bins on the reference interpreter (ragged and parity n)."""
    from paper_2007_01277_b200 import pairs
    for n in (1001, 2 * 8 * 56 * 56):
        digs = []
        for src in (cu("histogram_b200.cu"), pairs.source("b200", "histogram")):
            (tmp_path / "k.mk").write_text(hf.lower(src))
            (tmp_path / "k.img").write_text(pairs._hist(n, -4.5, 4.5)(0).image)
            digs.append(oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img", "--grid", 4)[0])
        assert digs[0] == digs[1], n


@pytest.mark.gpu
def test_cuda_member_fused_with_mkplus_member_on_device(gpu):
    """Mixed input languages: the CUDA Hist fused with the MK+ BatchNorm at 512/512 reproduces
    the reference's sequential run of the MK+ pair (members.json fixture) bit for bit."""
    from paper_2007_01277_b200 import pairs
    hf = gpu
    G = golden("members.json")
    m = hf.Module.fused(pairs.source("b200", "batchnorm"), cu("histogram_b200.cu"), 512, 512, grid=G["grid"])
    img = hf.Image(pairs.MEMBERS["bn"].sizes["parity"](0).image).merge(
        hf.Image(pairs.MEMBERS["hist"].sizes["parity"](0).image)).upload()
    m.run(img, G["grid"])
    img.download()
    assert img.digest_hex() == G["pairs"]["bn+hist"]["512"]["digest"]


TERNARY = r"""
__global__ void __launch_bounds__(64) sel(const int* __restrict__ x, int* y, unsigned* z) {
  int t = threadIdx.x;
  int v = x[t];
  y[t] = v > 0 ? v * 2 : (v < -100 ? -1 : v);
  unsigned u = (unsigned)v;
  z[t] = (t & 1) ? u : u >> 3;
}
"""


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_cuda_integer_conditional_as_select(hf, tmp_path):
    """`c ? a : b` on integer operands lowers to a branch-free select (nested, unsigned arms)."""
    img = "array x int32 64 seed 4 range -300 300\narray y int32 64 zero\narray z int32 64 zero\n"
    (tmp_path / "k.mk").write_text(hf.lower(TERNARY))
    (tmp_path / "k.img").write_text(img)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    out, _ = oracle.parse_image(dump)
    x = [int(v) for v in oracle.parse_image(img)[0]["x"]]
    assert [int(v) for v in out["y"]] == [v * 2 if v > 0 else (-1 if v < -100 else v) for v in x]
    want_z = [(v & 0xFFFFFFFF) if t & 1 else (v & 0xFFFFFFFF) >> 3 for t, v in enumerate(x)]
    assert [int(v) & 0xFFFFFFFF for v in out["z"]] == want_z


LOOPS = r"""
__global__ void __launch_bounds__(64) loops(const int* __restrict__ x, int* y) {
  int t = threadIdx.x;
  int acc = 0;
  for (int i = 0; i < 16; ++i) {
    if (i == t % 7) continue;
    if (x[t] + i > 250) break;
    int j = 0;
    while (1) {
      j++;
      if (j > i % 3) break;
      acc += j;
    }
    acc += i;
  }
  y[t] = acc;
}
"""


def loops_reference(x):
    out = []
    for t, v in enumerate(x):
        acc = 0
        for i in range(16):
            if i == t % 7:
                continue
            if v + i > 250:
                break
            j = 0
            while True:
                j += 1
                if j > i % 3:
                    break
                acc += j
            acc += i
        out.append(acc)
    return out


@pytest.mark.skipif(not oracle.have_ref(), reason="reference build (oracle/_ref) not present")
def test_cuda_break_and_continue(hf, tmp_path):
    """break / continue (nested loops) lower to gotos to per-loop labels: the reference interpreter
    runs the translation with C's semantics, and two such kernels fuse (labels stay distinct)."""
    img = "array x int32 64 seed 8 range 200 260\narray y int32 64 zero\n"
    (tmp_path / "k.mk").write_text(hf.lower(LOOPS))
    (tmp_path / "k.img").write_text(img)
    _, _, dump = oracle.ref_run("run", tmp_path / "k.mk", "--mem", tmp_path / "k.img")
    out, _ = oracle.parse_image(dump)
    x = [int(v) for v in oracle.parse_image(img)[0]["x"]]
    assert [int(v) for v in out["y"]] == loops_reference(x)
    other = LOOPS.replace("loops(", "loops2(").replace("int* y", "int* z").replace("y[t]", "z[t]")
    src, _ = hf.fuse(LOOPS, other, 64, 64, style="structured")
    assert hf.check(src).startswith("ok")
    assert len(hf.Module.fused(LOOPS, other, 64, 64).cubin) > 1000


def test_cuda_stcs_is_vstore_cs(hf):
    src = r"""
__global__ void __launch_bounds__(64) cp(const float* __restrict__ x, float* y) {
  int t = threadIdx.x;
  float4 v = reinterpret_cast<const float4*>(x)[t];
  __stcs(reinterpret_cast<float4*>(y) + t, make_float4(v.w, v.z, v.y, v.x));
}
"""
    low = hf.normalize(src)
    assert "vstore_cs(y, t" in low
    assert "__stcs(" in hf.emit_kernel(src)
