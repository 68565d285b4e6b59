"""The C ABI boundary (include/hfuse.h): the in-tree library loads on a GPU-less host and
exports every declared entry point; no compute calls here."""
import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "hfuse.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hf_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(hf):
    lib = ctypes.CDLL(hf.LIB_PATH)
    names = declared()
    assert len(names) >= 35
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", hf.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hf_\w+)", out))
    assert set(names) <= exported


def test_python_mirror_binds_the_whole_header(hf):
    assert sorted(hf.EXPORTS) == declared()


def test_version_and_device_count_without_gpu(hf):
    assert "sm_100a" in hf.lib().hf_version().decode()
    assert hf.device_count() >= 0


def test_errors_cross_the_abi_as_codes(hf):
    try:
        hf.fuse("kernel a() dims (32, 1, 1) { x = 1; }", "kernel b() dims (32, 1, 1) { }", 32, 32)
    except hf.HFuseError as e:
        assert e.name == "UnknownIdentifier" and (e.line, e.col) == (1, 30)
    else:
        raise AssertionError("expected an error")


def test_cli_binary_present():
    exe = os.path.join(ROOT, "paper_2007_01277_b200", "bin", "hfuse")
    r = subprocess.run([exe, "nope"], capture_output=True, text=True)
    assert r.returncode == 1 and r.stderr.startswith("error[InvalidArgument]")


def test_param_read_flags_mark_pure_outputs(hf):
    """hf_module_param_reads: written arrays the kernel never loads (vstore/store only) are pure
    outputs; atomically updated ones (histogram bins) and inputs are read. Compile-only on CPU."""
    from paper_2007_01277_b200 import pairs
    m = hf.Module.fused(pairs.source("b200", "histogram"), pairs.source("b200", "upsample"), 512, 512, grid=296)
    p = {x["name"]: x for x in m.params if x["array"]}
    assert p["hi_x"]["read"] and not p["hi_x"]["written"]
    assert p["hi_out"]["read"] and p["hi_out"]["written"]      # atomic_add: read-modify-write
    assert p["us_y"]["written"] and not p["us_y"]["read"]      # pure output: no upload needed
    assert p["us_x"]["read"]
    m = hf.Module.kernel(pairs.source("b200", "maxpool"), grid=296)
    p = {x["name"]: x for x in m.params if x["array"]}
    assert not p["mp_y"]["read"] and not p["mp_idx"]["read"] and p["mp_x"]["read"]


def test_requires_annotation_checked_before_launch(hf):
    """`//@ requires` (MK+): printed back, dropped by the lowering, carried into fused kernels,
    refused at hf_launch when false (checked before the device is touched, so this runs on CPU)
    and at build time when every scalar it names is JIT-specialized."""
    from paper_2007_01277_b200 import pairs
    bn, up = pairs.source("b200", "batchnorm"), pairs.source("b200", "upsample")
    assert "requires" not in hf.lower(bn)
    src, _ = hf.fuse(bn, up, 512, 512, style="structured", sm="b200")
    assert "//@ requires bn_HW % 4 == 0\n" in src and "//@ requires us_OH == 2 * us_IH" in src
    m = hf.Module.fused(bn, up, 512, 512, grid=8)
    args = {p["name"]: 0 for p in m.params}
    args.update(bn_N=2, bn_C=3, bn_HW=18, us_NC=1, us_IH=4, us_IW=4, us_OH=8, us_OW=8)
    with pytest.raises(hf.HFuseError) as e:
        m.launch(args, grid=8)
    assert e.value.name == "InvalidArgument" and "requires bn_HW % 4 == 0 (bn_HW = 18)" in str(e.value)
    args["bn_HW"] = 16
    with pytest.raises(hf.HFuseError) as e:   # precondition holds: now it is the missing GPU
        m.launch(args, grid=8)
    assert e.value.name != "InvalidArgument"
    bad = hf.Image(pairs._bn(2, 3, 18)(0).image)
    with pytest.raises(hf.HFuseError) as e:
        hf.Module.kernel(bn, grid=4, specialize=bad)
    assert e.value.name == "InvalidArgument" and "specialized" in str(e.value)
    for text, code in [("//@ requires bn_x[0] == 1\n", "TypeMismatch"), ("//@ requires nope > 1\n", "TypeMismatch"),
                       ("//@ requires bn_HW %\n", "Syntax")]:
        with pytest.raises(hf.HFuseError) as e:
            hf.check(text + bn[bn.index("kernel bn_stats"):])
        assert e.value.name == code, text
