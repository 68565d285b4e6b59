"""TEST INFRASTRUCTURE ONLY: ctypes view of the C restatement (hf_oracle.c) and a
driver for the reference interpreter (oracle/_ref/mkfuse_ref). Imported only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs."""
import ctypes as C
import os
import subprocess
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libhforacle.so")
REF = os.path.join(HERE, "_ref", "mkfuse_ref")

_lib = C.CDLL(LIB)
_f, _i32, _i64, _u64, _d = C.c_float, C.c_int32, C.c_int64, C.c_uint64, C.c_double
_P = C.c_void_p
for name, res, args in [
    ("hfo_mix_seed", _u64, [_u64, C.c_int, _u64]),
    ("hfo_fill_uniform", None, [_P, _i64, _u64, _f, _f]),
    ("hfo_fill_range", None, [_P, _i64, _u64, _i32, _i32]),
    ("hfo_fnv_init", _u64, []),
    ("hfo_fnv_array", _u64, [_u64, C.c_char_p, C.c_int, _i64, _P]),
    ("hfo_fnv_scalar", _u64, [_u64, C.c_char_p, C.c_int, C.c_uint32]),
    ("hfo_occupancy", C.c_int, [C.c_int, _i64, C.c_int, _i64, _i64, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    ("hfo_register_bound", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, _i64, _i64, _i64, C.c_int]),
    ("hfo_bn_stats", None, [_P, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("hfo_hist", None, [_P, _i64, _P]),
    ("hfo_maxpool", None, [_P, C.c_int, C.c_int, C.c_int, _P, _P]),
    ("hfo_upsample", None, [_P, C.c_int, C.c_int, C.c_int, _P]),
    ("hfo_im2col", None, [_P, C.c_int, C.c_int, C.c_int, _P]),
    ("hfo_threads", C.c_int, []),
]:
    fn = getattr(_lib, name)
    fn.restype, fn.argtypes = res, args

PASCAL = dict(regs_per_sm=65536, shmem_per_sm=98304, max_threads_per_sm=2048, max_blocks_per_sm=32)


def threads():
    return _lib.hfo_threads()


def mix_seed(file_seed, override=None):
    return _lib.hfo_mix_seed(file_seed, override is not None, override or 0)


def fill_uniform(n, seed, lo, hi):
    out = np.empty(n, np.float32)
    _lib.hfo_fill_uniform(out.ctypes.data, n, seed, lo, hi)
    return out


def fill_range(n, seed, lo, hi):
    out = np.empty(n, np.int32)
    _lib.hfo_fill_range(out.ctypes.data, n, seed, lo, hi)
    return out


def parse_image(text, seed=None):
    """memimage.cpp:74-155 for the subset the tests use -> ({name: array}, {name: scalar})."""
    arrays, scalars = {}, {}
    for line in text.splitlines():
        line = line.split("#")[0].split()
        if not line:
            continue
        if line[0] == "scalar":
            scalars[line[1]] = (np.int32 if line[2] == "int32" else np.float32)(float(line[3]) if line[2] != "int32" else int(line[3]))
            continue
        name, typ, n, mode = line[1], line[2], int(line[3]), line[4]
        if mode == "zero":
            arrays[name] = np.zeros(n, np.int32 if typ == "int32" else np.float32)
        elif mode == "values":
            arrays[name] = np.array(line[5:5 + n], np.int32 if typ == "int32" else np.float32)
        else:
            s = mix_seed(int(line[5]), seed)
            if typ == "int32":
                arrays[name] = fill_range(n, s, int(line[7]), int(line[8]))
            else:
                arrays[name] = fill_uniform(n, s, float(line[7]), float(line[8]))
    return arrays, scalars


def digest(arrays, scalars):
    h = _lib.hfo_fnv_init()
    for name in sorted(arrays):
        a = np.ascontiguousarray(arrays[name])
        h = _lib.hfo_fnv_array(h, name.encode(), int(a.dtype == np.float32), a.size, a.ctypes.data)
    for name in sorted(scalars):
        v = scalars[name]
        bits = int(np.array(v, dtype=np.float32).view(np.uint32)) if isinstance(v, np.float32) else int(np.uint32(np.int32(v)))
        h = _lib.hfo_fnv_scalar(h, name.encode(), int(isinstance(v, np.float32)), bits)
    return h


def register_bound(r1, t1, r2, t2, shmem, sm=PASCAL):
    return _lib.hfo_register_bound(r1, t1, r2, t2, shmem, sm["regs_per_sm"], sm["shmem_per_sm"], sm["max_threads_per_sm"])


def occupancy(regs, shmem, threads, sm=PASCAL):
    lim = C.c_int()
    b = _lib.hfo_occupancy(regs, shmem, threads, sm["regs_per_sm"], sm["shmem_per_sm"], sm["max_threads_per_sm"],
                           sm["max_blocks_per_sm"], C.byref(lim))
    return b, ["registers", "shared_memory", "threads", "block_slots"][lim.value]


def bn_stats(x, N, C_, HW):
    mean, var = np.empty(C_, np.float64), np.empty(C_, np.float64)
    _lib.hfo_bn_stats(np.ascontiguousarray(x, np.float32).ctypes.data, N, C_, HW, mean.ctypes.data, var.ctypes.data)
    return mean, var


def hist(x):
    out = np.empty(64, np.int32)
    x = np.ascontiguousarray(x, np.float32)
    _lib.hfo_hist(x.ctypes.data, x.size, out.ctypes.data)
    return out


def maxpool(x, NC, H, W):
    OH, OW = (H - 1) // 2 + 1, (W - 1) // 2 + 1
    y, idx = np.empty(NC * OH * OW, np.float32), np.empty(NC * OH * OW, np.int32)
    _lib.hfo_maxpool(np.ascontiguousarray(x, np.float32).ctypes.data, NC, H, W, y.ctypes.data, idx.ctypes.data)
    return y, idx


def upsample(x, NC, IH, IW):
    y = np.empty(NC * 4 * IH * IW, np.float32)
    _lib.hfo_upsample(np.ascontiguousarray(x, np.float32).ctypes.data, NC, IH, IW, y.ctypes.data)
    return y


def im2col(x, NC, H, W):
    col = np.empty(NC * 9 * H * W, np.float32)
    _lib.hfo_im2col(np.ascontiguousarray(x, np.float32).ctypes.data, NC, H, W, col.ctypes.data)
    return col


# ---- the reference interpreter (run_functional, exec.cpp:958-965) ----------------------

def have_ref():
    return os.path.exists(REF)


def ref_run(cmd, *args, timeout=600):
    """Run oracle/_ref/mkfuse_ref; returns (digest, seconds, dump_text)."""
    with tempfile.TemporaryDirectory() as d:
        dump = os.path.join(d, "dump.img")
        r = subprocess.run([REF, cmd, *map(str, args), "--dump", dump, "--time"], capture_output=True, text=True,
                           timeout=timeout)
        if r.returncode != 0:
            raise RuntimeError(r.stderr.strip())
        kv = dict(line.split(" = ") for line in r.stdout.strip().splitlines())
        return kv["digest"], float(kv["seconds"]), open(dump).read()
