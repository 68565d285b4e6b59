"""Python host mirror of the hfuse C ABI (include/hfuse.h) over ctypes.

The names follow the reference interfaces they replace (mkfuse, /root/reference/proj):
``fuse`` = generate_fused + emit_source (fuser.hpp:70-77), ``Image`` = MemoryImage
(memimage.hpp:36-68), ``run`` = run_functional on the device (sim.hpp:43-52),
``search`` = search_config / fixed_partition_fuse (search.hpp:66-77). Errors raise
``HFuseError`` carrying the reference ErrCode name and source position, like the
reference's ``Error`` (error.hpp:43-57).

There is no CPU fallback: every device entry point goes through libhfuse.so, and importing
this module fails loudly when the in-tree library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhfuse.so")
CLI_PATH = os.path.join(_HERE, "bin", "hfuse")

CODE_NAMES = [
    "Ok", "Syntax", "UnknownIdentifier", "TypeMismatch", "DuplicateName", "UnresolvedCall",
    "UnresolvedLabel", "Recursion", "BadBarrierId", "MisalignedCount", "DimensionMismatch",
    "GridMismatch", "ThreadBudgetExceeded", "SharedMemoryOverflow", "DoesNotFit", "OutOfBounds",
    "DivideByZero", "BarrierDeadlock", "BarrierOverflow", "DivergentBarrier", "NothingFeasible",
    "IncompatibleFixedDims", "InvalidArgument", "Io", "Compile", "Device",
]

STYLES = {"structured": 0, "goto": 1, "sm100": 2}
TIME_MODES = {"single": 0, "sequential": 1, "two_stream": 2}

# Every symbol include/hfuse.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "hf_free", "hf_version", "hf_fuse", "hf_fuse_report", "hf_normalize", "hf_check", "hf_lower",
    "hf_emit_kernel", "hf_register_bound", "hf_occupancy", "hf_combined_utilization", "hf_device_count",
    "hf_get_device_props", "hf_build_fused", "hf_build_fused_opts", "hf_build_fused_regs", "hf_build_kernel", "hf_build_naive", "hf_build_vertical",
    "hf_module_get_info",
    "hf_module_source", "hf_module_entry", "hf_module_param", "hf_module_param_reads", "hf_module_barrier",
    "hf_module_cubin", "hf_launch", "hf_launch_ex", "hf_run_ex", "hf_module_free", "hf_image_parse", "hf_image_merge",
    "hf_image_materialize", "hf_image_upload", "hf_image_download", "hf_image_digest",
    "hf_image_serialize", "hf_image_count", "hf_image_entry", "hf_image_find",
    "hf_image_set_host", "hf_image_bytes", "hf_image_free", "hf_run", "hf_time", "hf_time_graph", "hf_profile",
    "hf_search", "hf_shard_pack", "hf_shard_reduce",
]

SLOT_KINDS = {"hist": 0, "bn": 1, "crypto": 2}


class HFuseError(Exception):
    def __init__(self, code: int, line: int, col: int, message: str):
        self.code = code
        self.name = CODE_NAMES[code] if 0 <= code < len(CODE_NAMES) else "Unknown"
        self.line, self.col, self.message = line, col, message
        where = f"{line}:{col}: " if line > 0 else ""
        super().__init__(f"[{self.name}] {where}{message}")


class _Err(C.Structure):
    _fields_ = [("code", C.c_int), ("line", C.c_int), ("col", C.c_int), ("message", C.c_char * 512)]


class _Barrier(C.Structure):
    _fields_ = [("id", C.c_int), ("count", C.c_int), ("owner", C.c_int), ("original", C.c_int)]


class _Occ(C.Structure):
    _fields_ = [("blocks_per_sm", C.c_int), ("limiting", C.c_int), ("achieved_warps", C.c_int),
                ("occupancy_fraction", C.c_double)]


class _ModInfo(C.Structure):
    _fields_ = [("threads", C.c_int), ("grid", C.c_int), ("smem_bytes", C.c_longlong),
                ("regs", C.c_int), ("local_bytes", C.c_int), ("blocks_per_sm", C.c_int),
                ("n_params", C.c_int), ("n_barriers", C.c_int), ("launch_regs", C.c_int),
                ("interval_regs", C.c_int * 2)]


class _FuseOpts(C.Structure):
    _fields_ = [("regcap", C.c_int), ("regs1", C.c_int), ("regs2", C.c_int), ("vgrid1", C.c_int),
                ("vgrid2", C.c_int), ("grid", C.c_int), ("min_blocks", C.c_int), ("split_grid", C.c_int)]


class _Timing(C.Structure):
    _fields_ = [("median_us", C.c_double), ("min_us", C.c_double), ("mean_us", C.c_double),
                ("max_us", C.c_double), ("reps", C.c_int), ("iqm_us", C.c_double)]


class _GraphTiming(C.Structure):
    _fields_ = [("mean_us", C.c_double), ("median_us", C.c_double), ("min_us", C.c_double),
                ("max_us", C.c_double), ("ci95_us", C.c_double), ("samples", C.c_int), ("reps", C.c_int)]


class _Eval(C.Structure):
    _fields_ = [("cycles", C.c_longlong), ("occupancy", C.c_double), ("utilization", C.c_double),
                ("us", C.c_double), ("regs", C.c_int)]


class _SearchOpts(C.Structure):
    _fields_ = [("d0", C.c_int), ("granularity", C.c_int), ("backend", C.c_int),
                ("profiler_cmd", C.c_char_p), ("grid", C.c_int), ("warmup", C.c_int),
                ("reps", C.c_int), ("flush_l2", C.c_int), ("measured_registers", C.c_int),
                ("specialize", C.c_int), ("n_extra_caps", C.c_int), ("extra_caps", C.POINTER(C.c_int)),
                ("out_style", C.c_int), ("interval_regs", C.c_int), ("budget_points", C.c_int),
                ("best_regs1", C.c_int), ("best_regs2", C.c_int), ("prefilter", C.c_int),
                ("prefilter_tol", C.c_double), ("model_csv", C.c_void_p)]


class _PackSrc(C.Structure):
    _fields_ = [("src", C.c_void_p), ("offset", C.c_longlong), ("cells", C.c_longlong)]


class _ReduceSlot(C.Structure):
    _fields_ = [("kind", C.c_int), ("channels", C.c_int), ("offset", C.c_longlong), ("cells", C.c_longlong),
                ("out_offset", C.c_longlong)]


class _Props(C.Structure):
    _fields_ = [("sms", C.c_int), ("cc_major", C.c_int), ("cc_minor", C.c_int),
                ("smem_per_sm", C.c_longlong), ("smem_per_block_optin", C.c_longlong),
                ("regs_per_sm", C.c_int), ("max_threads_per_sm", C.c_int), ("clock_khz", C.c_int),
                ("l2_bytes", C.c_longlong), ("name", C.c_char * 128)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"hfuse: {LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    vp, cp, ip = C.c_void_p, C.c_char_p, C.c_int
    E = C.POINTER(_Err)
    sig = {
        "hf_free": (None, [vp]),
        "hf_version": (cp, []),
        "hf_fuse": (ip, [cp, cp, ip, ip, ip, ip, cp, C.POINTER(vp), C.POINTER(_Barrier), ip, C.POINTER(ip), E]),
        "hf_fuse_report": (ip, [cp, cp, ip, ip, ip, cp, C.POINTER(vp), E]),
        "hf_normalize": (ip, [cp, cp, C.POINTER(vp), E]),
        "hf_check": (ip, [cp, ip, C.POINTER(vp), E]),
        "hf_lower": (ip, [cp, C.POINTER(vp), E]),
        "hf_emit_kernel": (ip, [cp, ip, C.POINTER(vp), E]),
        "hf_register_bound": (ip, [ip, ip, ip, ip, C.c_longlong, cp, C.POINTER(ip), E]),
        "hf_occupancy": (ip, [ip, C.c_longlong, ip, cp, C.POINTER(_Occ), E]),
        "hf_combined_utilization": (C.c_double, [C.c_double, C.c_longlong, C.c_double, C.c_longlong]),
        "hf_device_count": (ip, []),
        "hf_get_device_props": (ip, [C.POINTER(_Props), E]),
        "hf_build_fused": (ip, [cp, cp, ip, ip, ip, ip, ip, vp, C.POINTER(vp), E]),
        "hf_build_fused_opts": (ip, [cp, cp, ip, ip, C.POINTER(_FuseOpts), vp, C.POINTER(vp), E]),
        "hf_build_fused_regs": (ip, [cp, cp, ip, ip, ip, ip, ip, vp, C.POINTER(vp), E]),
        "hf_build_kernel": (ip, [cp, ip, ip, ip, vp, C.POINTER(vp), E]),
        "hf_build_naive": (ip, [cp, cp, ip, ip, ip, C.POINTER(vp), E]),
        "hf_build_vertical": (ip, [cp, cp, ip, vp, C.POINTER(vp), E]),
        "hf_module_get_info": (ip, [vp, C.POINTER(_ModInfo)]),
        "hf_module_source": (cp, [vp]),
        "hf_module_entry": (cp, [vp]),
        "hf_module_param": (ip, [vp, ip, C.POINTER(cp), C.POINTER(ip), C.POINTER(ip), C.POINTER(ip),
                                 C.POINTER(ip)]),
        "hf_module_param_reads": (ip, [vp, ip, C.POINTER(ip)]),
        "hf_module_barrier": (ip, [vp, ip, C.POINTER(_Barrier)]),
        "hf_module_cubin": (ip, [vp, C.POINTER(vp), C.POINTER(C.c_size_t)]),
        "hf_launch": (ip, [vp, ip, C.POINTER(vp), vp, E]),
        "hf_launch_ex": (ip, [vp, ip, C.POINTER(vp), vp, ip, E]),
        "hf_run_ex": (ip, [vp, vp, ip, vp, ip, E]),
        "hf_module_free": (None, [vp]),
        "hf_image_parse": (ip, [cp, ip, C.c_ulonglong, C.POINTER(vp), E]),
        "hf_image_merge": (ip, [vp, vp, E]),
        "hf_image_materialize": (ip, [vp, E]),
        "hf_image_upload": (ip, [vp, vp, E]),
        "hf_image_download": (ip, [vp, vp, E]),
        "hf_image_digest": (ip, [vp, C.POINTER(C.c_ulonglong), E]),
        "hf_image_serialize": (ip, [vp, C.POINTER(vp), E]),
        "hf_image_count": (ip, [vp]),
        "hf_image_entry": (ip, [vp, ip, C.POINTER(cp), C.POINTER(vp), C.POINTER(C.POINTER(C.c_int32)),
                                C.POINTER(C.c_longlong), C.POINTER(ip)]),
        "hf_image_find": (ip, [vp, cp, C.POINTER(vp), C.POINTER(C.POINTER(C.c_int32)),
                               C.POINTER(C.c_longlong), C.POINTER(ip)]),
        "hf_image_set_host": (ip, [vp, cp, vp, C.c_longlong, E]),
        "hf_image_bytes": (C.c_longlong, [vp]),
        "hf_image_free": (None, [vp]),
        "hf_run": (ip, [vp, vp, ip, vp, E]),
        "hf_time": (ip, [ip, vp, vp, vp, ip, ip, ip, ip, ip, vp, C.POINTER(_Timing), E]),
        "hf_time_graph": (ip, [ip, vp, vp, vp, ip, ip, ip, ip, vp, C.POINTER(_GraphTiming), E]),
        "hf_profile": (ip, [cp, cp, ip, ip, ip, vp, ip, ip, ip, ip, ip, C.POINTER(_Eval), E]),
        "hf_shard_pack": (ip, [C.POINTER(_PackSrc), ip, vp, vp, E]),
        "hf_shard_reduce": (ip, [vp, ip, C.c_longlong, C.POINTER(_ReduceSlot), ip, C.POINTER(C.c_double), vp, vp,
                                 E]),
        "hf_search": (ip, [cp, cp, vp, C.POINTER(_SearchOpts), C.POINTER(ip), C.POINTER(ip), C.POINTER(ip),
                           C.POINTER(C.c_longlong), C.POINTER(vp), C.POINTER(vp), E]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


def lib() -> C.CDLL:
    return _lib


def _check(rc: int, err: _Err) -> None:
    if rc != 0:
        raise HFuseError(err.code, err.line, err.col, err.message.decode(errors="replace"))


def _take(p: C.c_void_p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    _lib.hf_free(p)
    return s


def _b(s: Optional[str]) -> Optional[bytes]:
    return None if s is None else s.encode()


def _regcap(regcap) -> int:
    if regcap in (None, "off"):
        return -1
    if regcap == "auto":
        return 0
    return int(regcap)


@dataclass
class Barrier:
    id: int
    count: int
    owner: int
    original: int


# ---- compiler ---------------------------------------------------------------------------

def fuse(src1: str, src2: str, d1: int, d2: int, style: str = "goto", regcap="auto",
         sm: str = "pascal-like") -> Tuple[str, List[Barrier]]:
    out = C.c_void_p()
    table = (_Barrier * 16)()
    n = C.c_int()
    err = _Err()
    rc = _lib.hf_fuse(src1.encode(), src2.encode(), d1, d2, STYLES[style], _regcap(regcap), _b(sm),
                      C.byref(out), table, 16, C.byref(n), C.byref(err))
    _check(rc, err)
    return _take(out), [Barrier(t.id, t.count, t.owner, t.original) for t in table[: n.value]]


def fuse_report(src1: str, src2: str, d1: int, d2: int, regcap="auto", sm: str = "pascal-like") -> str:
    out, err = C.c_void_p(), _Err()
    _check(_lib.hf_fuse_report(src1.encode(), src2.encode(), d1, d2, _regcap(regcap), _b(sm),
                               C.byref(out), C.byref(err)), err)
    return _take(out)


def _text_call(fn, *args) -> str:
    out, err = C.c_void_p(), _Err()
    _check(fn(*args, C.byref(out), C.byref(err)), err)
    return _take(out)


def normalize(src: str, prefix: str = "") -> str:
    return _text_call(_lib.hf_normalize, src.encode(), prefix.encode())


def check(src: str, strict: bool = False) -> str:
    return _text_call(_lib.hf_check, src.encode(), int(strict))


def lower(src: str) -> str:
    """MK+ (B200 dialect) -> reference Mini-Kernel with identical semantics."""
    return _text_call(_lib.hf_lower, src.encode())


def emit_kernel(src: str, min_blocks: int = 0) -> str:
    return _text_call(_lib.hf_emit_kernel, src.encode(), min_blocks)


def register_bound(regs1: int, threads1: int, regs2: int, threads2: int, fused_shmem: int,
                   sm: str = "pascal-like") -> int:
    out, err = C.c_int(), _Err()
    _check(_lib.hf_register_bound(regs1, threads1, regs2, threads2, fused_shmem, _b(sm), C.byref(out),
                                  C.byref(err)), err)
    return out.value


def combined_utilization(u1: float, c1: int, u2: float, c2: int) -> float:
    """machine.cpp:285-289: cycle-weighted utilization of two kernels run back to back."""
    return _lib.hf_combined_utilization(u1, c1, u2, c2)


LIMITS = ["registers", "shared_memory", "threads", "block_slots"]


def occupancy(regs: int, shmem: int, threads: int, sm: str = "pascal-like") -> dict:
    o, err = _Occ(), _Err()
    _check(_lib.hf_occupancy(regs, shmem, threads, _b(sm), C.byref(o), C.byref(err)), err)
    return {"blocks_per_sm": o.blocks_per_sm, "limiting": LIMITS[o.limiting],
            "achieved_warps": o.achieved_warps, "occupancy_fraction": o.occupancy_fraction}


# ---- runtime ----------------------------------------------------------------------------

def device_count() -> int:
    return _lib.hf_device_count()


def device_props() -> dict:
    p, err = _Props(), _Err()
    _check(_lib.hf_get_device_props(C.byref(p), C.byref(err)), err)
    return {k: (getattr(p, k).decode() if k == "name" else getattr(p, k)) for k, _ in _Props._fields_}


def _stream(stream) -> Optional[int]:
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):  # torch.cuda.Stream
        return stream.cuda_stream
    return int(stream)


class Image:
    """A memory image (arrays + scalars) whose seeded arrays are generated in HBM."""

    def __init__(self, text: str = "", seed: Optional[int] = None):
        h, err = C.c_void_p(), _Err()
        _check(_lib.hf_image_parse(text.encode(), int(seed is not None), seed or 0, C.byref(h), C.byref(err)), err)
        self._h = h

    @classmethod
    def load(cls, *paths: str, seed: Optional[int] = None) -> "Image":
        img = cls("", seed)
        for p in paths:
            img.merge(cls(open(p).read(), seed))
        return img

    def merge(self, other: "Image") -> "Image":
        err = _Err()
        _check(_lib.hf_image_merge(self._h, other._h, C.byref(err)), err)
        return self

    def materialize(self) -> "Image":
        err = _Err()
        _check(_lib.hf_image_materialize(self._h, C.byref(err)), err)
        return self

    def upload(self, stream=None) -> "Image":
        err = _Err()
        _check(_lib.hf_image_upload(self._h, _stream(stream), C.byref(err)), err)
        return self

    def download(self, stream=None) -> "Image":
        err = _Err()
        _check(_lib.hf_image_download(self._h, _stream(stream), C.byref(err)), err)
        return self

    def digest(self) -> int:
        out, err = C.c_ulonglong(), _Err()
        _check(_lib.hf_image_digest(self._h, C.byref(out), C.byref(err)), err)
        return out.value

    def digest_hex(self) -> str:
        return f"{self.digest():016x}"

    def serialize(self) -> str:
        return _text_call(_lib.hf_image_serialize, self._h)

    def names(self) -> List[str]:
        out = []
        for i in range(_lib.hf_image_count(self._h)):
            n = C.c_char_p()
            _lib.hf_image_entry(self._h, i, C.byref(n), None, None, None, None)
            out.append(n.value.decode())
        return out

    def _find(self, name: str):
        dev, host, n, fl = C.c_void_p(), C.POINTER(C.c_int32)(), C.c_longlong(), C.c_int()
        rc = _lib.hf_image_find(self._h, name.encode(), C.byref(dev), C.byref(host), C.byref(n), C.byref(fl))
        if rc != 0:
            raise KeyError(name)
        return dev.value, host, n.value, bool(fl.value)

    def device_ptr(self, name: str) -> int:
        dev, _, _, _ = self._find(name)
        if not dev:
            raise HFuseError(22, 0, 0, f"array '{name}' is not on the device")
        return dev

    def array(self, name: str) -> np.ndarray:
        """Host copy (after download()/materialize()) as int32 or float32 numpy array."""
        _, host, n, fl = self._find(name)
        if not host:
            raise HFuseError(22, 0, 0, f"array '{name}' has no host copy")
        raw = np.ctypeslib.as_array(host, shape=(n,)).copy()
        return raw.view(np.float32) if fl else raw

    def set_array(self, name: str, values: np.ndarray) -> None:
        v = np.ascontiguousarray(values)
        assert v.itemsize == 4
        err = _Err()
        _check(_lib.hf_image_set_host(self._h, name.encode(), v.ctypes.data, v.size, C.byref(err)), err)

    @property
    def nbytes(self) -> int:
        return _lib.hf_image_bytes(self._h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:  # at interpreter exit the module globals may be gone
            _lib.hf_image_free(h)
            self._h = None


@dataclass
class ModuleInfo:
    threads: int
    grid: int
    smem_bytes: int
    regs: int
    local_bytes: int
    blocks_per_sm: int
    n_params: int
    n_barriers: int
    launch_regs: int = 0                 # per-interval budgets: registers per thread at launch
    interval_regs: Tuple[int, int] = (0, 0)


class Module:
    """A compiled sm_100a kernel (fused or unfused) bound to parameter names."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @classmethod
    def fused(cls, src1: str, src2: str, d1: int, d2: int, regcap="off", grid: int = 0,
              min_blocks: int = 0, specialize: Optional["Image"] = None) -> "Module":
        """specialize: fold that image's scalar values into the code (JIT specialization)."""
        h, err = C.c_void_p(), _Err()
        _check(_lib.hf_build_fused(src1.encode(), src2.encode(), d1, d2, _regcap(regcap), grid, min_blocks,
                                   specialize._h if specialize else None, C.byref(h), C.byref(err)), err)
        return cls(h)

    @classmethod
    def fused_opts(cls, src1: str, src2: str, d1: int, d2: int, regcap="off", regs=None, vgrid=None,
                   grid: int = 0, min_blocks: int = 0, specialize: Optional["Image"] = None,
                   split_grid: int = 0) -> "Module":
        """Every B200 option (hf_build_fused_opts): regcap, per-interval budgets regs=(r1, r2),
        dynamic interval scheduling vgrid=(virtual grid of member 1, of member 2), heterogeneous
        CTA partition split_grid (blocks below it fused, above it member 2 only)."""
        r1, r2 = regs or (0, 0)
        v1, v2 = vgrid or (0, 0)
        o = _FuseOpts(_regcap(regcap), r1, r2, v1, v2, grid, min_blocks, split_grid)
        h, err = C.c_void_p(), _Err()
        _check(_lib.hf_build_fused_opts(src1.encode(), src2.encode(), d1, d2, C.byref(o),
                                        specialize._h if specialize else None, C.byref(h), C.byref(err)), err)
        return cls(h)

    @classmethod
    def from_config(cls, src1: str, src2: str, cfg: dict, specialize: Optional["Image"] = None) -> "Module":
        """The fused module of a search / bench configuration dict: d1, d2, grid and one of
        reg_cap (None = uncapped), interval_regs (per-interval budgets) or split_grid
        (heterogeneous CTA partition, with reg_cap)."""
        if cfg.get("interval_regs"):
            return cls.fused_regs(src1, src2, cfg["d1"], cfg["d2"], *cfg["interval_regs"], grid=cfg["grid"],
                                  specialize=specialize)
        if cfg.get("split_grid"):
            return cls.fused_opts(src1, src2, cfg["d1"], cfg["d2"], regcap=cfg.get("reg_cap") or "off",
                                  grid=cfg["grid"], split_grid=cfg["split_grid"], specialize=specialize)
        return cls.fused(src1, src2, cfg["d1"], cfg["d2"], regcap=cfg.get("reg_cap") or "off", grid=cfg["grid"],
                         specialize=specialize)

    @classmethod
    def fused_regs(cls, src1: str, src2: str, d1: int, d2: int, regs1: int, regs2: int, grid: int = 0,
                   specialize: Optional["Image"] = None) -> "Module":
        """Per-interval register budgets: interval 1 runs with regs1, interval 2 with regs2
        registers per thread (setmaxnreg), instead of one cap for the whole fused kernel."""
        h, err = C.c_void_p(), _Err()
        _check(_lib.hf_build_fused_regs(src1.encode(), src2.encode(), d1, d2, regs1, regs2, grid,
                                        specialize._h if specialize else None, C.byref(h), C.byref(err)), err)
        return cls(h)

    @classmethod
    def kernel(cls, src: str, regcap=None, grid: int = 0, min_blocks: int = 0,
               specialize: Optional["Image"] = None) -> "Module":
        h, err = C.c_void_p(), _Err()
        # None: the kernel's own `//@ regcap=` annotation (if any); "off": no cap at all
        cap = -1 if regcap == "off" else (0 if regcap is None else int(regcap))
        _check(_lib.hf_build_kernel(src.encode(), cap, grid, min_blocks, specialize._h if specialize else None,
                                    C.byref(h), C.byref(err)), err)
        return cls(h)

    @classmethod
    def naive(cls, src1: str, src2: str, d1: int, d2: int, grid: int = 0) -> "Module":
        """The reference's goto-style fusion text compiled as-is (timing baseline only)."""
        h, err = C.c_void_p(), _Err()
        _check(_lib.hf_build_naive(src1.encode(), src2.encode(), d1, d2, grid, C.byref(h), C.byref(err)), err)
        return cls(h)

    @classmethod
    def vertical(cls, src1: str, src2: str, grid: int = 0, specialize: Optional["Image"] = None) -> "Module":
        """VFuse: both bodies back to back in one block (equal block dims)."""
        h, err = C.c_void_p(), _Err()
        _check(_lib.hf_build_vertical(src1.encode(), src2.encode(), grid, specialize._h if specialize else None,
                                      C.byref(h), C.byref(err)), err)
        return cls(h)

    @property
    def info(self) -> ModuleInfo:
        i = _ModInfo()
        _lib.hf_module_get_info(self._h, C.byref(i))
        vals = [getattr(i, f) for f, _ in _ModInfo._fields_]
        vals[-1] = tuple(vals[-1])
        return ModuleInfo(*vals)

    @property
    def source(self) -> str:
        return _lib.hf_module_source(self._h).decode()

    @property
    def entry(self) -> str:
        return _lib.hf_module_entry(self._h).decode()

    @property
    def params(self) -> List[dict]:
        out = []
        for i in range(self.info.n_params):
            n, a, f, w, sp, rd = C.c_char_p(), C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
            _lib.hf_module_param(self._h, i, C.byref(n), C.byref(a), C.byref(f), C.byref(w), C.byref(sp))
            _lib.hf_module_param_reads(self._h, i, C.byref(rd))
            # "read": an array whose prior contents the kernel observes (needs uploading)
            out.append({"name": n.value.decode(), "array": bool(a.value), "float": bool(f.value),
                        "written": bool(w.value), "specialized": bool(sp.value), "read": bool(rd.value)})
        return out

    @property
    def barriers(self) -> List[Barrier]:
        out = []
        for i in range(self.info.n_barriers):
            b = _Barrier()
            _lib.hf_module_barrier(self._h, i, C.byref(b))
            out.append(Barrier(b.id, b.count, b.owner, b.original))
        return out

    @property
    def cubin(self) -> bytes:
        p, n = C.c_void_p(), C.c_size_t()
        _lib.hf_module_cubin(self._h, C.byref(p), C.byref(n))
        return C.string_at(p, n.value)

    def run(self, img: Image, grid: int = 0, stream=None, overlap: bool = False) -> None:
        """overlap: programmatic dependent launch (HF_LAUNCH_OVERLAP) -- may start while the
        previous kernel of the stream drains; only for kernels independent of that one."""
        err = _Err()
        _check(_lib.hf_run_ex(self._h, img._h, grid, _stream(stream), int(overlap), C.byref(err)), err)

    def launch(self, args: Dict[str, object], grid: int = 0, stream=None, overlap: bool = False) -> None:
        """Raw launch: args maps parameter name -> device pointer (int / torch tensor) or scalar."""
        keep, ptrs = [], []
        for p in self.params:
            v = args[p["name"]]
            if p["array"]:
                cell = C.c_void_p(v.data_ptr() if hasattr(v, "data_ptr") else int(v))
            elif p["float"]:
                cell = C.c_float(float(v))
            else:
                cell = C.c_int32(int(v))
            keep.append(cell)
            ptrs.append(C.cast(C.pointer(cell), C.c_void_p))
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        err = _Err()
        _check(_lib.hf_launch_ex(self._h, grid, arr, _stream(stream), int(overlap), C.byref(err)), err)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.hf_module_free(h)
            self._h = None


def time(mode: str, a: Module, b: Optional[Module], img: Image, grid_a: int = 0, grid_b: int = 0,
         warmup: int = 3, reps: int = 10, flush_l2: bool = True, stream=None) -> dict:
    t, err = _Timing(), _Err()
    _check(_lib.hf_time(TIME_MODES[mode], a._h, b._h if b else None, img._h, grid_a, grid_b, warmup, reps,
                        int(flush_l2), _stream(stream), C.byref(t), C.byref(err)), err)
    return {"median_us": t.median_us, "min_us": t.min_us, "mean_us": t.mean_us, "max_us": t.max_us,
            "reps": t.reps, "iqm_us": t.iqm_us}


def shard_pack(sources, packed_ptr: int, stream=None) -> None:
    """One launch copying int32 device arrays into a packed buffer: sources = [(device pointer,
    cell offset, cells)] (the multi-GPU step's send buffer, include/hfuse.h hf_shard_pack)."""
    arr = (_PackSrc * max(1, len(sources)))(*[_PackSrc(p, o, n) for p, o, n in sources])
    err = _Err()
    _check(_lib.hf_shard_pack(arr, len(sources), C.c_void_p(packed_ptr), _stream(stream), C.byref(err)), err)


def shard_reduce(gathered_ptr: int, world: int, cells: int, slots, counts, out_ptr: int, stream=None) -> None:
    """One launch reducing an all-gathered [world, cells] int32 buffer: slots = [(kind, channels,
    cell offset, cells, out offset in 8-byte elements)], kind in SLOT_KINDS; counts = per-rank
    elements per channel for bn slots (include/hfuse.h hf_shard_reduce)."""
    arr = (_ReduceSlot * max(1, len(slots)))(*[_ReduceSlot(SLOT_KINDS.get(k, k), ch, o, n, oo)
                                                for k, ch, o, n, oo in slots])
    cnt = (C.c_double * max(1, len(counts or [])))(*(counts or [0.0]))
    err = _Err()
    _check(_lib.hf_shard_reduce(C.c_void_p(gathered_ptr), world, cells, arr, len(slots), cnt if counts else None,
                                C.c_void_p(out_ptr), _stream(stream), C.byref(err)), err)


def time_graph(mode: str, a: Module, b: Optional[Module], img: Image, grid_a: int = 0, grid_b: int = 0,
               reps: int = 20, samples: int = 7, stream=None) -> dict:
    """Graph protocol (hf_time_graph): `reps` back-to-back repetitions captured as one CUDA graph,
    launched `samples` times between consecutive events; per-repetition statistics over samples."""
    t, err = _GraphTiming(), _Err()
    _check(_lib.hf_time_graph(TIME_MODES[mode], a._h, b._h if b else None, img._h, grid_a, grid_b, reps, samples,
                              _stream(stream), C.byref(t), C.byref(err)), err)
    return {k: getattr(t, k) for k, _ in _GraphTiming._fields_}


def profile(src1: str, src2: str, d1: int, d2: int, img: Image, regcap="off", grid: int = 0,
            warmup: int = 3, reps: int = 10, flush_l2: bool = True, specialize: bool = False) -> dict:
    e, err = _Eval(), _Err()
    _check(_lib.hf_profile(src1.encode(), src2.encode(), d1, d2, _regcap(regcap), img._h, grid, warmup, reps,
                           int(flush_l2), int(specialize), C.byref(e), C.byref(err)), err)
    return {"cycles": e.cycles, "occupancy": e.occupancy, "utilization": e.utilization, "us": e.us,
            "regs": e.regs}


def _model(p) -> dict:
    """Pre-filter model rows: {"model": d1 -> predicted us, "member_us": d1 -> (t1, t2), with
    d1 = 0 holding the full-block times (T1, T2)}."""
    if not p:
        return {"model": {}, "member_us": {}}
    rows = [line.split(",") for line in _take(C.c_void_p(p)).strip().splitlines()[1:]]
    return {"model": {int(r[0]): float(r[1]) for r in rows if int(r[0]) > 0},
            "member_us": {int(r[0]): (float(r[2]), float(r[3])) for r in rows}}


def search(src1: str, src2: str, img: Optional[Image] = None, d0: int = 1024, granularity: int = 128,
           profiler_cmd: Optional[str] = None, grid: int = 0, warmup: int = 3, reps: int = 10,
           flush_l2: bool = True, measured_registers: bool = True, extra_caps: Sequence[int] = (),
           out_style: str = "structured", specialize: bool = False, interval_regs: bool = False,
           budget_points: int = 5, prefilter: int = 0, prefilter_tol: float = -1.0) -> dict:
    """interval_regs: also sweep per-interval register budgets (setmaxnreg) for warpgroup-
    aligned partitions; the best point's budgets come back as "interval_regs" (or None).
    prefilter: keep only the k partitions the B200 model predicts fastest (max of the two
    constituents timed alone at each interval size) plus those predicted within prefilter_tol
    (default 3 %) of the best; "model" maps d1 -> predicted us."""
    caps = (C.c_int * max(1, len(extra_caps)))(*extra_caps)
    o = _SearchOpts(d0, granularity, 1 if profiler_cmd else 0, _b(profiler_cmd), grid, warmup, reps,
                    int(flush_l2), int(measured_registers), int(specialize), len(extra_caps), caps,
                    STYLES[out_style], int(interval_regs), budget_points, 0, 0, prefilter, prefilter_tol,
                    None)
    d1, d2, cap, best = C.c_int(), C.c_int(), C.c_int(), C.c_longlong()
    trace, src, err = C.c_void_p(), C.c_void_p(), _Err()
    _check(_lib.hf_search(src1.encode(), src2.encode(), img._h if img else None, C.byref(o), C.byref(d1),
                          C.byref(d2), C.byref(cap), C.byref(best), C.byref(trace), C.byref(src),
                          C.byref(err)), err)
    csv = _take(trace)
    rows = []
    lines = csv.strip().splitlines()
    keys = lines[0].split(",")
    for line in lines[1:]:
        vals = line.split(",")
        rows.append({k: (v if k == "reg_cap" else float(v) if "." in v else int(v)) for k, v in zip(keys, vals)})
    return {"d1": d1.value, "d2": d2.value, "reg_cap": None if cap.value < 0 else cap.value,
            "interval_regs": (o.best_regs1, o.best_regs2) if o.best_regs1 > 0 else None,
            **_model(o.model_csv),
            "best_time": best.value, "trace_csv": csv, "trace": rows, "source": _take(src)}
