"""ctypes binding of libfcg.so (the C ABI in include/fcg.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every entry point of the package raises.  The library is loaded
from the package directory (built in-tree by _build.py).
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libfcg.so"

FCG_D, FCG_DR, FCG_RH, FCG_MAX_BLOCKS = 128, 64, 64, 8
FCG_OK, FCG_ERR_CAPACITY, FCG_ERR_ARG, FCG_ERR_CUDA = 0, 1, 2, 3
FCG_FMT_FP32, FCG_FMT_W16 = 0, 1
FCG_STATUS_WORDS = 8
FCG_SCHED_SEGRED, FCG_SCHED_SCATTER = 0, 1   # include/fcg.h
ST_EDGES, ST_OVERFLOW, ST_MAXDEG, ST_BLOWUP, ST_BLOWUP_STEP, ST_EDGE_SUM, ST_BUILDS, ST_ARRIVE = range(8)

_f = C.POINTER(C.c_float)
_u16 = C.POINTER(C.c_uint16)
_i32 = C.POINTER(C.c_int32)


class FcgBlock(C.Structure):
    _fields_ = [(n, _f) for n in (
        "pre_w", "pre_wt", "pre_b", "f0_w", "f0_wt", "f0_b", "f1_w", "f1_wt", "f1_b",
        "p0_w", "p0_wt", "p0_b", "p1_w", "p1_wt", "p1_b")] + \
        [(n, _u16) for n in ("pre_h", "f0_h", "f1_h", "p0_h", "p1_h")] + \
        [(n, _f) for n in ("pre_s", "f0_s", "f1_s", "p0_s", "p1_s")] + \
        [("f0_img", _u16), ("f1_img", _u16), ("f0_exp", C.c_int), ("f1_exp", C.c_int),
         ("pre_img", _u16), ("p0_img", _u16), ("p1_img", _u16),
         ("pre_exp", C.c_int), ("p0_exp", C.c_int), ("p1_exp", C.c_int),
         ("f_hexp", C.c_int), ("f_dbexp", C.c_int), ("f1_qmax", C.c_float),
         ("f_vexp", C.c_int)]


class FcgModel(C.Structure):
    _fields_ = [
        ("format", C.c_int), ("num_blocks", C.c_int), ("num_types", C.c_int),
        ("cutoff", C.c_float), ("gamma", C.c_float),
        ("centers", _f), ("embedding", _f),
        ("blocks", FcgBlock * FCG_MAX_BLOCKS),
        ("r0_w", _f), ("r0_wt", _f), ("r0_b", _f), ("r1_w", _f), ("r1_b", C.c_float),
        ("r0_h", _u16), ("r0_s", _f), ("r1_h", _u16), ("r1_s", C.c_float),
        ("r0_img", _u16), ("r0_exp", C.c_int),
        ("pre0_table", _f), ("pre0_amax", C.c_float),
    ]


class FcgPrior(C.Structure):
    _fields_ = [("num_bonds", C.c_int), ("bond_i", _i32), ("bond_j", _i32),
                ("k", _f), ("r0", _f), ("inc_ptr", _i32), ("inc_bond", _i32),
                ("inc_sign", _i32)]


class FcgMdParams(C.Structure):
    _fields_ = [("half_dt", C.c_float), ("c1", C.c_float), ("c2_num", C.c_float),
                ("seed", C.c_uint64), ("rep_offset", C.c_int), ("neighbor_stride", C.c_int),
                ("schedule", C.c_int)]


_VP = C.c_void_p
_SIGS = {
    "fcg_abi_version": (C.c_int, []),
    "fcg_memcpy_async": (C.c_int, [_VP, _VP, C.c_size_t, _VP]),
    "fcg_last_error": (C.c_char_p, []),
    "fcg_profile_enable": (C.c_int, [C.c_int]),
    "fcg_debug_phase_buffer": (C.c_int, [_VP]),
    "fcg_profile_read": (C.c_int, [C.c_int, C.c_char_p, C.POINTER(C.c_double),
                                   C.POINTER(C.c_int)]),
    "fcg_nbr_workspace_bytes": (C.c_size_t, [C.c_int, C.c_int]),
    "fcg_nbr_build": (C.c_int, [_VP, C.c_int, C.c_int, C.c_double, C.c_int64, _VP, _VP, _VP,
                                _VP, _VP, _VP, C.c_size_t, _VP]),
    "fcg_nbr_build_f64": (C.c_int, [_VP, C.c_int, C.c_int, C.c_double, C.c_int64, _VP, _VP,
                                    _VP, _VP, _VP, _VP, C.c_size_t, _VP]),
    "fcg_group_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int]),
    "fcg_group_by": (C.c_int, [_VP, C.c_int64, C.c_int, _VP, _VP, _VP, C.c_size_t, _VP]),
    "fcg_segment_reduce_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int, C.c_int]),
    "fcg_segment_reduce": (C.c_int, [_VP, C.c_int64, C.c_int, _VP, C.c_int, _VP, _VP,
                                     C.c_size_t, _VP]),
    "fcg_segment_reduce_f64": (C.c_int, [_VP, C.c_int64, C.c_int, _VP, C.c_int, _VP, _VP,
                                         C.c_size_t, _VP]),
    "fcg_ef_workspace_bytes": (C.c_size_t, [C.POINTER(FcgModel), C.c_int, C.c_int, C.c_int64]),
    "fcg_energy_forces": (C.c_int, [C.POINTER(FcgModel), _VP, _VP, C.c_int, C.c_int, _VP, _VP,
                                    _VP, _VP, C.c_int64, _VP, _VP, _VP, _VP, C.c_size_t, _VP]),
    "fcg_energy_forces_sched": (C.c_int, [C.POINTER(FcgModel), _VP, _VP, C.c_int, C.c_int, _VP,
                                          _VP, _VP, _VP, C.c_int64, _VP, _VP, _VP, _VP,
                                          C.c_size_t, C.c_int, _VP]),
    "fcg_normal_noise": (C.c_int, [C.c_uint64, C.c_int, _VP, C.c_int, C.c_int, _VP, _VP]),
    "fcg_calib_errors": (C.c_int, [_VP, C.c_int, C.c_int, _VP, C.c_int, _VP, _VP, _VP]),
    "fcg_langevin_baoa": (C.c_int, [C.POINTER(FcgMdParams), _VP, C.c_int, C.c_int, _VP, _VP,
                                    _VP, _VP, _VP]),
    "fcg_half_kick": (C.c_int, [C.POINTER(FcgMdParams), _VP, C.c_int, C.c_int, _VP, _VP, _VP]),
    "fcg_prior_forces": (C.c_int, [C.POINTER(FcgPrior), _VP, C.c_int, C.c_int, _VP, _VP, _VP]),
    "fcg_selftest_mma": (C.c_int, [_VP, _VP, _VP, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_int, C.c_int, C.c_int, _VP]),
    "fcg_kabsch": (C.c_int, [_VP, _VP, C.c_int, C.c_int, _VP, _VP, _VP, _VP, _VP]),
    "fcg_gdt_counts": (C.c_int, [_VP, _VP, C.c_int, C.c_int, _VP, C.c_int, _VP, _VP, _VP]),
    "fcg_native_q": (C.c_int, [_VP, C.c_int, C.c_int, _VP, _VP, C.c_int, C.c_double, C.c_double,
                               _VP, _VP]),
    "fcg_format_xyz": (C.c_int64, [_VP, _VP, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_char_p,
                                   C.c_int64, C.c_int]),
    "fcg_md_workspace_bytes": (C.c_size_t, [C.POINTER(FcgModel), C.c_int, C.c_int, C.c_int64]),
    "fcg_md_step": (C.c_int, [C.POINTER(FcgModel), C.POINTER(FcgPrior), C.POINTER(FcgMdParams),
                              _VP, _VP, C.c_int, C.c_int, C.c_double, C.c_int64, _VP, _VP, _VP,
                              _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, C.c_size_t, _VP]),
}

EXPORTED = tuple(_SIGS)


class CapacityError(RuntimeError):
    """Edge capacity exceeded; buffers must grow (FCG_ERR_CAPACITY)."""


_lib = None


def load(path: os.PathLike | None = None):
    """Load (once) and return the ctypes handle; raises if the .so is absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # FCG_LIB_PATH: diagnostic A/B override (another in-tree build of the same ABI)
    p = Path(path) if path else Path(os.environ.get("FCG_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"libfcg.so not found at {p}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fcg_abi_version() != 1:
        raise RuntimeError("libfcg.so ABI version mismatch")
    if path is None:
        _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == FCG_OK:
        return
    msg = (load().fcg_last_error() or b"").decode()
    if rc == FCG_ERR_ARG:
        raise ValueError(f"{what}: {msg}")
    if rc == FCG_ERR_CAPACITY:
        raise CapacityError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def fptr(t) -> C.POINTER(C.c_float):
    return C.cast(C.c_void_p(t.data_ptr()), _f) if t is not None else _f()


def u16ptr(t):
    return C.cast(C.c_void_p(t.data_ptr()), _u16) if t is not None else _u16()


def i32ptr(t):
    return C.cast(C.c_void_p(t.data_ptr()), _i32) if t is not None else _i32()


def vp(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p()


def format_xyz(positions, types, step: int, replica0: int = 0, nthreads: int = 0) -> bytes:
    """Trajectory frames of positions[R][N][3] (host float32) in the
    reference's bytes (md.py:224-228), formatted in C (no GIL held)."""
    import numpy as np
    pos = np.ascontiguousarray(positions, dtype=np.float32)
    if pos.ndim == 2:
        pos = pos[None]
    typ = np.ascontiguousarray(types, dtype=np.int32)
    R, N = pos.shape[0], pos.shape[1]
    lib = load()
    args = (C.c_void_p(pos.ctypes.data), C.c_void_p(typ.ctypes.data), R, N, int(step),
            int(replica0))
    need = -lib.fcg_format_xyz(*args, None, 0, nthreads)
    if need < 0:
        raise ValueError((lib.fcg_last_error() or b"").decode())
    buf = C.create_string_buffer(int(need))
    n = lib.fcg_format_xyz(*args, buf, need, nthreads)
    if n < 0:
        raise RuntimeError("fcg_format_xyz: buffer too small")
    return buf.raw[:n]


def profile_read(max_classes: int = 32) -> dict:
    """{kernel class: (total_ms, launches)} from the built-in profiler."""
    lib = load()
    names = C.create_string_buffer(32 * max_classes)
    tot = (C.c_double * max_classes)()
    cnt = (C.c_int * max_classes)()
    k = lib.fcg_profile_read(max_classes, names, tot, cnt)
    out = {}
    for i in range(max(k, 0)):
        nm = names.raw[32 * i:32 * (i + 1)].split(b"\0", 1)[0].decode()
        out[nm] = (float(tot[i]), int(cnt[i]))
    return out
