"""ctypes binding of libhx.so (include/hx.h).  No CPU fallback: a missing or unusable library raises.

The library is built in-tree by `make` (or `__graft_entry__.build()`) for sm_100a.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("HX_LIB", _HERE / "libhx.so"))

HX_PENCIL_STANDARD = 0
HX_PENCIL_COMMUTING = 1
HX_PENCIL_GENERAL = 2
HX_ST_OK, HX_ST_NOT_PD, HX_ST_NONFINITE, HX_ST_EMPTY = 0, 1, 2, 3

# every symbol declared in include/hx.h (checked by tests/test_boundary.py)
EXPORTED = (
    "hx_abi_version", "hx_last_error", "hx_device_count", "hx_ctx_create", "hx_ctx_create_priority",
    "hx_ctx_destroy",
    "hx_ctx_synchronize", "hx_cell_create", "hx_cell_destroy", "hx_eval_idos_batch",
    "hx_eval_idos_batch_device", "hx_eval_idos_batch_k", "hx_eval_idos_batch_device_k", "hx_eigvalsh_batch_device", "hx_smoothed_counts_device",
    "hx_sharp_counts_device", "hx_level_moments_device", "hx_sample_masks", "hx_sample_masks_device",
    "hx_uniforms", "hx_restrict_masks", "hx_assemble_device", "hx_restrict_masks_device",
    "hx_kernel_launches", "hx_set_option", "hx_clear_option", "hx_get_option",
    "hx_level_sums_fixed_device", "hx_fixed_finalize_device", "hx_level_sums_fixed", "hx_fixed_finalize",
)

HX_FX_LIMBS = 6  # include/hx.h: fixed-point limbs per grid point of the exact level sums


class HxError(RuntimeError):
    """A libhx call failed (CUDA error, bad argument, no device)."""


class CellDesc(C.Structure):
    _fields_ = [
        ("ndof", C.c_int32), ("nunits", C.c_int32),
        ("unit_of_dof", C.c_void_p), ("onsite", C.c_void_p),
        ("h_row_ptr", C.c_void_p), ("h_col", C.c_void_p), ("h_amp", C.c_void_p), ("h_disp", C.c_void_p),
        ("s_row_ptr", C.c_void_p), ("s_col", C.c_void_p), ("s_amp", C.c_void_p), ("s_disp", C.c_void_p),
        ("pencil", C.c_int32), ("eps0", C.c_double), ("t", C.c_double), ("s", C.c_double),
        ("area", C.c_double), ("sublattice", C.c_void_p), ("dof_pos", C.c_void_p),
    ]


class EGrid(C.Structure):
    _fields_ = [("e0", C.c_double), ("step", C.c_double), ("npts", C.c_int32), ("delta", C.c_double)]


_lib = None
_lock = threading.Lock()


def load():
    """Load libhx.so once; raise HxError if it is absent (never fall back to CPU code)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise HxError(f"libhx.so not found at {LIB_PATH}; build it with `make` (sm_100a CUDA extension)")
        lib = C.CDLL(str(LIB_PATH))
        vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
        sig = {
            "hx_abi_version": (C.c_int, []),
            "hx_kernel_launches": (C.c_int, [C.POINTER(u64)]),
            "hx_last_error": (C.c_char_p, []),
            "hx_set_option": (C.c_int, [C.c_char_p, i64]),
            "hx_clear_option": (C.c_int, [C.c_char_p]),
            "hx_get_option": (C.c_int, [C.c_char_p, i64, C.POINTER(i64)]),
            "hx_device_count": (C.c_int, [C.POINTER(i32)]),
            "hx_ctx_create": (C.c_int, [i32, C.POINTER(vp)]),
            "hx_ctx_create_priority": (C.c_int, [i32, i32, C.POINTER(vp)]),
            "hx_ctx_destroy": (C.c_int, [vp]),
            "hx_ctx_synchronize": (C.c_int, [vp]),
            "hx_cell_create": (C.c_int, [vp, C.POINTER(CellDesc), C.POINTER(vp)]),
            "hx_cell_destroy": (C.c_int, [vp]),
            "hx_eval_idos_batch": (C.c_int, [vp, vp, vp, i32, vp, i64, C.POINTER(EGrid), vp, vp, vp]),
            "hx_eval_sharp_batch": (C.c_int, [vp, vp, vp, i32, vp, i64, C.POINTER(EGrid), vp, vp, vp]),
            "hx_eval_idos_batch_device": (C.c_int, [vp, vp, vp, i32, vp, i64, C.POINTER(EGrid), vp, vp, vp, vp]),
            "hx_eval_idos_batch_k": (C.c_int, [vp, vp, vp, vp, i32, vp, i64, C.POINTER(EGrid), vp, vp]),
            "hx_eval_idos_batch_device_k": (C.c_int, [vp, vp, vp, vp, i32, vp, i64, C.POINTER(EGrid), vp, vp, vp]),
            "hx_eigvalsh_batch_device": (C.c_int, [vp, i32, i64, vp, vp, vp, vp, vp]),
            "hx_smoothed_counts_device": (C.c_int, [vp, vp, i64, C.POINTER(EGrid), vp, vp]),
            "hx_sharp_counts_device": (C.c_int, [vp, vp, i64, C.POINTER(EGrid), vp, vp]),
            "hx_level_moments_device": (C.c_int, [vp, vp, i64, i32, vp, vp, vp, vp]),
            "hx_level_sums_fixed_device": (C.c_int, [vp, vp, i64, i32, vp, vp, vp]),
            "hx_fixed_finalize_device": (C.c_int, [vp, i32, dbl, vp, vp]),
            "hx_level_sums_fixed": (C.c_int, [vp, vp, i64, i32, vp, vp]),
            "hx_fixed_finalize": (C.c_int, [vp, i32, dbl, vp]),
            "hx_sample_masks": (C.c_int, [u64, u64, u64, i64, dbl, i32, vp, i32]),
            "hx_sample_masks_device": (C.c_int, [u64, u64, u64, i64, dbl, i32, vp, vp]),
            "hx_uniforms": (C.c_int, [u64, u64, u64, i64, vp]),
            "hx_restrict_masks": (C.c_int, [vp, i64, i32, vp, vp, i32, vp]),
            "hx_assemble_device": (C.c_int, [vp, vp, vp, i32, vp, i64, vp, vp, vp, vp]),
            "hx_restrict_masks_device": (C.c_int, [vp, i64, i32, vp, vp, i32, vp, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str):
    if rc != 0:
        msg = load().hx_last_error().decode(errors="replace")
        raise HxError(f"{what} failed (rc={rc}): {msg}")


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a is not None and a.size else 0


def host_sample_masks(seed: int, level: int, rep0: int, count: int, p: float, nunits: int, threads: int = 0):
    """uint64 words [count, words] of vacancy masks (disorder.py:71-81), bit-exact with numpy."""
    words = max(1, (nunits + 63) // 64)
    out = np.zeros((count, words), dtype=np.uint64)
    check(load().hx_sample_masks(seed, level, rep0, count, p, nunits, ptr(out), threads), "hx_sample_masks")
    return out


def uniforms(seed: int, level: int, rep: int, count: int) -> np.ndarray:
    out = np.empty(count)
    check(load().hx_uniforms(seed, level, rep, count, ptr(out)), "hx_uniforms")
    return out


def restrict_masks(parent_words: np.ndarray, parent_units: int, assign: np.ndarray, umap: np.ndarray,
                   sub_units: int) -> np.ndarray:
    """[n, 4, sub_words] quarter masks (disorder.py:84-94)."""
    parent_words = np.ascontiguousarray(parent_words, dtype=np.uint64)
    n = parent_words.shape[0]
    sw = max(1, (sub_units + 63) // 64)
    out = np.zeros((n, 4, sw), dtype=np.uint64)
    a = np.ascontiguousarray(assign, dtype=np.int32)
    m = np.ascontiguousarray(umap, dtype=np.int32)
    check(load().hx_restrict_masks(ptr(parent_words), n, parent_units, ptr(a), ptr(m), sub_units, ptr(out)),
          "hx_restrict_masks")
    return out


def fixed_sums(full: np.ndarray, quarters: np.ndarray | None = None, center: np.ndarray | None = None) -> np.ndarray:
    """Exact fixed-point limbs [npts, HX_FX_LIMBS] of sum_m term_m (center None) or sum_m (term_m - center)^2,
    term = full - 0.25 * sum_r quarters[:, r] (hx_level_sums_fixed, host twin of the device kernel)."""
    full = np.ascontiguousarray(full, dtype=np.float64)
    M, npts = full.shape
    q = None if quarters is None else np.ascontiguousarray(quarters, dtype=np.float64).reshape(M, 4, npts)
    c = None if center is None else np.ascontiguousarray(center, dtype=np.float64).reshape(npts)
    out = np.zeros((npts, HX_FX_LIMBS), dtype=np.int64)
    check(load().hx_level_sums_fixed(ptr(full), ptr(q) if q is not None else 0, M, npts,
                                     ptr(c) if c is not None else 0, ptr(out)), "hx_level_sums_fixed")
    return out


def fixed_finalize(limbs: np.ndarray, divisor: float) -> np.ndarray:
    """value(limbs) / divisor per grid point (NaN for divisor <= 0)."""
    limbs = np.ascontiguousarray(limbs, dtype=np.int64).reshape(-1, HX_FX_LIMBS)
    out = np.empty(limbs.shape[0])
    check(load().hx_fixed_finalize(ptr(limbs), limbs.shape[0], float(divisor), ptr(out)), "hx_fixed_finalize")
    return out


def set_option(name: str, value: int):
    check(load().hx_set_option(name.encode(), int(value)), f"hx_set_option({name})")


def clear_option(name: str | None = None):
    check(load().hx_clear_option(None if name is None else name.encode()), "hx_clear_option")


def get_option(name: str, default: int = -1) -> int:
    v = C.c_int64(0)
    check(load().hx_get_option(name.encode(), int(default), C.byref(v)), "hx_get_option")
    return int(v.value)


class options:
    """Context manager forcing libhx path knobs (hx_set_option), restoring them on exit:
    `with options(HX_CHASE_RNW=4): ...`."""

    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        for k, v in self.kv.items():
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k in self.kv:
            clear_option(k)


def kernel_launches() -> int:
    n = C.c_uint64(0)
    check(load().hx_kernel_launches(C.byref(n)), "hx_kernel_launches")
    return int(n.value)


class Device:
    """One hx_ctx per CUDA device (created lazily, process-wide)."""

    _ctxs: dict = {}

    @classmethod
    def ctx(cls, device: int = 0):
        if device not in cls._ctxs:
            lib = load()
            h = C.c_void_p()
            check(lib.hx_ctx_create(device, C.byref(h)), "hx_ctx_create")
            cls._ctxs[device] = h
        return cls._ctxs[device]

    _pools: dict = {}

    @classmethod
    def new_ctx(cls, device: int = 0, priority: int = 0):
        """An additional, independent context (own buffers and work stream) for concurrent work."""
        h = C.c_void_p()
        check(load().hx_ctx_create_priority(device, priority, C.byref(h)), "hx_ctx_create_priority")
        return h

    @classmethod
    def lane(cls, device: int, i: int, high=None):
        """Context i of the per-device pool used to evaluate independent groups concurrently.  Default:
        lane 0 on a high-priority stream, the others normal; `high` picks the pool explicitly: True / False
        (greatest / default priority) or an int stream priority (clamped to the device's range)."""
        if high is None:
            high = i == 0
        prio = high if isinstance(high, int) and not isinstance(high, bool) else (-100 if high else 0)
        pool = cls._pools.setdefault((device, prio), [])
        while len(pool) <= i:
            pool.append(cls.new_ctx(device, prio))  # -100: clamped to the greatest priority
        return pool[i]

    @classmethod
    def count(cls) -> int:
        n = C.c_int32(0)
        load().hx_device_count(C.byref(n))
        return int(n.value)
