"""ctypes binding of libetc_b200.so (the C ABI declared in include/etc_b200.h).

There is no CPU fallback: if the shared library is missing, cannot be
loaded, or no CUDA device is visible, every entry point raises
`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libetc_b200.so"

ETC_OK, ETC_BREAKDOWN, ETC_CONFIG, ETC_CUDA, ETC_PIVOT = range(5)
PRECOND_KINDS = {"fct": 0, "jacobi": 1, "none": 2}  # ETC_PRECOND_* (include/etc_b200.h)

# every symbol include/etc_b200.h declares (tests check the .so exports them)
EXPORTS = (
    "etc_last_error", "etc_version", "etc_plan_create", "etc_plan_destroy",
    "etc_plan_device_bytes", "etc_load_field", "etc_select_axis",
    "etc_coefficient_stats", "etc_set_reference", "etc_solve", "etc_keep_solution",
    "etc_set_precond", "etc_set_precision", "etc_get_solution",
    "etc_apply_operator", "etc_dct2_xy", "etc_dct3_xy", "etc_thomas",
    "etc_apply_precond", "etc_build_rhs", "etc_profile", "etc_profile_read",
    "etc_voxelize_balls", "etc_voxelize_fibres", "etc_fill_channels", "etc_slab_create", "etc_slab_load", "etc_slab_plane",
    "etc_slab_init", "etc_slab_run", "etc_slab_status", "etc_slab_fused", "etc_slab_p2p_ok", "etc_slab_xbuf",
    "etc_slab_set_peers", "etc_slab_set_ends_peers", "etc_slab_plane_ptr", "etc_ipc_handle", "etc_ipc_open", "etc_ipc_close",
    "etc_plan_bare", "etc_dct2_xy_f32", "etc_dct3_xy_f32", "etc_apply_precond_f32",
    "etc_op_last_error", "etc_op_reduce_parts", "etc_op_stencil", "etc_op_diagonal", "etc_op_faces", "etc_op_scale",
    "etc_op_permute", "etc_op_rhs", "etc_op_flux", "etc_op_thomas", "etc_op_elementwise", "etc_op_dots",
    "etc_op_pcg_update", "etc_op_xpby", "etc_op_minmax", "etc_op_dense", "etc_op_ssor",
)


class NativeUnavailable(RuntimeError):
    """The CUDA extension could not be loaded (no fallback exists)."""


class SolveInfo(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("status", C.c_int),
        ("breakdown_iter", C.c_int),
        ("breakdown_kind", C.c_int),
        ("pad_", C.c_int),
        ("kappa_eff", C.c_double),
        ("flux_sum", C.c_double),
        ("norm_b", C.c_double),
        ("device_ms", C.c_double),
    ]


_lib = None
_lock = threading.Lock()

_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_DP = C.POINTER(C.c_double)
_L = C.c_longlong

_SIGS = {
    "etc_last_error": (C.c_char_p, []),
    "etc_version": (_I, []),
    "etc_plan_create": (_I, [C.POINTER(_P), _I, _I, _I, _D, _D, _D, _P]),
    "etc_plan_destroy": (_I, [_P]),
    "etc_plan_device_bytes": (C.c_size_t, [_P]),
    "etc_load_field": (_I, [_P, _P, _P, _P, _I]),
    "etc_select_axis": (_I, [_P, _I, C.POINTER(_I), _DP]),
    "etc_coefficient_stats": (_I, [_P, _DP]),
    "etc_set_reference": (_I, [_P, _DP, _DP, _DP, _DP]),
    "etc_solve": (_I, [_P, _D, _D, _D, _I, C.POINTER(SolveInfo), _DP]),
    "etc_keep_solution": (_I, [_P, _I]),
    "etc_set_precond": (_I, [_P, _I]),
    "etc_set_precision": (_I, [_P, _I]),
    "etc_get_solution": (_I, [_P, _P, _I]),
    "etc_apply_operator": (_I, [_P, _P, _P]),
    "etc_dct2_xy": (_I, [_P, _P, _P]),
    "etc_dct3_xy": (_I, [_P, _P, _P]),
    "etc_thomas": (_I, [_P, _P]),
    "etc_apply_precond": (_I, [_P, _P, _P]),
    "etc_build_rhs": (_I, [_P, _D, _D, _P]),
    "etc_profile": (_I, [_P, _I]),
    "etc_profile_read": (_I, [_P, _DP, C.POINTER(C.c_longlong), _I]),
    "etc_voxelize_balls": (_I, [_P, _I, _DP, _I, _D, _P]),
    "etc_voxelize_fibres": (_I, [_P, _I, _DP, _I, _D, _I, _P]),
    "etc_fill_channels": (_I, [_P, _P, _P, _I, _I, _D, _D, _D, _P]),
    "etc_slab_create": (_I, [C.POINTER(_P), _I, _I, _I, _I, _I, _I, _I, _D, _D, _D, _P]),
    "etc_slab_load": (_I, [_P, _P, _P, _P, _I]),
    "etc_slab_plane": (_I, [_P, _I, _I, _P, _I]),
    "etc_slab_init": (_I, [_P, _D, _D, _D, _I, _P]),
    "etc_slab_run": (_I, [_P, _I, _I, _P]),
    "etc_slab_status": (_I, [_P, C.POINTER(SolveInfo), _DP]),
    "etc_slab_fused": (_I, [_P]),
    "etc_slab_p2p_ok": (_I, [_P]),
    "etc_slab_xbuf": (_I, [_P, _I, C.POINTER(_P)]),
    "etc_slab_set_peers": (_I, [_P, C.POINTER(_P), C.POINTER(_P)]),
    "etc_slab_set_ends_peers": (_I, [_P, C.POINTER(_P)]),
    "etc_slab_plane_ptr": (_I, [_P, _I, _I, C.POINTER(_P)]),
    "etc_ipc_handle": (_I, [_P, _P, _P, C.POINTER(C.c_size_t)]),
    "etc_ipc_open": (_I, [_P, C.POINTER(_P)]),
    "etc_ipc_close": (_I, [_P]),
    "etc_plan_bare": (_I, [_P]),
    "etc_dct2_xy_f32": (_I, [_P, _P, _P]),
    "etc_dct3_xy_f32": (_I, [_P, _P, _P]),
    "etc_apply_precond_f32": (_I, [_P, _P, _P]),
    "etc_op_last_error": (C.c_char_p, []),
    "etc_op_reduce_parts": (_I, [_L]),
    "etc_op_stencil": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "etc_op_diagonal": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "etc_op_faces": (_I, [_I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P]),
    "etc_op_scale": (_I, [_I, _L, _P, _D, _P, _P]),
    "etc_op_permute": (_I, [_I, _I, _I, _I, _I, _P, _P, _P]),
    "etc_op_rhs": (_I, [_I, _I, _I, _I, _P, _P, _P, _D, _P, _D, _P, _P]),
    "etc_op_flux": (_I, [_I, _I, _I, _I, _P, _D, _P, _D, _I, _P, _P]),
    "etc_op_thomas": (_I, [_I, _I, _I, _I, _P, _P, _D, _P, _P, _P, C.POINTER(_I), _P]),
    "etc_op_elementwise": (_I, [_I, _I, _L, _P, _P, _P, _P]),
    "etc_op_dots": (_I, [_I, _I, _L, _P, _P, _P, _P, _P]),
    "etc_op_pcg_update": (_I, [_I, _L, _D, _P, _P, _P, _P, _P, _P, _P]),
    "etc_op_xpby": (_I, [_I, _L, _P, _D, _P, _P]),
    "etc_op_minmax": (_I, [_I, _L, _P, _P, _DP, _P]),
    "etc_op_dense": (_I, [_I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "etc_op_ssor": (_I, [_I, _I, _I, _P, _P, _P, _P, _D, _P, _P, _P]),
}


def load_library(path: Path | str | None = None) -> C.CDLL:
    """Load (once) and type the shared library.  Loading needs no GPU."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(
                f"{p} not found: build it with `python -m paper_2404_02433_b200.build`"
            )
        try:
            lib = C.CDLL(str(p))
        except OSError as exc:  # pragma: no cover - environment specific
            raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib() -> C.CDLL:
    return load_library()


def last_error() -> str:
    msg = lib().etc_last_error()
    return msg.decode() if msg else ""
