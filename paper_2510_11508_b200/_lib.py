"""ctypes binding of ``libnormint_b200.so`` (the C ABI in include/normint_b200.h).

The product path has no CPU fallback: if the library cannot be loaded, or no
CUDA device is present, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnormint_b200.so")

# status codes (include/normint_b200.h)
NI_OK = 0
NI_ERR_INVALID_ARG = 1
NI_ERR_EMPTY_MASK = 2
NI_ERR_NONUNIT_NORMAL = 3
NI_ERR_NONFINITE = 4
NI_ERR_WORKSPACE = 5
NI_ERR_CUDA = 6
NI_ERR_UNSUPPORTED = 7

# every exported symbol and its signature
_P = C.c_void_p
_I = C.c_int
_D = C.c_double
_SZ = C.c_size_t
_PSZ = C.POINTER(C.c_size_t)
_PI32 = C.POINTER(C.c_int32)

SIGNATURES = {
    "ni_last_error": ([], C.c_char_p),
    "ni_version": ([], C.c_char_p),
    "ni_launch_count": ([], C.c_longlong),
    "ni_fill_last_report": ([C.POINTER(C.c_double), C.POINTER(C.c_longlong), _PI32, _PI32, _PI32,
                             _PI32], _I),
    "ni_normalize": ([_P, _I, _P, _I, _I, _I, _P, _P, _P, _P], _I),
    "ni_components_workspace_size": ([_I, _I, _I, _PSZ], _I),
    "ni_components": ([_P, _P, _I, _I, _I, _I, _D, _I, _P, _P, _P, _P, _P, _SZ, _P], _I),
    "ni_coefficients": ([_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "ni_fill_workspace_size": ([_I, _I, _I, _I, _I, _I, _PSZ], _I),
    "ni_fill": ([_P, _I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _D, _I, _P, _P, _P, _P, _SZ,
                 _P], _I),
    "ni_fill_mg_workspace_size": ([_I, _I, _I, _I, _I, _PSZ], _I),
    "ni_fill_mg": ([_P, _I, _P, _P, _P, _P, _I, _I, _I, _I, _I, _D, _I, _P, _P, _P, _P, _SZ, _PSZ,
                    _P], _I),
    "ni_fill_mg_last_report": ([_PI32, _PI32, _PI32], _I),
    "ni_set_fill_profiling": ([_I], _I),
    "ni_fill_mg_last_profile": ([C.POINTER(C.c_double), C.POINTER(C.c_longlong)], _I),
    "ni_edge_weights": ([_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _D, _D, _D, _P, _P, _P],
                        _I),
    "ni_pair_energy_workspace_size": ([_I, _PSZ], _I),
    "ni_pair_energy": ([_P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _SZ, _P], _I),
    "ni_inter_edges_workspace_size": ([_I, _I, _I, _I, _PSZ], _I),
    "ni_inter_edges": ([_P, _P, _I, _I, _I, _I, _P, _P, _P, _SZ, _P], _I),
    "ni_keys_filter_workspace_size": ([_I, _PSZ], _I),
    "ni_keys_filter": ([_P, _I, _P, _P, _I, _I, _I, _P, _P, _P, _SZ, _P], _I),
    "ni_quotient_workspace_size": ([_I, _I, _I, _PSZ], _I),
    "ni_quotient_build": ([_P, _I, _P, _I, _I, _I, _I, _I, _P, _SZ, _PI32, _P, _P], _I),
    "ni_scale_step_workspace_size": ([_I, _I, _I, _PSZ], _I),
    "ni_scale_step": ([_P, _SZ, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _I, _I, _I, _I,
                       _I, _I, _I, _D, _D, _D, _D, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ,
                       _P], _I),
    "ni_loop_decide": ([_P, _P, _P, _I, _I, _I, _I, _D, _P, _P, _P, _P, _P, _I, _P, _P], _I),
    "ni_apply_shift": ([_P, _P, _P, _I, _I, _I, _P, _I, _P, _SZ, _P], _I),
    "ni_scale_step_fused": ([_P, _SZ, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P, _P, _P, _I, _I,
                             _I, _I, _I, _I, _I, _I, _D, _D, _D, _D, _I, _P, _P, _P, _P, _P,
                             _P, _P, _I, _D, _P, _P, _P, _P, _P, _I, _P, _P, _SZ, _P], _I),
    "ni_scale_fused_limits": ([_PI32, _PI32], _I),
    "ni_merge_workspace_size": ([_I, _I, _I, _PSZ], _I),
    "ni_merge": ([_P, _SZ, _I, _I, _I, _P, _P, _P, _I, _P, _I, _I, _P, _P, _P, _P, _P, _SZ, _P],
                 _I),
    "ni_decode_png16": ([_P, _I, _I, _I, _P, _P, _P], _I),
    "ni_evaluate_workspace_size": ([_I, _I, _I, _PSZ], _I),
    "ni_evaluate": ([_P, _P, _P, _I, _I, _I, _P, _P, _SZ, _P], _I),
    "ni_min_theoretical_made_workspace_size": ([_I, _I, _I, _PSZ], _I),
    "ni_min_theoretical_made": ([_P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _SZ, _P], _I),
    "ni_gauge_workspace_size": ([_I, _I, _I, _PSZ], _I),
    "ni_gauge": ([_P, _P, _I, _I, _I, _D, _P, _P, _SZ, _P], _I),
    "ni_copy_to_host": ([_P, _P, _SZ, _I, _P], _I),
    "ni_copy_from_host": ([_P, _P, _SZ, _I, _P], _I),
}

_lib = None


def load(path: str | None = None):
    """Load (once) and return the library handle; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("NI_LIB") or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"{p} is missing: build it with `python -m paper_2510_11508_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(p)
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def last_error() -> str:
    return load().ni_last_error().decode(errors="replace")


def check(status: int, what: str) -> None:
    """Map an ni_status to the reference's exception types."""
    if status == NI_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == NI_ERR_EMPTY_MASK:
        raise errors.EmptyMask(last_error())
    if status in (NI_ERR_NONUNIT_NORMAL, NI_ERR_NONFINITE, NI_ERR_INVALID_ARG):
        raise ValueError(last_error())
    raise errors.DeviceError(msg)


def size_query(fn, *args) -> int:
    out = C.c_size_t(0)
    check(fn(*args, C.byref(out)), fn.__name__)
    return int(out.value)


def launch_count() -> int:
    """Kernels this library has launched so far (host-side counter)."""
    return int(load().ni_launch_count())


def mg_report() -> dict:
    """Multigrid statistics of the last ni_fill_mg on this thread."""
    lv, vc = C.c_int32(0), C.c_int32(0)
    n = (C.c_int32 * 16)()
    load().ni_fill_mg_last_report(C.byref(lv), C.byref(vc), n)
    return {"levels": lv.value, "vcycles": vc.value, "unknowns": [n[i] for i in range(1, lv.value + 1)]}


def set_fill_profiling(on: bool) -> None:
    """Bracket the multigrid fill's stages with CUDA events (measurement only)."""
    check(load().ni_set_fill_profiling(int(bool(on))), "ni_set_fill_profiling")


def mg_profile() -> dict:
    """Per-stage device time of the last profiled ni_fill_mg on this thread:
    pass A, coarse levels, pass B, scalar step (ms summed over V-cycles), and
    the active unit pixels summed over V-cycles."""
    ms = (C.c_double * 4)()
    pxv = C.c_longlong(0)
    load().ni_fill_mg_last_profile(ms, C.byref(pxv))
    return {"pass_a_ms": ms[0], "coarse_ms": ms[1], "pass_b_ms": ms[2], "scalar_ms": ms[3],
            "px_vcycles": pxv.value}


def fill_report() -> dict:
    """Diagnostics of the last fill on this thread (see ni_fill_last_report)."""
    ms, pxi = C.c_double(0), C.c_longlong(0)
    mx, g, nt, npart = C.c_int32(0), C.c_int32(0), C.c_int32(0), C.c_int32(0)
    load().ni_fill_last_report(C.byref(ms), C.byref(pxi), C.byref(mx), C.byref(g), C.byref(nt),
                               C.byref(npart))
    return {"cg_ms": ms.value, "px_iters": pxi.value, "max_iters": mx.value, "grid": g.value,
            "ntiles": nt.value, "npartials": npart.value}
