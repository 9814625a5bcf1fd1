"""ctypes binding of the C ABI declared in include/loopforge_b200.h.

The shared library is the product: if it cannot be loaded the executor
raises -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

from ._loopforge import CodegenError, InterpError
from .build import LIB

ABI_VERSION = 1
LFB_OK, LFB_ERR_UNSUPPORTED, LFB_ERR_LAUNCH, LFB_ERR_ARG = 0, 1, 2, 3


class LfbLaunch(C.Structure):
    """Mirror of ``struct lfb_launch``."""

    _fields_ = [
        ("abi_version", C.c_int32),
        ("guard", C.c_int32),
        ("group_extent", C.c_int64 * 3),
        ("local_extent", C.c_int32 * 3),
        ("npts", C.c_int32),
        ("sm_count", C.c_int32),
        ("ctas_per_sm", C.c_int32),
        ("variant", C.c_int32),
        ("reserved", C.c_int32),
        ("sumsq", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_len", C.c_int64),
    ]


P = C.c_void_p
I32 = C.c_int
D = C.c_double
F = C.c_float
LP = C.POINTER(LfbLaunch)

# name -> argtypes (restype int unless listed in _RESTYPES)
SIGNATURES = {
    "lfb_abi_version": [],
    "lfb_last_error": [],
    "lfb_device_sm_count": [],
    "lfb_fill_f64": [P, D, I32, LP, P],
    "lfb_fill_f32": [P, F, I32, LP, P],
    "lfb_axpy_f64": [P, P, D, I32, LP, P],
    "lfb_axpy_f32": [P, P, F, I32, LP, P],
    "lfb_matvec_f64": [P, P, P, I32, LP, P],
    "lfb_semlap_f64": [P, P, P, P, I32, LP, P],
    "lfb_semlap_workspace": [I32, I32, LP],
    "lfb_dssum_f64": [P, I32, I32, I32, I32, I32, I32, I32, P, P, P],
    "lfb_sgemm_f32": [F, P, P, P, I32, I32, I32, LP, P],
    "lfb_sgemm_workspace": [I32, I32, I32],
    "lfb_dgemm_f64": [D, P, P, P, I32, I32, I32, LP, P],
    "lfb_probe_fp64": [P, I32, I32, I32, P],
    "lfb_probe_stream": [P, P, P, C.c_int64, P],
    "lfb_rtc_compile": [C.c_char_p, C.c_char_p, C.POINTER(C.c_char_p), I32,
                        P, C.POINTER(C.c_int64)],
    "lfb_module_load": [P, C.c_int64, C.c_char_p, C.POINTER(P)],
    "lfb_module_launch": [P, C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                          C.c_int32, C.POINTER(P), P],
    "lfb_module_unload": [P],
    "lfb_tmap_encode": [P, I32, I32, C.POINTER(C.c_int64),
                        C.POINTER(C.c_int64), C.POINTER(C.c_int32), I32, P],
}
_RESTYPES = {"lfb_last_error": C.c_char_p, "lfb_semlap_workspace": C.c_int64,
             "lfb_sgemm_workspace": C.c_int64}

_lib = None


def library_path():
    return LIB


def load(path=None):
    """Load (once) and type the shared library."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB
    if not os.path.exists(path):
        raise InterpError(
            f"B200 executor library missing ({path}); run "
            "`python -m paper_1503_07659_b200.build` (no CPU fallback)")
    lib = C.CDLL(path)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = _RESTYPES.get(name, C.c_int)
    if lib.lfb_abi_version() != ABI_VERSION:
        raise InterpError(
            f"ABI version mismatch: library {lib.lfb_abi_version()} "
            f"!= bindings {ABI_VERSION}")
    _lib = lib
    return lib


def last_error():
    return load().lfb_last_error().decode(errors="replace")


def check(rc, what):
    """Map an LFB status to the reference's exception types."""
    if rc == LFB_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == LFB_ERR_UNSUPPORTED:
        raise CodegenError(msg)
    raise InterpError(msg)


def make_launch(geometry=None, npts=0, variant=0, ctas_per_sm=0,
                sumsq=None, workspace=None, workspace_len=0):
    """Build an ``lfb_launch`` from a :class:`launch.Geometry`."""
    g = LfbLaunch()
    g.abi_version = ABI_VERSION
    if geometry is not None and geometry.parallel:
        g.guard = int(geometry.guard)
        for a in range(3):
            g.group_extent[a] = int(geometry.group_extent[a])
            g.local_extent[a] = int(geometry.local_extent[a])
    else:
        # no parallel tags (untransformed kernel): group_extent[0] = 0 lets
        # the executor choose its own decomposition
        for a in range(3):
            g.group_extent[a] = 0 if a == 0 else 1
            g.local_extent[a] = 1
    g.npts = int(npts)
    g.variant = int(variant)
    g.ctas_per_sm = int(ctas_per_sm)
    g.sumsq = sumsq
    g.workspace = workspace
    g.workspace_len = int(workspace_len)
    return g
