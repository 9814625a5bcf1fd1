"""ctypes front of the CPU oracle (lf_oracle.c) and of the reference's own
emitted C (oracle/_ref, built by make_ref.py).

TEST INFRASTRUCTURE ONLY -- the checker for tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs.  The product package
never imports this module.

Both libraries are compiled exactly as the reference compiles its emitted C
(``cc -std=c99 -O1``, /root/reference/pkg/tests/c_oracle.py:95-97): no FP
contraction, IEEE double/float arithmetic, so results are bitwise those of
``loopforge.interp.interpret`` (pinned by tests/test_oracle.py).
"""

from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import os
import shutil
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "lf_oracle.c")
LIB = os.path.join(HERE, "liblf_oracle.so")
REF_DIR = os.path.join(HERE, "_ref")
REF_LIB = os.path.join(REF_DIR, "libref_kernels.so")

CFLAGS = ["-std=c99", "-O1", "-shared", "-fPIC"]


def cc():
    return shutil.which("cc") or shutil.which("gcc")


def build(force=False):
    if not force and os.path.exists(LIB) and \
            os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    subprocess.run([cc()] + CFLAGS + ["-o", LIB, SRC], check=True)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        P, I64, D, F = C.c_void_p, C.c_int64, C.c_double, C.c_float
        sig = {
            "lfo_fill_f64": [P, D, I64], "lfo_fill_f32": [P, F, I64],
            "lfo_axpy_f64": [P, P, D, I64], "lfo_axpy_f32": [P, P, F, I64],
            "lfo_matvec_f64": [P, P, P, I64, I64, I64],
            "lfo_semlap_f64": [P, P, P, P, I64, I64, I64],
            "lfo_sgemm_f32": [F, P, P, P, I64, I64, I64, I64, I64],
            "lfo_dgemm_f64": [D, P, P, P, I64, I64, I64, I64, I64],
            "lfo_sumsq_f64": [P, I64],
            "lfo_dssum_f64": [P, I64, I64, I64, I64, I64, I64, I64, P, P],
        }
        for name, args in sig.items():
            getattr(L, name).argtypes = args
            getattr(L, name).restype = None
        L.lfo_sumsq_f64.restype = D
        _lib = L
    return _lib


def _p(a):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(C.c_void_p)


def _parallel(fn, lo, hi, threads):
    """Run fn(a, b) over [lo, hi) split into `threads` chunks (ctypes drops
    the GIL during the C call, so chunks run on separate cores)."""
    threads = max(1, min(threads, hi - lo))
    if threads == 1:
        fn(lo, hi)
        return
    cuts = [lo + (hi - lo) * t // threads for t in range(threads + 1)]
    with cf.ThreadPoolExecutor(threads) as pool:
        list(pool.map(lambda t: fn(cuts[t], cuts[t + 1]), range(threads)))


# {{{ numpy-level oracle (flat buffers in the reference's layouts)

def fill(out, a):
    f = lib().lfo_fill_f64 if out.dtype == np.float64 else lib().lfo_fill_f32
    f(_p(out), a, out.size)
    return out


def axpy(y, x, alpha):
    f = lib().lfo_axpy_f64 if y.dtype == np.float64 else lib().lfo_axpy_f32
    f(_p(y), _p(x), alpha, y.size)
    return y


def matvec(y, a, x, n, rows=None, threads=1):
    lo, hi = rows or (0, n)
    _parallel(lambda r0, r1: lib().lfo_matvec_f64(_p(y), _p(a), _p(x), n,
                                                  r0, r1), lo, hi, threads)
    return y


def semlap(w, u, d, g, n, nelt, elems=None, threads=1):
    lo, hi = elems or (0, nelt)
    _parallel(lambda e0, e1: lib().lfo_semlap_f64(_p(w), _p(u), _p(d), _p(g),
                                                  n, e0, e1), lo, hi, threads)
    return w


def sgemm(alpha, a, b, c, l, m, n, cols=None, threads=1):
    lo, hi = cols or (0, n)
    f = lib().lfo_sgemm_f32 if c.dtype == np.float32 else lib().lfo_dgemm_f64
    _parallel(lambda j0, j1: f(alpha, _p(a), _p(b), _p(c), l, m, n, j0, j1),
              lo, hi, threads)
    return c


def dssum(w, n, ex, ey, ez, zlo=0, zhi=None, mode=0, plane_in=None,
          plane_out=None):
    """Q Q^T on element-local w (lf_oracle.c lfo_dssum_f64), in place."""
    p = n - 1
    if zhi is None:
        zhi = ez * p
    lib().lfo_dssum_f64(_p(w), n, ex, ey, ez, zlo, zhi, mode,
                        None if plane_in is None else _p(plane_in),
                        None if plane_out is None else _p(plane_out))
    return w


def sumsq(w):
    return lib().lfo_sumsq_f64(_p(w), w.size)

# }}}


# {{{ the reference's own emitted C (oracle/_ref)

_ref = None


def have_ref():
    return os.path.exists(REF_LIB)


def ref_lib():
    """The reference's emitted C for the fixture kernels (make_ref.py)."""
    global _ref
    if _ref is None:
        if not have_ref():
            raise FileNotFoundError(
                f"{REF_LIB} missing: run `python oracle/make_ref.py` in a "
                "container that has /root/reference")
        _ref = C.CDLL(REF_LIB)
    return _ref


def ref_fn(name, argtypes):
    f = getattr(ref_lib(), name)
    f.argtypes = argtypes
    f.restype = None
    return f

# }}}
