"""Pin the CPU oracle (oracle/lf_oracle.c) to the reference.

1. against the goldens the reference interpreter produced
   (tests/golden/make_golden.py), bitwise;
2. against the reference's own emitted C (oracle/_ref, make_ref.py) on
   larger seeded inputs, bitwise -- skipped when oracle/_ref was not built.
"""

import ctypes as C

import numpy as np
import pytest

import oracle
from conftest import Golden, golden_names


def _run_oracle(g):
    fam = g.meta["generator"].replace("_source", "")
    p = g.params
    bufs = {a: g.inp(a).copy() for a in g.args}
    if fam == "fill":
        oracle.fill(bufs["out"], bufs["a"].reshape(())[()])
        return {"out": bufs["out"]}
    if fam == "axpy":
        oracle.axpy(bufs["y"], bufs["x"], bufs["alpha"].reshape(())[()])
        return {"y": bufs["y"]}
    if fam == "matvec":
        oracle.matvec(bufs["y"], bufs["a"], bufs["x"], p["n"])
        return {"y": bufs["y"]}
    if fam == "semlap":
        n = g.meta["kwargs"]["n"]
        oracle.semlap(bufs["w"], bufs["u"], bufs["d"], bufs["g"], n,
                      p["nelt"])
        return {"w": bufs["w"]}
    if fam == "gemm":
        oracle.sgemm(bufs["alpha"].reshape(())[()], bufs["a"], bufs["b"],
                     bufs["c"], p["l"], p["m"], p["n"])
        return {"c": bufs["c"]}
    raise AssertionError(fam)


@pytest.mark.parametrize("name", [n for n in golden_names()
                                  if not n.startswith("gen_")])
def test_oracle_matches_reference_interpreter(name):
    g = Golden(name)
    got = _run_oracle(g)
    for out in g.outputs():
        want = g.out(out)
        assert got[out].dtype == want.dtype
        assert got[out].tobytes() == want.tobytes(), out


def test_golden_inputs_follow_make_env_recipe():
    """Seeded inputs are the reference's rng.random(shape)*2-1 in arg order
    (interp.py:115-119) -- the device env reproduces them the same way."""
    g = Golden("axpy_f64_n300")
    rng = np.random.default_rng(g.meta["seed"])
    x = rng.random((300,)) * 2 - 1       # y is in/out: never randomised
    assert np.array_equal(g.inp("x"), x)
    y = np.random.default_rng(100 + g.meta["seed"]).random((300,)) * 2 - 1
    assert np.array_equal(g.inp("y"), y)


needs_ref = pytest.mark.skipif(not oracle.have_ref(),
                               reason="oracle/_ref not built")

P, D, F, I = C.c_void_p, C.c_double, C.c_float, C.c_int


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


@needs_ref
def test_oracle_matches_emitted_c_semlap_n8():
    nelt, n = 96, 8
    rng = np.random.default_rng(11)
    u = rng.random(nelt * n**3) * 2 - 1
    g = rng.random(6 * nelt * n**3)
    d = rng.random(n * n) * 2 - 1
    w_ref = np.zeros_like(u)
    oracle.ref_fn("ref_semlap_n8", [P, P, P, P, I])(
        _p(w_ref), _p(u), _p(d), _p(g), nelt)
    w = np.zeros_like(u)
    oracle.semlap(w, u, d, g, n, nelt)
    assert w.tobytes() == w_ref.tobytes()


@needs_ref
@pytest.mark.parametrize("n", [2, 3, 4, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15,
                               16])
def test_oracle_matches_emitted_c_semlap_orders(n):
    nelt = 32
    rng = np.random.default_rng(n)
    u = rng.random(nelt * n**3) * 2 - 1
    g = rng.random(6 * nelt * n**3)
    d = rng.random(n * n) * 2 - 1
    w_ref = np.zeros_like(u)
    oracle.ref_fn(f"ref_semlap_n{n}", [P, P, P, P, I])(
        _p(w_ref), _p(u), _p(d), _p(g), nelt)
    w = np.zeros_like(u)
    oracle.semlap(w, u, d, g, n, nelt)
    assert w.tobytes() == w_ref.tobytes()


@needs_ref
def test_oracle_matches_emitted_c_streams_and_matvec():
    n = 1024 + 77
    rng = np.random.default_rng(5)
    x = rng.random(n) * 2 - 1
    y0 = rng.random(n) * 2 - 1
    out_ref = np.zeros(n)
    oracle.ref_fn("ref_fill_f64", [P, D, I])(_p(out_ref), 0.3, n)
    assert oracle.fill(np.zeros(n), 0.3).tobytes() == out_ref.tobytes()
    y_ref = y0.copy()
    oracle.ref_fn("ref_axpy_f64", [P, P, D, I])(_p(y_ref), _p(x), 1.7, n)
    assert oracle.axpy(y0.copy(), x, 1.7).tobytes() == y_ref.tobytes()
    nm = 512  # the matvec fixture assumes n mod 128 = 0
    a = rng.random(nm * nm)
    xv = rng.random(nm)
    y_ref = np.zeros(nm)
    oracle.ref_fn("ref_matvec_f64", [P, P, P, I])(_p(y_ref), _p(a), _p(xv),
                                                  nm)
    y = oracle.matvec(np.zeros(nm), a, xv, nm)
    assert y.tobytes() == y_ref.tobytes()


@needs_ref
@pytest.mark.parametrize("fn", ["ref_sgemm_f32", "ref_sgemm_raw_f32"])
def test_oracle_matches_emitted_c_sgemm(fn):
    m, n, l = 48, 24, 64
    rng = np.random.default_rng(9)
    a = rng.random(m * l).astype(np.float32)
    b = rng.random(l * n).astype(np.float32)
    c0 = rng.random(m * n).astype(np.float32)
    c_ref = c0.copy()
    oracle.ref_fn(fn, [F, P, P, P, I, I, I])(
        F(1.5), _p(a), _p(b), _p(c_ref), l, m, n)
    c = oracle.sgemm(np.float32(1.5), a, b, c0.copy(), l, m, n)
    assert c.tobytes() == c_ref.tobytes()


def test_oracle_sharded_semlap_equals_whole():
    """Elements are independent: chunked/threaded runs are bitwise equal
    (the basis of element sharding)."""
    nelt, n = 20, 4
    rng = np.random.default_rng(3)
    u = rng.random(nelt * n**3)
    g = rng.random(6 * nelt * n**3)
    d = rng.random(n * n)
    w1 = oracle.semlap(np.zeros_like(u), u, d, g, n, nelt)
    w2 = oracle.semlap(np.zeros_like(u), u, d, g, n, nelt, threads=4)
    assert w1.tobytes() == w2.tobytes()
