"""The reference's own known-answer and compiled-C-vs-interpreter tests,
restated through the B200 device path.

Each case is the reference test's kernel, inputs and seed, run through the
drop-in ``interpret()`` -- with ``engine="generic"`` (CUDA generated from the
schedule) always, and with ``engine="kernels"`` (the hand-written kernel)
where the recognizer matches it -- and checked bitwise against the
reference test's own expected value, and against the reference interpreter
itself (loopforge.interp from the installed front end, baseline/_ref) on the
same env:

* /root/reference/pkg/tests/test_interp.py:51-56   fill -> 7.0
* test_interp.py:59-64    cond -> [4.0, 1350.0]
* test_interp.py:85-103   DGEMM 4x4x4 seed 7 vs the naive sequential loop
* test_interp.py:106-116  reduction order and dtype (f32 sum)
* test_interp.py:119-125  min / max reductions
* test_interp.py:128-136  parallel tags do not change results
* test_codegen.py:255-264 cond n=32 seed 17 (emitted C == interp)
* test_codegen.py:267-274 section 5.1 forward difference f32 n=48 seed 23
* test_codegen.py:277-288 dbl with g.0/l.0 + tag_instructions n=20 seed 29
"""

import numpy as np
import pytest
import torch

import paper_1503_07659_b200 as lfb
from paper_1503_07659_b200._loopforge import (CodegenError, fortran, interp,
                                              transforms)
from paper_1503_07659_b200._loopforge import kernel as lfk

pytestmark = pytest.mark.gpu

COND_F = """
subroutine cond(out, inp, n)
  implicit none
  real*8 out(n), inp(n)
  integer n

  do i = 1, n
    a = inp(i)
    if (a.ge.3) then
        b = 2*a
        do j = 1,3
            b = 3 * b
        end do
        out(i) = 5*b
    else
        out(i) = 4*a
    endif
  end do
end
"""

DGEMM_F = """
subroutine dgemm(m,n,l,alpha,a,b,c)
  implicit none
  real*8 temp, a(m,l),b(l,n),c(m,n), alpha
  integer m,n,k,i,j,l

  do j = 1,n
    do k = 1,l
      do i = 1,m
        c(i,j) = c(i,j) + alpha*b(k,j)*a(i,k)
      end do
    end do
  end do
end subroutine
"""


def _recognized(knl):
    try:
        lfb.recognize(knl)
        return True
    except CodegenError:
        return False


def _run_all(knl, params, inputs, outputs, cuda, need_kernels=False,
             seed=None):
    """interpret() through every engine that takes *knl*, plus the
    reference interpreter on the same inputs; returns {engine: {name: np}}
    and checks every engine equals the reference bitwise."""
    ref_env = interp.make_env(knl, params, dict(inputs), seed=seed)
    ref = interp.interpret(knl, ref_env)
    engines = ["generic"]
    if _recognized(knl):
        engines.append("kernels")
    elif need_kernels:
        raise AssertionError(f"{knl.name} should hit a hand-written kernel")
    res = {}
    for eng in engines:
        env = lfb.make_device_env(knl, params, dict(inputs), seed=seed,
                                  device=cuda)
        out = lfb.interpret(knl, env, engine=eng)
        torch.cuda.synchronize()
        res[eng] = {o: lfb.get_output(out, o) for o in outputs}
        for o in outputs:
            want = interp.get_output(ref, o)
            assert res[eng][o].dtype == want.dtype, (eng, o)
            assert res[eng][o].tobytes() == want.tobytes(), (eng, o)
    return res


def test_fill_kernel(cuda):
    """test_interp.py:51-56: a bare float literal binding is f32."""
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = a", name="fill")
    res = _run_all(knl, {"n": 4}, {"a": 7.0}, ["out"], cuda,
                   need_kernels=True)
    for r in res.values():
        assert np.array_equal(r["out"], np.full(4, 7.0, dtype=np.float32))
        assert r["out"].dtype == np.float32


def test_conditional_example_values(cuda):
    """test_interp.py:59-64."""
    raw, _t, _u = fortran.translate_file_text(COND_F, "cond.f")
    res = _run_all(raw, {"n": 2}, {"inp": np.array([1.0, 5.0])}, ["out"],
                   cuda)
    for r in res.values():
        assert np.array_equal(r["out"], np.array([4.0, 1350.0]))


@pytest.mark.parametrize("transformed", [False, True])
def test_dgemm_against_naive_matmul(cuda, transformed):
    """test_interp.py:85-103 (4x4x4, seed 7), the raw kernel and the same
    text through a g.N/l.N split: bitwise vs the naive triple loop in the
    reference's update order, on both engines."""
    raw, _t, _u = fortran.translate_file_text(DGEMM_F, "dgemm.f")
    knl = raw
    if transformed:
        knl = transforms.split_iname(knl, "i", 2, outer_tag="g.0",
                                     inner_tag="l.0")
        knl = transforms.split_iname(knl, "j", 2, outer_tag="g.1",
                                     inner_tag="l.1")
    m, n, l = 4, 4, 4
    rng = np.random.default_rng(7)
    a = rng.random((m, l))
    b = rng.random((l, n))
    c0 = rng.random((m, n))
    alpha = 1.5
    res = _run_all(knl, {"m": m, "n": n, "l": l},
                   {"a": a, "b": b, "c": c0, "alpha": alpha}, ["c"], cuda,
                   need_kernels=True)
    want = c0.copy()
    for j in range(n):
        for k in range(l):
            for i in range(m):
                want[i, j] = want[i, j] + alpha * b[k, j] * a[i, k]
    for r in res.values():
        assert np.array_equal(r["c"], want)


def test_reduction_order_and_dtype(cuda):
    """test_interp.py:106-116: sum() accumulates in f32, in j order."""
    knl = lfk.make_kernel(["{[i,j]: 0<=i<1 and 0<=j<5}"],
                          "out[i] = sum(j, a[j])")
    a = np.array([1e8, 1.0, -1e8, 1.0, 1.0], dtype=np.float32)
    res = _run_all(knl, {}, {"a": a}, ["out"], cuda)
    acc = np.float32(0)
    for v in a:
        acc = acc + v
    for r in res.values():
        assert r["out"][0] == acc and r["out"].dtype == np.float32


def test_min_max_reductions(cuda):
    """test_interp.py:119-125."""
    knl = lfk.make_kernel(["{[i,j]: 0<=i<1 and 0<=j<6}"],
                          "lo[i] = min(j, a[j])\nhi[i] = max(j, a[j])")
    a = np.array([3., -2., 7., 0., 7., -2.], dtype=np.float32)
    res = _run_all(knl, {}, {"a": a}, ["lo", "hi"], cuda)
    for r in res.values():
        assert r["lo"][0] == np.float32(-2.0)
        assert r["hi"][0] == np.float32(7.0)


def test_parallel_tags_do_not_change_results(cuda):
    """test_interp.py:128-136: tagged and untagged splits."""
    base = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = 2*a[i]")
    tagged = transforms.split_iname(base, "i", 8, outer_tag="g.0",
                                    inner_tag="l.0")
    untagged = transforms.split_iname(base, "i", 8)
    a = np.arange(24, dtype=np.float32)
    for knl in (tagged, untagged):
        res = _run_all(knl, {"n": 24}, {"a": a}, ["out"], cuda)
        for r in res.values():
            assert np.array_equal(r["out"], 2 * a)


def test_compiled_cond_matches_interpreter(cuda):
    """test_codegen.py:255-264: cond, n = 32, seed 17."""
    raw, _t, _u = fortran.translate_file_text(COND_F, "cond.f")
    rng = np.random.default_rng(17)
    inp = rng.random(32) * 6
    _run_all(raw, {"n": 32}, {"inp": inp}, ["out"], cuda)


def _sec51():
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "result[i] = u[i+1]-u[i]",
                          name="fwd_diff")
    knl = transforms.split_iname(knl, "i", 16)
    knl = transforms.assume(knl, "n mod 16 = 0")
    knl = transforms.extract_subst(knl, "u_acc", "u[j]", parameters="j")
    return transforms.precompute(knl, "u_acc", "i_inner", default_tag=None)


def test_compiled_sec51_matches_interpreter(cuda):
    """test_codegen.py:267-274: the paper's section 5.1 forward difference
    with a precomputed u tile, f32, n = 48, seed 23 (and the checked build,
    test_interp.py:164-171)."""
    knl = _sec51()
    rng = np.random.default_rng(23)
    u = rng.random(49).astype(np.float32)
    res = _run_all(knl, {"n": 48}, {"u": u}, ["result"], cuda)
    for r in res.values():
        assert np.array_equal(r["result"], u[1:] - u[:-1])
    env = lfb.make_device_env(knl, {"n": 48}, {"u": u}, device=cuda)
    got = lfb.get_output(lfb.interpret_bounds_checked(knl, env), "result")
    assert got.tobytes() == (u[1:] - u[:-1]).tobytes()


def test_compiled_parallel_emulation_matches(cuda):
    """test_codegen.py:277-288: dbl with g.0/l.0 and tag_instructions,
    n = 20 (ragged: 20 is not a multiple of 8), seed 29."""
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = 2*a[i]", name="dbl")
    knl = transforms.split_iname(knl, "i", 8, outer_tag="g.0",
                                 inner_tag="l.0")
    knl = transforms.tag_instructions(knl, "*", "touched")
    rng = np.random.default_rng(29)
    a = rng.random(20).astype(np.float32)
    res = _run_all(knl, {"n": 20}, {"a": a}, ["out"], cuda)
    for r in res.values():
        assert np.array_equal(r["out"], 2 * a)


def test_seeded_env_matches_reference_recipe(cuda):
    """make_device_env(seed=...) binds exactly the reference's make_env
    values (interp.py:115-119), so seeded cases compare like for like."""
    raw, _t, _u = fortran.translate_file_text(DGEMM_F, "dgemm.f")
    params = {"m": 5, "n": 3, "l": 7}
    ref = interp.make_env(raw, params, {"alpha": 0.5}, seed=4)
    dev = lfb.make_device_env(raw, params, {"alpha": 0.5}, seed=4,
                              device=cuda)
    for name in ("a", "b", "c"):
        assert interp.get_output(ref, name).tobytes() == \
            lfb.get_output(dev, name).tobytes(), name
    _run_all(raw, params, {"alpha": 0.5}, ["c"], cuda, need_kernels=True,
             seed=4)


@pytest.mark.parametrize("n", [3, 4])
def test_real4_semlap_on_the_generic_engine(cuda, n):
    """A real*4 SEM Laplacian (the Appendix-A fixture with real*8 -> real*4
    and the fixture script): no hand-written kernel matches it, so it runs
    as CUDA generated from its schedule -- bitwise the reference
    interpreter's f32 result on the same seeded env."""
    from paper_1503_07659_b200 import fixtures as fx
    src = fx.semlap_source(n, block=1).replace("real*8", "real*4")
    _raw, knl, _u = fortran.translate_file_text(src, "semlap4.f")
    with pytest.raises(CodegenError):
        lfb.interpret(knl, lfb.make_device_env(knl, {"nelt": 3}, seed=5,
                                               device=cuda),
                      engine="kernels")
    _run_all(knl, {"nelt": 3}, {}, ["w"], cuda, seed=5)
