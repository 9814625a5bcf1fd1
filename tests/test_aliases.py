"""The paper's transform names (north star: tag_inames, add_prefetch,
assignment_to_subst, fix_parameters, unr / ilp tags) lowered to the
reference's verbs (script.py).  CPU: each lowering gives the kernel the
reference's own verbs give (same canonical form, same interpreter bits);
scripts using the aliases run through ``translate_file_text``; the same
error behaviour as the reference's script runner (fortran.py:798-834).
GPU: the Appendix-B matvec written with ``add_prefetch`` and the SEM
fixture with a symbolic order fixed by ``fix_parameters`` hit the
hand-written kernels and match the oracle bitwise."""

import re

import numpy as np
import pytest
import torch

import paper_1503_07659_b200 as lfb
from paper_1503_07659_b200 import fixtures as fx
from paper_1503_07659_b200._loopforge import (fortran, interp, transforms)
from paper_1503_07659_b200._loopforge import kernel as lfk
from loopforge.errors import ParseError, TransformError

MATVEC_PREFETCH = fx.matvec_source("f64", script=False) + """\
!$loopy begin transform
! matvec = lp.split_iname(matvec, "i", 128, outer_tag="g.0", inner_tag="l.0")
! matvec = lp.split_iname(matvec, "j", 32)
! matvec = lp.assume(matvec, "n mod 128 = 0")
! matvec = lp.add_prefetch(matvec, "x", "j_inner")
!$loopy end transform
"""


def semlap_symbolic(order_name="npt", value=8, extra=""):
    """The Appendix-A SEM text with its order as an integer argument (the
    reference rejects it: strides n*n are not affine) fixed by
    fix_parameters in the script."""
    src = fx.semlap_source(value, script=False)
    src = re.sub(r"(?<!\*)\b%d\b" % value, order_name, src)
    src = src.replace("nelt)\n", f"nelt, {order_name})\n", 1)
    src = src.replace("integer nelt,", f"integer {order_name}, nelt,")
    return src + f"""!$loopy begin transform
! semlap = lp.fix_parameters(semlap, {order_name}={value})
! semlap = lp.split_iname(semlap, "e", 32, outer_tag="g.0", inner_tag="l.0")
! semlap = lp.assume(semlap, "nelt mod 32 = 0")
! semlap = lp.extract_subst(semlap, "gf", "g[c, p, q, r, ee]", parameters="c, p, q, r, ee")
{extra}!$loopy end transform
"""


def _run_ref(knl, params, seed=1, **inputs):
    env = interp.make_env(knl, params, inputs, seed=seed)
    return interp.interpret(knl, env)


def test_add_prefetch_is_appendix_b():
    """add_prefetch(x, j_inner) == extract_subst(x[jj]) + precompute: the
    same canonical form as the Appendix-B script, the hand-written matvec,
    the same interpreter bits."""
    _raw, k = fx.translate(MATVEC_PREFETCH)
    _raw, ref = fx.translate(fx.matvec_source("f64"))
    assert "x_fetch_0" in k.temporaries
    assert lfb.canonicalize(k).form == lfb.canonicalize(ref).form
    assert lfb.recognize(k).workload.name == "matvec"
    a = interp.get_output(_run_ref(k, {"n": 128}), "y")
    b = interp.get_output(_run_ref(ref, {"n": 128}), "y")
    assert a.tobytes() == b.tobytes()


def test_fix_parameters_symbolic_order():
    """The reference cannot lower a symbolic SEM order; with
    fix_parameters(npt=8) it is the order-7 fixture exactly."""
    src = semlap_symbolic()
    no_fix = src.replace("fix_parameters(semlap, npt=8)",
                         'assume(semlap, "nelt mod 32 = 0")')
    with pytest.raises(ParseError, match="not affine"):
        fortran.translate_file_text(no_fix, "s.f")
    _raw, k = fx.translate(src)
    _raw, ref = fx.translate(fx.semlap_source(8))
    assert k.param_names == ("nelt",)
    assert lfb.recognize(k).workload.npts == 8
    assert lfb.canonicalize(k).form == lfb.canonicalize(ref).form


def test_fix_parameters_on_the_ir():
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = 2*a[i] + n")
    knl = transforms.assume(knl, "n mod 4 = 0")
    fixed = lfb.fix_parameters(knl, n=12)
    assert fixed.param_names == ()
    assert [a.shape[0].constant for a in fixed.args] == [12, 12]
    a = np.arange(12, dtype=np.float32)
    got = interp.get_output(_run_ref(fixed, {}, a=a), "out")
    want = interp.get_output(_run_ref(knl, {"n": 12}, a=a), "out")
    assert got.tobytes() == want.tobytes()
    with pytest.raises(TransformError, match="mod 4"):
        lfb.fix_parameters(knl, n=10)
    with pytest.raises(TransformError, match="unknown parameter"):
        lfb.fix_parameters(knl, m=3)


def test_tag_inames_and_tag_aliases():
    base = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = 2*a[i]")
    split = transforms.split_iname(base, "i", 8)
    k = lfb.tag_inames(split, "i_outer:g.0, i_inner:l.0")
    ref = transforms.split_iname(base, "i", 8, outer_tag="g.0",
                                 inner_tag="l.0")
    assert k.iname_tags == ref.iname_tags
    assert lfb.canonicalize(k).form == lfb.canonicalize(ref).form
    assert lfb.tag_inames(split, {"i_inner": "unr"}).iname_tags == \
        {"i_inner": "unroll"}
    assert lfb.tag_inames(split, [("i_inner", "ilp")]).iname_tags == \
        {"i_inner": "unroll"}
    with pytest.raises(TransformError, match="bad iname tag"):
        lfb.tag_inames(split, "i_inner:vec")
    with pytest.raises(TransformError, match="unknown iname"):
        lfb.tag_inames(split, "q:g.0")
    with pytest.raises(TransformError, match="already tagged"):
        lfb.tag_inames(k, "i_outer:g.1")


def test_assignment_to_subst():
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "<> t = 3*a[i]\nout[i] = t + 1")
    k = lfb.assignment_to_subst(knl, "t")
    ref = transforms.temporary_to_subst(knl, "t")
    assert lfb.canonicalize(k).form == lfb.canonicalize(ref).form
    a = np.arange(6, dtype=np.float32)
    assert interp.get_output(_run_ref(k, {"n": 6}, a=a), "out").tobytes() \
        == interp.get_output(_run_ref(knl, {"n": 6}, a=a), "out").tobytes()


def test_script_runner_errors_match_the_reference():
    """Unknown verbs, missing kernels and bad arguments fail before any
    transform runs, with the reference's messages."""
    src = fx.fill_source("f64", script=False)
    for script, msg in (
            ('! fill = lp.vectorize(fill, "i")\n', "unknown transform"),
            ('! fill = lp.split_iname(other, "i", 4)\n', "unknown kernel"),
            ('! fill = lp.add_prefetch(fill, x)\n', "unexpected identifier"),
            ('! fill = lp.tag_inames(fill, "i:g.0", 1, 2, 3)\n',
             "bad arguments")):
        text = src + "!$loopy begin transform\n" + script + \
            "!$loopy end transform\n"
        with pytest.raises(TransformError, match=msg):
            fx.translate(text)


def test_reference_scripts_unchanged():
    """Scripts of the reference's own verbs give the reference's kernels."""
    for src in (fx.gemm_source("f32"), fx.semlap_source(8),
                fx.matvec_source("f64"), fx.axpy_source("f64")):
        _r, ref, _u = fortran.translate_file_text(src, "x.f")
        _r, ours = fx.translate(src, "x.f")
        assert ours == ref


@pytest.mark.gpu
def test_add_prefetch_matvec_on_device(cuda):
    """the Appendix-B matvec written with add_prefetch
    is recognised (hand-written kernel) and bitwise on the B200 (variant 3,
    the bitwise TMA kernel; the split-j default within 1e-12)."""
    import oracle
    _raw, k = fx.translate(MATVEC_PREFETCH)
    n = 4096
    rng = np.random.default_rng(4)
    a = rng.random((n, n))
    x = rng.random(n)
    env = lfb.make_device_env(k, {"n": n}, {"a": a, "x": x}, device=cuda)
    ref = oracle.matvec(np.zeros(n), np.asfortranarray(a).reshape(-1,
                                                                  order="F"),
                        x, n, threads=8)
    out = lfb.interpret(k, env, engine="kernels", variant=3)
    assert lfb.get_output(out, "y").tobytes() == ref.tobytes()
    out = lfb.interpret(k, env, engine="kernels")
    got = lfb.get_output(out, "y")
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.gpu
def test_fix_parameters_semlap_on_device(cuda):
    """The symbolic-order SEM text fixed by fix_parameters runs the
    hand-written order-7 kernel, bitwise the reference interpreter's."""
    import oracle
    _raw, k = fx.translate(semlap_symbolic())
    nelt = 64
    env = lfb.make_device_env(k, {"nelt": nelt}, seed=2, device=cuda)
    out = lfb.interpret(k, env, engine="kernels")
    u, d, g = (env.arrays[a].data.cpu().numpy() for a in ("u", "d", "g"))
    ref = oracle.semlap(np.zeros_like(u), u, d, g, 8, nelt)
    assert out.arrays["w"].data.cpu().numpy().tobytes() == ref.tobytes()
