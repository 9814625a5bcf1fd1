"""Host-side logic (CPU): recognizer and launch geometry.

The recognizer must accept exactly the kernels whose reference execution the
sm_100a kernels reproduce, whatever the transform script did to names,
splits, tags and prefetch tiles -- and reject anything else with the
reference's own errors (ScheduleError from the reference scheduler,
CodegenError otherwise).
"""

import pytest

from paper_1503_07659_b200 import fixtures as fx
from paper_1503_07659_b200._loopforge import (CodegenError, ScheduleError,
                                              codegen, transforms)
from paper_1503_07659_b200.launch import launch_geometry
from paper_1503_07659_b200.recognize import canonicalize, recognize


@pytest.mark.parametrize("src,family,npts", [
    (fx.fill_source("f64"), "fill", 0),
    (fx.fill_source("f64", assume=True), "fill", 0),
    (fx.fill_source("f32", block=256), "fill", 0),
    (fx.axpy_source("f64"), "axpy", 0),
    (fx.axpy_source("f32", block=64, assume=True), "axpy", 0),
    (fx.matvec_source("f64"), "matvec", 0),
    (fx.matvec_source("f64", block=32, jtile=16), "matvec", 0),
    (fx.semlap_source(8), "semlap", 8),
    (fx.semlap_source(8, block=1, gf=False), "semlap", 8),
    (fx.semlap_source(4, block=7, assume=False), "semlap", 4),
    (fx.semlap_source(16), "semlap", 16),
    (fx.semlap_source(5), "semlap", 5),
    (fx.gemm_source("f32"), "gemm", 0),
    (fx.gemm_source("f32", tiles=(32, 16, 8)), "gemm", 0),
])
def test_fixtures_recognised_raw_and_transformed(src, family, npts):
    raw, knl = fx.translate(src)
    for k in (raw, knl):
        m = recognize(k)
        assert m.workload.name == family
        assert m.workload.npts == npts


def test_renamed_kernel_maps_roles():
    src = fx.axpy_source("f64").replace("(y, x, alpha, n)", "(zz, xx, b, n)") \
        .replace("y(n), x(n), alpha", "zz(n), xx(n), b") \
        .replace("y(i) = y(i) + alpha*x(i)", "zz(i) = zz(i) + b*xx(i)") \
        .replace('"i"', '"i"')
    _raw, knl = fx.translate(src)
    m = recognize(knl)
    assert m.arg_map == {"y": "zz", "x": "xx", "alpha": "b"}


def test_semlap_parallel_k_is_rejected_by_reference_scheduler():
    raw, _k = fx.translate(fx.semlap_source(4, script=False))
    with pytest.raises(ScheduleError):
        recognize(transforms.split_iname(raw, "k", 4, outer_tag="g.1"))


def test_matvec_parallel_reduction_is_rejected():
    """j tagged l.0 makes the interpreter run j outermost (interp.py:385):
    y(i) would only see the last j -- not the matvec semantics."""
    raw, _k = fx.translate(fx.matvec_source(script=False))
    with pytest.raises(CodegenError):
        recognize(transforms.split_iname(raw, "j", 4, inner_tag="l.0"))


def test_commuted_single_node_is_accepted():
    """a*b == b*a and a+b == b+a bitwise in IEEE arithmetic (one node):
    these hit the hand-written kernels."""
    for body in ("y(i) + x(i)*alpha", "x(i)*alpha + y(i)"):
        src = fx.axpy_source("f64").replace("y(i) + alpha*x(i)", body)
        raw, _k = fx.translate(src)
        assert recognize(raw).workload.name == "axpy"
    src = fx.semlap_source(8).replace("d(i,l)*u(l,j,k,e)", "u(l,j,k,e)*d(i,l)")
    raw, _k = fx.translate(src)
    assert recognize(raw).workload.npts == 8


def test_reassociated_expression_is_rejected():
    src = fx.axpy_source("f64").replace("y(i) + alpha*x(i)",
                                        "(y(i) + alpha)*x(i)")
    raw, _k = fx.translate(src)
    with pytest.raises(CodegenError, match="no CPU fallback"):
        recognize(raw)
    src = fx.semlap_source(4).replace(
        "s = s + d(l,i)*wr(l,j,k) + d(l,j)*ws(i,l,k) + d(l,k)*wt(i,j,l)",
        "s = s + (d(l,i)*wr(l,j,k) + d(l,j)*ws(i,l,k)) + d(l,k)*wt(i,j,l)")
    raw, _k = fx.translate(src)
    with pytest.raises(CodegenError):
        recognize(raw)


def test_gemm_permuted_nest_is_canonical():
    """The paper's script runs (i, j, k) where the source nests (j, k, i);
    each c(i,j) still sees k ascending, so both canonicalise equal."""
    raw, knl = fx.translate(fx.gemm_source("f32"))
    assert canonicalize(raw).form == canonicalize(knl).form


def test_sem_split_merges_to_raw():
    raw, knl = fx.translate(fx.semlap_source(8))
    c = canonicalize(knl)
    assert c.form == canonicalize(raw).form
    (logical, (outer, inner, f)), = c.splits.items()
    assert (outer, inner, f) == ("e_outer", "e_inner", 32)


@pytest.mark.parametrize("src,params,groups,local,guard", [
    (fx.fill_source("f64"), {"n": 1 << 24}, (131072, 1, 1), (128, 1, 1),
     True),
    (fx.fill_source("f64", assume=True), {"n": 1 << 24}, (131072, 1, 1),
     (128, 1, 1), False),
    (fx.fill_source("f64"), {"n": 300}, (3, 1, 1), (128, 1, 1), True),
    (fx.semlap_source(8), {"nelt": 65536}, (2048, 1, 1), (32, 1, 1), False),
    (fx.matvec_source("f64"), {"n": 4096}, (32, 1, 1), (128, 1, 1), False),
    (fx.gemm_source("f32"), {"m": 8192, "n": 8192, "l": 8192},
     (512, 1024, 1), (8, 16, 1), True),
])
def test_geometry(src, params, groups, local, guard):
    _raw, knl = fx.translate(src)
    geo = launch_geometry(knl, params)
    assert geo.group_extent == groups
    assert geo.local_extent == local
    assert geo.guard == guard


@pytest.mark.parametrize("src", [fx.fill_source("f64"),
                                 fx.fill_source("f64", assume=True),
                                 fx.semlap_source(8),
                                 fx.semlap_source(8, block=7, assume=False),
                                 fx.gemm_source("f32")])
def test_guard_matches_reference_opencl(src):
    """The guard the executor derives is the one the reference's OpenCL
    emitter writes (codegen.py:590-612)."""
    _raw, knl = fx.translate(src)
    geo = launch_geometry(knl, {p: 64 for p in knl.param_names})
    text = codegen.emit(knl, "opencl")
    if geo.guard:
        assert f"if ({geo.guard_text})" in text
    else:
        assert "\n  if (" not in text


def test_untransformed_geometry_has_no_axes():
    raw, _k = fx.translate(fx.fill_source("f64"))
    geo = launch_geometry(raw, {"n": 100})
    assert geo.parallel == () and not geo.guard
