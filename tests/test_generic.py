"""The generic path: CUDA generated from the schedule (cudagen.py), compiled
by NVRTC for sm_100a, launched through the C-ABI.

CPU: every fixture (raw and transformed) emits and compiles for sm_100a;
structure of the paper's DGEMM (shared tiles, real barriers, cooperative
fetch).  GPU: every golden the reference interpreter produced
(tests/golden/) is reproduced through ``interpret(..., engine="generic")``
-- bitwise, except rotnorm's sin/cos (libdevice vs numpy, a few ulp).
"""

import numpy as np
import pytest
import torch

import paper_1503_07659_b200 as lfb
from conftest import Golden, golden_names
from paper_1503_07659_b200 import fixtures as fx
from paper_1503_07659_b200._loopforge import CodegenError
from paper_1503_07659_b200.cudagen import emit_cuda
from paper_1503_07659_b200.generic import compile_program


def _fixture_kernels():
    out = []
    for name in fx.GENERIC_FORTRAN:
        raw, knl = fx.translate(fx.generic_source(name), f"{name}.f")
        out += [(f"{name}-raw", raw), (name, knl)]
    for name in fx.GENERIC_NATIVE:
        raw, knl = fx.generic_native(name)
        out += [(f"{name}-raw", raw), (name, knl)]
    for name, src in (("dgemm", fx.gemm_source("f64")),
                      ("sgemm", fx.gemm_source("f32")),
                      ("semlap7", fx.semlap_source(7, block=4)),
                      ("matvec", fx.matvec_source("f64")),
                      ("axpy32", fx.axpy_source("f32"))):
        raw, knl = fx.translate(src, f"{name}.f")
        out += [(f"{name}-raw", raw), (name, knl)]
    return out


FIXTURES = _fixture_kernels()


@pytest.mark.parametrize("name,knl", FIXTURES, ids=[n for n, _ in FIXTURES])
def test_emits_and_compiles_for_sm100a(name, knl):
    prog = emit_cuda(knl)
    for narrow in (False, True):    # 64-bit and 32-bit index builds
        cubin = compile_program(prog, narrow)
        assert cubin[:4] == b"\x7fELF"
    assert prog.entry in prog.source


def test_paper_dgemm_uses_shared_tiles_and_barriers():
    _raw, knl = fx.translate(fx.gemm_source("f64"), "dgemm.f")
    prog = emit_cuda(knl)
    assert prog.shared == ("a_acc_0", "b_acc_0") and not prog.demoted
    assert prog.cooperative == 2          # both tile fetches spread over CTA
    assert prog.block == (8, 16, 1)       # l.0 = j_inner, l.1 = i_inner
    # 16 x 32 tile laid out as TMA writes it, two buffers
    assert "__shared__ __align__(1024) double a_acc_0[1024];" in prog.source
    # c[i,j] accumulated in a register across k_inner (scalar replacement)
    assert "lfb_r0_0 = (lfb_r0_0 + " in prog.source
    # constant footprint box: no 64-bit division in the fetch
    assert "lfb_q0 < 512" in prog.source
    assert prog.source.count("__syncthreads();") >= 2
    # the guard became a per-statement predicate so barriers stay uniform
    assert "const bool lfb_in =" in prog.source


def test_untransformed_kernel_is_one_thread():
    raw, _knl = fx.translate(fx.generic_source("cond"), "cond.f")
    prog = emit_cuda(raw)
    assert prog.block == (1, 1, 1)
    assert "blockIdx" not in prog.source.split("lfb_tid")[0]


def test_literal_and_promotion_semantics():
    """interp.py:140-187: a bare float literal is f32 (hex-exact); int32 op
    float32 computes in float64 (numpy promotion) before the f32 store."""
    _raw, knl = fx.translate(fx.generic_source("mixed"), "mixed.f")
    src = emit_cuda(knl).source
    assert "0x1.0000000000000p-1f" in src          # 0.5 as float32
    assert "((double)(x[" in src                   # x(i)*i in float64


def test_symbolic_private_temporary_is_codegen_error():
    import dataclasses

    from paper_1503_07659_b200._loopforge import kernel as lfk, polyset
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = 2*a[i]")
    t = lfk.TemporaryDecl("t", "f64", (polyset.AffineExpr.var("n"),))
    bad = dataclasses.replace(knl, temporaries={"t": t})
    with pytest.raises(CodegenError, match="symbolic extent"):
        emit_cuda(bad)


# {{{ device parity

TOL = {"gen_rotnorm_n300": 1e-14}


def _env(g, knl, dev):
    env = lfb.make_device_env(knl, g.params, device=dev)
    for a in knl.args:
        buf = g.inp(a.name)
        if a.kind == "scalar-value":
            env.scalars[a.name] = buf.reshape(-1)[0]
        else:
            env.arrays[a.name].data.copy_(torch.from_numpy(buf.copy()))
    return env


@pytest.mark.gpu
@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("which", ["transformed", "raw"])
def test_generic_engine_matches_reference(name, which, cuda):
    """Every golden, through the generated CUDA (the hand-written kernels
    are bypassed): bitwise against the reference interpreter."""
    g = Golden(name)
    raw, knl = g.kernels()
    k = knl if which == "transformed" else raw
    if which == "raw" and name.startswith("semlap"):
        pytest.skip("untransformed SEM is one thread per launch: slow")
    env = _env(g, k, cuda)
    out = lfb.interpret(k, env, engine="generic")
    torch.cuda.synchronize()
    for o in g.outputs():
        got = out.arrays[o].data.cpu().numpy()
        want = g.out(o)
        assert got.dtype == want.dtype
        if name in TOL:
            rel = np.max(np.abs(got - want)) / np.max(np.abs(want))
            assert rel <= TOL[name], (o, rel)
        else:
            assert got.tobytes() == want.tobytes(), f"{name}:{o}"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gen_dgemm_m20_n12_l40", "gen_mvacc_n64",
                                  "gen_transpose_n37_m21", "gen_cond_n300"])
def test_generic_wide_index_build(name, cuda, monkeypatch):
    """The 64-bit index build (chosen when an array or parameter passes
    2^31) gives the same bits as the 32-bit one the small goldens use."""
    from paper_1503_07659_b200 import generic
    monkeypatch.setattr(generic.GenericLauncher, "narrow",
                        lambda self, env: False)
    g = Golden(name)
    _raw, knl = g.kernels()
    out = lfb.interpret(knl, _env(g, knl, cuda), engine="generic")
    torch.cuda.synchronize()
    for o in g.outputs():
        assert out.arrays[o].data.cpu().numpy().tobytes() == \
            g.out(o).tobytes(), f"{name}:{o}"


@pytest.mark.gpu
def test_auto_engine_routes_unrecognised_kernels(cuda):
    g = Golden("gen_mvacc_n64")
    _raw, knl = g.kernels()
    env = _env(g, knl, cuda)
    with pytest.raises(CodegenError):
        lfb.interpret(knl, env, engine="kernels")
    out = lfb.interpret(knl, env)            # auto -> generated CUDA
    assert out.arrays["y"].data.cpu().numpy().tobytes() == \
        g.out("y").tobytes()


def test_precompute_footprints_become_tma_loads():
    """the paper's DGEMM tiles (a_acc_0 16x32,
    b_acc_0 32x8 from precompute) are fetched by TMA, one elected thread
    per tile, 128-B swizzled rows (b split into two 128-B pieces)."""
    _raw, knl = fx.translate(fx.gemm_source("f64"), "dgemm.f")
    prog = emit_cuda(knl)
    # a is read along its contiguous dim (dense rows), b down its columns
    # (128-B swizzle, split into two 128-B pieces)
    assert [(m.array, m.box, m.swizzle) for m in prog.tma] == \
        [("a", (16, 32), 0), ("b", (16, 8), 128)]
    # double-buffered over k_outer: prologue + prefetch, 3 TMAs each
    assert prog.source.count("lfb_tma2(") == 3 + 3 + 1
    assert "lfb_expect_tx(&lfb_bars[0], 6144u);" in prog.source
    assert "__shared__ __align__(1024) double a_acc_0[1024];" in prog.source
    assert prog.arg_order[-3:] == ("lfb_tma", "lfb_tm0", "lfb_tm1")
    # sgemm: 16 floats = 64-B rows for a (no swizzle), 128-B rows for b
    _raw, ks = fx.translate(fx.gemm_source("f32"), "sgemm.f")
    assert [(m.array, m.box, m.swizzle) for m in emit_cuda(ks).tma] == \
        [("a", (16, 32), 0), ("b", (32, 8), 128)]


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,l,tma", [(250, 120, 200, True),
                                       (251, 120, 200, False),
                                       (64, 40, 96, True)])
def test_generic_dgemm_larger(m, n, l, tma, cuda):
    """The paper's DGEMM script with ragged tiles against a sequential-k
    numpy restatement (c + (alpha*b)*a per k, f64).  Odd m breaks the
    tensor-map stride rule: the same kernel then fetches cooperatively."""
    from paper_1503_07659_b200.generic import GenericLauncher
    _raw, knl = fx.translate(fx.gemm_source("f64"), "dgemm.f")
    rng = np.random.default_rng(3)
    a, b, c = rng.random((m, l)), rng.random((l, n)), rng.random((m, n))
    env = lfb.make_device_env(knl, {"m": m, "n": n, "l": l},
                              {"a": a, "b": b, "c": c, "alpha": 1.5},
                              device=cuda)
    assert GenericLauncher(knl, env).tensor_maps(env)[1] is tma
    got = lfb.get_output(lfb.interpret(knl, env, engine="generic"), "c")
    want = c.copy()
    for k in range(l):
        want = want + (1.5 * b[k, :])[None, :] * a[:, k][:, None]
    assert got.tobytes() == want.tobytes()

# }}}


@pytest.mark.gpu
@pytest.mark.parametrize("name,tma", [("gen_smooth_n320", True),
                                      ("gen_ttile_n40_m21", True),
                                      ("gen_ttile_n37_m21", False),
                                      ("gen_dgemm_m20_n12_l40", True)])
def test_precompute_footprint_paths(name, tma, cuda):
    """Which fetch path the goldens exercise: TMA tensor maps when the
    array meets the tensor-map rules, else the cooperative fetch of the
    same kernel (both bitwise the reference, test above)."""
    from paper_1503_07659_b200.generic import GenericLauncher
    g = Golden(name)
    _raw, knl = g.kernels()
    env = _env(g, knl, cuda)
    launcher = GenericLauncher(knl, env)
    assert launcher.program.tma
    assert launcher.tensor_maps(env)[1] is tma


@pytest.mark.gpu
def test_group_prefetch_large(cuda):
    """Enough work-groups that every CTA walks several: the next group's
    tiles are TMA-prefetched into the second buffer (128-B / 1024-B
    aligned); results against numpy restatements, bitwise."""
    n = 64 * 10000
    _raw, km = fx.translate(fx.generic_source("smooth"), "smooth.f")
    u = np.random.default_rng(1).random(n + 2)
    env = lfb.make_device_env(km, {"n": n}, {"u": u}, device=cuda)
    got = lfb.get_output(lfb.interpret(km, env), "r")
    want = (u[:-2] + 2.0 * u[1:-1]) + u[2:]
    assert got.tobytes() == want.tobytes()
    nt, mt = 1040, 1000
    _raw, kt = fx.translate(fx.generic_source("ttile"), "ttile.f")
    a = np.random.default_rng(2).random((nt, mt))
    env = lfb.make_device_env(kt, {"n": nt, "m": mt}, {"a": a}, device=cuda)
    got = lfb.get_output(lfb.interpret(kt, env), "b")
    assert got.tobytes() == np.ascontiguousarray(a.T).tobytes()


@pytest.mark.gpu
def test_generic_launch_in_cuda_graph(cuda):
    """A generated kernel with TMA tiles captured in a CUDA graph and
    replayed: the tensor maps travel as kernel parameters by value."""
    from paper_1503_07659_b200.generic import GenericLauncher
    m, n, l = 64, 40, 96
    _raw, knl = fx.translate(fx.gemm_source("f64"), "dgemm.f")
    rng = np.random.default_rng(9)
    a, b, c = rng.random((m, l)), rng.random((l, n)), rng.random((m, n))
    env = lfb.make_device_env(knl, {"m": m, "n": n, "l": l},
                              {"a": a, "b": b, "c": c, "alpha": 1.5},
                              device=cuda)
    launcher = GenericLauncher(knl, env)
    c0 = env.arrays["c"].data.clone()
    s = torch.cuda.Stream(cuda)
    s.wait_stream(torch.cuda.current_stream(cuda))
    with torch.cuda.stream(s):
        launcher.launch()           # warm: compile + module load
    torch.cuda.current_stream(cuda).wait_stream(s)
    torch.cuda.synchronize()
    env.arrays["c"].data.copy_(c0)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        launcher.launch()
    env.arrays["c"].data.copy_(c0)
    graph.replay()
    graph.replay()                  # c accumulates twice
    torch.cuda.synchronize()
    want = c.copy()
    for _ in range(2):
        for k in range(l):
            want = want + (1.5 * b[k, :])[None, :] * a[:, k][:, None]
    got = lfb.get_output(env, "c")
    assert got.tobytes() == want.tobytes()


@pytest.mark.gpu
def test_generic_wide_build_past_2_31(cuda):
    """An array of 2^31 + 5 elements: the launcher picks the 64-bit index
    build and the elements past the int range are written."""
    from paper_1503_07659_b200.generic import GenericLauncher
    n = (1 << 31) + 5
    _raw, kf = fx.translate(fx.fill_source("f32"), "fill.f")
    out = torch.zeros(n, dtype=torch.float32, device=cuda)
    env = lfb.env_from_buffers(kf, {"n": n}, {"out": out}, {"a": 0.75})
    launcher = GenericLauncher(kf, env)
    assert launcher.narrow(env) is False
    launcher.launch()
    torch.cuda.synchronize()
    idx = torch.tensor([0, (1 << 31) - 1, 1 << 31, n - 1], device=cuda)
    assert bool((out[idx] == 0.75).all())
    assert int((out != 0.75).sum()) == 0


REV_F = """subroutine rev(y, x, n)
  implicit none
  real*8 y(n), x(n), t(n)
  integer n, i

  do i = 1, n
    t(i) = 2*x(i)
  end do
  do i = 1, n
    y(i) = t(n + 1 - i) + x(i)
  end do
end
"""


def test_temporaries_sized_by_parameters_compile():
    """A local array sized by a parameter (the reference allocates it from
    the call's parameters, interp.py:332-338): the program is specialised
    to the launch's values; without values it is a CodegenError."""
    _raw, knl = fx.translate(REV_F)
    with pytest.raises(CodegenError, match="symbolic extent"):
        emit_cuda(knl)
    for n in (5, 300):
        prog = emit_cuda(knl, params={"n": n})
        assert f"double t[{n}];" in prog.source
        assert compile_program(prog, True)[:4] == b"\x7fELF"
    with pytest.raises(CodegenError, match="budget"):
        emit_cuda(knl, params={"n": 1 << 20})


@pytest.mark.gpu
@pytest.mark.parametrize("n", [5, 37, 300])
def test_temporaries_sized_by_parameters_run(cuda, n):
    from paper_1503_07659_b200._loopforge import interp
    _raw, knl = fx.translate(REV_F)
    x = np.random.default_rng(n).random(n)
    ref = interp.interpret(knl, interp.make_env(knl, {"n": n}, {"x": x}))
    env = lfb.make_device_env(knl, {"n": n}, {"x": x}, device=cuda)
    out = lfb.interpret(knl, env)
    assert lfb.get_output(out, "y").tobytes() == \
        interp.get_output(ref, "y").tobytes()
