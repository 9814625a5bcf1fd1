"""Device parity: the sm_100a kernels against the reference.

* every golden (made by the reference interpreter, tests/golden/) is
  reproduced bit for bit through the drop-in ``interpret``;
* at BASELINE sizes, outputs are compared with the CPU oracle (pinned to the
  reference by tests/test_oracle.py) on full arrays or on element/row/column
  samples, bitwise;
* geometry variants (block sizes, guards, ragged extents) and the error
  behaviour of the reference (InterpError / CodegenError) are covered.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1503_07659_b200 as lfb
from conftest import Golden, golden_names
from paper_1503_07659_b200 import fixtures as fx
from paper_1503_07659_b200._loopforge import CodegenError, InterpError

pytestmark = pytest.mark.gpu


def _env_from_golden(g, knl, dev):
    env = lfb.make_device_env(knl, g.params, device=dev)
    for a in knl.args:
        buf = g.inp(a.name)
        if a.kind == "scalar-value":
            env.scalars[a.name] = buf.reshape(-1)[0]
        else:
            env.arrays[a.name].data.copy_(torch.from_numpy(buf.copy()))
    return env


@pytest.mark.parametrize("name", golden_names())
def test_golden_bitwise(name, cuda):
    g = Golden(name)
    _raw, knl = g.kernels()
    env = _env_from_golden(g, knl, cuda)
    before = {k: v.data.clone() for k, v in env.arrays.items()}
    out = lfb.interpret(knl, env)
    torch.cuda.synchronize()
    for o in g.outputs():
        got = out.arrays[o].data.cpu().numpy()
        want = g.out(o)
        assert got.dtype == want.dtype
        assert got.tobytes() == want.tobytes(), f"{name}:{o}"
    # interpret never mutates its input env (interp.py:329 env.copy())
    for k, v in env.arrays.items():
        assert torch.equal(v.data, before[k]), k


@pytest.mark.parametrize("name", ["semlap_n8_b2_nelt2", "matvec_f64_n128",
                                  "sgemm_m20_n12_l40", "axpy_f64_n300"])
def test_golden_untransformed_kernel(name, cuda):
    """The raw (untransformed) lowering of the same text gives the same
    bits -- transforms do not change results (test_interp.py:128-136)."""
    g = Golden(name)
    raw, _knl = g.kernels()
    env = _env_from_golden(g, raw, cuda)
    out = lfb.interpret(raw, env)
    for o in g.outputs():
        assert out.arrays[o].data.cpu().numpy().tobytes() == \
            g.out(o).tobytes()


def _sem_inputs(n, nelt, dev, seed=0):
    gen = torch.Generator(device=dev).manual_seed(seed)
    u = torch.rand(nelt * n**3, dtype=torch.float64, device=dev,
                   generator=gen) * 2 - 1
    g = torch.rand(6 * nelt * n**3, dtype=torch.float64, device=dev,
                   generator=gen)
    d = torch.rand(n * n, dtype=torch.float64, device=dev,
                   generator=gen) * 2 - 1
    return u, d, g


def _sem_check(n, nelt, src, dev, samples, variant=0, seed=0):
    _raw, knl = fx.translate(src)
    u, d, g = _sem_inputs(n, nelt, dev, seed)
    w = torch.full_like(u, float("nan"))
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    lfb.interpret(knl, env, inplace=True, variant=variant)
    torch.cuda.synchronize()
    uh, dh, gh, wh = (t.cpu().numpy() for t in (u, d, g, w))
    np3 = n**3
    for lo, hi in samples:
        ref = np.zeros_like(uh)
        oracle.semlap(ref, uh, dh, gh, n, nelt, elems=(lo, hi), threads=8)
        assert wh[lo * np3:hi * np3].tobytes() == \
            ref[lo * np3:hi * np3].tobytes(), (lo, hi)
    assert not np.isnan(wh).any()


def test_semlap_o7_65536_elements(cuda):
    """BASELINE config 3 (order 7, 65,536 elements, the fixture script)."""
    nelt = 65536
    _sem_check(8, nelt, fx.semlap_source(8), cuda,
               [(0, 1024), (30000, 31000), (nelt - 1024, nelt)])


@pytest.mark.parametrize("variant", [1, 2, 3, 4, 5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 39, 40, 41, 42])  # bitwise ones
def test_semlap_o7_variants(cuda, variant):
    nelt = 4096
    _sem_check(8, nelt, fx.semlap_source(8), cuda, [(0, nelt)],
               variant=variant)


@pytest.mark.parametrize("n", list(range(2, 17)))
def test_semlap_orders(cuda, n):
    """The order sweep of BASELINE config 5 (p = 1..15): staged kernel for
    even n <= 10, k-slab kernel for odd n and n >= 12."""
    nelt = 640 if n <= 10 else 96
    _sem_check(n, nelt, fx.semlap_source(n), cuda, [(0, nelt)], seed=n)


GEN_VARIANTS = [(4, 20), (4, 21), (5, 20), (5, 21), (5, 22), (6, 20),
                (6, 21), (6, 22), (7, 20), (7, 21), (7, 22), (8, 20),
                (8, 21), (8, 22), (9, 20), (9, 21), (10, 20), (10, 21),
                (11, 20), (7, 60), (9, 60), (10, 60), (11, 60), (12, 60)]


@pytest.mark.parametrize("n,variant", GEN_VARIANTS)
def test_semlap_gen_variants(cuda, n, variant):
    """The E-element-chunk kernel (semlap_gen.cu) in every tabulated
    configuration; nelt leaves a partial last chunk and, for odd n, a last
    u span that must be copied by the threads."""
    nelt = 331
    _sem_check(n, nelt, fx.semlap_source(n, block=1), cuda, [(0, nelt)],
               variant=variant, seed=variant + n)


SLAB_VARIANTS = [(12, 30), (12, 31), (13, 31), (14, 30), (14, 31),
                 (15, 30), (16, 30), (16, 31)]


@pytest.mark.parametrize("n,variant", SLAB_VARIANTS)
def test_semlap_slab_variants(cuda, n, variant):
    """k-slab kernel tuning alternatives for the large orders."""
    _sem_check(n, 53, fx.semlap_source(n, block=1), cuda, [(0, 53)],
               variant=variant, seed=variant + n)


@pytest.mark.parametrize("n,variant", [(n, v) for n in range(9, 17)
                                       for v in (70, 72)])
@pytest.mark.parametrize("nelt", [1, 53, 300])
def test_semlap_line_kernel(cuda, n, variant, nelt):
    """Line-owner kernel (semlap_line.cu): phase 1 by the owners of the
    u lines, bitwise; one element, a partial last round of groups, and
    enough elements that every group wraps the slice ring several times."""
    _sem_check(n, nelt, fx.semlap_source(n, block=1), cuda, [(0, nelt)],
               variant=variant, seed=variant + n + nelt)


@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 9, 10, 11])
def test_semlap_slab_kernel_small_orders(cuda, n):
    """Variant 9 forces the k-slab kernel for orders the chunk kernel
    serves by default."""
    _sem_check(n, 97, fx.semlap_source(n, block=1), cuda, [(0, 97)],
               variant=9, seed=n)


@pytest.mark.parametrize("n,nelt", [(5, 3), (7, 1), (9, 37), (15, 5),
                                    (3, 101), (3, 6), (5, 11), (6, 7),
                                    (2, 9)])
def test_semlap_odd_order_tail(cuda, n, nelt):
    """Odd n and odd nelt: the last element's 16-byte-rounded u copy would
    run past the array, so the threads copy it themselves."""
    src = fx.semlap_source(n, block=1)
    _sem_check(n, nelt, src, cuda, [(0, nelt)], seed=nelt)


@pytest.mark.parametrize("block,nelt", [(1, 37), (7, 100), (32, 33),
                                        (32, 1), (3, 448)])
def test_semlap_ragged_and_guarded(cuda, block, nelt):
    """Blocks that do not divide nelt: the reference emits a guard; no
    assume() so any nelt is legal."""
    src = fx.semlap_source(8, block=block, assume=False)
    _sem_check(8, nelt, src, cuda, [(0, nelt)], seed=block)


@pytest.mark.parametrize("n,variant", [(n, 50) for n in range(2, 17)]
                         + [(n, 51) for n in range(9, 17)]
                         + [(n, 61) for n in (7, 9, 10, 11, 12)]
                         + [(n, 52) for n in range(7, 17)]
                         + [(n, 71) for n in range(9, 17)] + [(8, 53),
                                                              (8, 55),
                                                              (16, 54)])
def test_semlap_fma_mode(cuda, n, variant):
    """variant 50: the default kernel with every multiply-add fused (DFMA);
    variant 51: the FP64 tensor-core (DMMA) kernel for even n >= 10;
    52: the interleaved-phase DMMA kernel (n = 16: u staged by a swizzled
    2-D TMA), 54: the same with the plain bulk-copy staging.
    Tolerance parity (north star: 1e-12 relative fp64): per point against
    the magnitude of the terms it sums -- the same operator on |u|, |d|,
    |g| -- and normwise."""
    nelt = max(3, 4096 // n ** 3 * 4 + 3)
    _raw, knl = fx.translate(fx.semlap_source(n, block=1))
    u, d, g = _sem_inputs(n, nelt, cuda, 40 + n)
    w = torch.full_like(u, float("nan"))
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    lfb.Launcher(knl, env, variant=variant).launch()
    torch.cuda.synchronize()
    uh, dh, gh = u.cpu().numpy(), d.cpu().numpy(), g.cpu().numpy()
    ref = oracle.semlap(np.zeros_like(uh), uh, dh, gh, n, nelt)
    mag = oracle.semlap(np.zeros_like(uh), np.abs(uh), np.abs(dh),
                        np.abs(gh), n, nelt)
    got = w.cpu().numpy()
    err = np.abs(got - ref)
    assert (err <= 1e-12 * mag).all()
    assert err.max() <= 1e-12 * np.abs(ref).max()
    assert got.tobytes() != ref.tobytes() or n < 3  # really the fused path


def test_semlap_constant_d_slots_across_streams(cuda):
    """The n = 8 default keeps d in a ring of constant-bank slots: launches
    with different d on two streams, more launches than slots, each result
    bitwise the oracle's (no slot overwritten while a kernel reads it)."""
    n, nelt = 8, 2048
    _raw, knl = fx.translate(fx.semlap_source(n))
    streams = [torch.cuda.Stream(cuda), torch.cuda.Stream(cuda)]
    cases = []
    for c in range(6):
        u, d, g = _sem_inputs(n, nelt, cuda, 100 + c)
        w = torch.full_like(u, float("nan"))
        env = lfb.env_from_buffers(knl, {"nelt": nelt},
                                   {"u": u, "d": d, "g": g, "w": w})
        cases.append((env, u, d, g, w))
    for s in streams:
        s.wait_stream(torch.cuda.current_stream(cuda))
    for rep in range(3):
        for c, (env, *_rest) in enumerate(cases):
            s = streams[c % 2]
            with torch.cuda.stream(s):
                lfb.Launcher(knl, env).launch(stream=s.cuda_stream)
    torch.cuda.synchronize()
    for env, u, d, g, w in cases:
        ref = oracle.semlap(np.zeros(nelt * n ** 3), u.cpu().numpy(),
                            d.cpu().numpy(), g.cpu().numpy(), n, nelt)
        assert w.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("n,variant", [(8, 50), (8, 0), (12, 50),
                                       (12, 0), (16, 50), (5, 0),
                                       (16, 0), (13, 0)])
def test_semlap_graph_replay_mixed_with_eager_launches(cuda, n, variant):
    """a CUDA graph captured with one d, replayed on one
    stream while eager launches of the same order with other d run on a
    second stream (and a second graph on a third) -- every kernel reads its
    d from a constant-bank slot.  Captured launches wait on / record the
    slot events as graph event nodes, so no slot is overwritten under a
    running kernel: each result is the oracle's for its own d (bitwise,
    or within 1e-12 of the summed-term magnitude in DFMA mode)."""
    nelt = 8192 if n <= 8 else 2048
    _raw, knl = fx.translate(fx.semlap_source(n))
    cur = torch.cuda.current_stream(cuda)
    cases = []
    for c in range(4):
        u, d, g = _sem_inputs(n, nelt, cuda, 300 + c)
        w = torch.full_like(u, float("nan"))
        env = lfb.env_from_buffers(knl, {"nelt": nelt},
                                   {"u": u, "d": d, "g": g, "w": w})
        cases.append((env, u, d, g, w))
    s_graph, s_eager, s_graph2 = (torch.cuda.Stream(cuda) for _ in range(3))
    graphs = []
    for c, s in ((0, s_graph), (2, s_graph2)):
        L = lfb.Launcher(knl, cases[c][0], variant=variant)
        L.launch()  # warm up outside the capture
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            L.launch()
        graphs.append((gr, s))
    for s in (s_graph, s_eager, s_graph2):
        s.wait_stream(cur)
    eager = [lfb.Launcher(knl, cases[c][0], variant=variant) for c in (1, 3)]
    for rep in range(6):
        for q, (gr, s) in enumerate(graphs):
            with torch.cuda.stream(s):
                gr.replay()
            with torch.cuda.stream(s_eager):
                eager[q].launch(stream=s_eager.cuda_stream)
    torch.cuda.synchronize()
    for env, u, d, g, w in cases:
        uh, dh, gh = u.cpu().numpy(), d.cpu().numpy(), g.cpu().numpy()
        ref = oracle.semlap(np.zeros(nelt * n ** 3), uh, dh, gh, n, nelt,
                            threads=8)
        got = w.cpu().numpy()
        if variant == 0:
            assert got.tobytes() == ref.tobytes()
        else:
            mag = oracle.semlap(np.zeros(nelt * n ** 3), np.abs(uh),
                                np.abs(dh), np.abs(gh), n, nelt, threads=8)
            assert (np.abs(got - ref) <= 1e-12 * mag).all()


@pytest.mark.parametrize("n", [8, 5])
def test_semlap_sumsq_epilogue(cuda, n):
    _raw, knl = fx.translate(fx.semlap_source(n))
    nelt = 3008  # the fixture assumes nelt mod 32 = 0
    u, d, g = _sem_inputs(n, nelt, cuda, 5)
    w = torch.empty_like(u)
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    sumsq = torch.zeros(1, dtype=torch.float64, device=cuda)
    ws = torch.zeros(4096, dtype=torch.float64, device=cuda)
    lfb.Launcher(knl, env, sumsq=sumsq, workspace=ws).launch()
    torch.cuda.synchronize()
    ref = float((w.double() ** 2).sum())
    assert abs(float(sumsq) - ref) <= 1e-12 * abs(ref)


def test_fill_axpy_2_24(cuda):
    """BASELINE config 1 at full size: bitwise against numpy, which rounds
    each operation exactly like the reference (interp.py:169-187)."""
    n = 1 << 24
    _r, kf = fx.translate(fx.fill_source("f64"))
    env = lfb.make_device_env(kf, {"n": n}, {"a": 1.5}, device=cuda)
    out = lfb.interpret(kf, env)
    assert bool((out.arrays["out"].data == 1.5).all())
    _r, ka = fx.translate(fx.axpy_source("f64"))
    gen = torch.Generator(device=cuda).manual_seed(1)
    x = torch.rand(n, dtype=torch.float64, device=cuda, generator=gen)
    y = torch.rand(n, dtype=torch.float64, device=cuda, generator=gen)
    y0 = y.cpu().numpy().copy()
    env = lfb.env_from_buffers(ka, {"n": n}, {"x": x, "y": y},
                               {"alpha": 1.25})
    lfb.interpret(ka, env, inplace=True)
    want = y0 + np.float64(1.25) * x.cpu().numpy()
    assert y.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("n", [1, 5, 127, 129, 1000003])
def test_fill_axpy_ragged(cuda, n):
    for dt, npt in (("f64", np.float64), ("f32", np.float32)):
        _r, ka = fx.translate(fx.axpy_source(dt))
        env = lfb.make_device_env(ka, {"n": n}, {"alpha": 0.3}, seed=n,
                                  device=cuda)
        y = np.random.default_rng(n).random(n).astype(npt)
        env.arrays["y"].data.copy_(torch.from_numpy(y))
        x = env.arrays["x"].data.cpu().numpy()
        out = lfb.interpret(ka, env)
        want = y + npt(0.3) * x
        assert out.arrays["y"].data.cpu().numpy().tobytes() == want.tobytes()
        _r, kf = fx.translate(fx.fill_source(dt))
        env = lfb.make_device_env(kf, {"n": n}, {"a": 0.1}, device=cuda)
        out = lfb.interpret(kf, env)
        assert (out.arrays["out"].data.cpu().numpy() == npt(0.1)).all()


@pytest.mark.parametrize("n", [1 << 20, (1 << 20) + 2, 1000003, 4097])
@pytest.mark.parametrize("variant", [0, 1])
def test_fill_no_overrun(cuda, n, variant):
    """The bulk-copy fill (variant 0) and the vector-store fill (variant 1)
    write exactly out[0, n): a canary after the end stays untouched."""
    for dt, tdt in (("f64", torch.float64), ("f32", torch.float32)):
        _r, kf = fx.translate(fx.fill_source(dt))
        base = torch.zeros(n + 64, dtype=tdt, device=cuda)
        env = lfb.env_from_buffers(kf, {"n": n}, {"out": base[:n]},
                                   {"a": 0.75})
        lfb.interpret(kf, env, inplace=True, variant=variant)
        h = base.cpu().numpy()
        assert (h[:n] == 0.75).all() and (h[n:] == 0).all()


def test_fill_misaligned_pointer(cuda):
    _r, kf = fx.translate(fx.fill_source("f64"))
    base = torch.zeros(1001, dtype=torch.float64, device=cuda)
    env = lfb.env_from_buffers(kf, {"n": 1000}, {"out": base[1:]},
                               {"a": 2.0})
    lfb.interpret(kf, env, inplace=True)
    h = base.cpu().numpy()
    assert h[0] == 0 and (h[1:] == 2.0).all()


@pytest.mark.parametrize("n", [4096, 128, 256, 1024 + 128, 1000, 4094])
def test_matvec(cuda, n):
    """BASELINE config 2 at n=4096: full bitwise comparison (ragged n: the
    untransformed kernel, same entry point)."""
    raw, knl = fx.translate(fx.matvec_source("f64"))
    knl = knl if n % 128 == 0 else raw
    gen = torch.Generator(device=cuda).manual_seed(n)
    a = torch.rand(n * n, dtype=torch.float64, device=cuda, generator=gen)
    x = torch.rand(n, dtype=torch.float64, device=cuda, generator=gen)
    y = torch.full((n,), float("nan"), dtype=torch.float64, device=cuda)
    env = lfb.env_from_buffers(knl, {"n": n}, {"a": a, "x": x, "y": y})
    lfb.interpret(knl, env, inplace=True, variant=3)  # bitwise TMA kernel
    ref = oracle.matvec(np.zeros(n), a.cpu().numpy(), x.cpu().numpy(), n,
                        threads=8)
    assert y.cpu().numpy().tobytes() == ref.tobytes()
    y.fill_(float("nan"))
    lfb.interpret(knl, env, inplace=True, variant=4)  # 28-row panels
    assert y.cpu().numpy().tobytes() == ref.tobytes()

    y.fill_(float("nan"))
    lfb.interpret(knl, env, inplace=True, variant=1)  # bitwise direct loads
    assert y.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("variant", [0, 2])
@pytest.mark.parametrize("n", [4096, 256, 1024 + 128, 1000, 2050])
def test_matvec_split_j(cuda, n, variant):
    """Default / variant 2: W column parts per row, summed in part order -- tolerance
    parity (north star: 1e-12 relative for fp64), here normwise and per row
    on [-1, 1) data like make_env's."""
    raw, knl = fx.translate(fx.matvec_source("f64", script=n % 128 == 0))
    knl = knl if n % 128 == 0 else raw
    gen = torch.Generator(device=cuda).manual_seed(n + 1)
    a = torch.rand(n * n, dtype=torch.float64, device=cuda, generator=gen)
    x = torch.rand(n, dtype=torch.float64, device=cuda, generator=gen)
    a = a * 2 - 1
    x = x * 2 - 1
    y = torch.full((n,), float("nan"), dtype=torch.float64, device=cuda)
    env = lfb.env_from_buffers(knl, {"n": n}, {"a": a, "x": x, "y": y})
    lfb.interpret(knl, env, inplace=True, variant=variant)
    ah, xh = a.cpu().numpy(), x.cpu().numpy()
    ref = oracle.matvec(np.zeros(n), ah, xh, n, threads=8)
    got = y.cpu().numpy()
    assert np.isfinite(got).all()
    err = np.abs(got - ref)
    assert err.max() <= 1e-12 * np.abs(ref).max()
    # per row against the magnitude the row sums over
    scale = np.abs(ah.reshape(n, n).T) @ np.abs(xh)
    assert (err <= 1e-12 * scale).all()


@pytest.mark.parametrize("n", [97, 130, 4095])
def test_matvec_untransformed_odd_sizes(cuda, n):
    """Odd n (TMA cannot describe the stride): direct-load path."""
    src = fx.matvec_source("f64", script=False)
    raw, _k = fx.translate(src)
    gen = torch.Generator(device=cuda).manual_seed(n)
    a = torch.rand(n * n, dtype=torch.float64, device=cuda, generator=gen)
    x = torch.rand(n, dtype=torch.float64, device=cuda, generator=gen)
    y = torch.zeros(n, dtype=torch.float64, device=cuda)
    env = lfb.env_from_buffers(raw, {"n": n}, {"a": a, "x": x, "y": y})
    lfb.interpret(raw, env, inplace=True)
    ref = oracle.matvec(np.zeros(n), a.cpu().numpy(), x.cpu().numpy(), n)
    assert y.cpu().numpy().tobytes() == ref.tobytes()


@pytest.mark.parametrize("m,n,l", [(256, 128, 64), (200, 72, 100),
                                   (1024, 512, 768)])
def test_sgemm_exact(cuda, m, n, l):
    """variant=1: the bit-exact CUDA-core path."""
    _r, knl = fx.translate(fx.gemm_source("f32"))
    rng = np.random.default_rng(m + n + l)
    a = rng.random(m * l).astype(np.float32)
    b = rng.random(l * n).astype(np.float32)
    c = rng.random(m * n).astype(np.float32)
    env = lfb.env_from_buffers(
        knl, {"m": m, "n": n, "l": l},
        {"a": torch.from_numpy(a).to(cuda), "b": torch.from_numpy(b).to(cuda),
         "c": torch.from_numpy(c.copy()).to(cuda)}, {"alpha": 1.5})
    out = lfb.interpret(knl, env, variant=1)
    ref = oracle.sgemm(np.float32(1.5), a, b, c.copy(), l, m, n, threads=8)
    assert out.arrays["c"].data.cpu().numpy().tobytes() == ref.tobytes()


# {{{ error behaviour mirrors the reference

def test_assumption_violation_is_interp_error(cuda):
    _r, knl = fx.translate(fx.semlap_source(8))
    with pytest.raises(InterpError, match="assumption"):
        lfb.make_device_env(knl, {"nelt": 33}, device=cuda)


def test_commuted_operands_hit_the_hand_written_kernel(cuda):
    """`y(i) + x(i)*alpha` is bit-identical to the template's
    `y(i) + alpha*x(i)` (one IEEE multiply commutes exactly; association,
    expr.py:243-255, is kept), so it runs lfb_axpy_f64 -- bitwise."""
    for body in ("y(i) + x(i)*alpha", "x(i)*alpha + y(i)",
                 "alpha*x(i) + y(i)"):
        src = fx.axpy_source("f64").replace("y(i) + alpha*x(i)", body)
        _r, knl = fx.translate(src)
        assert lfb.recognize(knl).workload.name == "axpy"
        env = lfb.make_device_env(knl, {"n": 1000}, {"alpha": 1.7}, seed=1,
                                  device=cuda)
        out = lfb.interpret(knl, env, engine="kernels")
        y = env.arrays["y"].data.cpu().numpy()
        x = env.arrays["x"].data.cpu().numpy()
        alpha = env.scalars["alpha"]
        assert out.arrays["y"].data.cpu().numpy().tobytes() == \
            (y + alpha * x).tobytes(), body


def test_unrecognised_kernel_is_codegen_error(cuda):
    """A re-associated body is a different computation: CodegenError from
    the hand-written engine, generated CUDA under the default engine."""
    src = fx.axpy_source("f64").replace("y(i) + alpha*x(i)",
                                        "alpha*(x(i) + y(i))")
    _r, knl = fx.translate(src)
    env = lfb.make_device_env(knl, {"n": 256}, {"alpha": 1.7}, seed=1,
                              device=cuda)
    with pytest.raises(CodegenError, match="no CPU fallback"):
        lfb.interpret(knl, env, engine="kernels")
    out = lfb.interpret(knl, env)
    y = env.arrays["y"].data.cpu().numpy()
    x = env.arrays["x"].data.cpu().numpy()
    alpha = env.scalars["alpha"]
    assert out.arrays["y"].data.cpu().numpy().tobytes() == \
        (alpha * (x + y)).tobytes()


def test_parameters_past_2_31_run_on_the_64_bit_build(cuda):
    """fill with n = 2^31 + 5: the emitted-C ABI's int cannot hold n (the
    reference interpreter's Python ints can), so interpret() routes the
    recognised kernel to the generic engine's 64-bit build instead of
    raising -- every element written, the tail past 2^31 included."""
    n = (1 << 31) + 5
    _r, knl = fx.translate(fx.fill_source("f32"))
    out = torch.zeros(n, dtype=torch.float32, device=cuda)
    env = lfb.env_from_buffers(knl, {"n": n}, {"out": out}, {"a": 0.75})
    with pytest.raises(CodegenError, match="C int"):
        lfb.Launcher(knl, env)
    lfb.interpret(knl, env, inplace=True)
    torch.cuda.synchronize()
    assert int((out == 0.75).sum()) == n
    assert float(out[-1]) == 0.75 and float(out[(1 << 31) - 1]) == 0.75
    del out, env
    torch.cuda.empty_cache()


def test_wrong_shape_input_is_interp_error(cuda):
    _r, knl = fx.translate(fx.fill_source("f64"))
    with pytest.raises(InterpError, match="expected shape"):
        lfb.make_device_env(knl, {"n": 10}, {"out": np.zeros(11)},
                            device=cuda)

# }}}


# {{{ sgemm on tensor cores (tolerance parity)

@pytest.mark.parametrize("variant", [2, 3, 4])
@pytest.mark.parametrize("m,n,l", [(128, 256, 32), (256, 512, 256),
                                   (1024, 768, 4096), (384, 256, 8192),
                                   (3200, 3072, 64), (4096, 2048, 512)])
def test_sgemm_tensor_cores(cuda, m, n, l, variant):
    """variant=2: tcgen05 kind::tf32 with the 3xTF32 split (persistent,
    double-buffered TMEM; variant 3 the first one-tile-per-CTA kernel).  Tolerance
    (north star: 1e-5 relative for fp32), normwise against the reference's
    own fp32 sequential result (the oracle), and the same bound against an
    exact fp64 product; the reference's own rounding error is printed."""
    _r, knl = fx.translate(fx.gemm_source("f32"))
    rng = np.random.default_rng(m * 7 + n * 3 + l)
    a = rng.random(m * l).astype(np.float32)
    b = rng.random(l * n).astype(np.float32)
    c = rng.random(m * n).astype(np.float32)
    alpha = np.float32(1.5)
    env = lfb.env_from_buffers(
        knl, {"m": m, "n": n, "l": l},
        {"a": torch.from_numpy(a).to(cuda), "b": torch.from_numpy(b).to(cuda),
         "c": torch.from_numpy(c.copy()).to(cuda)}, {"alpha": alpha})
    out = lfb.interpret(knl, env, variant=variant)
    got = out.arrays["c"].data.cpu().numpy().astype(np.float64)
    ref = oracle.sgemm(alpha, a, b, c.copy(), l, m, n, threads=8) \
        .astype(np.float64)
    A = a.astype(np.float64).reshape(l, m).T      # column major (m, l)
    B = b.astype(np.float64).reshape(n, l).T      # column major (l, n)
    exact = (c.astype(np.float64).reshape(n, m).T
             + float(alpha) * (A @ B)).T.reshape(-1)
    err_ref = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    err_exact = np.linalg.norm(got - exact) / np.linalg.norm(exact)
    ref_own = np.linalg.norm(ref - exact) / np.linalg.norm(exact)
    print(f"m={m} n={n} l={l}: |tc-ref|/|ref|={err_ref:.2e} "
          f"|tc-exact|={err_exact:.2e} |ref-exact|={ref_own:.2e} "
          f"max rel={np.max(np.abs(got - ref) / np.abs(ref)):.2e}")
    assert err_ref <= 1e-5
    assert err_exact <= 1e-5


@pytest.mark.parametrize("m,n,l,variant", [(128, 128, 16, 0),
                                           (256, 384, 512, 0),
                                           (1024, 512, 2048, 0),
                                           (512, 256, 8192, 0),
                                           (256, 384, 512, 3),
                                           (384, 256, 1040, 0)])
def test_dgemm_tensor_cores(cuda, m, n, l, variant):
    """The paper's DGEMM in real*8 on the FP64 tensor cores (DMMA):
    tolerance parity (north star: 1e-12 relative fp64) against the
    reference's sequential-k result -- normwise, and per entry against the
    magnitude sum_k |alpha b a| + |c| on [-1, 1) data."""
    _r, knl = fx.translate(fx.gemm_source("f64"))
    rng = np.random.default_rng(m + n + l)
    a = rng.random(m * l) * 2 - 1
    b = rng.random(l * n) * 2 - 1
    c = rng.random(m * n) * 2 - 1
    alpha = 1.5
    env = lfb.env_from_buffers(
        knl, {"m": m, "n": n, "l": l},
        {"a": torch.from_numpy(a).to(cuda), "b": torch.from_numpy(b).to(cuda),
         "c": torch.from_numpy(c.copy()).to(cuda)}, {"alpha": alpha})
    out = lfb.interpret(knl, env, variant=variant)  # 3: 16 x 4 k tiles
    got = out.arrays["c"].data.cpu().numpy()
    ref = oracle.sgemm(alpha, a, b, c.copy(), l, m, n, threads=8)
    mag = oracle.sgemm(alpha, np.abs(a), np.abs(b), np.abs(c), l, m, n,
                       threads=8)
    err = np.abs(got - ref)
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    assert (err <= 1e-12 * mag).all()
    assert got.tobytes() != ref.tobytes()  # really the fused path


@pytest.mark.parametrize("m,n,l", [(128, 128, 16), (100, 60, 33),
                                   (300, 130, 70)])
def test_dgemm_exact(cuda, m, n, l):
    """variant 1 (and every shape the tensor-core path cannot take): the
    reference's chain c + (alpha*b)*a per k on the FP64 CUDA cores,
    bitwise."""
    _r, knl = fx.translate(fx.gemm_source("f64", script=False))
    rng = np.random.default_rng(m * n + l)
    a, b, c = rng.random(m * l), rng.random(l * n), rng.random(m * n)
    env = lfb.env_from_buffers(
        knl, {"m": m, "n": n, "l": l},
        {"a": torch.from_numpy(a).to(cuda), "b": torch.from_numpy(b).to(cuda),
         "c": torch.from_numpy(c.copy()).to(cuda)}, {"alpha": 1.25})
    variant = 1 if m % 128 == 0 else 0
    out = lfb.interpret(knl, env, variant=variant)
    ref = oracle.sgemm(1.25, a, b, c.copy(), l, m, n, threads=8)
    assert out.arrays["c"].data.cpu().numpy().tobytes() == ref.tobytes()


def test_sgemm_default_dispatch(cuda):
    """Default variant: tensor cores for 128/256/32-aligned shapes, the
    bit-exact kernel otherwise -- both on the device."""
    _r, knl = fx.translate(fx.gemm_source("f32"))
    m, n, l = 100, 36, 50
    rng = np.random.default_rng(1)
    a = rng.random(m * l).astype(np.float32)
    b = rng.random(l * n).astype(np.float32)
    c = rng.random(m * n).astype(np.float32)
    env = lfb.env_from_buffers(
        knl, {"m": m, "n": n, "l": l},
        {"a": torch.from_numpy(a).to(cuda), "b": torch.from_numpy(b).to(cuda),
         "c": torch.from_numpy(c.copy()).to(cuda)}, {"alpha": 0.5})
    out = lfb.interpret(knl, env)
    ref = oracle.sgemm(np.float32(0.5), a, b, c.copy(), l, m, n)
    assert out.arrays["c"].data.cpu().numpy().tobytes() == ref.tobytes()

@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_gemm_8192_cubed_vs_oracle(cuda, dtype):
    """BASELINE config 5 at its own size: the paper's GEMM script, 8192^3,
    default dispatch through interpret() (sgemm: tcgen05 3xTF32; dgemm:
    DMMA), checked on 64 FULL columns (4 spread groups of 16) against the
    oracle's restatement of the reference's sequential chain
    c + (alpha*b)*a over ascending k (test_fortran.py:72-103, interp.py:
    169-187; the oracle is pinned to the reference's emitted C by
    test_oracle.py).  Tolerance (north star): normwise max|d|/max|ref| <=
    1e-5 for fp32, 1e-12 for fp64; the fp64 case also per entry against
    the magnitude sum (|c| + sum_k |alpha b a|)."""
    m = n = l = 8192
    np_dt = np.float32 if dtype == "f32" else np.float64
    _r, knl = fx.translate(fx.gemm_source(dtype))
    gen = torch.Generator(device=cuda).manual_seed(81)
    tdt = torch.float32 if dtype == "f32" else torch.float64
    a = torch.rand(m * l, dtype=tdt, device=cuda, generator=gen)
    b = torch.rand(l * n, dtype=tdt, device=cuda, generator=gen)
    c = torch.rand(m * n, dtype=tdt, device=cuda, generator=gen)
    alpha = np_dt(1.5)
    env = lfb.env_from_buffers(knl, {"m": m, "n": n, "l": l},
                               {"a": a, "b": b, "c": c}, {"alpha": alpha})
    out = lfb.interpret(knl, env)
    torch.cuda.synchronize()
    got_all = out.arrays["c"].data
    ah = a.cpu().numpy()
    bh = b.cpu().numpy()
    per = 16
    worst = 0.0
    for j0 in (0, 2731, 5461, n - per):
        cols = slice(j0 * m, (j0 + per) * m)
        ref = c[cols].cpu().numpy()
        oracle.sgemm(alpha, ah, np.ascontiguousarray(bh[j0 * l:(j0 + per) * l]),
                     ref, l, m, per, threads=16)
        got = got_all[cols].cpu().numpy()
        d = np.abs(got.astype(np.float64) - ref.astype(np.float64))
        normwise = d.max() / np.abs(ref).max()
        worst = max(worst, normwise)
        if dtype == "f32":
            assert normwise <= 1e-5, (j0, normwise)
        else:
            assert normwise <= 1e-12, (j0, normwise)
            mag = oracle.sgemm(alpha, np.abs(ah),
                               np.abs(bh[j0 * l:(j0 + per) * l]).copy(),
                               np.abs(c[cols].cpu().numpy()), l, m, per,
                               threads=16)
            assert (d <= 1e-12 * mag).all(), j0
    print(f"{dtype} 8192^3: worst normwise error vs the oracle {worst:.2e}")


# }}}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 50])
def test_semlap_offsets_past_2_31(cuda, variant):
    """Full-size indexing: 2^20 + 37 elements at n = 8, so g holds
    3.2e9 doubles and its flat index passes 2^31 at element 699,051 (where
    the reference's emitted C overflows its int).  Every element is
    written (no NaN left), and sampled elements on both sides of that
    boundary, the ends and random places match the oracle: bitwise in the
    default mode, within 1e-12 of the summed-term magnitude in DFMA mode."""
    n, nelt = 8, (1 << 20) + 37
    np3 = n ** 3
    _raw, knl = fx.translate(fx.semlap_source(n, block=1))
    u, d, g = _sem_inputs(n, nelt, cuda, 77)
    w = torch.full_like(u, float("nan"))
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    lfb.interpret(knl, env, inplace=True, variant=variant)
    torch.cuda.synchronize()
    assert not bool(torch.isnan(w).any())
    cross = (1 << 31) // (6 * np3)
    es = np.unique(np.concatenate([
        [0, 1, nelt - 2, nelt - 1, cross - 1, cross, cross + 1,
         (1 << 31) // np3 % nelt],
        np.random.default_rng(5).integers(0, nelt, 120)]))
    dh = d.cpu().numpy()
    for e in es.tolist():
        ue = u[e * np3:(e + 1) * np3].cpu().numpy()
        ge = g[6 * e * np3:6 * (e + 1) * np3].cpu().numpy()
        we = w[e * np3:(e + 1) * np3].cpu().numpy()
        ref = oracle.semlap(np.zeros(np3), ue, dh, ge, n, 1)
        if variant == 0:
            assert we.tobytes() == ref.tobytes(), e
        else:
            mag = oracle.semlap(np.zeros(np3), np.abs(ue), np.abs(dh),
                                np.abs(ge), n, 1)
            assert (np.abs(we - ref) <= 1e-12 * mag).all(), e


@pytest.mark.gpu
@pytest.mark.parametrize("n,variant", [(16, 0), (15, 0), (13, 0), (16, 50)])
def test_semlap_high_order_offsets_past_2_31(cuda, n, variant):
    """The high-order defaults (line-owner kernel bitwise, DMMA kernel in
    DFMA mode) past the 2^31 flat index of g: nelt just above
    2^31 / (6 n^3), every element written, sampled elements around the
    boundary, the ends and random places against the oracle."""
    np3 = n ** 3
    cross = (1 << 31) // (6 * np3)
    nelt = cross + 53
    _raw, knl = fx.translate(fx.semlap_source(n, block=1))
    u, d, g = _sem_inputs(n, nelt, cuda, 78 + n)
    w = torch.full_like(u, float("nan"))
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    lfb.interpret(knl, env, inplace=True, variant=variant)
    torch.cuda.synchronize()
    assert not bool(torch.isnan(w).any())
    es = np.unique(np.concatenate([
        [0, 1, nelt - 2, nelt - 1, cross - 1, cross, cross + 1],
        np.random.default_rng(n).integers(0, nelt, 24)]))
    dh = d.cpu().numpy()
    for e in es.tolist():
        ue = u[e * np3:(e + 1) * np3].cpu().numpy()
        ge = g[6 * e * np3:6 * (e + 1) * np3].cpu().numpy()
        we = w[e * np3:(e + 1) * np3].cpu().numpy()
        ref = oracle.semlap(np.zeros(np3), ue, dh, ge, n, 1)
        if variant == 0:
            assert we.tobytes() == ref.tobytes(), e
        else:
            mag = oracle.semlap(np.zeros(np3), np.abs(ue), np.abs(dh),
                                np.abs(ge), n, 1)
            assert (np.abs(we - ref) <= 1e-12 * mag).all(), e
    del u, d, g, w, env
    torch.cuda.empty_cache()
