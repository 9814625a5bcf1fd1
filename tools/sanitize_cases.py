"""Small launches of every hand-written kernel family, for
compute-sanitizer (memcheck / racecheck / synccheck): tools/gpu_sanitize.sh.
Each case also checks its result against the oracle so a sanitizer run is a
parity run too."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402

dev = torch.device("cuda", 0)


def sem(n, nelt, variant, exact=True):
    _r, knl = fx.translate(fx.semlap_source(n, block=1))
    g = torch.Generator(device=dev).manual_seed(n)
    u = torch.rand(nelt * n ** 3, dtype=torch.float64, device=dev,
                   generator=g) * 2 - 1
    gg = torch.rand(6 * nelt * n ** 3, dtype=torch.float64, device=dev,
                    generator=g)
    d = torch.rand(n * n, dtype=torch.float64, device=dev, generator=g)
    w = torch.zeros_like(u)
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": gg, "w": w})
    lfb.Launcher(knl, env, variant=variant).launch()
    torch.cuda.synchronize()
    ref = oracle.semlap(np.zeros(u.numel()), u.cpu().numpy(), d.cpu().numpy(),
                        gg.cpu().numpy(), n, nelt)
    got = w.cpu().numpy()
    ok = got.tobytes() == ref.tobytes() if exact else \
        np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    print(f"semlap n={n} nelt={nelt} variant={variant}: "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def gemm(dt, m, n, l, variant, exact):
    _r, knl = fx.translate(fx.gemm_source(dt))
    npt = np.float32 if dt == "f32" else np.float64
    rng = np.random.default_rng(1)
    a, b, c = (rng.random(s).astype(npt) for s in (m * l, l * n, m * n))
    env = lfb.env_from_buffers(
        knl, {"m": m, "n": n, "l": l},
        {"a": torch.from_numpy(a).to(dev), "b": torch.from_numpy(b).to(dev),
         "c": torch.from_numpy(c.copy()).to(dev)}, {"alpha": 1.5})
    out = lfb.interpret(knl, env, variant=variant)
    got = out.arrays["c"].data.cpu().numpy()
    ref = oracle.sgemm(npt(1.5), a, b, c.copy(), l, m, n, threads=8)
    tol = 1e-5 if dt == "f32" else 1e-12
    ok = got.tobytes() == ref.tobytes() if exact else \
        np.linalg.norm(got - ref) <= tol * np.linalg.norm(ref)
    print(f"{dt}gemm {m}x{n}x{l} variant={variant}: "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def streams():
    n = 100003
    _r, kf = fx.translate(fx.fill_source("f64"))
    env = lfb.make_device_env(kf, {"n": n}, {"a": 0.5}, device=dev)
    ok = bool((lfb.interpret(kf, env).arrays["out"].data == 0.5).all())
    _r, km = fx.translate(fx.matvec_source("f64"))
    nn = 2048  # every stage ring wraps several times
    a = torch.rand(nn * nn, dtype=torch.float64, device=dev)
    x = torch.rand(nn, dtype=torch.float64, device=dev)
    for v in (0, 3):
        y = torch.zeros(nn, dtype=torch.float64, device=dev)
        env = lfb.env_from_buffers(km, {"n": nn}, {"a": a, "x": x, "y": y})
        lfb.interpret(km, env, inplace=True, variant=v)
        ref = oracle.matvec(np.zeros(nn), a.cpu().numpy(), x.cpu().numpy(),
                            nn)
        ok &= float(np.abs(y.cpu().numpy() - ref).max()) <= 1e-12 * nn
    print(f"fill/matvec: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def generic_gemm(m, n, l, want_tma):
    """The generic engine on the paper's DGEMM script: TMA-fetched,
    double-buffered tiles (even m) or the cooperative fallback (odd m)."""
    from paper_1503_07659_b200.generic import GenericLauncher
    _r, knl = fx.translate(fx.gemm_source("f64"))
    rng = np.random.default_rng(m)
    a, b, c = rng.random((m, l)), rng.random((l, n)), rng.random((m, n))
    env = lfb.make_device_env(knl, {"m": m, "n": n, "l": l},
                              {"a": a, "b": b, "c": c, "alpha": 1.5},
                              device=dev)
    tma = GenericLauncher(knl, env).tensor_maps(env)[1]
    got = lfb.get_output(lfb.interpret(knl, env, engine="generic"), "c")
    want = c.copy()
    for k in range(l):
        want = want + (1.5 * b[k, :])[None, :] * a[:, k][:, None]
    ok = tma == want_tma and got.tobytes() == want.tobytes()
    print(f"generic dgemm {m}x{n}x{l} tma={tma}: "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def generic_prefetch():
    """Work-group-level TMA prefetch rings (smoother, tiled transpose) with
    several groups per CTA."""
    n = 64 * 6000
    _r, km = fx.translate(fx.generic_source("smooth"))
    u = np.random.default_rng(1).random(n + 2)
    env = lfb.make_device_env(km, {"n": n}, {"u": u}, device=dev)
    got = lfb.get_output(lfb.interpret(km, env), "r")
    ok = got.tobytes() == ((u[:-2] + 2.0 * u[1:-1]) + u[2:]).tobytes()
    _r, kt = fx.translate(fx.generic_source("ttile"))
    a = np.random.default_rng(2).random((560, 600))
    env = lfb.make_device_env(kt, {"n": 560, "m": 600}, {"a": a}, device=dev)
    got = lfb.get_output(lfb.interpret(kt, env), "b")
    ok &= got.tobytes() == np.ascontiguousarray(a.T).tobytes()
    print(f"generic prefetch rings: {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def assembly():
    """dssum (every mode through the 2-slab protocol) and a traced run."""
    from paper_1503_07659_b200.assembly import BoxMesh, _launch, dssum
    mesh = BoxMesh(3, 2, 4, 5)
    w = torch.rand(mesh.nelt * 125, dtype=torch.float64, device=dev)
    ref = oracle.dssum(w.cpu().numpy(), 5, 3, 2, 4)
    whole = w.clone()
    dssum(whole, mesh)
    per = 3 * 2 * 125
    lo, hi = w[:2 * per], w[2 * per:]
    s_lo, s_hi = mesh.slab(0, 2), mesh.slab(1, 2)
    _launch(lo, s_lo, 0, s_lo.top - 1, 0)
    _launch(hi, s_hi, 1, s_hi.top, 0)
    part = torch.empty(mesh.plane, dtype=torch.float64, device=dev)
    tot = torch.empty_like(part)
    _launch(lo, s_lo, s_lo.top, s_lo.top, 1, None, part)
    _launch(hi, s_hi, 0, 0, 2, part, tot)
    _launch(lo, s_lo, s_lo.top, s_lo.top, 3, tot, None)
    torch.cuda.synchronize()
    ok = whole.cpu().numpy().tobytes() == ref.tobytes() and \
        torch.equal(w, whole)
    _r, kg = fx.translate(fx.gemm_source("f64"))
    env = lfb.make_device_env(kg, {"m": 20, "n": 12, "l": 40},
                              {"alpha": 0.5}, seed=3, trace=True, device=dev)
    out = lfb.interpret(kg, env)
    ok &= len(out.write_trace) > 0
    print(f"dssum modes / write trace: {'ok' if ok else 'MISMATCH'}",
          flush=True)
    return ok


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    oks = []
    if which in ("all", "sem"):
        oks += [sem(8, 37, 0), sem(8, 37, 50, False), sem(8, 37, 39),
                sem(4, 33, 0), sem(7, 9, 61, False), sem(9, 5, 0),
                sem(12, 5, 0), sem(15, 3, 51, False), sem(16, 3, 51, False),
                sem(16, 5, 52, False), sem(16, 5, 54, False),
                sem(16, 7, 0), sem(13, 7, 70), sem(12, 4, 71, False),
                sem(15, 3, 72)]
    if which in ("all", "gemm"):
        oks += [gemm("f32", 256, 256, 64, 0, False),
                gemm("f32", 256, 256, 512, 0, False),  # the ring wraps
                gemm("f32", 100, 60, 33, 1, True),
                gemm("f64", 256, 128, 64, 0, False),
                gemm("f64", 128, 256, 256, 0, False),  # ring wraps
                gemm("f64", 128, 128, 48, 0, False),   # 16 x 5 ring
                gemm("f64", 100, 60, 33, 1, True)]
    if which in ("all", "stream"):
        oks.append(streams())
    if which in ("all", "assembly"):
        oks.append(assembly())
    if which in ("all", "generic"):
        oks += [generic_gemm(64, 40, 96, True), generic_gemm(37, 20, 45, False),
                generic_prefetch()]
    sys.exit(0 if all(oks) else 1)
