"""Edge cases the reference defines (③): empty and ragged
extents.

* ``make_env`` rejects a non-positive array extent with InterpError
  (interp.py:107-112); ``make_device_env`` does the same.
* The emitted-C ABI (codegen.py:511-527) at a zero extent runs no
  iterations and touches nothing; every C-ABI launcher and ``interpret`` on
  wrapped buffers (``env_from_buffers``) are the same no-op.
* Ragged extents (not a multiple of the tile) are covered by the parity
  suites (test_gpu_parity.py, test_generic.py); here one odd size per
  workload is run through both engines against the oracle.
"""

import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import paper_1503_07659_b200 as lfb
from paper_1503_07659_b200 import abi, fixtures as fx
from paper_1503_07659_b200._loopforge import InterpError

ZERO = [("fill", fx.fill_source("f64"), {"n": 0}),
        ("axpy", fx.axpy_source("f64"), {"n": 0}),
        ("matvec", fx.matvec_source("f64"), {"n": 0}),
        ("semlap", fx.semlap_source(4, block=2), {"nelt": 0}),
        ("sgemm", fx.gemm_source("f32"), {"m": 16, "n": 8, "l": 0}),
        ("dgemm", fx.gemm_source("f64"), {"m": 0, "n": 8, "l": 32})]


@pytest.mark.parametrize("name,src,params", ZERO, ids=[z[0] for z in ZERO])
def test_make_device_env_rejects_empty_arrays(name, src, params):
    _raw, knl = fx.translate(src, f"{name}.f")
    with pytest.raises(InterpError, match="non-positive shape"):
        lfb.make_device_env(knl, params, device="cpu")


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["auto", "generic"])
@pytest.mark.parametrize("name,src,params", ZERO, ids=[z[0] for z in ZERO])
def test_zero_extent_is_a_noop(name, src, params, engine, cuda):
    """Zero-size work through interpret() on caller buffers: no launch
    error, outputs untouched (a sentinel buffer keeps its bits)."""
    _raw, knl = fx.translate(src, f"{name}.f")
    bufs = {}
    for a in knl.args:
        if a.kind == "global-array":
            dt = torch.float32 if a.dtype == "f32" else torch.float64
            bufs[a.name] = torch.full((512,), 7.25, dtype=dt, device=cuda)
    scal = {a.name: 1.5 for a in knl.args if a.kind == "scalar-value"}
    env = lfb.env_from_buffers(knl, params, bufs, scal)
    lfb.interpret(knl, env, inplace=True, engine=engine)
    torch.cuda.synchronize()
    for t in bufs.values():
        assert bool((t == 7.25).all())


@pytest.mark.gpu
def test_c_abi_zero_extent(cuda):
    """Each launcher at n = 0 returns LFB_OK without touching memory."""
    lib = abi.load()
    t = torch.full((8,), 3.0, dtype=torch.float64, device=cuda)
    f = torch.full((8,), 3.0, dtype=torch.float32, device=cuda)
    p, q = t.data_ptr(), f.data_ptr()
    s = torch.cuda.current_stream().cuda_stream
    assert lib.lfb_fill_f64(p, 1.0, 0, None, s) == abi.LFB_OK
    assert lib.lfb_fill_f32(q, 1.0, 0, None, s) == abi.LFB_OK
    assert lib.lfb_axpy_f64(p, p, 2.0, 0, None, s) == abi.LFB_OK
    assert lib.lfb_axpy_f32(q, q, 2.0, 0, None, s) == abi.LFB_OK
    assert lib.lfb_matvec_f64(p, p, p, 0, None, s) == abi.LFB_OK
    geo = abi.make_launch(npts=4)
    assert lib.lfb_semlap_f64(p, p, p, p, 0, C.byref(geo), s) == abi.LFB_OK
    for m, n, l in ((0, 8, 8), (8, 0, 8), (8, 8, 0)):
        assert lib.lfb_dgemm_f64(1.0, p, p, p, l, m, n, None, s) == \
            abi.LFB_OK
    torch.cuda.synchronize()
    assert bool((t == 3.0).all()) and bool((f == 3.0).all())


RAGGED = [("fill", fx.fill_source("f64"), {"n": 1}),
          ("axpy", fx.axpy_source("f64"), {"n": 129}),
          ("matvec", fx.matvec_source("f64", block=16), {"n": 48}),
          ("semlap", fx.semlap_source(5, block=2, assume=False), {"nelt": 3})]


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["auto", "generic"])
@pytest.mark.parametrize("name,src,params", RAGGED,
                         ids=[r[0] for r in RAGGED])
def test_ragged_extents_match_the_oracle(name, src, params, engine, cuda):
    _raw, knl = fx.translate(src, f"{name}.f")
    env = lfb.make_device_env(knl, params, seed=5, device=cuda)
    if "a" in env.scalars:
        env.scalars["a"] = np.float64(1.5)
    if "alpha" in env.scalars:
        env.scalars["alpha"] = np.float64(1.25)
    host = {k: v.data.cpu().numpy().copy() for k, v in env.arrays.items()}
    out = lfb.interpret(knl, env, engine=engine)
    got = {k: v.data.cpu().numpy() for k, v in out.arrays.items()}
    if name == "fill":
        want = host["out"].copy()
        oracle.fill(want, 1.5)
        assert got["out"].tobytes() == want.tobytes()
    elif name == "axpy":
        want = host["y"].copy()
        oracle.axpy(want, host["x"], 1.25)
        assert got["y"].tobytes() == want.tobytes()
    elif name == "matvec":
        nn = params["n"]
        want = oracle.matvec(host["y"].copy(), host["a"], host["x"], nn)
        # the split-j default reassociates; the generic engine does not
        if engine == "generic":
            assert got["y"].tobytes() == want.tobytes()
        else:
            assert np.abs(got["y"] - want).max() <= \
                1e-12 * nn * np.abs(want).max()
    else:
        n, nelt = 5, params["nelt"]
        want = oracle.semlap(host["w"].copy(), host["u"], host["d"],
                             host["g"], n, nelt)
        assert got["w"].tobytes() == want.tobytes()
