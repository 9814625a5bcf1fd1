"""The reference's run-time checks, on the device (race
detection / sanitizers; the reference's tests/test_interp.py:139-192).

* ``interpret(kernel, env, bounds_check=False)`` keeps the reference's
  signature (interp.py:323); ``interpret_bounds_checked`` (403-405) exists.
* Out-of-bounds subscripts raise InterpError naming the instruction: the
  checked build of the generated CUDA records the first violation of a
  launch (cudagen.py ``checked``), the host raises the reference's message.
* A read of a temporary no instruction writes raises "never-written".
* ``make_env(trace=True)``'s write trace: the trace build records every
  store on the device, the host sorts the records into the sequential
  interpreter's order -- the same list the reference builds.
"""

import dataclasses
import inspect

import numpy as np
import pytest
import torch

import paper_1503_07659_b200 as lfb
from conftest import Golden
from paper_1503_07659_b200 import fixtures as fx
from paper_1503_07659_b200._loopforge import (InterpError, kernel as lfk,
                                              polyset, transforms)
from paper_1503_07659_b200.cudagen import emit_cuda
from paper_1503_07659_b200.generic import compile_program


def sec51_precomputed():
    """The reference's §5.1 forward difference with a precomputed tile
    (tests/test_interp.py sec51_precomputed)."""
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "result[i] = u[i+1]-u[i]",
                          name="fwd_diff")
    knl = transforms.split_iname(knl, "i", 16)
    knl = transforms.assume(knl, "n mod 16 = 0")
    knl = transforms.extract_subst(knl, "u_acc", "u[j]", parameters="j")
    return transforms.precompute(knl, "u_acc", "i_inner", default_tag=None)


def test_interpret_keeps_the_reference_signature():
    params = list(inspect.signature(lfb.interpret).parameters)
    assert params[:3] == ["kernel", "env", "bounds_check"]
    assert callable(lfb.interpret_bounds_checked)


def test_read_never_written_temporary():
    knl = lfk.make_kernel(["{[i]: 0<=i<4}"], "<> t = a[i]\nout[i] = t")
    reader = dataclasses.replace(knl.instructions[1],
                                 depends_on=frozenset())
    broken = knl.copy(instructions=(reader,))
    env = lfb.make_device_env(broken, {}, {"a": np.ones(4, np.float32)},
                              device="cpu")
    with pytest.raises(InterpError, match="never-written"):
        lfb.interpret(broken, env)


def test_trace_build_compiles():
    """make_env(trace=True) runs the trace build of the generated CUDA:
    every store also appends a record; workgroup tiles are per work-item
    (each work-item runs its own fetch, as in the reference interpreter)."""
    for src in (fx.gemm_source("f64"), fx.generic_source("cond"),
                fx.semlap_source(4, block=2)):
        _raw, knl = fx.translate(src)
        prog = emit_cuda(knl, checked="plain", trace=True)
        assert prog.trace and "lfb_trace(" in prog.source
        assert not prog.shared and not prog.tma
        assert compile_program(prog, True)[:4] == b"\x7fELF"


@pytest.mark.parametrize("mode", ["plain", "dims"])
def test_checked_builds_compile(mode):
    for src in (fx.gemm_source("f64"), fx.generic_source("matvec_acc"),
                fx.semlap_source(4, block=2)):
        _raw, knl = fx.translate(src)
        prog = emit_cuda(knl, checked=mode)
        assert prog.checked == mode and "lfb_oob(" in prog.source
        assert not prog.tma                 # plain layouts when checked
        assert compile_program(prog, True)[:4] == b"\x7fELF"


@pytest.mark.gpu
def test_out_of_bounds_reports_instruction(cuda):
    """tests/test_interp.py:139-147: the env lies about a's extent."""
    knl = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = a[i+3]")
    env = lfb.make_device_env(knl, {"n": 6},
                              {"a": np.ones(9, dtype=np.float32)},
                              device=cuda)
    env.arrays["a"].shape = (4,)
    with pytest.raises(InterpError, match="insn_0"):
        lfb.interpret(knl, env)


@pytest.mark.gpu
def test_bounds_checked_forward_diff_ok(cuda):
    knl = sec51_precomputed()
    u = np.random.default_rng(11).random(33).astype(np.float32)
    env = lfb.make_device_env(knl, {"n": 32}, {"u": u}, device=cuda)
    out = lfb.interpret_bounds_checked(knl, env)
    want = u[1:] - u[:-1]
    assert np.array_equal(lfb.get_output(out, "result"), want)


@pytest.mark.gpu
def test_bounds_checked_detects_shrunk_temp(cuda):
    knl = sec51_precomputed()
    temp = knl.temporaries["u_acc_0"]
    shrunk = lfk.TemporaryDecl(temp.name, temp.dtype,
                               (polyset.AffineExpr.const(16),),
                               temp.address_space, temp.base_offsets)
    bad = knl.copy(temporaries={**knl.temporaries, "u_acc_0": shrunk})
    env = lfb.make_device_env(bad, {"n": 32},
                              {"u": np.ones(33, dtype=np.float32)},
                              device=cuda)
    with pytest.raises(InterpError, match="u_acc_0"):
        lfb.interpret_bounds_checked(bad, env)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["gen_dgemm_m20_n12_l40", "gen_mvacc_n64",
                                  "gen_stencil_n250", "gen_rowsum_n40_m17",
                                  "semlap_n5_b2_nelt2"])
def test_bounds_checked_same_results(name, cuda):
    """In-bounds kernels: the checked build gives the reference's bits."""
    g = Golden(name)
    _raw, knl = g.kernels()
    env = lfb.make_device_env(knl, g.params, device=cuda)
    for a in knl.args:
        buf = g.inp(a.name)
        if a.kind == "scalar-value":
            env.scalars[a.name] = buf.reshape(-1)[0]
        else:
            env.arrays[a.name].data.copy_(torch.from_numpy(buf.copy()))
    out = lfb.interpret_bounds_checked(knl, env)
    for o in g.outputs():
        assert out.arrays[o].data.cpu().numpy().tobytes() == \
            g.out(o).tobytes(), f"{name}:{o}"


OOB_F = """subroutine shift(y, x, n)
  implicit none
  real*8 y(n), x(n)
  integer n, i

  do i = 1, n
    y(i) = x(i+1)
  end do
end
"""


def test_in_bounds_proof():
    """inbounds.unproven_access: every fixture kernel is proved in bounds
    (so the fast kernels may run unchecked); a subscript that leaves its
    declaration is reported."""
    from paper_1503_07659_b200.inbounds import unproven_access
    for src in (fx.fill_source("f64"), fx.axpy_source("f32"),
                fx.matvec_source("f64"), fx.gemm_source("f32"),
                fx.semlap_source(8), fx.semlap_source(5, block=2)):
        for knl in fx.translate(src):
            assert unproven_access(knl) is None
    _raw, knl = fx.translate(OOB_F)
    msg = unproven_access(knl)
    assert msg is not None and "upper bound of x" in msg
    # an index the rational engine cannot bound: x(2*i) over i <= n
    _raw, knl = fx.translate(OOB_F.replace("x(i+1)", "x(2*i)"))
    assert unproven_access(knl) is not None


@pytest.mark.gpu
def test_unproven_kernel_raises_the_reference_error(cuda):
    """`y(i) = x(i+1)` with x(n) declared.  The reference raises
    at the first out-of-bounds read (interp.py:293-308, checked whatever
    bounds_check is); the device path cannot prove the subscript in bounds,
    so it runs the checked build and raises the same InterpError instead of
    reading past the buffer."""
    from paper_1503_07659_b200._loopforge import interp
    _raw, knl = fx.translate(OOB_F)
    x = np.arange(8, dtype=np.float64)
    with pytest.raises(InterpError) as ref_exc:
        interp.interpret(knl, interp.make_env(knl, {"n": 8}, {"x": x}))
    env = lfb.make_device_env(knl, {"n": 8}, {"x": x}, device=cuda)
    with pytest.raises(InterpError) as dev_exc:
        lfb.interpret(knl, env)
    assert str(dev_exc.value) == str(ref_exc.value)


@pytest.mark.gpu
def test_side_stream_launch_orders_after_the_clones(cuda):
    """interpret(..., stream=s) clones the outputs on the current
    stream, then launches on s; s must wait for the clones (and the
    allocator must know s uses them).  A big clone makes a missing wait
    visible; the result is bitwise the oracle's."""
    import oracle
    n = 1 << 26
    _r, knl = fx.translate(fx.axpy_source("f64"))
    gen = torch.Generator(device=cuda).manual_seed(3)
    x = torch.rand(n, dtype=torch.float64, device=cuda, generator=gen)
    y = torch.rand(n, dtype=torch.float64, device=cuda, generator=gen)
    env = lfb.env_from_buffers(knl, {"n": n}, {"x": x, "y": y},
                               {"alpha": 1.25})
    s = torch.cuda.Stream(cuda)
    for stream in (s, s.cuda_stream):
        out = lfb.interpret(knl, env, stream=stream)
        torch.cuda.synchronize()
        ref = oracle.axpy(y.cpu().numpy(), x.cpu().numpy(), 1.25)
        assert out.arrays["y"].data.cpu().numpy().tobytes() == ref.tobytes()
    # checked mode on a side stream still reports the first violation
    k2 = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = a[i+3]")
    env2 = lfb.make_device_env(k2, {"n": 6},
                               {"a": np.ones(9, dtype=np.float32)},
                               device=cuda)
    env2.arrays["a"].shape = (4,)
    with pytest.raises(InterpError, match="insn_0"):
        lfb.interpret(k2, env2, stream=s)


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


@pytest.mark.gpu
def test_conditional_write_trace_exactly_one_branch(cuda):
    """tests/test_interp.py:67-82 restated on the device: every out[i] is
    written exactly once, by the branch the input selects -- and the whole
    trace equals the reference interpreter's, order included."""
    from paper_1503_07659_b200._loopforge import fortran, interp
    raw, _t, _u = fortran.translate_file_text(COND_F, "cond.f")
    rng = np.random.default_rng(3)
    inp = rng.random(8) * 6
    env = lfb.make_device_env(raw, {"n": 8}, {"inp": inp}, trace=True,
                              device=cuda)
    out = lfb.interpret(raw, env)
    then_id = [i.id for i in raw.instructions
               if ("loopy_cond0", False) in i.predicates
               and i.assignee_name() == "out"][0]
    else_id = [i.id for i in raw.instructions
               if ("loopy_cond0", True) in i.predicates][0]
    for i in range(8):
        writes = [iid for (iid, name, idx) in out.write_trace
                  if name == "out" and idx == (i,)]
        assert len(writes) == 1
        assert writes[0] == (then_id if inp[i] >= 3 else else_id)
    ref = interp.interpret(raw, interp.make_env(raw, {"n": 8},
                                                {"inp": inp}, trace=True))
    assert out.write_trace == ref.write_trace
    assert lfb.get_output(out, "out").tobytes() == \
        interp.get_output(ref, "out").tobytes()


def _trace_cases():
    from paper_1503_07659_b200._loopforge import transforms
    out = []
    _r, k = fx.translate(fx.gemm_source("f64"))          # workgroup tiles
    out.append(("dgemm_paper", k, {"m": 20, "n": 12, "l": 40},
                {"alpha": 0.75}))
    out.append(("sec51", sec51_precomputed(), {"n": 32}, {}))
    base = lfk.make_kernel(["{[i]: 0<=i<n}"], "out[i] = 2*a[i]")
    out.append(("dbl_ragged", transforms.split_iname(
        base, "i", 8, outer_tag="g.0", inner_tag="l.0"), {"n": 20}, {}))
    _r, k = fx.translate(fx.semlap_source(4, block=2))
    out.append(("semlap4", k, {"nelt": 2}, {}))
    _r, k = fx.translate(fx.generic_source("matvec_acc"))
    out.append(("mvacc", k, {"n": 16}, {}))
    knl = lfk.make_kernel(["{[i,j]: 0<=i<3 and 0<=j<5}"],
                          "out[i] = sum(j, a[i,j])")
    out.append(("rowsum", knl, {}, {}))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("case", _trace_cases(), ids=lambda c: c[0])
def test_write_trace_equals_the_reference(cuda, case):
    """The device write trace of transformed kernels (work-group tiles,
    ragged guards, parallel tags, SEM temporaries, reductions) equals the
    reference interpreter's trace exactly, and a second traced run appends
    to it (env.copy() keeps the trace, interp.py:66-70)."""
    from paper_1503_07659_b200._loopforge import interp
    _name, knl, params, scalars = case
    ref_env = interp.make_env(knl, params, dict(scalars), seed=5,
                              trace=True)
    ref = interp.interpret(knl, ref_env)
    env = lfb.make_device_env(knl, params, dict(scalars), seed=5,
                              trace=True, device=cuda)
    out = lfb.interpret(knl, env)
    assert out.write_trace == ref.write_trace
    for a in knl.args:
        if a.kind == "global-array" and a.is_output:
            assert lfb.get_output(out, a.name).tobytes() == \
                interp.get_output(ref, a.name).tobytes()
    again = lfb.interpret(knl, out)
    assert again.write_trace == ref.write_trace * 2
    assert env.write_trace == []
