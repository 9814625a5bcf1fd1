"""Device execution environment and the ``interpret`` drop-in.

Mirrors the reference's execution API one for one
(/root/reference/pkg/src/loopforge/interp.py):

=====================================  ======================================
reference                              B200 executor
=====================================  ======================================
``make_env(kernel, params, inputs,      ``make_device_env(...)`` -- same
seed, trace)`` interp.py:79-123         checks, same flat strided layout, the
                                        same seeded inputs, buffers in HBM
``interpret(kernel, env)``              ``interpret(kernel, env)`` -- runs
interp.py:323-400                       the recognised sm_100a kernel on the
                                        current CUDA stream; returns a new env
``get_output(env, name)`` 417-419       ``get_output`` (numpy, logical shape)
                                        / ``get_device_output`` (torch view)
``FlatArray`` interp.py:31-57           ``DeviceArray`` (flat torch tensor +
                                        logical shape/strides)
=====================================  ======================================

Like the reference, ``interpret`` does not mutate its input env (interp.py:329
``env.copy()``): output arrays are cloned first unless ``inplace=True``.
Errors are the reference's: ``InterpError`` for bad bindings and device
faults, ``CodegenError`` for kernels the executor cannot run.  There is no
CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import abi
from ._loopforge import CodegenError, InterpError
from .inbounds import unproven_access
from .launch import check_assumptions, launch_geometry
from .recognize import recognize

NP_DTYPE = {"f32": np.float32, "f64": np.float64, "i32": np.int32}
TORCH_DTYPE = {"f32": torch.float32, "f64": torch.float64, "i32": torch.int32}


def _flat_size(shape, strides):
    """interp.py:73-76."""
    if not shape:
        return 1
    return sum(s * (n - 1) for s, n in zip(strides, shape)) + 1


@dataclass
class DeviceArray:
    dtype: str
    data: torch.Tensor       # flat, element strided, on the device
    shape: tuple
    strides: tuple

    def logical(self):
        """Logical-shape strided view (no copy)."""
        if not self.shape:
            return self.data[:1]
        return torch.as_strided(self.data, self.shape, self.strides)

    def copy(self):
        return DeviceArray(self.dtype, self.data.clone(), self.shape,
                           self.strides)


@dataclass
class DeviceEnv:
    params: dict = field(default_factory=dict)
    arrays: dict = field(default_factory=dict)   # name -> DeviceArray
    scalars: dict = field(default_factory=dict)  # name -> numpy scalar
    device: torch.device = None
    # make_env(trace=True): (insn id, name, index) per write, in the
    # sequential interpreter's order (interp.py:79, 381-382)
    write_trace: list = None


def _device(device):
    if device is None:
        if not torch.cuda.is_available():
            raise InterpError("the B200 executor needs a CUDA device "
                              "(no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def make_device_env(kernel, params, inputs=None, seed=None, trace=False,
                    device=None):
    """Bind parameters and device arrays for a kernel run (interp.py:79-123).

    *inputs* maps argument names to numpy arrays / torch tensors of logical
    shape, or scalars.  Unspecified arrays are zero filled, or -- with *seed*
    -- filled with the reference's recipe (``rng.random(shape)*2-1`` for
    floats, ``rng.integers(-10, 10)`` for i32, non-output arrays only, in
    argument order), so a seeded device env holds exactly the values of the
    seeded reference env.
    """
    dev = _device(device)
    inputs = dict(inputs or {})
    params = {k: int(v) for k, v in params.items()}
    check_assumptions(kernel, params)
    rng = np.random.default_rng(seed) if seed is not None else None
    env = DeviceEnv(params=params, device=dev,
                    write_trace=[] if trace else None)
    for a in kernel.args:
        npt = NP_DTYPE[a.dtype]
        if a.kind == "scalar-value":
            env.scalars[a.name] = npt(inputs.pop(a.name, 0))
            continue
        shape = tuple(s.eval(params) for s in a.shape)
        strides = tuple(s.eval(params) for s in a.strides)
        if any(n <= 0 for n in shape):
            raise InterpError(
                f"array '{a.name}' has non-positive shape {shape}")
        flat = torch.zeros(_flat_size(shape, strides),
                           dtype=TORCH_DTYPE[a.dtype], device=dev)
        arr = DeviceArray(a.dtype, flat, shape, strides)
        src = None
        if a.name in inputs:
            src = inputs.pop(a.name)
            if isinstance(src, torch.Tensor):
                src = src.to(device=dev, dtype=TORCH_DTYPE[a.dtype])
            else:
                src = torch.from_numpy(np.ascontiguousarray(
                    np.asarray(src, dtype=npt))).to(dev)
            if tuple(src.shape) != shape:
                raise InterpError(
                    f"array '{a.name}': expected shape {shape}, "
                    f"got {tuple(src.shape)}")
        elif rng is not None and not a.is_output:
            vals = rng.random(shape) * 2 - 1 if a.dtype != "i32" \
                else rng.integers(-10, 10, shape)
            src = torch.from_numpy(np.ascontiguousarray(
                vals.astype(npt))).to(dev)
        if src is not None:
            arr.logical().copy_(src)
        env.arrays[a.name] = arr
    if inputs:
        raise InterpError(f"unknown input arrays: {sorted(inputs)}")
    return env


def env_from_buffers(kernel, params, buffers, scalars=None):
    """Wrap existing flat device tensors (no copy) -- the ``run`` boundary
    of SURVEY.md §8(b)."""
    params = {k: int(v) for k, v in params.items()}
    check_assumptions(kernel, params)
    env = DeviceEnv(params=params)
    scalars = dict(scalars or {})
    for a in kernel.args:
        if a.kind == "scalar-value":
            env.scalars[a.name] = NP_DTYPE[a.dtype](scalars.pop(a.name, 0))
            continue
        if a.name not in buffers:
            raise InterpError(f"missing buffer for array '{a.name}'")
        t = buffers[a.name]
        shape = tuple(s.eval(params) for s in a.shape)
        strides = tuple(s.eval(params) for s in a.strides)
        need = _flat_size(shape, strides)
        if t.dtype != TORCH_DTYPE[a.dtype] or not t.is_cuda \
                or t.dim() != 1 or t.numel() < need \
                or not t.is_contiguous():
            raise InterpError(
                f"buffer '{a.name}' must be a contiguous 1-D CUDA "
                f"{a.dtype} tensor of >= {need} elements")
        env.arrays[a.name] = DeviceArray(a.dtype, t, shape, strides)
        env.device = t.device
    return env


# {{{ recognition cache

_PLAN_CACHE = {}


def plan_for(kernel):
    """Cached :func:`recognize.recognize` (kernels are immutable)."""
    hit = _PLAN_CACHE.get(id(kernel))
    if hit is not None and hit[0] is kernel:
        return hit[1]
    match = recognize(kernel)
    if len(_PLAN_CACHE) > 256:
        _PLAN_CACHE.clear()
    _PLAN_CACHE[id(kernel)] = (kernel, match)
    return match

# }}}


def _ptr(arr):
    return arr.data.data_ptr()


def _int_param(v, name):
    if not -2**31 <= v < 2**31:
        raise InterpError(f"parameter {name}={v} does not fit the C int of "
                          "the emitted-C ABI")
    return v


class Launcher:
    """One prepared launch: recognised workload + geometry + pointers."""

    def __init__(self, kernel, env, variant=0, sumsq=None, workspace=None):
        self.kernel = kernel
        self.match = plan_for(kernel)
        self.geometry = launch_geometry(kernel, env.params)
        self.variant = variant
        self.env = env
        w = self.match.workload
        self.npts = w.npts
        for tp, user in self.match.param_map.items():
            v = env.params[user]
            if not -2**31 <= v < 2**31:
                # the emitted-C ABI passes parameters as C int
                # (codegen.py:523-525); interp.py uses Python ints, so the
                # reference runs such a kernel -- make_launcher sends it to
                # the generic engine's 64-bit build instead
                raise CodegenError(
                    f"parameter {user}={v} does not fit the C int of the "
                    f"{w.name} entry point (emitted-C ABI)")
        self._sumsq = sumsq
        self._workspace = workspace
        if w.name == "gemm" and w.dtype == "f32" and workspace is None \
                and variant != 1:
            # tf32 hi/lo operand split for the tensor-core path
            pm = self.match.param_map
            l, m, n = (env.params[pm[p]] for p in ("l", "m", "n"))
            need = abi.load().lfb_sgemm_workspace(l, m, n)
            if need > 0:
                self._workspace = torch.empty(need, dtype=torch.float64,
                                              device=env.device)

    def workload(self):
        return self.match.workload

    def launch(self, env=None, stream=None):
        env = env or self.env
        lib = abi.load()
        m = self.match
        w = m.workload
        am, pm = m.arg_map, m.param_map
        arrays, scalars, params = env.arrays, env.scalars, env.params
        if stream is None:
            stream = torch.cuda.current_stream(env.device).cuda_stream
        elif not isinstance(stream, int):
            stream = stream.cuda_stream
        geom = abi.make_launch(
            self.geometry, npts=w.npts, variant=self.variant,
            sumsq=None if self._sumsq is None else self._sumsq.data_ptr(),
            workspace=None if self._workspace is None
            else self._workspace.data_ptr(),
            workspace_len=0 if self._workspace is None
            else self._workspace.numel())
        gp = abi.C.byref(geom)

        def P(name):
            return abi.C.c_void_p(_ptr(arrays[am[name]]))

        def S(name):
            return scalars[am[name]]

        def I(name):
            user = pm[name]
            return _int_param(params[user], user)

        fam, dt = w.name, w.dtype
        if fam == "fill":
            fn = lib.lfb_fill_f64 if dt == "f64" else lib.lfb_fill_f32
            rc = fn(P("out"), float(S("a")), I("n"), gp, stream)
        elif fam == "axpy":
            fn = lib.lfb_axpy_f64 if dt == "f64" else lib.lfb_axpy_f32
            rc = fn(P("y"), P("x"), float(S("alpha")), I("n"), gp, stream)
        elif fam == "matvec":
            rc = lib.lfb_matvec_f64(P("y"), P("a"), P("x"), I("n"), gp,
                                    stream)
        elif fam == "semlap":
            rc = lib.lfb_semlap_f64(P("w"), P("u"), P("d"), P("g"),
                                    I("nelt"), gp, stream)
        elif fam == "gemm":
            fn = lib.lfb_sgemm_f32 if dt == "f32" else lib.lfb_dgemm_f64
            rc = fn(float(S("alpha")), P("a"), P("b"), P("c"), I("l"),
                    I("m"), I("n"), gp, stream)
        else:
            raise CodegenError(f"no entry point for workload {fam}")
        abi.check(rc, f"{fam}_{dt}")


ENGINES = ("auto", "kernels", "generic")


def make_launcher(kernel, env, variant=0, engine="auto"):
    """The launcher for *kernel*.

    ``engine="kernels"``: the hand-written sm_100a kernel of the recognised
    workload, else ``CodegenError``.  ``"generic"``: CUDA generated from the
    kernel's schedule (cudagen.py).  ``"auto"`` (default): the hand-written
    kernel when the recognizer matches, otherwise the generated one.  Both
    run on the device; there is no CPU path.
    """
    if engine not in ENGINES:
        raise CodegenError(f"unknown engine {engine!r}; one of {ENGINES}")
    if engine == "generic":
        from .generic import GenericLauncher
        return GenericLauncher(kernel, env)
    try:
        return Launcher(kernel, env, variant=variant)
    except CodegenError as exc:
        if engine == "kernels":
            raise
        from .generic import GenericLauncher
        try:
            return GenericLauncher(kernel, env)
        except CodegenError as exc2:
            raise CodegenError(f"{exc}; generic CUDA emitter: {exc2} "
                               "(no CPU fallback)") from exc2


_CHECKED_KERNELS = {}  # id(kernel) -> kernel that passed _never_written


def _never_written(kernel):
    """interp.py:272-291 raises on a read of a temporary no instruction
    wrote; here the same condition is found before the launch: a
    temporary read by some instruction and written by none."""
    hit = _CHECKED_KERNELS.get(id(kernel))
    if hit is kernel:
        return
    _never_written_scan(kernel)
    if len(_CHECKED_KERNELS) > 512:
        _CHECKED_KERNELS.clear()
    _CHECKED_KERNELS[id(kernel)] = kernel


def _never_written_scan(kernel):
    from ._loopforge import ex, transforms
    k = transforms.expand_all_rules(kernel) if kernel.rules else kernel
    written = set()
    for insn in k.instructions:
        lhs = insn.lhs
        written.add(lhs.array if isinstance(lhs, ex.Subscript) else lhs.name)
    for insn in k.instructions:
        for e in insn.read_expressions():
            for name in ex.free_variables(e):
                if name in k.temporaries and name not in written:
                    raise InterpError(f"read of never-written temporary "
                                      f"'{name}' in {insn.id}")


def _shapes_as_declared(kernel, env):
    for a in kernel.args:
        if a.kind != "global-array":
            continue
        want = tuple(s.eval(env.params) for s in a.shape)
        if tuple(env.arrays[a.name].shape) != want:
            return False
    return True


def interpret(kernel, env, bounds_check=False, *, inplace=False, variant=0,
              stream=None, engine="auto"):
    """Run *kernel* on the B200 (drop-in for interp.py:323, same
    ``interpret(kernel, env, bounds_check=False)`` signature).

    Returns a new :class:`DeviceEnv` whose output arrays hold the results;
    the launch is asynchronous on the current CUDA stream (or *stream*).

    ``bounds_check=True`` (``interpret_bounds_checked``, interp.py:403) runs
    the checked build of the generated CUDA: every argument subscript
    checked per dimension against the env's shapes and every temporary
    subscript per dimension; the first violation raises the reference's
    InterpError naming the instruction.  The same checked build (temporaries
    by flat offset, the reference's plain mode) runs whenever the
    reference's always-on argument checks could fire: when an env's array
    shapes no longer match the kernel's declarations, or when
    :func:`inbounds.unproven_access` cannot prove every subscript inside
    its declared extent over the iteration domain.  Otherwise the
    recognised hand-written kernel (or the unchecked generated one) runs.
    """
    check_assumptions(kernel, env.params)
    _never_written(kernel)
    out = DeviceEnv(dict(env.params), dict(env.arrays), dict(env.scalars),
                    env.device)
    cloned = []
    if not inplace:
        for a in kernel.args:
            if a.kind == "global-array" and a.is_output:
                out.arrays[a.name] = env.arrays[a.name].copy()
                cloned.append(out.arrays[a.name].data)
    if env.write_trace is not None:
        return _interpret_traced(kernel, env, out, bounds_check, stream)
    if stream is not None:
        # the clones above run on the current stream; a launch on another
        # stream must start after them, and the allocator must know the
        # clones are used there
        dev = env.device if env.device is not None else _device(None)
        cur = torch.cuda.current_stream(dev)
        s = stream if isinstance(stream, torch.cuda.Stream) else \
            torch.cuda.ExternalStream(int(stream), device=dev)
        if s.cuda_stream != cur.cuda_stream:
            s.wait_stream(cur)
            for t in cloned:
                t.record_stream(s)
        stream = s.cuda_stream
    if bounds_check or not _shapes_as_declared(kernel, env) \
            or unproven_access(kernel) is not None:
        from .generic import GenericLauncher
        launcher = GenericLauncher(kernel, out,
                                   checked="dims" if bounds_check
                                   else "plain")
    else:
        launcher = make_launcher(kernel, out, variant=variant, engine=engine)
    launcher.launch(stream=stream)
    return out


def _interpret_traced(kernel, env, out, bounds_check, stream):
    """make_env(trace=True): the trace build of the generated CUDA
    (cudagen ``trace``) records every store with the values of its
    enclosing inames; the records are sorted into the reference
    interpreter's sequential order and appended to a copy of the env's
    trace (interp.py:66-70, 381-382).  Synchronises: a debugging mode."""
    from .generic import GenericLauncher, TraceOverflow
    launcher = GenericLauncher(kernel, out,
                               checked="dims" if bounds_check else "plain",
                               trace=True)
    originals = {n: a.data.clone() for n, a in out.arrays.items()
                 if any(x.name == n and x.is_output for x in kernel.args)}
    while True:
        try:
            launcher.launch(stream=stream)
            break
        except TraceOverflow:
            # larger buffer (the launcher grew it); outputs back to their
            # pre-launch values, then run again
            for n, t in originals.items():
                out.arrays[n].data.copy_(t)
    out.write_trace = list(env.write_trace) + launcher.last_trace
    return out


def interpret_bounds_checked(kernel, env, **kw):
    """As :func:`interpret`, with every temporary access checked per
    dimension (interp.py:403-405)."""
    return interpret(kernel, env, bounds_check=True, **kw)


def get_device_output(env, name):
    """Logical-shape torch view of an array (interp.py:417-419)."""
    if name in env.scalars:
        return env.scalars[name]
    return env.arrays[name].logical()


def get_output(env, name):
    """Logical-shape numpy copy of an array (interp.py:417-419)."""
    if name in env.scalars:
        return env.scalars[name]
    return get_device_output(env, name).cpu().numpy()


def flat_outputs(kernel, env):
    """Flat host copies of every output array (tests/c_oracle.py:114-117)."""
    return {a.name: env.arrays[a.name].data.cpu().numpy()
            for a in kernel.args if a.kind == "global-array" and a.is_output}
