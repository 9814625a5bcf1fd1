"""Generic execution path: schedule -> CUDA (cudagen) -> NVRTC -> launch.

For kernels outside the hand-written set (recognize.py).  Compiles once per
distinct generated source (in-process cache keyed by its hash), loads the
cubin into the current CUDA context and launches it with the reference's
logical geometry: grid = the g.N extents, CTA = the l.N extents
(launch.py / codegen.py:580-612).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import abi
from ._loopforge import InterpError
from .cudagen import NVRTC_OPTIONS, emit_cuda, temp_params
from .launch import launch_geometry

_CUBINS = {}    # program key -> cubin bytes
_MODULES = {}   # (program key, device index) -> lfb_module handle
_PROGRAMS = {}  # id(kernel) -> (kernel, Program)


def program_for(kernel, checked=None, trace=False, params=None):
    """The generated program of *kernel* (cached per kernel and build
    flavour).  Temporaries whose extents depend on parameters specialise
    the program to those parameters' values (*params*), as the reference
    sizes them per call (interp.py:332-338)."""
    tp = temp_params(kernel)
    spec = tuple((p, int(params[p])) for p in tp) if tp and params else ()
    key = (id(kernel), checked, trace, spec)
    hit = _PROGRAMS.get(key)
    if hit is not None and hit[0] is kernel:
        return hit[1]
    prog = emit_cuda(kernel, checked=checked, trace=trace,
                     params=dict(spec) if spec else None)
    if len(_PROGRAMS) > 256:
        _PROGRAMS.clear()
    _PROGRAMS[key] = (kernel, prog)
    return prog


class TraceOverflow(Exception):
    """The write-trace buffer was too small; *needed* records were made."""

    def __init__(self, needed):
        super().__init__(f"write trace needs {needed} records")
        self.needed = needed


def _schedule_paths(kernel):
    """insn id -> path through the reference interpreter's schedule tree
    (codegen.schedule, interp.py:341-363): ('c', child index) per tree level
    and ('l', iname) per loop, outermost first."""
    from ._loopforge import codegen, transforms
    k = transforms.expand_all_rules(kernel) if kernel.rules else kernel
    paths = {}

    def walk(node, path):
        for c, child in enumerate(node.children):
            if isinstance(child, codegen.Statement):
                paths[child.insn_id] = path + [("c", c)]
            elif isinstance(child, codegen.Loop):
                walk(child, path + [("c", c), ("l", child.iname)])
            else:
                walk(child, path + [("c", c)])

    walk(codegen.schedule(k), [])
    return paths, list(codegen.parallel_inames_of(k))


def decode_trace(kernel, prog, records):
    """Device write-trace records -> the reference's ``write_trace`` list of
    (insn id, name, index tuple), in the sequential interpreter's order:
    parallel inames outermost in domain order (interp.py:385-399), then the
    schedule tree's order and loop values (interp.py:341-363)."""
    paths, parallel = _schedule_paths(kernel)
    keyed = []
    for r in records:
        insn = prog.insn_ids[int(r[0])]
        name = prog.trace_names[int(r[1])]
        idx = tuple(int(x) for x in r[3:3 + int(r[2])])
        vis = prog.trace_vis[int(r[0])]
        vals = dict(zip(vis, (int(x) for x in r[9:9 + int(r[8])])))
        key = [vals[p] for p in parallel]
        for kind, v in paths[insn]:
            key.append(v if kind == "c" else vals[v])
        keyed.append((tuple(key), (insn, name, idx)))
    keyed.sort(key=lambda t: t[0])
    return [w for _k, w in keyed]


def compile_program(prog, narrow=False):
    """NVRTC -> sm_100a cubin (no device needed).  *narrow*: 32-bit index
    arithmetic (``LFB_IX=int``), valid when every index fits (launcher)."""
    cub = _CUBINS.get((prog.key, narrow))
    if cub is not None:
        return cub
    lib = abi.load()
    names = NVRTC_OPTIONS + (("-DLFB_IX=int",) if narrow else ())
    opts = (C.c_char_p * len(names))(*[o.encode() for o in names])
    n = C.c_int64(0)
    abi.check(lib.lfb_rtc_compile(prog.source.encode(),
                                  f"{prog.entry}.cu".encode(), opts,
                                  len(names), None, C.byref(n)),
              f"NVRTC {prog.entry}")
    buf = C.create_string_buffer(n.value)
    abi.check(lib.lfb_rtc_compile(prog.source.encode(),
                                  f"{prog.entry}.cu".encode(), opts,
                                  len(names), buf, C.byref(n)),
              f"NVRTC {prog.entry}")
    cub = buf.raw[:n.value]
    _CUBINS[(prog.key, narrow)] = cub
    return cub


def _module(prog, device_index, narrow):
    key = (prog.key, device_index, narrow)
    mod = _MODULES.get(key)
    if mod is None:
        cub = compile_program(prog, narrow)
        h = C.c_void_p()
        abi.check(abi.load().lfb_module_load(cub, len(cub),
                                             prog.entry.encode(),
                                             C.byref(h)),
                  f"load {prog.entry}")
        mod = h
        _MODULES[key] = mod
    return mod


_CTY = {"f64": C.c_double, "f32": C.c_float, "i32": C.c_int32}


_SMS = {}


def _sm_count(index):
    if index not in _SMS:
        _SMS[index] = torch.cuda.get_device_properties(index) \
            .multi_processor_count
    return _SMS[index]


class GenericLauncher:
    """Prepared launch of the generated kernel (same interface as
    executor.Launcher)."""

    def __init__(self, kernel, env, checked=None, trace=False):
        self.kernel = kernel
        self.env = env
        self.program = program_for(kernel, checked, trace, env.params)
        self.trace_cap = 1 << 14
        self.last_trace = None
        self.geometry = launch_geometry(kernel, env.params)
        self._narrow = {}

    def narrow(self, env):
        """32-bit index arithmetic when every flat array size, parameter
        value and the work-group count stay below 2^31 (2^30 for the
        parameters, which bound expressions combine)."""
        key = (tuple(sorted(env.params.items())),
               tuple(sorted((n, a.data.numel())
                            for n, a in env.arrays.items())))
        hit = self._narrow.get(key)
        if hit is None:
            lim = 1 << 31
            g = self.geometry
            ng = 1
            for x in g.group_extent:
                ng *= max(1, int(x))
            hit = (all(abs(int(v)) < (1 << 30) for v in env.params.values())
                   and all(a.data.numel() < lim for a in env.arrays.values())
                   and ng < lim)
            self._narrow[key] = hit
        return hit

    def tensor_maps(self, env):
        """TMA descriptors of the program's precompute footprints
        (cudagen._plan_tma) for *env*'s buffers.  All-or-nothing: when one
        array breaks the tensor-map rules (odd leading dimension, unaligned
        base) the kernel runs its cooperative fetch for every tile."""
        lib = abi.load()
        args = {a.name: a for a in self.kernel.args}
        maps, ok = [], True
        for m in self.program.tma:
            a = args[m.array]
            buf = (C.c_uint64 * 16)()
            maps.append(buf)
            if not ok:
                continue
            t = env.arrays[m.array].data
            esize = t.element_size()
            dims = [int(x.eval(env.params)) for x in a.shape]
            strides = [int(x.eval(env.params)) * esize for x in a.strides[1:]]
            rank = len(dims)
            rc = lib.lfb_tmap_encode(
                buf, {"f64": 0, "f32": 1, "i32": 2}[m.dtype], rank,
                (C.c_int64 * rank)(*dims), (C.c_int64 * max(1, rank - 1))(
                    *(strides or [0])), (C.c_int32 * rank)(*m.box),
                m.swizzle, C.c_void_p(t.data_ptr()))
            if rc == abi.LFB_ERR_UNSUPPORTED:
                ok = False
            else:
                abi.check(rc, f"tensor map for '{m.array}'")
        return maps, ok

    def launch(self, env=None, stream=None):
        env = env or self.env
        if env is not self.env and temp_params(self.kernel):
            # temporaries sized by parameters: the program of these values
            self.program = program_for(self.kernel, self.program.checked,
                                       self.program.trace, env.params)
        prog = self.program
        dev = env.device if env.device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        narrow = self.narrow(env)
        with torch.cuda.device(dev):
            mod = _module(prog, dev.index, narrow)
            cur = torch.cuda.current_stream(dev)
            if stream is None:
                stream = cur.cuda_stream
            elif not isinstance(stream, int):
                stream = stream.cuda_stream
        geo = self.geometry
        if any(int(x) <= 0 for x in geo.group_extent):
            # an empty g.N range: the reference's loop over it runs no
            # iterations (the residual guard omits what launch sizing
            # guarantees, so launching one group anyway would be wrong)
            if prog.trace:
                self.last_trace = []
            return
        vals = []
        args = {a.name: a for a in self.kernel.args}
        gext = [max(1, int(x)) for x in geo.group_extent]
        maps, tma_ok = self.tensor_maps(env) if prog.tma else ((), False)
        for name in prog.arg_order:
            a = args.get(name)
            if name.startswith("lfb_G"):       # logical work-group extents
                vals.append(C.c_int64(gext[int(name[5:])]))
            elif name == "lfb_tma":
                vals.append(C.c_int32(1 if tma_ok else 0))
            elif name == "lfb_err":
                err = torch.zeros(16, dtype=torch.int64, device=dev)
                if stream != cur.cuda_stream:
                    # zeroed on the current stream, written on `stream`
                    ext = torch.cuda.ExternalStream(stream, device=dev)
                    ext.wait_stream(cur)
                    err.record_stream(ext)
                vals.append(C.c_void_p(err.data_ptr()))
            elif name == "lfb_tr":
                tr = torch.zeros(8 + 24 * self.trace_cap, dtype=torch.int64,
                                 device=dev)
                if stream != cur.cuda_stream:
                    ext = torch.cuda.ExternalStream(stream, device=dev)
                    ext.wait_stream(cur)
                    tr.record_stream(ext)
                vals.append(C.c_void_p(tr.data_ptr()))
            elif name == "lfb_trcap":
                vals.append(C.c_int64(self.trace_cap))
            elif name.startswith("lfb_x_"):   # checked mode: env extents
                arr, d = name[6:].rsplit("_", 1)
                vals.append(C.c_int64(int(env.arrays[arr].shape[int(d)])))
            elif name.startswith("lfb_tm"):
                vals.append(maps[int(name[6:])])
            elif a is None:                    # a parameter (int64)
                vals.append(C.c_int64(int(env.params[name])))
            elif a.kind == "global-array":
                vals.append(C.c_void_p(env.arrays[name].data.data_ptr()))
            else:
                vals.append(_CTY[a.dtype](env.scalars[name]))
        argv = (C.c_void_p * len(vals))(
            *[C.cast(C.pointer(v), C.c_void_p) for v in vals])
        nthreads = prog.block[0] * prog.block[1] * prog.block[2]
        ngroups = gext[0] * gext[1] * gext[2]
        idx = dev.index if dev.index is not None \
            else torch.cuda.current_device()
        cap = _sm_count(idx) * max(1, 2048 // max(32, nthreads))
        grid = (C.c_int64 * 3)(min(ngroups, cap), 1, 1)
        block = (C.c_int32 * 3)(*prog.block)
        abi.check(abi.load().lfb_module_launch(mod, grid, block, 0, argv,
                                               stream),
                  f"launch {prog.entry}")
        if prog.checked:
            self._raise_first_oob(err, env)
        if prog.trace:
            torch.cuda.synchronize(dev)
            count = int(tr[0].item())
            if count > self.trace_cap:
                self.trace_cap = count
                raise TraceOverflow(count)
            recs = tr[8:8 + 24 * count].view(count, 24).cpu().numpy() \
                if count else []
            self.last_trace = decode_trace(self.kernel, prog, recs)

    def _raise_first_oob(self, err, env):
        """The reference's InterpError for the recorded access
        (interp.py:293-308 check_bounds messages)."""
        # the kernel may run on another stream than the current one:
        # wait for the whole device (a debugging mode) before reading
        torch.cuda.synchronize(err.device)
        rec = err.cpu().tolist()
        if not rec[0]:
            return
        prog = self.program
        insn = prog.insn_ids[rec[1]] if rec[1] >= 0 else None
        name = prog.arr_names[rec[2]]
        rank = rec[4]
        idx = tuple(rec[5:5 + rank])
        if rec[3] == -1:          # temporary, flat offset (plain mode)
            raise InterpError(f"out-of-bounds subscript {idx} of '{name}' "
                              f"in instruction {insn}")
        if name in env.arrays:
            shape = tuple(int(x) for x in env.arrays[name].shape)
        else:
            shape = tuple(rec[10:10 + rank])
        d = next((i for i, (v, n) in enumerate(zip(idx, shape))
                  if not 0 <= v < n), 0)
        raise InterpError(f"out-of-bounds subscript {idx} of '{name}' "
                          f"(extent {shape}) in instruction {insn}, dim {d}")


__all__ = ["GenericLauncher", "program_for", "compile_program"]
