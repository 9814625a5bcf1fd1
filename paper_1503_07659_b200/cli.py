"""Command line: the reference's specified but
unimplemented CLI (pyproject.toml:15-16 names ``loopforge.cli:main``; the
command set is SPEC.md:703-742), with ``run`` executing on the B200.

    python -m paper_1503_07659_b200 run <file.f> --param n=32 \\
        --in u=u.bin [--scalar alpha=1.5] --out result=r.bin [--flat-out]

An input file holds either the logical array or, 1-D, the flat strided
buffer (interp.py FlatArray.data / the emitted C's arrays).
    python -m paper_1503_07659_b200 translate <file.f> --target c|opencl|cuda
    python -m paper_1503_07659_b200 dump-ir <file.f> --stage raw|transformed|expanded
    python -m paper_1503_07659_b200 check <file.f> [--param n=32 [--smoke]]

``--transforms <script>`` (any mode) applies an extra transform script after
the embedded ``!$loopy`` blocks, in that order.  Array
files use the reference's format (interp.py:426-449, arrayio.py).  Exit
codes: 0 success, 1 user error (diagnostic with its
file:line:col span on stderr), 2 internal failure.
"""

from __future__ import annotations

import argparse
import json
import sys
import time


def _kv(items, what, conv):
    out = {}
    for it in items or ():
        if "=" not in it:
            raise SystemExit(f"{what} '{it}': expected name=value")
        k, v = it.split("=", 1)
        out[k.strip()] = conv(v.strip())
    return out


def _translate(args):
    from . import script
    with open(args.file) as f:
        src = f.read()
    extra = ()
    if args.transforms:
        with open(args.transforms) as f:
            extra = (f.read(),)
    raw, knl, _unit = script.translate_file_text(src, args.file,
                                                 extra_scripts=extra)
    return raw, knl


def _write(args, text):
    if getattr(args, "output", None):
        with open(args.output, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text if text.endswith("\n") else text + "\n")


def cmd_translate(args):
    from ._loopforge import codegen
    _raw, knl = _translate(args)
    if args.target == "cuda":
        from .cudagen import emit_cuda
        text = emit_cuda(knl).source
    else:
        text = codegen.emit(knl, args.target)
    _write(args, text)
    return 0


def cmd_dump_ir(args):
    from ._loopforge import kernel as lfk, transforms
    raw, knl = _translate(args)
    k = {"raw": raw, "transformed": knl,
         "expanded": transforms.expand_all_rules(knl)}[args.stage]
    _write(args, lfk.ir_dump(k))
    return 0


def cmd_check(args):
    """Validate, then report how the B200 executor would run the kernel."""
    from ._loopforge import kernel as lfk
    from .executor import plan_for
    from .launch import launch_geometry
    raw, knl = _translate(args)
    lfk.validate_kernel(raw)
    lfk.validate_kernel(knl)
    report = {"kernel": knl.name, "valid": True}
    try:
        m = plan_for(knl)
        report["engine"] = "kernels"
        report["workload"] = m.workload.name
        report["dtype"] = m.workload.dtype
        if m.workload.npts:
            report["npts"] = m.workload.npts
    except Exception as exc:  # not a hand-written workload
        from .cudagen import emit_cuda
        prog = emit_cuda(knl)
        report["engine"] = "generic"
        report["why_not_kernels"] = str(exc)[:200]
        report["cuda_entry"] = prog.entry
        report["block"] = list(prog.block)
    params = _kv(args.param, "--param", int)
    rc = 0
    if params:
        g = launch_geometry(knl, params)
        report["launch"] = {"group_extent": list(g.group_extent),
                            "local_extent": list(g.local_extent),
                            "guard": bool(g.guard)}
        if args.smoke:
            report["smoke"] = _engine_smoke(knl, params, args)
            rc = 0 if report["smoke"]["agree"] else 1
    print(json.dumps(report))
    return rc


def _engine_smoke(knl, params, args):
    """The check mode's property smoke test (SPEC.md cli: "validate +
    property smoke tests"): the same seeded inputs through the hand-written
    kernel (when recognised) and the generated CUDA, both on the device;
    their outputs must agree -- bitwise where both keep the reference's
    arithmetic, within the north star's tolerance where the default kernel
    reassociates (matvec split-j, tensor-core GEMM)."""
    import numpy as np
    import torch

    from ._loopforge import InterpError
    from .executor import interpret, make_device_env
    if not torch.cuda.is_available():
        raise InterpError("check --smoke runs on the B200: no CUDA device")
    dev = torch.device("cuda", args.device)
    env = make_device_env(knl, params, seed=args.seed or 0, device=dev)
    outs = [a.name for a in knl.args
            if a.kind == "global-array" and a.is_output]
    res = {}
    for engine in ("auto", "generic"):
        o = interpret(knl, env, engine=engine)
        res[engine] = {n: o.arrays[n].data.cpu().numpy() for n in outs}
    worst, bitwise = 0.0, True
    for n in outs:
        x, y = res["auto"][n], res["generic"][n]
        bitwise &= x.tobytes() == y.tobytes()
        if x.size and np.issubdtype(x.dtype, np.floating):
            scale = float(np.max(np.abs(y))) or 1.0
            worst = max(worst, float(np.max(np.abs(x - y))) / scale)
        elif x.tobytes() != y.tobytes():
            worst = float("inf")
    tol = 1e-5 if any(a.dtype == "f32" for a in knl.args) else 1e-12
    return {"outputs": outs, "bitwise": bitwise,
            "max_rel_diff": worst, "tolerance": tol,
            "agree": bitwise or worst <= tol}


def cmd_run(args):
    import torch

    from . import arrayio
    from .executor import (_flat_size, get_device_output, interpret,
                           make_device_env)
    _raw, knl = _translate(args)
    params = _kv(args.param, "--param", int)
    missing = [p for p in knl.param_names if p not in params]
    if missing:
        from ._loopforge import InterpError
        raise InterpError(f"run mode needs --param bindings for "
                          f"{', '.join(missing)} (SPEC.md CliConfig)")
    if not torch.cuda.is_available():
        from ._loopforge import InterpError
        raise InterpError("run mode executes on the B200: no CUDA device "
                          "(there is no CPU fallback)")
    dev = torch.device("cuda", args.device)
    inputs, flat = {}, {}
    argmap = {a.name: a for a in knl.args}
    for name, path in _kv(args.inputs, "--in", str).items():
        if name not in argmap:
            from ._loopforge import InterpError
            raise InterpError(f"--in {name}: the kernel has no argument "
                              f"'{name}'")
        a = argmap[name]
        t = arrayio.read_array_file(path, dev, a.dtype)
        if a.kind == "scalar-value":
            inputs[name] = t.item()
            continue
        shape = tuple(s.eval(params) for s in a.shape)
        strides = tuple(s.eval(params) for s in a.strides)
        if t.dim() == 1 and tuple(t.shape) != shape and \
                t.numel() == _flat_size(shape, strides):
            flat[name] = t  # the flat strided buffer itself (FlatArray.data)
        else:
            inputs[name] = t  # logical shape
    for name, v in _kv(args.scalar, "--scalar", float).items():
        inputs[name] = v
    env = make_device_env(knl, params, inputs, seed=args.seed, device=dev)
    for name, t in flat.items():
        env.arrays[name].data.copy_(t)
    t0 = time.perf_counter()
    out = interpret(knl, env, args.bounds_check, variant=args.variant,
                    engine=args.engine)
    torch.cuda.synchronize(dev)
    t1 = time.perf_counter()
    outs = _kv(args.outputs, "--out", str)
    for name, path in outs.items():
        arrayio.write_array_file(path, out.arrays[name].data if args.flat_out
                                 else get_device_output(out, name))
    if args.verbose:
        print(json.dumps({"kernel": knl.name, "params": params,
                          "outputs": sorted(outs), "seconds": t1 - t0}),
              file=sys.stderr)
    return 0


def _diagnostic(exc):
    """``file:line:col: message`` (errors.py:9-28); tolerant of the shorter
    spans some reference errors carry."""
    span = getattr(exc, "span", None) or ()
    msg = getattr(exc, "message", None) or str(exc)
    loc = ":".join(str(p) for p in span if p is not None)
    return f"{loc}: {msg}" if loc else msg


def main(argv=None):
    ap = argparse.ArgumentParser(
        prog="python -m paper_1503_07659_b200",
        description="loopforge kernels on the B200 (SPEC.md cli module)")
    sub = ap.add_subparsers(dest="mode", required=True)

    def common(p):
        p.add_argument("file")
        p.add_argument("--transforms", help="extra transform script")

    p = sub.add_parser("translate")
    common(p)
    p.add_argument("--target", choices=["c", "opencl", "cuda"], default="c")
    p.add_argument("-o", "--output")
    p.set_defaults(fn=cmd_translate)
    p = sub.add_parser("dump-ir")
    common(p)
    p.add_argument("--stage", choices=["raw", "transformed", "expanded"],
                   default="transformed")
    p.add_argument("-o", "--output")
    p.set_defaults(fn=cmd_dump_ir)
    p = sub.add_parser("check")
    common(p)
    p.add_argument("--param", action="append")
    p.add_argument("--smoke", action="store_true",
                   help="with --param: run both device engines on seeded "
                        "inputs and compare (exit 1 on disagreement)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--device", type=int, default=0)
    p.set_defaults(fn=cmd_check)
    p = sub.add_parser("run")
    common(p)
    p.add_argument("--param", action="append")
    p.add_argument("--in", dest="inputs", action="append")
    p.add_argument("--scalar", action="append")
    p.add_argument("--out", dest="outputs", action="append")
    p.add_argument("--flat-out", action="store_true",
                   help="write the flat strided buffers (the emitted C's "
                        "arrays) instead of logical-shape arrays")
    p.add_argument("--seed", type=int, default=None,
                   help="fill unspecified inputs like make_env(seed=...)")
    p.add_argument("--engine", choices=["auto", "kernels", "generic"],
                   default="auto")
    p.add_argument("--variant", type=int, default=0)
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--bounds-check", action="store_true",
                   help="interpret_bounds_checked: every subscript checked "
                        "on the device (interp.py:403)")
    p.add_argument("-v", "--verbose", action="store_true")
    p.set_defaults(fn=cmd_run)
    args = ap.parse_args(argv)
    try:
        from ._loopforge import LoopforgeError
    except ImportError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    try:
        return args.fn(args)
    except LoopforgeError as exc:
        print(f"error: {_diagnostic(exc)}", file=sys.stderr)
        return 1
    except (OSError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 1
    except SystemExit:
        raise
    except Exception as exc:  # internal invariant failure
        print(f"internal error: {type(exc).__name__}: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
