"""Launch geometry: how a kernel's g.N / l.N tags map onto a B200 launch.

The reference gives parallel tags a hardware meaning only in its OpenCL text
(/root/reference/pkg/src/loopforge/codegen.py:580-612): ``g.N`` inames become
``get_group_id(N)``, ``l.N`` inames ``get_local_id(N)``, the host is expected
to size the group counts from the projected domain bounds, and a residual
guard covers whatever the launch does not enforce.  This module computes that
*logical* geometry with the reference's own bound machinery
(``loop_bounds`` codegen.py:241-248 -> ``BasicSet.bounds_for`` polyset.py:515,
``launch_guaranteed_constraints`` codegen.py:251-274, ``constraint_implied``
polyset.py:341) and hands it to the C-ABI in an ``lfb_launch`` record:

* ``group_extent[N]`` = upper bound of the g.N iname + 1 at the bound params
  (= CUDA gridDim[N] of a literal launch);
* ``local_extent[N]`` = constant extent of the l.N iname (= blockDim[N]);
* ``guard`` = 1 iff the reference would emit an ``if (...)`` guard.

The sm_100a kernels honour the logical index space exactly (every point the
guarded OpenCL program would execute, and no other) but are free to coarsen:
streaming kernels keep ``l.0`` as the CTA size and let each CTA cover several
logical groups; the SEM kernel is persistent and walks logical element blocks
(DESIGN.md §Launch mapping).
"""

from __future__ import annotations

from dataclasses import dataclass

from ._loopforge import CodegenError, codegen, kernel as lfk, polyset, \
    transforms


@dataclass(frozen=True)
class Geometry:
    group_extent: tuple      # g.0, g.1, g.2 (1 if unused)
    local_extent: tuple      # l.0, l.1, l.2 (1 if unused)
    n_group_axes: int
    n_local_axes: int
    guard: bool
    guard_text: str
    parallel: tuple          # ((iname, tag), ...) in domain order


def _expanded(kernel):
    return transforms.expand_all_rules(kernel) if kernel.rules else kernel


def opencl_guard_constraints(kernel):
    """The constraints the reference's OpenCL guard would test.

    Restates ``_Emitter.opencl_guard`` (codegen.py:590-612) on the public
    helpers so the executor can tell whether partial work-groups exist.
    """
    k = _expanded(kernel)
    parallel = codegen.parallel_inames_of(k)
    if not parallel:
        return []
    context, seen = [], []
    for iname in parallel:
        context.extend(codegen.launch_guaranteed_constraints(k, iname, seen))
        seen.append(iname)
    guards = []
    pset = set(parallel)
    seq = set(k.all_inames) - pset
    for node in k.domains.nodes:
        for c in node.constraints:
            if not (c.expr.variables & pset):
                continue
            if c.expr.variables & seq:
                continue
            if not polyset.constraint_implied(c, context, k.assumptions):
                guards.append(c)
    return guards


_STATIC = {}  # id(kernel) -> (kernel, per-iname bounds, guards, guard text)


def _static_geometry(kernel):
    """The parameter-independent part of the geometry: the reference's
    bounds (``loop_bounds``, Fourier-Motzkin on the domain, SURVEY.md §8(a)
    row a5: ~81 % of interpret() time) and the guard constraints, computed
    once per kernel (kernels are immutable) instead of on every launch."""
    hit = _STATIC.get(id(kernel))
    if hit is not None and hit[0] is kernel:
        return hit[1:]
    k = _expanded(kernel)
    bounds = []
    for iname in codegen.parallel_inames_of(k):
        tag = k.iname_tags[iname]
        kind, axis = tag.split(".")
        axis = int(axis)
        if axis > 2:
            raise CodegenError(f"tag {tag} on '{iname}': CUDA has 3 axes")
        lowers, uppers = codegen.loop_bounds(k, iname, [])
        bounds.append((iname, tag, kind, axis, lowers, uppers))
    guards = opencl_guard_constraints(kernel)
    text = " && ".join(codegen.render_constraint_c(c) for c in guards)
    if len(_STATIC) > 512:
        _STATIC.clear()
    _STATIC[id(kernel)] = (kernel, tuple(bounds), tuple(guards), text)
    return tuple(bounds), tuple(guards), text


def launch_geometry(kernel, params):
    """Logical launch geometry of *kernel* at parameter values *params*."""
    bounds, guards, text = _static_geometry(kernel)
    groups = [1, 1, 1]
    local = [1, 1, 1]
    ng = nl = 0
    tags = []
    for iname, tag, kind, axis, lowers, uppers in bounds:
        lo = max(b.eval(params) for b in lowers)
        hi = min(b.eval(params) for b in uppers)
        if lo != 0:
            raise CodegenError(
                f"parallel iname '{iname}' has nonzero lower bound {lo}")
        if kind == "l":
            if not all(b.is_plain_affine() and b.as_affine().is_constant()
                       for b in uppers):
                raise CodegenError(
                    f"l.{axis} iname '{iname}' needs a constant extent "
                    "(work-group size is a launch constant)")
            local[axis] = hi + 1
            nl = max(nl, axis + 1)
        else:
            groups[axis] = max(hi + 1, 0)
            ng = max(ng, axis + 1)
        tags.append((iname, tag))
    return Geometry(tuple(groups), tuple(local), ng, nl, bool(guards), text,
                    tuple(tags))


def check_assumptions(kernel, params):
    """``make_env``'s assumption check (interp.py:88-90)."""
    from ._loopforge import InterpError
    if not kernel.assumptions.satisfied_by(params):
        raise InterpError(
            f"parameter binding {params} violates the kernel assumptions")


__all__ = ["Geometry", "launch_geometry", "opencl_guard_constraints",
           "check_assumptions", "lfk"]
