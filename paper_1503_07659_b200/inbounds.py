"""Static proof that a kernel's subscripts stay inside their declarations.

The reference interpreter checks every argument subscript per dimension on
every access, whatever ``bounds_check`` says (``check_bounds``,
/root/reference/pkg/src/loopforge/interp.py:293-308), and every temporary
subscript by flat offset.  The fast device kernels do no such check, so they
may only run a kernel whose accesses are in bounds for every execution the
reference would make.  This module proves that once per kernel (kernels are
immutable), with the reference's own integer-set engine:

for every instruction, every subscript ``A[..., f(i, p), ...]`` it reads or
writes, and every dimension d, the constraints

    f >= 0        and        extent_d(p) - 1 - f >= 0

must be implied (``polyset.constraint_implied``: rational Fourier-Motzkin on
``context and not c``, polyset.py:341-352) by the instruction's iteration
domain -- the domain nodes with every iname the instruction is not inside
projected out (``BasicSet.project_out``, polyset.py:497-508) -- plus the
kernel's assumptions.  Inside a ``sum/product/min/max`` reduction the
reduction iname counts as an enclosing iname.

The proof is sound and conservative: rational projection over-approximates
the integer iteration set, predicates (if-branches) are ignored, and a
non-affine subscript fails the proof.  A kernel it cannot prove runs the
checked build of the generated CUDA instead (executor.interpret), which
raises the reference's InterpError at the first out-of-bounds access.
"""

from __future__ import annotations

from ._loopforge import ex, polyset, transforms

_CACHE = {}  # id(kernel) -> (kernel, result)


def _subscripts(e, red=frozenset()):
    """Yield (Subscript, reduction inames in scope) for every subscript of
    an expression."""
    if isinstance(e, ex.Subscript):
        yield e, red
        for i in e.index:
            yield from _subscripts(i, red)
    elif isinstance(e, ex.Reduction):
        yield from _subscripts(e.body, red | {e.iname})
    elif isinstance(e, (ex.BinOp, ex.Compare)):
        yield from _subscripts(e.left, red)
        yield from _subscripts(e.right, red)
    elif isinstance(e, ex.UnOp):
        yield from _subscripts(e.operand, red)
    elif isinstance(e, ex.Call):
        for a in e.args:
            yield from _subscripts(a, red)


def _context(k, inames):
    """Constraints of the iteration set over *inames* (and params)."""
    cs = []
    for node in k.domains.nodes:
        bs = node
        for d in node.set_dims:
            if d not in inames:
                bs = bs.project_out(d)
        cs.extend(bs.constraints)
    return cs


def unproven_access(kernel):
    """None if every subscript of *kernel* is provably in bounds, else a
    description of the first access the proof could not cover."""
    hit = _CACHE.get(id(kernel))
    if hit is not None and hit[0] is kernel:
        return hit[1]
    res = _scan(kernel)
    if len(_CACHE) > 512:
        _CACHE.clear()
    _CACHE[id(kernel)] = (kernel, res)
    return res


def _scan(kernel):
    k = transforms.expand_all_rules(kernel) if kernel.rules else kernel
    args = {a.name: a for a in k.args}
    ctx_cache = {}
    for insn in k.instructions:
        within = frozenset(insn.within_inames or ())
        exprs = [insn.lhs] + list(insn.read_expressions())
        for e in exprs:
            for sub, red in _subscripts(e):
                if sub.array in args:
                    a = args[sub.array]
                    if a.kind != "global-array":
                        continue
                    shape = a.shape
                elif sub.array in k.temporaries:
                    shape = k.temporaries[sub.array].shape
                else:
                    continue
                scope = within | red
                if scope not in ctx_cache:
                    ctx_cache[scope] = _context(k, scope)
                ctx = ctx_cache[scope]
                if len(sub.index) != len(shape):
                    return (f"{insn.id}: {sub.array} subscripted with "
                            f"{len(sub.index)} indices, rank {len(shape)}")
                for d, (ix, ext) in enumerate(zip(sub.index, shape)):
                    f = ex.expression_to_affine(ix)
                    if f is None:
                        return (f"{insn.id}: non-affine subscript "
                                f"{ex.render_expr(ix)} of {sub.array}")
                    lo = polyset.Constraint(polyset.INEQ, f)
                    hi = polyset.Constraint(polyset.INEQ, ext - 1 - f)
                    for c, side in ((lo, "lower"), (hi, "upper")):
                        if not polyset.constraint_implied(c, ctx,
                                                          k.assumptions):
                            return (f"{insn.id}: {side} bound of "
                                    f"{sub.array} dim {d} "
                                    f"({ex.render_expr(ix)}) not implied "
                                    "by the domain")
    return None


__all__ = ["unproven_access"]
