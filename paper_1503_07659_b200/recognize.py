"""Recognizer: map a transformed reference kernel onto a B200 workload.

The executor never falls back to a CPU path: a kernel is
either recognised as one of the workloads in :mod:`.fixtures` -- in which case
a hand-written sm_100a kernel reproduces its arithmetic operation for
operation -- or it is rejected with ``CodegenError`` (mirrors the reference's
``_Emitter`` rejections, /root/reference/pkg/src/loopforge/codegen.py:470-472).

Recognition is structural, not name based.  Both the user's kernel and the
workload template (the *untransformed* lowering of the fixture text) are
reduced to a canonical form that is invariant under exactly the
transformations that cannot change the reference's results:

1. rule expansion -- ``expand_all_rules`` (transforms.py:490-503), which is
   also the reference interpreter's first step (interp.py:326-327);
2. precompute fetches -- a temporary written by one fetch instruction whose
   right-hand side reads only arguments is forward-substituted into its
   readers (precompute, transforms.py:541-684, only copies values);
3. ``split_iname`` -- ``i -> i_inner + F*i_outer`` with ``0 <= i_inner < F``
   (transforms.py:45-103, polyset.py:478-494) is merged back into one
   logical iname when the outer loop directly encloses the inner one in the
   *execution* order;
4. renaming -- inames, arguments, temporaries and parameters get canonical
   names by first appearance.

The execution order used is the interpreter's: parallel (g.N / l.N) inames
run as outermost loops in domain order around the sequential schedule tree
(interp.py:385-399, codegen.py:58-65, 89-159).  The only loop permutation
accepted is that of a perfect nest around one update statement whose
left-hand side is indexed by the non-reduction inames: there, every output
element sees its reduction loop(s) in the same ascending order whatever the
nest order (the paper's DGEMM script permutes (j,k,i) into (i,j,k)).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from ._loopforge import (CodegenError, codegen, ex, kernel as lfk, polyset,
                         transforms)
from . import fixtures

# {{{ affine helpers (tuples: ((name, coeff), ...), const)


def _aff(coeffs, const=0):
    return (tuple(sorted((n, c) for n, c in coeffs.items() if c)), int(const))


def _aff_from_ref(a):
    return _aff(a.coeffs, a.constant)


def _aff_vars(a):
    return [n for n, _c in a[0]]


def _aff_subst(a, mapping):
    """mapping: name -> affine tuple."""
    coeffs, const = dict(a[0]), a[1]
    out, oconst = {}, const
    for n, c in coeffs.items():
        if n in mapping:
            mc, mk = mapping[n]
            for mn, mv in mc:
                out[mn] = out.get(mn, 0) + c * mv
            oconst += c * mk
        else:
            out[n] = out.get(n, 0) + c
    return _aff(out, oconst)


def _aff_rename(a, names):
    return _aff({names.get(n, n): c for n, c in a[0]}, a[1])

# }}}


# {{{ expression encoding


def _encode(e, inames):
    """Reference expression -> nested tuples; integer-affine subtrees that
    mention inames become ('aff', affine)."""
    if isinstance(e, (ex.IntLit, ex.VarRef, ex.BinOp, ex.UnOp)):
        a = ex.expression_to_affine(e)
        if a is not None and (a.variables & inames):
            return ("aff", _aff_from_ref(a))
    if isinstance(e, ex.IntLit):
        return ("int", e.value)
    if isinstance(e, ex.FloatLit):
        return ("flt", e.value)
    if isinstance(e, ex.VarRef):
        return ("var", e.name)
    if isinstance(e, ex.Subscript):
        idx = []
        for i in e.index:
            a = ex.expression_to_affine(i)
            if a is None:
                raise CodegenError(
                    f"non-affine subscript {ex.render_expr(i)!r} of "
                    f"'{e.array}' is not supported by the B200 executor")
            idx.append(_aff_from_ref(a))
        return ("sub", e.array, tuple(idx))
    if isinstance(e, ex.BinOp):
        left, right = _encode(e.left, inames), _encode(e.right, inames)
        if e.op in _COMMUTATIVE and _skey(right) < _skey(left):
            # one IEEE multiply or add gives the same bits with its operands
            # swapped (and infer_expr_dtype, kernel.py:198-233, promotes
            # symmetrically), so `x(i)*alpha` is the template's `alpha*x(i)`.
            # Only this node commutes -- association (expr.py:243-255) is
            # kept.  The order is by a name-free structural key, so the
            # canonical renaming that follows stays alpha-invariant; equal
            # keys keep the written order.
            left, right = right, left
        return ("bin", e.op, left, right)
    if isinstance(e, ex.UnOp):
        return ("un", e.op, _encode(e.operand, inames))
    if isinstance(e, ex.Compare):
        return ("cmp", e.op, _encode(e.left, inames),
                _encode(e.right, inames))
    if isinstance(e, ex.Call):
        return ("call", e.function,
                tuple(_encode(a, inames) for a in e.args))
    if isinstance(e, ex.Reduction):
        return ("red", e.op, e.iname, _encode(e.body, inames))
    raise CodegenError(f"cannot encode expression {e!r}")


_COMMUTATIVE = ("+", "*")


def _skey(t):
    """Name-free structural key of an encoded expression: node kinds,
    operators, literals and affine coefficients, every name erased."""
    kind = t[0]
    if kind == "aff":
        return ("aff", tuple(sorted(c for _n, c in t[1][0])), t[1][1])
    if kind == "var":
        return ("var",)
    if kind == "sub":
        return ("sub", len(t[2]),
                tuple((tuple(sorted(c for _n, c in a[0])), a[1])
                      for a in t[2]))
    if kind in ("bin", "cmp"):
        return (kind, t[1], _skey(t[2]), _skey(t[3]))
    if kind == "un":
        return ("un", t[1], _skey(t[2]))
    if kind == "call":
        return ("call", t[1], tuple(_skey(a) for a in t[2]))
    if kind == "red":
        return ("red", t[1], _skey(t[3]))
    return (kind, repr(t[1:]))


def _map_affs(t, fn):
    """Apply fn to every affine leaf of an encoded expression."""
    kind = t[0]
    if kind == "aff":
        return ("aff", fn(t[1]))
    if kind == "sub":
        return ("sub", t[1], tuple(fn(a) for a in t[2]))
    if kind in ("bin", "cmp"):
        return (kind, t[1], _map_affs(t[2], fn), _map_affs(t[3], fn))
    if kind == "un":
        return ("un", t[1], _map_affs(t[2], fn))
    if kind == "call":
        return ("call", t[1], tuple(_map_affs(a, fn) for a in t[2]))
    if kind == "red":
        return ("red", t[1], t[2], _map_affs(t[3], fn))
    return t


def _walk(t):
    yield t
    kind = t[0]
    if kind in ("bin", "cmp"):
        yield from _walk(t[2])
        yield from _walk(t[3])
    elif kind == "un":
        yield from _walk(t[2])
    elif kind == "call":
        for a in t[2]:
            yield from _walk(a)
    elif kind == "red":
        yield from _walk(t[3])


def _replace_subs(t, array, fn):
    """Replace ('sub', array, idx) nodes by fn(idx)."""
    kind = t[0]
    if kind == "sub" and t[1] == array:
        return fn(t[2])
    if kind in ("bin", "cmp"):
        return (kind, t[1], _replace_subs(t[2], array, fn),
                _replace_subs(t[3], array, fn))
    if kind == "un":
        return ("un", t[1], _replace_subs(t[2], array, fn))
    if kind == "call":
        return ("call", t[1], tuple(_replace_subs(a, array, fn)
                                    for a in t[2]))
    if kind == "red":
        return ("red", t[1], t[2], _replace_subs(t[3], array, fn))
    return t

# }}}


# {{{ execution nest


@dataclass
class _Loop:
    iname: str
    children: list


@dataclass
class _Stmt:
    id: str
    lhs: tuple
    rhs: tuple
    within: frozenset
    preds: frozenset


@dataclass
class _Cond:
    preds: frozenset
    children: list


def _convert_tree(node, imap, inames):
    if isinstance(node, codegen.Block):
        out = []
        for c in node.children:
            out.extend(_convert_tree(c, imap, inames))
        return out
    if isinstance(node, codegen.Loop):
        kids = []
        for c in node.children:
            kids.extend(_convert_tree(c, imap, inames))
        return [_Loop(node.iname, kids)]
    if isinstance(node, codegen.Conditional):
        kids = []
        for c in node.children:
            kids.extend(_convert_tree(c, imap, inames))
        return [_Cond(frozenset(node.predicates), kids)]
    if isinstance(node, codegen.Statement):
        insn = imap[node.insn_id]
        return [_Stmt(insn.id, _encode(insn.lhs, inames),
                      _encode(insn.rhs, inames),
                      frozenset(insn.within_inames),
                      frozenset(insn.predicates))]
    raise AssertionError(node)


def _stmts(nodes):
    for n in nodes:
        if isinstance(n, _Stmt):
            yield n
        else:
            yield from _stmts(n.children)


def _map_nest(nodes, fn_stmt, fn_loop=None):
    out = []
    for n in nodes:
        if isinstance(n, _Stmt):
            s = fn_stmt(n)
            if s is not None:
                out.append(s)
        elif isinstance(n, _Loop):
            kids = _map_nest(n.children, fn_stmt, fn_loop)
            if kids:
                out.append(_Loop(fn_loop(n.iname) if fn_loop else n.iname,
                                 kids))
        else:
            kids = _map_nest(n.children, fn_stmt, fn_loop)
            if kids:
                out.append(_Cond(n.preds, kids))
    return out

# }}}


@dataclass
class Canonical:
    """Canonical form + the maps back to the kernel's own names."""

    form: tuple
    arg_names: dict          # canonical -> original
    param_names: dict        # canonical -> original
    temp_names: dict
    iname_names: dict        # canonical -> original (logical, post-merge)
    splits: dict = field(default_factory=dict)  # logical -> (outer, inner, F)


def canonicalize(kernel):
    """Canonical form of *kernel* (see module docstring)."""
    k = transforms.expand_all_rules(kernel) if kernel.rules else kernel
    lfk.validate_kernel(k)
    # the reference's own scheduler; raises ScheduleError exactly where the
    # reference interpreter/emitter would (codegen.py:115-133)
    tree = codegen.schedule(k)
    inames = set(k.all_inames)
    imap = k.instruction_map()
    nest = _convert_tree(tree, imap, inames)
    # parallel inames wrap the whole body, outermost, in domain order
    # (interp.py:385-399)
    for iname in reversed(codegen.parallel_inames_of(k)):
        nest = [_Loop(iname, nest)]

    temps = dict(k.temporaries)
    argmap = k.arg_map()
    removed_inames = set()

    # {{{ 2. forward-substitute precompute fetches

    changed = True
    while changed:
        changed = False
        stmts = list(_stmts(nest))
        for st in stmts:
            if st.lhs[0] != "sub" or st.lhs[1] not in temps:
                continue
            tname = st.lhs[1]
            if not temps[tname].shape or st.preds:
                continue
            writers = [s for s in stmts
                       if s.lhs[0] in ("sub", "var") and s.lhs[1] == tname]
            if len(writers) != 1:
                continue
            fetch_vars = []
            ok = True
            for a in st.lhs[2]:
                if a[1] != 0 or len(a[0]) != 1 or a[0][0][1] != 1:
                    ok = False
                    break
                fetch_vars.append(a[0][0][0])
            if not ok or len(set(fetch_vars)) != len(fetch_vars):
                continue
            others = [s for s in stmts if s is not st]
            if any(set(fetch_vars) & s.within for s in others):
                continue
            reads = {t[1] for t in _walk(st.rhs) if t[0] in ("sub", "var")}
            if reads & set(temps):
                continue
            # the fetch must run inside every loop enclosing its readers
            readers = [s for s in others
                       if any(t[0] == "sub" and t[1] == tname
                              for t in list(_walk(s.rhs)) + [s.lhs])]
            outer_within = st.within - set(fetch_vars)
            if any(not outer_within <= r.within for r in readers):
                continue

            def inline(idx, st=st, fetch_vars=fetch_vars):
                mapping = dict(zip(fetch_vars, idx))
                return _map_affs(st.rhs, lambda a: _aff_subst(a, mapping))

            def fix(s, st=st, tname=tname, inline=inline):
                if s is st:
                    return None
                return _Stmt(s.id, s.lhs, _replace_subs(s.rhs, tname, inline),
                             s.within, s.preds)

            nest = _map_nest(nest, fix)
            del temps[tname]
            removed_inames |= set(fetch_vars)
            changed = True
            break

    # }}}

    # {{{ collect domain constraints + affine forms

    constraints = []
    for node in k.domains.nodes:
        for c in node.constraints:
            cc = c.canonicalized()
            if cc.expr.variables & removed_inames:
                continue
            constraints.append((cc.kind, _aff_from_ref(cc.expr)))

    def all_affs():
        for s in _stmts(nest):
            for t in list(_walk(s.lhs)) + list(_walk(s.rhs)):
                if t[0] == "aff":
                    yield t[1]
                elif t[0] == "sub":
                    yield from t[2]
        for _kind, a in constraints:
            yield a

    # }}}

    # {{{ 3. merge split pairs

    splits = {}
    live = [i for i in k.all_inames if i not in removed_inames]
    while True:
        pair = None
        cset = set(constraints)
        for inner in live:
            box_lo = ("ineq", _aff({inner: 1}))
            if box_lo not in cset:
                continue
            for kind, a in constraints:
                if kind != "ineq" or a[0] != ((inner, -1),) or a[1] < 0:
                    continue
                factor = a[1] + 1
                box_hi = (kind, a)
                for outer in live:
                    if outer == inner:
                        continue
                    good = True
                    seen = False
                    for aa in all_affs():
                        co, ci = dict(aa[0]).get(outer, 0), \
                            dict(aa[0]).get(inner, 0)
                        if aa in (box_lo[1], box_hi[1]):
                            continue
                        if co or ci:
                            if co != factor * ci:
                                good = False
                                break
                            seen = seen or bool(co)
                    if good and seen and _nest_adjacent(nest, outer, inner):
                        pair = (outer, inner, factor, box_lo, box_hi)
                        break
                if pair:
                    break
            if pair:
                break
        if pair is None:
            break
        outer, inner, factor, box_lo, box_hi = pair
        logical = f"{inner}__L"
        repl = {inner: _aff({logical: 1}), outer: _aff({})}

        def sub_aff(a, outer=outer, inner=inner, logical=logical):
            d = dict(a[0])
            ci = d.pop(inner, 0)
            d.pop(outer, None)
            if ci:
                d[logical] = d.get(logical, 0) + ci
            return _aff(d, a[1])

        del repl
        constraints = [(kind, sub_aff(a)) for kind, a in constraints
                       if (kind, a) not in (box_lo, box_hi)]

        def fix(s, sub_aff=sub_aff, outer=outer, inner=inner,
                logical=logical):
            within = set(s.within)
            if inner in within or outer in within:
                within -= {inner, outer}
                within.add(logical)
            lhs = _map_affs(s.lhs, sub_aff)
            rhs = _map_affs(s.rhs, sub_aff)
            return _Stmt(s.id, lhs, rhs, frozenset(within), s.preds)

        nest = _merge_loops(_map_nest(nest, fix), outer, inner, logical)
        splits[logical] = (outer, inner, factor)
        live = [i for i in live if i not in (outer, inner)] + [logical]

    # }}}

    return _finish(k, nest, temps, argmap, constraints, live, splits)


def _nest_adjacent(nest, outer, inner):
    for n in nest:
        if isinstance(n, _Loop):
            if n.iname == outer:
                return (len(n.children) == 1
                        and isinstance(n.children[0], _Loop)
                        and n.children[0].iname == inner)
            if _nest_adjacent(n.children, outer, inner):
                return True
        elif isinstance(n, _Cond):
            if _nest_adjacent(n.children, outer, inner):
                return True
    return False


def _merge_loops(nest, outer, inner, logical):
    out = []
    for n in nest:
        if isinstance(n, _Loop):
            if n.iname == outer:
                inner_loop = n.children[0]
                out.append(_Loop(logical, _merge_loops(
                    inner_loop.children, outer, inner, logical)))
            else:
                out.append(_Loop(n.iname, _merge_loops(
                    n.children, outer, inner, logical)))
        elif isinstance(n, _Cond):
            out.append(_Cond(n.preds, _merge_loops(n.children, outer, inner,
                                                   logical)))
        else:
            out.append(n)
    return out


def _finish(k, nest, temps, argmap, constraints, live_inames, splits):
    # {{{ 4. canonical names by first appearance

    names = {}
    counters = {"i": 0, "a": 0, "t": 0, "p": 0}
    params = set(k.param_names)
    inames = set(live_inames)

    def name_of(n):
        if n in names:
            return names[n]
        if n in inames:
            kind = "i"
        elif n in argmap:
            kind = "a"
        elif n in temps:
            kind = "t"
        elif n in params:
            kind = "p"
        else:
            raise CodegenError(f"unknown name '{n}' in kernel")
        names[n] = f"{kind}{counters[kind]}"
        counters[kind] += 1
        return names[n]

    def visit_aff(a):
        for n, _c in sorted(a[0], key=lambda nc: (-abs(nc[1]), nc[0])):
            name_of(n)

    def visit(t):
        for node in _walk(t):
            if node[0] == "aff":
                visit_aff(node[1])
            elif node[0] == "sub":
                name_of(node[1])
                for a in node[2]:
                    visit_aff(a)
            elif node[0] == "var":
                name_of(node[1])

    for s in _stmts(nest):
        visit(s.lhs)
        visit(s.rhs)
        for flag, _neg in sorted(s.preds):
            name_of(flag)

    def visit_loops(nodes):
        for n in nodes:
            if isinstance(n, _Loop):
                name_of(n.iname)
                visit_loops(n.children)
            elif isinstance(n, _Cond):
                visit_loops(n.children)

    visit_loops(nest)
    for a in k.args:
        name_of(a.name)
    for a in sorted((a for a in k.args), key=lambda a: names[a.name]):
        for e in tuple(a.shape) + tuple(a.strides):
            visit_aff(_aff_from_ref(e))
    for _kind, a in constraints:
        visit_aff(a)
    for t in temps:
        name_of(t)

    def rn_aff(a):
        return _aff_rename(a, names)

    def rn(t):
        kind = t[0]
        if kind == "aff":
            return ("aff", rn_aff(t[1]))
        if kind == "var":
            return ("var", names.get(t[1], t[1]))
        if kind == "sub":
            return ("sub", names[t[1]], tuple(rn_aff(a) for a in t[2]))
        if kind in ("bin", "cmp"):
            return (kind, t[1], rn(t[2]), rn(t[3]))
        if kind == "un":
            return ("un", t[1], rn(t[2]))
        if kind == "call":
            return ("call", t[1], tuple(rn(a) for a in t[2]))
        if kind == "red":
            return ("red", t[1], names.get(t[2], t[2]), rn(t[3]))
        return t

    # }}}

    def emit(nodes):
        out = []
        for n in nodes:
            if isinstance(n, _Stmt):
                out.append(("S", rn(n.lhs), rn(n.rhs),
                            tuple(sorted(names[w] for w in n.within
                                         if w in names)),
                            tuple(sorted((names[f], g) for f, g in n.preds))))
            elif isinstance(n, _Loop):
                out.append(("L", names[n.iname], tuple(emit(n.children))))
            else:
                out.append(("C", tuple(sorted((names[f], g)
                                              for f, g in n.preds)),
                            tuple(emit(n.children))))
        return out

    body = tuple(_normalize_perfect(x) for x in emit(nest))

    args = tuple(sorted(
        (names[a.name], a.kind, a.dtype,
         tuple(rn_aff(_aff_from_ref(e)) for e in a.shape),
         tuple(rn_aff(_aff_from_ref(e)) for e in a.strides),
         bool(a.is_output))
        for a in k.args))
    tmps = tuple(sorted(
        (names[t.name], t.dtype,
         tuple(rn_aff(_aff_from_ref(e)) for e in t.shape))
        for t in temps.values()))
    doms = tuple(sorted(set((kind, rn_aff(a)) for kind, a in constraints)))
    inv = {v: kk for kk, v in names.items()}
    return Canonical(
        form=(args, tmps, doms, body),
        arg_names={c: inv[c] for c in inv if c[0] == "a"},
        param_names={c: inv[c] for c in inv if c[0] == "p"},
        temp_names={c: inv[c] for c in inv if c[0] == "t"},
        iname_names={c: inv[c] for c in inv if c[0] == "i"},
        splits=splits)


def _normalize_perfect(node):
    """Sort the loops of a perfect nest around one update statement."""
    if node[0] == "S":
        return node
    if node[0] == "C":
        return ("C", node[1], tuple(_normalize_perfect(c) for c in node[2]))
    chain = []
    cur = node
    while cur[0] == "L" and len(cur[2]) == 1:
        chain.append(cur[1])
        cur = cur[2][0]
    if cur[0] == "S" and len(chain) > 1:
        lhs = cur[1]
        if lhs[0] == "sub":
            lhs_inames = []
            ok = True
            for a in lhs[2]:
                if a[1] != 0 or len(a[0]) != 1 or a[0][0][1] != 1:
                    ok = False
                    break
                lhs_inames.append(a[0][0][0])
            reads = [t for t in _walk(cur[2])
                     if t[0] == "sub" and t[1] == lhs[1]]
            if ok and len(set(lhs_inames)) == len(lhs_inames) \
                    and all(t == lhs for t in reads) \
                    and set(chain) >= set(lhs_inames):
                outer = sorted(i for i in chain if i in lhs_inames)
                red = [i for i in chain if i not in lhs_inames]
                new = cur
                for iname in reversed(outer + red):
                    new = ("L", iname, (new,))
                return new
    return ("L", node[1], tuple(_normalize_perfect(c) for c in node[2]))


# {{{ workload registry


@dataclass(frozen=True)
class Workload:
    name: str          # entry-point family: fill, axpy, matvec, semlap, gemm
    dtype: str
    npts: int          # SEM points per direction; 0 otherwise
    source: str        # Fortran text of the template (no transform block)
    abi_args: tuple    # template arg names in emitted-C order
    abi_params: tuple  # template params, sorted (codegen.py:523-525)


def _templates():
    out = []
    for dt in ("f64", "f32"):
        out.append(Workload("fill", dt, 0,
                            fixtures.fill_source(dt, script=False),
                            ("out", "a"), ("n",)))
        out.append(Workload("axpy", dt, 0,
                            fixtures.axpy_source(dt, script=False),
                            ("y", "x", "alpha"), ("n",)))
    out.append(Workload("matvec", "f64", 0,
                        fixtures.matvec_source("f64", script=False),
                        ("y", "a", "x"), ("n",)))
    for n in range(2, 17):
        out.append(Workload("semlap", "f64", n,
                            fixtures.semlap_source(n, script=False),
                            ("w", "u", "d", "g"), ("nelt",)))
    for dt in ("f32", "f64"):
        out.append(Workload("gemm", dt, 0,
                            fixtures.gemm_source(dt, script=False),
                            ("alpha", "a", "b", "c"), ("l", "m", "n")))
    return out


_TEMPLATE_CACHE = {}


def _template_canon(w):
    if w not in _TEMPLATE_CACHE:
        raw, _t = fixtures.translate(w.source, f"{w.name}.f")
        _TEMPLATE_CACHE[w] = (raw, canonicalize(raw))
    return _TEMPLATE_CACHE[w]


WORKLOADS = tuple(_templates())


@dataclass
class Match:
    workload: Workload
    canon: Canonical
    arg_map: dict      # template arg name -> user arg name
    param_map: dict    # template param name -> user param name


def _prefilter(w, kernel):
    kinds = sorted((a.kind, a.dtype) for a in kernel.args)
    return kinds


def recognize(kernel):
    """Return the :class:`Match` for *kernel* or raise ``CodegenError``."""
    canon = canonicalize(kernel)
    user_kinds = _prefilter(None, kernel)
    for w in WORKLOADS:
        raw, tcanon = _template_canon(w)
        if sorted((a.kind, a.dtype) for a in raw.args) != user_kinds:
            continue
        if tcanon.form != canon.form:
            continue
        arg_map = {tcanon.arg_names[c]: canon.arg_names[c]
                   for c in tcanon.arg_names}
        param_map = {tcanon.param_names[c]: canon.param_names[c]
                     for c in tcanon.param_names}
        return Match(w, canon, arg_map, param_map)
    raise CodegenError(
        f"kernel '{kernel.name}' is not one of the B200 executor's "
        "workloads (fill, axpy, matvec, semlap n=2..16, sgemm, dgemm); the "
        "executor has no CPU fallback")

# }}}
