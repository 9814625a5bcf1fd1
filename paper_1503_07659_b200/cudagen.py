"""Generic CUDA emitter: a scheduled loopforge kernel -> sm_100a CUDA C++.

SURVEY.md §8(f) row 1.  The reference prints OpenCL text that it never
compiles (``_Emitter``, /root/reference/pkg/src/loopforge/codegen.py:469-753;
SPEC.md:14), and whose work-group barrier is a comment (codegen.py:707-710).
This module renders the same schedule as an executable CUDA kernel for the
kernels the hand-written sm_100a kernels (recognize.py) do not cover:

* schedule and loop nesting: ``schedule`` + ``group_predicates``
  (codegen.py:89-234); loop bounds from ``loop_bounds`` (241-248) rendered
  with 64-bit integers and floor division;
* tag -> hardware index exactly as ``emit_opencl_prologue`` (580-588):
  ``g.N`` -> the work-group index, ``l.N`` -> ``threadIdx``; the residual
  guard of ``opencl_guard`` (590-612, restated in launch.py).  Work-groups
  are walked by persistent CTAs (grid-stride over the logical g.0 x g.1 x
  g.2 space) so small work-groups are not CTA-launch bound;
* workgroup temporaries (``precompute`` with an ``l.*`` sweep iname,
  transforms.py:597-599) -> ``__shared__`` arrays with real
  ``__syncthreads()`` around the loop nests that write them.  A fetch nest
  that does not depend on ``l.*`` inames -- every work-item of the reference
  fetches the whole tile -- is distributed over the CTA's threads (same
  values, written once).  When a barrier cannot be placed uniformly the
  temporary is demoted to a per-thread array (still correct);
* arithmetic follows ``interpret`` (interp.py:140-256), the reference's
  semantic oracle, node for node: literal widths from the arithmetic context,
  ``/`` promoted to >= f32, numpy's scalar type promotion (int32 with
  float32 computes in float64), separate rounding of every operation
  (compiled with ``--fmad=false``), stores converting to the target dtype;
  ``**`` with a small integer exponent as repeated multiplication; int32
  arithmetic wraps like numpy's.  sqrt, +, -, *, / are IEEE correctly
  rounded, so such kernels are bitwise the reference's; sin/cos/exp/pow use
  CUDA's libdevice (within a few ulp).

Index arithmetic is 64-bit (the reference's emitted C uses ``int``).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

from ._loopforge import CodegenError, codegen, ex, kernel as lfk, polyset, \
    transforms
from .launch import opencl_guard_constraints

I32, F32, F64 = lfk.I32, lfk.F32, lfk.F64
CT = {I32: "int", F32: "float", F64: "double"}

PRELUDE = r"""
typedef long long i64;
typedef unsigned int u32;
static __device__ __forceinline__ i64 lfb_floordiv(i64 a, i64 b) {
  return (a >= 0 ? a : a - b + 1) / b;  /* b > 0 */
}
static __device__ __forceinline__ i64 lfb_max(i64 a, i64 b) { return a > b ? a : b; }
static __device__ __forceinline__ i64 lfb_min(i64 a, i64 b) { return a < b ? a : b; }
static __device__ __forceinline__ int lfb_ipow(int b, int e) {
  int r = 1;
  for (; e > 0; --e) r = (int)((u32)r * (u32)b);
  return r;
}
template <typename T> static __device__ __forceinline__ T lfb_npmin(T a, T b) {
  return (a != a) ? a : ((b != b) ? b : (b < a ? b : a));
}
template <typename T> static __device__ __forceinline__ T lfb_npmax(T a, T b) {
  return (a != a) ? a : ((b != b) ? b : (b > a ? b : a));
}
"""

NVRTC_OPTIONS = ("--gpu-architecture=sm_100a", "--fmad=false",
                 "--std=c++17", "-default-device", "-lineinfo")


def promote(a, b):
    """numpy (NEP 50) promotion of two scalar types among int32, float32,
    float64: equal types stay, any mixed pair computes in float64."""
    return a if a == b else F64


def _cast(text, have, want):
    return text if have == want else f"(({CT[want]})({text}))"


def _lit_int(v, t):
    if t == I32:
        return f"({v})" if v < 0 else str(v)
    if t == F32:
        return f"({float(v)!r}f)" if v < 0 else f"{float(v)!r}f"
    return f"({float(v)!r})" if v < 0 else f"{float(v)!r}"


def _lit_float(v, t):
    import numpy as np
    if t == F32:
        x = float(np.float32(v))
        return f"({x.hex()}f)" if x < 0 else f"{x.hex()}f"
    if t == F64:
        return f"({float(v).hex()})" if v < 0 else float(v).hex()
    return str(int(v))


def _aff(a):
    """AffineExpr -> i64 C expression."""
    parts = []
    for name in sorted(a.coeffs):
        c = a.coeffs[name]
        parts.append(f"(i64)({name})" if c == 1 else f"{c}LL * (i64)({name})")
    if a.constant or not parts:
        parts.append(f"({a.constant}LL)")
    return "(" + " + ".join(parts) + ")"


def _bound(b):
    if b.divisor == 1:
        return _aff(b.numerator + b.offset)
    if b.exact:
        core = f"({_aff(b.numerator)} / {b.divisor}LL)"
    else:
        core = f"lfb_floordiv({_aff(b.numerator)}, {b.divisor}LL)"
    return f"({core} + {b.offset}LL)" if b.offset else core


def _combine(texts, fn):
    out = texts[0]
    for t in texts[1:]:
        out = f"{fn}({out}, {t})"
    return out


def _temp_strides(shape):
    strides, acc = [], 1
    for n in reversed(shape):
        strides.append(acc)
        acc *= n
    return tuple(reversed(strides))


@dataclass
class Program:
    source: str
    entry: str
    arg_order: tuple        # kernel.args names, then params (sorted)
    params: tuple           # sorted param names (passed as int64)
    block: tuple            # CTA extents from the l.N tags
    shared: tuple           # workgroup temporaries kept in shared memory
    demoted: tuple          # workgroup temporaries demoted to per-thread
    cooperative: int        # fetch nests distributed over the CTA
    key: str                # content hash of the source


class _Emitter:
    def __init__(self, kernel):
        k = transforms.expand_all_rules(kernel) if kernel.rules else kernel
        lfk.validate_kernel(k)
        self.k = k
        self.imap = k.instruction_map()
        self.tree = codegen.group_predicates(codegen.schedule(k))
        self.parallel = codegen.parallel_inames_of(k)
        self.local = {i for i in self.parallel
                      if k.iname_tags[i].startswith("l.")}
        self.inames = set(k.all_inames)
        self.params = set(k.param_names)
        self.arrays = {}
        self.dtypes = {}
        self.scalars = set()
        for a in k.args:
            self.dtypes[a.name] = a.dtype
            if a.kind == "global-array":
                self.arrays[a.name] = a.strides
            else:
                self.scalars.add(a.name)
        self.temp_shapes = {}
        for t in k.temporaries.values():
            self.dtypes[t.name] = t.dtype
            if t.shape:
                shape = []
                for s in t.shape:
                    if not s.is_constant():
                        raise CodegenError(
                            f"temporary '{t.name}' has a symbolic extent; "
                            "the CUDA emitter needs constant extents")
                    shape.append(s.constant)
                self.temp_shapes[t.name] = tuple(shape)
                self.arrays[t.name] = tuple(
                    polyset.AffineExpr.const(s)
                    for s in _temp_strides(shape))
            else:
                self.scalars.add(t.name)
        self.lines = []
        self.ind = 1
        self.visible = list(self.parallel)
        self.tmp = 0
        self.cooperative = 0

    # {{{ typed expressions (interp.py:140-256)

    def dtype_of(self, e):
        return lfk.infer_expr_dtype(self.k, e)

    def rv(self, e, ctx=None):
        """(C text, numpy result type) of evaluating *e* with literal
        context *ctx*, as ``_Evaluator.eval`` does."""
        if isinstance(e, ex.IntLit):
            t = ctx or I32
            return _lit_int(e.value, t), t
        if isinstance(e, ex.FloatLit):
            t = ctx or F32
            return _lit_float(e.value, t), t
        if isinstance(e, ex.VarRef):
            n = e.name
            if n in self.inames or n in self.params:
                return f"((int)({n}))", I32
            if n in self.scalars:
                return n, self.dtypes[n]
            raise CodegenError(f"unbound name '{n}'")
        if isinstance(e, ex.Subscript):
            return f"{e.array}[{self.flat(e)}]", self.dtypes[e.array]
        if isinstance(e, ex.Compare):
            lt_, lt = self.rv(e.left)
            rt_, rt = self.rv(e.right)
            t = promote(lt, rt)
            return (f"((int)({_cast(lt_, lt, t)} {e.op} "
                    f"{_cast(rt_, rt, t)}))", I32)
        if isinstance(e, ex.UnOp):
            if e.op == "not":
                x, _t = self.rv(e.operand)
                return f"((int)!({x}))", I32
            x, t = self.rv(e.operand, ctx)
            if t == I32:
                return f"((int)(0u - (u32)({x})))", I32
            return f"(-({x}))", t
        if isinstance(e, ex.BinOp):
            return self.binop(e)
        if isinstance(e, ex.Call):
            return self.call(e)
        if isinstance(e, ex.Reduction):
            return self.reduction(e)
        raise CodegenError(f"cannot render {e!r} as CUDA")

    def binop(self, e):
        dtype = self.dtype_of(e)
        ctx = dtype if dtype in (F32, F64) else None
        if e.op == "**":
            return self.power(e, dtype, ctx)
        lt_, lt = self.rv(e.left, ctx)
        rt_, rt = self.rv(e.right, ctx)
        if e.op == "/" and ctx is not None:
            lt_, lt = _cast(lt_, lt, dtype), dtype
            rt_, rt = _cast(rt_, rt, dtype), dtype
        t = promote(lt, rt)
        a, b = _cast(lt_, lt, t), _cast(rt_, rt, t)
        if t == I32:
            if e.op == "/":
                raise CodegenError("integer '/' has no reference semantics")
            return f"((int)((u32)({a}) {e.op} (u32)({b})))", I32
        return f"({a} {e.op} {b})", t

    def power(self, e, dtype, ctx):
        if isinstance(e.right, ex.IntLit) and 0 <= e.right.value <= 4:
            n = e.right.value
            if n == 0:
                return _lit_int(1, dtype), dtype
            base, t = self.rv(e.left, ctx)
            if n == 1:
                return base, t
            if t == I32:
                acc = base
                for _ in range(n - 1):
                    acc = f"((int)((u32)({acc}) * (u32)({base})))"
                return acc, I32
            return "(" + " * ".join([base] * n) + ")", t
        base, bt = self.rv(e.left, ctx)
        expo, et = self.rv(e.right, ctx)
        t = promote(bt, et)
        if t == I32:
            return f"lfb_ipow({base}, {expo})", I32
        fn = "powf" if t == F32 else "pow"
        return f"{fn}({_cast(base, bt, t)}, {_cast(expo, et, t)})", t

    def call(self, e):
        dtype = self.dtype_of(e)
        ctx = dtype if dtype in (F32, F64) else None
        args = [self.rv(a, ctx) for a in e.args]
        fn = e.function
        if fn in ("sqrt", "sin", "cos", "exp"):
            (x, t), = args
            rt = F32 if t == F32 else F64
            name = fn + ("f" if rt == F32 else "")
            return f"{name}({_cast(x, t, rt)})", rt
        if fn == "abs":
            (x, t), = args
            name = {I32: "abs", F32: "fabsf", F64: "fabs"}[t]
            return f"{name}({x})", t
        if fn in ("min", "max"):
            (a, at), (b, bt) = args
            t = promote(at, bt)
            return (f"lfb_np{fn}<{CT[t]}>({_cast(a, at, t)}, "
                    f"{_cast(b, bt, t)})", t)
        raise CodegenError(f"no CUDA mapping for function '{fn}'")

    def reduction(self, e):
        """Accumulator loop in place (interp.py eval_reduction)."""
        dtype = self.dtype_of(e.body)
        n = self.tmp
        self.tmp += 1
        acc, first = f"lfb_red{n}", f"lfb_first{n}"
        lowers, uppers = codegen.loop_bounds(self.k, e.iname, self.visible)
        lo = _combine([_bound(b) for b in lowers], "lfb_max")
        up = _combine([_bound(b) for b in uppers], "lfb_min")
        ctx = dtype if dtype in (F32, F64) else None
        self.visible.append(e.iname)
        saved, self.lines = self.lines, []
        self.ind += 2
        body, vt = self.rv(e.body, ctx)
        inner = self.lines
        self.lines = saved
        self.ind -= 2
        self.visible.pop()
        t = promote(dtype, vt) if e.op in ("sum", "product") else vt
        ct = CT[t]
        init = {"sum": _lit_int(0, t), "product": _lit_int(1, t)}.get(
            e.op, _lit_int(0, t))
        self.line(f"{ct} {acc} = {init};")
        self.line(f"int {first} = 1;")
        self.line(f"for (i64 {e.iname} = {lo}; {e.iname} <= {up}; "
                  f"++{e.iname}) {{")
        self.ind += 1
        self.lines.extend(inner)
        self.line(f"{CT[vt]} lfb_v{n} = {body};")
        v = _cast(f"lfb_v{n}", vt, t)
        if e.op in ("sum", "product"):
            op = "+" if e.op == "sum" else "*"
            zero = _cast(_lit_int(0 if e.op == "sum" else 1, dtype), dtype, t)
            if t == I32:
                step = f"(int)((u32){acc} {op} (u32){v})"
                first_v = f"(int)((u32){zero} {op} (u32){v})"
            else:
                step, first_v = f"{acc} {op} {v}", f"{zero} {op} {v}"
            self.line(f"{acc} = {first} ? ({first_v}) : ({step});")
        else:
            self.line(f"{acc} = {first} ? {v} : lfb_np{e.op}<{ct}>({acc}, "
                      f"{v});")
        self.line(f"{first} = 0;")
        self.ind -= 1
        self.line("}")
        if e.op in ("min", "max"):
            self.line(f"if ({first}) __trap();  /* empty {e.op} reduction */")
        return acc, t

    def flat(self, e):
        strides = self.arrays.get(e.array)
        if strides is None:
            raise CodegenError(f"no strides known for array '{e.array}'")
        parts = []
        for idx, stride in zip(e.index, strides):
            aff = ex.expression_to_affine(idx)
            if aff is not None:
                it = _aff(aff)
            else:
                txt, _t = self.rv(idx)
                it = f"((i64)({txt}))"
            parts.append(it if stride == polyset.AffineExpr.const(1)
                         else f"{_aff(stride)} * {it}")
        return " + ".join(parts) if parts else "0"

    # }}}

    # {{{ structure

    def line(self, text):
        self.lines.append("  " * self.ind + text)

    def _stmts(self, node):
        if isinstance(node, codegen.Statement):
            yield self.imap[node.insn_id]
        else:
            for c in node.children:
                yield from self._stmts(c)

    def _reads(self, insn):
        names = set()
        for e in insn.read_expressions():
            names |= self._arrays_in(e)
        return names

    def _arrays_in(self, e):
        out = set()
        if isinstance(e, ex.Subscript):
            out.add(e.array)
        for c in ex.children(e):
            out |= self._arrays_in(c)
        return out

    def _writes(self, insn):
        return {insn.lhs.array} if isinstance(insn.lhs, ex.Subscript) \
            else set()

    def _loop_uniform(self, iname):
        lowers, uppers = codegen.loop_bounds(self.k, iname, self.visible)
        for b in lowers + uppers:
            if b.numerator.variables & (self.local | self._nonuniform):
                return False
        return True

    def plan(self, wg):
        """Decide shared (with barriers) vs per-thread for the workgroup
        temporaries *wg*.  Barriers must sit where every thread of the CTA
        arrives: outside predicates and outside loops whose bounds depend on
        l.* inames."""
        self._nonuniform = set()
        ok = [True]

        def walk(node, uniform):
            if isinstance(node, codegen.Statement):
                insn = self.imap[node.insn_id]
                if self._writes(insn) & wg and not uniform:
                    ok[0] = False
                return
            if isinstance(node, codegen.Conditional):
                for c in node.children:
                    walk(c, False)
                return
            if isinstance(node, codegen.Loop):
                u = uniform and self._loop_uniform(node.iname)
                if not u:
                    self._nonuniform.add(node.iname)
                self.visible.append(node.iname)
                for c in node.children:
                    walk(c, u)
                self.visible.pop()
                return
            for c in node.children:
                walk(c, uniform)

        walk(self.tree, True)
        return ok[0]

    def _cooperative(self, node, wg):
        """A pure fetch nest: loops over a single chain of statements that
        write *wg* arrays, read none, and mention no l.* iname."""
        if not isinstance(node, codegen.Loop):
            return False
        stmts = list(self._stmts(node))
        if not stmts:
            return False

        def no_cond(n):
            if isinstance(n, codegen.Conditional):
                return False
            if isinstance(n, codegen.Statement):
                return True
            return all(no_cond(c) for c in n.children)
        if not no_cond(node):
            return False
        for insn in stmts:
            if not (self._writes(insn) & wg) or (self._reads(insn) & wg):
                return False
            names = set()
            for e in [insn.lhs] + insn.read_expressions():
                names |= ex.free_variables(e)
            if names & self.local:
                return False
            lhs_names = set()
            for idx in insn.lhs.index:
                lhs_names |= ex.free_variables(idx)
            if node.iname not in lhs_names:
                return False
        # loop bounds inside the nest must not involve l.* inames either
        def bounds_ok(n):
            if isinstance(n, codegen.Loop):
                lo, up = codegen.loop_bounds(self.k, n.iname, self.visible)
                if any(b.numerator.variables & self.local for b in lo + up):
                    return False
                self.visible.append(n.iname)
                r = all(bounds_ok(c) for c in n.children)
                self.visible.pop()
                return r
            return True
        return bounds_ok(node)

    def emit_loop(self, node, body, strided=False):
        lowers, uppers = codegen.loop_bounds(self.k, node.iname, self.visible)
        lo = _combine([_bound(b) for b in lowers], "lfb_max")
        up = _combine([_bound(b) for b in uppers], "lfb_min")
        if self.k.iname_tags.get(node.iname) == "unroll":
            self.line("#pragma unroll")
        if strided:
            self.line(f"for (i64 {node.iname} = {lo} + lfb_tid; "
                      f"{node.iname} <= {up}; {node.iname} += lfb_nthreads) {{")
        else:
            self.line(f"for (i64 {node.iname} = {lo}; {node.iname} <= {up}; "
                      f"++{node.iname}) {{")
        self.ind += 1
        self.visible.append(node.iname)
        body()
        self.visible.pop()
        self.ind -= 1
        self.line("}")

    def emit_stmt(self, insn, guarded):
        if guarded:
            self.line("if (lfb_in) {")
            self.ind += 1
        tgt = insn.lhs.name if isinstance(insn.lhs, ex.VarRef) \
            else insn.lhs.array
        rhs, rt = self.rv(insn.rhs)
        if isinstance(insn.lhs, ex.VarRef):
            lhs = insn.lhs.name
        else:
            lhs = f"{insn.lhs.array}[{self.flat(insn.lhs)}]"
        self.line(f"{lhs} = {_cast(rhs, rt, self.dtypes[tgt])};  "
                  f"/* {insn.id} */")
        if guarded:
            self.ind -= 1
            self.line("}")

    def walk(self, node, ctx):
        """ctx: dict(wg=set of shared temporaries, guard='all'|'stmt'|None)"""
        if isinstance(node, codegen.Block):
            self.walk_children(node.children, ctx)
        elif isinstance(node, codegen.Loop):
            self.emit_loop(node, lambda: self.walk_children(node.children,
                                                            ctx))
        elif isinstance(node, codegen.Conditional):
            cond = " && ".join(f"!{f}" if neg else f"({f} != 0)"
                               for f, neg in sorted(node.predicates))
            self.line(f"if ({cond}) {{")
            self.ind += 1
            self.walk_children(node.children, ctx)
            self.ind -= 1
            self.line("}")
        else:
            self.emit_stmt(self.imap[node.insn_id], ctx["guard"] == "stmt")

    def _touches(self, node, wg):
        w = r = False
        for insn in self._stmts(node):
            w |= bool(self._writes(insn) & wg)
            r |= bool(self._reads(insn) & wg)
        return w, r

    def barrier(self):
        if not self.lines or self.lines[-1].strip() != "__syncthreads();":
            self.line("__syncthreads();")

    def walk_children(self, children, ctx):
        wg = ctx["wg"]
        i = 0
        while i < len(children):
            c = children[i]
            w, r = self._touches(c, wg) if wg else (False, False)
            if w and not r:
                # a run of pure writers between two barriers
                j = i
                while j < len(children):
                    wj, rj = self._touches(children[j], wg)
                    if not wj or rj:
                        break
                    j += 1
                self.barrier()
                for c2 in children[i:j]:
                    if self._cooperative(c2, wg):
                        self.cooperative += 1
                        self._emit_strided(c2, ctx)
                    else:
                        self.walk(c2, ctx)
                self.barrier()
                i = j
                continue
            if w and r:
                self.barrier()
                self.walk(c, ctx)
                self.barrier()
            else:
                self.walk(c, ctx)
            i += 1

    def _emit_strided(self, node, ctx):
        """A cooperative fetch nest: every thread of the CTA helps, no guard
        (the nest's own bounds keep its reads in the domain), no barriers
        inside.  A 2-deep perfect nest with independent bounds is flattened,
        the loop indexing the contiguous (first, column-major) dimension of
        the source array varying fastest across threads."""
        sub = dict(ctx, guard=None, wg=set())
        inner = node.children[0] if len(node.children) == 1 else None
        if isinstance(inner, codegen.Loop) and all(
                isinstance(c, codegen.Statement) for c in inner.children):
            lo1, up1 = codegen.loop_bounds(self.k, node.iname, self.visible)
            self.visible.append(node.iname)
            lo2, up2 = codegen.loop_bounds(self.k, inner.iname, self.visible)
            self.visible.pop()
            if not any(node.iname in b.numerator.variables
                       for b in lo2 + up2):
                self._emit_flat2(node, inner, (lo1, up1), (lo2, up2), sub)
                return
        self.emit_loop(node, lambda: self.walk_children(node.children, sub),
                       strided=True)

    def _fast_iname(self, outer, inner):
        for insn in self._stmts(inner):
            for e in insn.read_expressions():
                for sub in self._subscripts(e):
                    if sub.index and sub.array not in self.temp_shapes:
                        first = ex.free_variables(sub.index[0])
                        if outer.iname in first and inner.iname not in first:
                            return outer.iname
        return inner.iname

    def _subscripts(self, e):
        if isinstance(e, ex.Subscript):
            yield e
        for c in ex.children(e):
            yield from self._subscripts(c)

    def _emit_flat2(self, outer, inner, b1, b2, ctx):
        n = self.tmp
        self.tmp += 1
        rng = []
        for (lo, up), nm in ((b1, outer.iname), (b2, inner.iname)):
            lo_t = _combine([_bound(b) for b in lo], "lfb_max")
            up_t = _combine([_bound(b) for b in up], "lfb_min")
            rng.append((nm, lo_t, up_t))
        fast = self._fast_iname(outer, inner)
        order = rng if fast == inner.iname else rng[::-1]
        (sn, slo, sup), (fn_, flo, fup) = order
        self.line("{")
        self.ind += 1
        self.line(f"const i64 lfb_s{n} = {slo}, lfb_f{n} = {flo};")
        self.line(f"const i64 lfb_ns{n} = lfb_max({sup} - lfb_s{n} + 1, 0LL);")
        self.line(f"const i64 lfb_nf{n} = lfb_max({fup} - lfb_f{n} + 1, 0LL);")
        self.line(f"for (i64 lfb_q{n} = lfb_tid; lfb_q{n} < lfb_ns{n} * "
                  f"lfb_nf{n}; lfb_q{n} += lfb_nthreads) {{")
        self.ind += 1
        self.line(f"const i64 {sn} = lfb_s{n} + lfb_q{n} / lfb_nf{n};")
        self.line(f"const i64 {fn_} = lfb_f{n} + lfb_q{n} % lfb_nf{n};")
        self.visible += [outer.iname, inner.iname]
        self.walk_children(inner.children, ctx)
        del self.visible[-2:]
        self.ind -= 1
        self.line("}")
        self.ind -= 1
        self.line("}")

    # }}}

    def emit(self):
        k = self.k
        wg = {t.name for t in k.temporaries.values()
              if t.address_space == "workgroup" and t.shape}
        shared = set(wg)
        if wg and not self.plan(wg):
            shared = set()
        demoted = wg - shared
        self.visible = list(self.parallel)

        guards = opencl_guard_constraints(k)
        guard_text = " && ".join(
            f"({_aff(c.expr)} {'==' if c.kind == 'eq' else '>='} 0)"
            for c in guards)

        decl = []
        for name in sorted(k.temporaries):
            t = k.temporaries[name]
            ct = CT[t.dtype]
            if not t.shape:
                decl.append(f"{ct} {name} = 0;")
            else:
                size = 1
                for s in self.temp_shapes[name]:
                    size *= s
                q = "__shared__ " if name in shared else ""
                decl.append(f"{q}{ct} {name}[{size}];")

        pro = []
        gnames = {}   # g axis -> iname
        block = [1, 1, 1]
        for iname in self.parallel:
            kind, axis = k.iname_tags[iname].split(".")
            comp = "xyz"[int(axis)]
            if kind == "g":
                gnames[int(axis)] = iname
                continue
            pro.append(f"const i64 {iname} = (i64)threadIdx.{comp};")
            if kind == "l":
                _lo, ups = codegen.loop_bounds(k, iname, [])
                if not all(b.is_plain_affine() and b.as_affine().is_constant()
                           for b in ups):
                    raise CodegenError(
                        f"l.{axis} iname '{iname}' needs a constant extent")
                block[int(axis)] = min(b.as_affine().constant
                                       for b in ups) + 1
        pro.append("const i64 lfb_tid = (i64)threadIdx.x + (i64)blockDim.x * "
                   "((i64)threadIdx.y + (i64)blockDim.y * (i64)threadIdx.z);")
        pro.append("const i64 lfb_nthreads = (i64)blockDim.x * blockDim.y * "
                   "blockDim.z;")

        # work-groups in a grid-stride loop over a capped 1-D grid: the
        # logical g.0 x g.1 x g.2 space (extents lfb_G0..2) is walked by
        # persistent CTAs, so tiny work-groups do not leave the GPU
        # CTA-launch bound; barriers stay uniform (every thread of a CTA
        # walks the same groups), shared tiles get a barrier between groups
        self.lines = []
        self.ind = 1
        self.line("const i64 lfb_ng = lfb_G0 * lfb_G1 * lfb_G2;")
        self.line("for (i64 lfb_g = (i64)blockIdx.x; lfb_g < lfb_ng; "
                  "lfb_g += (i64)gridDim.x) {")
        self.ind += 1
        for axis, iname in sorted(gnames.items()):
            div = " * ".join(f"lfb_G{a}" for a in range(axis)) or "1"
            self.line(f"const i64 {iname} = (lfb_g / ({div})) % lfb_G{axis};")
        for name in sorted(k.temporaries):
            t = k.temporaries[name]
            if not t.shape:
                self.line(f"{name} = 0;")
        if shared and guard_text:
            self.line(f"const bool lfb_in = {guard_text};")
            self.walk(self.tree, {"wg": shared, "guard": "stmt"})
        elif guard_text:
            self.line(f"if ({guard_text}) {{")
            self.ind += 1
            self.walk(self.tree, {"wg": shared, "guard": None})
            self.ind -= 1
            self.line("}")
        else:
            self.walk(self.tree, {"wg": shared, "guard": None})
        if shared:
            self.line("__syncthreads();  // tiles free for the next group")
        self.ind -= 1
        self.line("}")
        body = self.lines

        params = tuple(sorted(k.param_names))
        sig, order = [], []
        for a in k.args:
            ct = CT[a.dtype]
            order.append(a.name)
            if a.kind == "global-array":
                const = "" if a.is_output else "const "
                sig.append(f"{const}{ct} *__restrict__ {a.name}")
            else:
                sig.append(f"{ct} {a.name}")
        argnames = {a.name for a in k.args}
        for p in params:
            if p not in argnames:
                sig.append(f"i64 {p}")
                order.append(p)
        for a in range(3):  # logical work-group extents (launch geometry)
            sig.append(f"i64 lfb_G{a}")
            order.append(f"lfb_G{a}")
        nthreads = block[0] * block[1] * block[2]
        if nthreads > 1024:
            raise CodegenError(
                f"work-group of {nthreads} work-items (l.N tags) exceeds "
                "1024 threads per CTA")
        entry = f"lfb_gen_{k.name}"
        src = "\n".join(
            [PRELUDE,
             f'extern "C" __global__ void __launch_bounds__({nthreads})',
             f"{entry}({', '.join(sig)})", "{"]
            + ["  " + d for d in decl] + ["  " + p for p in pro]
            + body + ["}", ""])
        key = hashlib.sha256(src.encode()).hexdigest()[:16]
        return Program(src, entry, tuple(order), params, tuple(block),
                       tuple(sorted(shared)), tuple(sorted(demoted)),
                       self.cooperative, key)


def emit_cuda(kernel):
    """Render *kernel* (transformed, rules expanded or not) as one CUDA
    kernel; returns a :class:`Program`."""
    return _Emitter(kernel).emit()


__all__ = ["Program", "emit_cuda", "NVRTC_OPTIONS", "promote"]
