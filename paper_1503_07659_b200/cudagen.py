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
/* index arithmetic width: int when every array, parameter and work-group
   count fits (the reference's emitted C uses int throughout), else 64-bit;
   the launcher picks the build (generic.py) */
#ifndef LFB_IX
#define LFB_IX long long
#endif
typedef LFB_IX lfb_ix;
static __device__ __forceinline__ lfb_ix lfb_floordiv(lfb_ix a, lfb_ix b) {
  return (a >= 0 ? a : a - b + 1) / b;  /* b > 0 */
}
static __device__ __forceinline__ lfb_ix lfb_max(lfb_ix a, lfb_ix b) { return a > b ? a : b; }
static __device__ __forceinline__ lfb_ix lfb_min(lfb_ix a, lfb_ix b) { return a < b ? a : b; }
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

CHECK_PRELUDE = r"""
/* checked execution: the first out-of-bounds access of the launch is
   recorded -- [flag, insn, array, mode, rank, idx0..4, ext0..4] -- and the
   access skipped (loads read 0); the host raises InterpError */
static __device__ __noinline__ void lfb_oob(long long *err, int insn, int arr,
    int mode, int rank, i64 i0, i64 i1, i64 i2, i64 i3, i64 i4,
    i64 x0, i64 x1, i64 x2, i64 x3, i64 x4) {
  if (atomicCAS((unsigned long long *)err, 0ull, 1ull) != 0ull) return;
  err[1] = insn; err[2] = arr; err[3] = mode; err[4] = rank;
  err[5] = i0; err[6] = i1; err[7] = i2; err[8] = i3; err[9] = i4;
  err[10] = x0; err[11] = x1; err[12] = x2; err[13] = x3; err[14] = x4;
  __threadfence();
}
"""

TRACE_PRELUDE = r"""
/* write trace (make_env(trace=True), interp.py:79, 381-382): every store
   appends [insn, array, rank, idx0..4, nv, v0..v11] -- the instruction, the
   subscript and the values of the inames enclosing the store -- at slot
   atomicAdd(count); the host sorts the records into the sequential
   interpreter's order.  tr[0] counts every store, also past the capacity
   (the host then re-runs with a larger buffer). */
static __device__ __noinline__ void lfb_trace(long long *tr, i64 cap, int insn,
    int arr, int rank, i64 i0, i64 i1, i64 i2, i64 i3, i64 i4, int nv,
    i64 v0, i64 v1, i64 v2, i64 v3, i64 v4, i64 v5, i64 v6, i64 v7, i64 v8,
    i64 v9, i64 v10, i64 v11) {
  const unsigned long long s = atomicAdd((unsigned long long *)tr, 1ull);
  if ((i64)s >= cap) return;
  long long *r = tr + 8 + 24 * (i64)s;
  r[0] = insn; r[1] = arr; r[2] = rank;
  r[3] = i0; r[4] = i1; r[5] = i2; r[6] = i3; r[7] = i4; r[8] = nv;
  r[9] = v0; r[10] = v1; r[11] = v2; r[12] = v3; r[13] = v4; r[14] = v5;
  r[15] = v6; r[16] = v7; r[17] = v8; r[18] = v9; r[19] = v10; r[20] = v11;
}
"""

TMA_PRELUDE = r"""
/* precompute footprints by TMA (SURVEY.md §8(f) row 3) */
struct __align__(64) lfb_tmap { unsigned long long v[16]; };
static __device__ __forceinline__ unsigned lfb_smem(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void lfb_bar_init(unsigned long long *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(lfb_smem(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
static __device__ __forceinline__ void lfb_expect_tx(unsigned long long *bar,
                                                     unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(lfb_smem(bar)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void lfb_bar_wait(unsigned long long *bar,
                                                    unsigned ph) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n"
                 " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(lfb_smem(bar)), "r"(ph) : "memory");
}
"""


def _tma_fn(rank):
    cs = ", ".join(f"int c{i}" for i in range(rank))
    regs = ", ".join(f"%{i + 2}" for i in range(rank))
    ops = ", ".join(f'"r"(c{i})' for i in range(rank))
    return (f"static __device__ __forceinline__ void lfb_tma{rank}(void *dst, "
            f"const lfb_tmap *m, {cs}, unsigned long long *bar) {{\n"
            f'  asm volatile("cp.async.bulk.tensor.{rank}d.shared::cluster.'
            f"global.tile.mbarrier::complete_tx::bytes [%0], [%1, {{{regs}}}],"
            f' [%{rank + 2}];"\n'
            f'               :: "r"(lfb_smem(dst)), '
            f'"l"((unsigned long long)m), {ops}, "r"(lfb_smem(bar)) '
            f': "memory");\n}}\n')


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
    """AffineExpr -> index-typed C expression."""
    parts = []
    for name in sorted(a.coeffs):
        c = a.coeffs[name]
        parts.append(f"(lfb_ix)({name})" if c == 1
                     else f"{c} * (lfb_ix)({name})")
    if a.constant or not parts:
        parts.append(f"({a.constant})")
    return "(" + " + ".join(parts) + ")"


def _bound(b):
    if b.divisor == 1:
        return _aff(b.numerator + b.offset)
    if b.exact:
        core = f"({_aff(b.numerator)} / {b.divisor})"
    else:
        core = f"lfb_floordiv({_aff(b.numerator)}, {b.divisor})"
    return f"({core} + {b.offset})" if b.offset else core


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
class TmaMap:
    """A precompute footprint fetched by TMA: the tensor map the launcher
    encodes for argument *array* (lfb_tmap_encode)."""
    array: str
    dtype: str
    box: tuple              # box extents per array dim (dim 0 contiguous)
    swizzle: int            # 0 or 128 (bytes)


@dataclass
class _TmaPlan:
    temp: str
    array: str
    esize: int
    sdim: tuple             # temp dim -> array dim
    fetch: tuple            # temp dim -> fetch iname
    ext: tuple              # box extent per array dim
    width: int              # inner-dim piece (elements)
    pieces: int
    rows: int               # product of the box extents of dims 1..
    swizzle: int
    coord: tuple            # array dim -> AffineExpr origin (fetch inames 0)


def _buf_stride(p):
    """Elements between the two buffers of a double-buffered TMA tile: the
    tile rounded up to TMA's 128-B destination alignment, or to the
    1024-B swizzle atom for a swizzled tile (the pattern is of the absolute
    shared address)."""
    unit = (1024 if p.swizzle else 128) // p.esize
    return (p.ext[0] * p.rows + unit - 1) // unit * unit


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
    tma: tuple = ()         # tensor maps (TmaMap), kernel params after lfb_G*
    checked: str = None     # None, "plain" or "dims"
    insn_ids: tuple = ()    # checked mode: instruction ids by index
    arr_names: tuple = ()   # checked mode: array names by index
    trace: bool = False     # write-trace build
    trace_names: tuple = ()  # trace: written names by record id
    trace_vis: tuple = ()   # trace: per insn index, the inames recorded


class _Emitter:
    # per-work-item (local memory) / per-work-group (shared memory) bytes of
    # one temporary
    TEMP_BYTES_MAX = 48 * 1024

    def __init__(self, kernel, checked=None, trace=False, params=None):
        k = transforms.expand_all_rules(kernel) if kernel.rules else kernel
        lfk.validate_kernel(k)
        self.k = k
        # trace: every store also appends a write-trace record; workgroup
        # temporaries become per-work-item (each work-item then runs the
        # whole schedule, fetches included, like one iteration of the
        # reference interpreter's parallel loops, interp.py:385-399)
        self.trace = trace
        self.trace_names = []
        self.trace_vis = {}
        # checked=None: the fast kernel.  "plain" / "dims": every array
        # access checked like the reference's _Evaluator.check_bounds
        # (interp.py:293-308) -- arguments per dimension against the env's
        # shapes, temporaries by flat offset ("plain", interpret()) or per
        # dimension ("dims", interpret_bounds_checked) -- the first
        # violation recorded for the host to raise; no layout tricks then
        self.checked = checked
        self.cur_insn = None
        self.insn_ids = [insn.id for insn in k.instructions]
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
        self.temp_alloc = {}
        self.tma_plan = {} if checked else self._plan_tma(k)
        self.tma_maps = []     # TmaMap per emitted footprint
        self.tma_index = {}    # temp -> map index
        self.pipes = 0         # double-buffered (prefetching) loops
        self.pipe_runs = {}    # id(first fetch nest) -> (K, loop, plans)
        self.pipe_buf = {}     # temp -> current-buffer variable
        self.pipe_temps = set()
        self.pipe_nbuf = {}    # temp -> buffers (default 2)
        self.bar_next = 0      # mbarriers handed out (one per buffer/run)
        for t in k.temporaries.values():
            self.dtypes[t.name] = t.dtype
            if t.shape:
                shape = []
                for s in t.shape:
                    if s.is_constant():
                        shape.append(s.constant)
                    elif params is not None and s.variables <= set(params):
                        # extent from the launch's parameters, as the
                        # reference allocates it (interp.py:332-338): the
                        # program is specialised to those values
                        shape.append(int(s.eval(params)))
                    else:
                        raise CodegenError(
                            f"temporary '{t.name}' has a symbolic extent; "
                            "the CUDA emitter needs constant extents (or "
                            "the parameter values)")
                if any(x <= 0 for x in shape):
                    raise CodegenError(
                        f"temporary '{t.name}' has non-positive extent "
                        f"{tuple(shape)}")
                size = 8
                for x in shape:
                    size *= x
                if size > self.TEMP_BYTES_MAX:
                    raise CodegenError(
                        f"temporary '{t.name}' of {size} bytes exceeds the "
                        f"{self.TEMP_BYTES_MAX}-byte per-work-item / "
                        "work-group budget of the CUDA emitter")
                self.temp_shapes[t.name] = tuple(shape)
                alloc = list(shape)
                if t.address_space == "workgroup" and len(shape) >= 2 \
                        and shape[-1] % 2 == 0 and t.name not in \
                        self.tma_plan and not checked:
                    # odd row pitch: work-items reading down a column of a
                    # shared tile hit distinct banks (the layout of a
                    # temporary is the executor's choice, interp.py:408-414)
                    alloc[-1] += 1
                self.temp_alloc[t.name] = alloc
                self.arrays[t.name] = tuple(
                    polyset.AffineExpr.const(s)
                    for s in _temp_strides(alloc))
            else:
                self.scalars.add(t.name)
        self.lines = []
        self.ind = 1
        self.visible = list(self.parallel)
        self.tmp = 0
        self.cooperative = 0
        self.arr_names = []   # checked mode: array ids in error records
        self.ext_args = set()  # checked mode: arguments needing extents
        self.promoted = {}    # array -> (subscript, register name)
        self.n_promoted = 0
        self.written = set()
        for insn in k.instructions:
            if isinstance(insn.lhs, ex.Subscript):
                self.written.add(insn.lhs.array)

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
            hit = self.promoted.get(e.array)
            if hit is not None and hit[0] == e:
                return hit[1], self.dtypes[e.array]
            if self.checked:
                cond, rec = self._bounds(e)
                z = _lit_int(0, self.dtypes[e.array])
                return (f"(({cond}) ? {e.array}[{self.flat(e)}] : "
                        f"({rec}, {z}))", self.dtypes[e.array])
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
        self.line(f"for (lfb_ix {e.iname} = {lo}; {e.iname} <= {up}; "
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
        if e.array in self.tma_plan:
            return self._tma_flat(e)
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
                it = f"((lfb_ix)({txt}))"
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
            self.line(f"for (lfb_ix {node.iname} = {lo} + lfb_tid; "
                      f"{node.iname} <= {up}; {node.iname} += lfb_nthreads) {{")
        else:
            self.line(f"for (lfb_ix {node.iname} = {lo}; {node.iname} <= {up}; "
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
        self.cur_insn = self.insn_ids.index(insn.id)
        rhs, rt = self.rv(insn.rhs)
        hit = self.promoted.get(tgt)
        store_if = None
        if isinstance(insn.lhs, ex.VarRef):
            lhs = insn.lhs.name
        elif hit is not None and hit[0] == insn.lhs:
            lhs = hit[1]
        else:
            lhs = f"{insn.lhs.array}[{self.flat(insn.lhs)}]"
            if self.checked:
                store_if = self._bounds(insn.lhs)
        val = _cast(rhs, rt, self.dtypes[tgt])
        tr = self._trace_call(insn) if self.trace else ""
        if store_if is not None:
            # the value first (its loads are checked before the store, the
            # reference's evaluation order), then the checked store
            cond, rec = store_if
            ct = CT[self.dtypes[tgt]]
            self.line(f"{{ const {ct} lfb_v = {val}; if ({cond}) {{ {lhs} = "
                      f"lfb_v; {tr}}} else {rec}; }}  /* {insn.id} */")
        else:
            self.line(f"{lhs} = {val};  /* {insn.id} */")
            if tr:
                self.line(tr)
        if guarded:
            self.ind -= 1
            self.line("}")

    def _trace_call(self, insn):
        """The write-trace record of *insn*'s store (interp.py:381-382:
        (insn id, array, index)) plus the values of the inames visible at
        the store, from which the host rebuilds the sequential order."""
        if isinstance(insn.lhs, ex.VarRef):
            name, idx = insn.lhs.name, []
        else:
            name = insn.lhs.array
            idx = []
            for ix in insn.lhs.index:
                aff = ex.expression_to_affine(ix)
                if aff is not None:
                    idx.append(f"(i64)({_aff(aff)})")
                else:
                    txt, _t = self.rv(ix)
                    idx.append(f"(i64)({txt})")
        if len(idx) > 5:
            raise CodegenError("write trace: arrays of rank > 5")
        if name not in self.trace_names:
            self.trace_names.append(name)
        vis = list(self.visible)
        if len(vis) > 12:
            raise CodegenError("write trace: more than 12 enclosing inames")
        self.trace_vis[self.cur_insn] = tuple(vis)
        args = ([str(self.cur_insn), str(self.trace_names.index(name)),
                 str(len(idx))] + idx + ["0"] * (5 - len(idx))
                + [str(len(vis))] + [f"(i64){v}" for v in vis]
                + ["0"] * (12 - len(vis)))
        return f"lfb_trace(lfb_tr, lfb_trcap, {', '.join(args)}); "

    def walk(self, node, ctx):
        """ctx: dict(wg=set of shared temporaries, guard='all'|'stmt'|None)"""
        if isinstance(node, codegen.Block):
            self.walk_children(node.children, ctx)
        elif isinstance(node, codegen.Loop):
            if ctx["guard"] == "stmt" and not (
                    ctx["wg"] and self._touches(node, ctx["wg"])[0]):
                # no shared writes inside, so no barriers: the residual
                # guard can enclose the whole nest instead of every statement
                self.line("if (lfb_in) {")
                self.ind += 1
                self.walk(node, dict(ctx, guard=None))
                self.ind -= 1
                self.line("}")
                return
            pipe = self._pipeline(node, ctx)
            if pipe is not None:
                self._emit_pipelined(node, ctx, *pipe)
                return
            promo = self._promotions(node)
            if promo:
                self._emit_promoted(node, ctx, promo)
            else:
                self.emit_loop(node, lambda: self.walk_children(
                    node.children, ctx))
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

    # {{{ precompute footprints by TMA

    def _plan_tma(self, k):
        """Workgroup temporaries whose one fetch instruction is a plain copy
        of a rectangular box of a column-major argument -- what ``precompute``
        builds (transforms.py:541-684: temporary extents = footprint box,
        fetch ``T[f0, f1, ..] = A[base + f..]``).  Such a tile can be loaded
        by one thread with the Tensor Memory Accelerator instead of by every
        work-item; the temporary is then laid out the way TMA writes it (the
        array's contiguous dimension innermost, 128-B rows swizzled so
        column reads stay conflict-free)."""
        plan = {}
        args = {a.name: a for a in k.args}
        writers = {}
        for insn in k.instructions:
            if isinstance(insn.lhs, ex.Subscript):
                writers.setdefault(insn.lhs.array, []).append(insn)
        written = set(writers)
        for t in k.temporaries.values():
            if t.address_space != "workgroup" or not t.shape or \
                    len(writers.get(t.name, ())) != 1:
                continue
            if not all(s.is_constant() for s in t.shape):
                continue
            shape = [s.constant for s in t.shape]
            insn = writers[t.name][0]
            lhs, rhs = insn.lhs, insn.rhs
            if not all(isinstance(i, ex.VarRef) for i in lhs.index):
                continue
            fetch = tuple(i.name for i in lhs.index)
            if len(set(fetch)) != len(fetch) or \
                    not isinstance(rhs, ex.Subscript):
                continue
            a = args.get(rhs.array)
            if a is None or a.kind != "global-array" or a.name in written \
                    or a.dtype != t.dtype or not 1 <= len(a.shape) <= 5:
                continue
            if a.strides[0] != polyset.AffineExpr.const(1):
                continue
            esize = 8 if t.dtype == F64 else 4
            sdim = [None] * len(fetch)
            ext = [1] * len(a.shape)
            coord = []
            ok = len(rhs.index) == len(a.shape)
            for d, idx in enumerate(rhs.index if ok else ()):
                aff = ex.expression_to_affine(idx)
                if aff is None:
                    ok = False
                    break
                here = [f for f in fetch if aff.coeff(f) != 0]
                if len(here) > 1 or any(aff.coeff(f) != 1 for f in here):
                    ok = False
                    break
                if here:
                    tdim = fetch.index(here[0])
                    sdim[tdim] = d
                    ext[d] = shape[tdim]
                coord.append(aff.substitute({f: polyset.AffineExpr.const(0)
                                             for f in here}))
            if not ok or None in sdim or ext[0] * esize % 16 or \
                    any(e > 256 for e in ext[1:]):
                continue
            rows = 1
            for e in ext[1:]:
                rows *= e
            # swizzle only if some consumer's work-items differ along a
            # non-contiguous dim (a column read down 128-B rows: bank
            # conflicts); reads whose work-items vary only along the
            # contiguous dim are conflict-free in the dense layout
            local = {i for i, tg in k.iname_tags.items()
                     if (tg or "").startswith("l.")}
            strided = False
            for other in k.instructions:
                if other is insn:
                    continue
                for e in other.read_expressions():
                    for sub in self._subscripts(e):
                        if sub.array != t.name:
                            continue
                        for tdim, idx in enumerate(sub.index):
                            if sdim[tdim] != 0 and \
                                    ex.free_variables(idx) & local:
                                strided = True
            width, swz = ext[0], 0
            if strided and ext[0] * esize % 128 == 0 and rows % 8 == 0:
                width, swz = 128 // esize, 128     # 128-B rows, swizzled
            elif ext[0] > 256:
                continue
            plan[t.name] = _TmaPlan(t.name, a.name, esize, tuple(sdim), fetch,
                                    tuple(ext), width, ext[0] // width, rows,
                                    swz, tuple(coord))
        return plan

    def _tma_flat(self, e):
        """Element offset of a TMA-laid-out temporary: pieces of *width*
        along the array's contiguous dim, each a dense [rows][width] block,
        128-B swizzle on top."""
        p = self.tma_plan[e.array]
        v = ["0"] * len(p.ext)
        for tdim, idx in enumerate(e.index):
            aff = ex.expression_to_affine(idx)
            if aff is not None:
                txt = _aff(aff)
            else:
                txt, _t = self.rv(idx)
            v[p.sdim[tdim]] = f"(int)({txt})"
        row = v[-1] if len(v) > 1 else "0"
        for d in range(len(v) - 2, 0, -1):
            row = f"({v[d]} + {p.ext[d]} * {row})"
        if p.pieces > 1:
            sh = p.width.bit_length() - 1
            inner = f"(int)((unsigned)({v[0]}) & {p.width - 1}u)"
            piece = (f" + {p.width * p.rows} * "
                     f"(int)((unsigned)({v[0]}) >> {sh})")
        else:
            inner, piece = f"({v[0]})", ""
        if p.swizzle:
            # 128-B swizzle (16-B chunk ^= row mod 8) written on the
            # (inner, row) split, so the row term hoists out of loops over
            # the contiguous index: (inner ^ ((row & 7) << s)) + width*row
            s_ = 1 if p.esize == 8 else 2
            inner = f"(({inner}) ^ ((({row}) & 7) << {s_}))"
        buf = self.pipe_buf.get(e.array)
        if buf is not None:
            piece += f" + {_buf_stride(p)} * {buf}"
        return f"({inner} + {p.width} * {row}{piece})"

    def _tma_nest(self, node):
        """The plan of a cooperative fetch nest TMA can replace: a perfect
        nest over exactly the plan's fetch inames, each from 0 with a
        constant upper candidate equal to the temporary's extent (the
        footprint box; a tighter domain clip only shortens what the
        reference fetches -- the consumers never read past it)."""
        if not isinstance(node, codegen.Loop):
            return None
        loops, cur = [], node
        while isinstance(cur, codegen.Loop):
            loops.append(cur)
            if len(cur.children) != 1:
                break
            cur = cur.children[0]
        last = loops[-1]
        if len(last.children) != 1 or \
                not isinstance(last.children[0], codegen.Statement):
            return None
        insn = self.imap[last.children[0].insn_id]
        if not isinstance(insn.lhs, ex.Subscript):
            return None
        p = self.tma_plan.get(insn.lhs.array)
        if p is None or sorted(l.iname for l in loops) != sorted(p.fetch):
            return None
        shape = self.temp_shapes[p.temp]
        vis = len(self.visible)
        try:
            for lp in loops:
                lo, up = codegen.loop_bounds(self.k, lp.iname, self.visible)
                if not lo or not all(b.is_plain_affine() and
                                     b.as_affine().is_constant() and
                                     b.as_affine().constant == 0 for b in lo):
                    return None
                ext = shape[p.fetch.index(lp.iname)]
                if not any(b.is_plain_affine() and b.as_affine().is_constant()
                           and b.as_affine().constant == ext - 1 for b in up):
                    return None
                self.visible.append(lp.iname)
        finally:
            del self.visible[vis:]
        return p

    def _emit_tma_issue(self, plans, cond="lfb_tid == 0", bar="0", buf=None,
                        subst=None, pre=()):
        """One elected work-item arms barrier *bar* with the byte count and
        issues one TMA per 128-B piece of every footprint (into buffer
        *buf* of a double-buffered tile; *subst* shifts the loop iname for
        a prefetch)."""
        total = sum(p.esize * p.ext[0] * p.rows for p in plans)
        self.line(f"if ({cond}) {{")
        self.ind += 1
        for ln in pre:
            self.line(ln)
        self.line(f"lfb_expect_tx(&lfb_bars[{bar}], {total}u);")
        for p in plans:
            if p.temp not in self.tma_index:
                self.tma_index[p.temp] = len(self.tma_maps)
                box = (p.width,) + p.ext[1:]
                self.tma_maps.append(TmaMap(p.array, self.dtypes[p.array],
                                            box, p.swizzle))
            m = self.tma_index[p.temp]
            rank = len(p.ext)
            self.tma_ranks.add(rank)
            coord = [c.substitute(subst) if subst else c for c in p.coord]
            for piece in range(p.pieces):
                cs = [f"(int)({_aff(c)})" for c in coord]
                if piece:
                    cs[0] = f"(int)({_aff(coord[0])} + {piece * p.width})"
                off = str(piece * p.width * p.rows)
                if buf is not None:
                    off = f"{off} + {_buf_stride(p)} * ({buf})"
                self.line(f"lfb_tma{rank}(&{p.temp}[{off}], &lfb_tm{m}, "
                          f"{', '.join(cs)}, &lfb_bars[{bar}]);")
        self.ind -= 1
        self.line("}")

    def _pipeline(self, node, ctx):
        """Double-buffer the TMA tiles of a sequential loop whose body
        starts a writer run of TMA-fetchable footprints that move with the
        loop's iname (the paper's k_outer): the next iteration's tiles are
        prefetched into the other buffer while this one is consumed.  Legal
        because the fetched arrays are never written by the kernel."""
        return self._pipeline_run(node.children, ctx, [node.iname], node)

    def _pipeline_run(self, kids, ctx, moving, node):
        """The first writer run of *kids* if it is all TMA footprints whose
        coordinates move with one of the inames *moving* (pushed visible
        while the nests are checked when *node* is a loop), and the temps
        are used nowhere outside *node* (None: the whole kernel)."""
        wg = ctx["wg"]
        if not wg or not self.tma_plan:
            return None
        i = 0
        while i < len(kids):
            w, r = self._touches(kids[i], wg)
            if w and not r:
                break
            i += 1
        if i == len(kids):
            return None
        j = i
        while j < len(kids):
            w, r = self._touches(kids[j], wg)
            if not w or r:
                break
            j += 1
        vis = len(self.visible)
        if node is not None:
            self.visible.append(node.iname)
        try:
            plans = []
            for c in kids[i:j]:
                if not self._cooperative(c, wg):
                    return None
                p = self._tma_nest(c)
                if p is None:
                    return None
                plans.append(p)
        finally:
            del self.visible[vis:]
        if not any(set(moving) & c.variables for p in plans
                   for c in p.coord):
            return None
        temps = {p.temp for p in plans}
        if node is not None:
            inside = {self.imap[st.insn_id].id
                      for st in self._walk_stmts(node)}
            for insn in self.k.instructions:
                if insn.id not in inside and (
                        (self._reads(insn) | self._writes(insn)) & temps):
                    return None
        for t in temps:
            if t in self.pipe_temps:
                return None
        return kids[i], plans

    def _walk_stmts(self, node):
        if isinstance(node, codegen.Statement):
            yield node
        else:
            for c in node.children:
                yield from self._walk_stmts(c)

    def _emit_pipelined(self, node, ctx, first, plans):
        k = self.pipes
        self.pipes += 1
        lowers, uppers = codegen.loop_bounds(self.k, node.iname, self.visible)
        lo = _combine([_bound(b) for b in lowers], "lfb_max")
        up = _combine([_bound(b) for b in uppers], "lfb_min")
        temps = {p.temp for p in plans}
        self.pipe_temps |= temps
        self.line("{")
        self.ind += 1
        self.line(f"const lfb_ix lfb_plo{k} = {lo}, lfb_pup{k} = {up};")
        self.barrier()
        base = self.bar_next
        self.bar_next += 2
        self._emit_tma_issue(
            plans, cond=f"lfb_tma && lfb_tid == 0 && lfb_plo{k} <= lfb_pup{k}",
            bar=f"{base}", buf="0",
            subst={node.iname: polyset.AffineExpr.var(f"lfb_plo{k}")})
        self.line(f"for (lfb_ix {node.iname} = lfb_plo{k}; {node.iname} <= "
                  f"lfb_pup{k}; ++{node.iname}) {{")
        self.ind += 1
        self.line(f"const int lfb_pb{k} = (int)(({node.iname} - lfb_plo{k}) "
                  "& 1);")
        self.visible.append(node.iname)
        for t in temps:
            self.pipe_buf[t] = f"lfb_pb{k}"
        self.pipe_runs[id(first)] = (k, node, plans, None, base)
        self.walk_children(node.children, ctx)
        del self.pipe_runs[id(first)]
        for t in temps:
            del self.pipe_buf[t]
        self.visible.pop()
        self.ind -= 1
        self.line("}")
        self.ind -= 1
        self.line("}")

    # }}}

    def _promotions(self, node):
        """Global array elements a sequential loop updates in place --
        ``c[i,j] = c[i,j] + ...`` with the subscript invariant in the loop
        -- kept in a register across the loop (scalar replacement): one load
        before, one store after, the same operations in the same order in
        between, so results stay bitwise.  Only statements that are direct,
        unconditional children of the loop qualify (then the element is
        touched on every trip, so hoisting the load adds no access the
        reference would not make), and every access to the array inside the
        loop must use that one subscript (arguments never alias: each is its
        own buffer)."""
        if self.checked:
            return []
        direct = [self.imap[c.insn_id] for c in node.children
                  if isinstance(c, codegen.Statement)]
        cands = {}
        for insn in direct:
            lhs = insn.lhs
            if isinstance(lhs, ex.Subscript) and lhs.array not in \
                    self.temp_shapes and lhs.array not in self.promoted:
                cands.setdefault(lhs.array, lhs)
        if not cands:
            return []
        outer = set(self.visible) | self.params
        out = []
        for name, sub in cands.items():
            fv = set()
            for idx in sub.index:
                fv |= ex.free_variables(idx)
            if not fv <= outer or node.iname in fv:
                continue
            ok = True
            for insn in self._stmts(node):
                subs = [x for e in [insn.lhs] + insn.read_expressions()
                        for x in self._subscripts(e) if x.array == name]
                if not subs:
                    continue
                if insn not in direct or any(x != sub for x in subs):
                    ok = False
                    break
            if ok:
                out.append((name, sub))
        return out

    def _emit_promoted(self, node, ctx, promo):
        lowers, uppers = codegen.loop_bounds(self.k, node.iname, self.visible)
        lo = _combine([_bound(b) for b in lowers], "lfb_max")
        up = _combine([_bound(b) for b in uppers], "lfb_min")
        n = self.n_promoted
        self.n_promoted += 1
        self.line("{")
        self.ind += 1
        self.line(f"const lfb_ix lfb_lo{n} = {lo}, lfb_up{n} = {up};")
        cond = f"lfb_lo{n} <= lfb_up{n}"
        if ctx["guard"] == "stmt":
            cond += " && lfb_in"
        self.line(f"const bool lfb_run{n} = {cond};")
        regs = []
        for k, (name, sub) in enumerate(promo):
            reg = f"lfb_r{n}_{k}"
            self.line(f"{CT[self.dtypes[name]]} {reg};")
            self.line(f"if (lfb_run{n}) {reg} = {name}[{self.flat(sub)}];")
            regs.append((name, sub, reg))
        for name, sub, reg in regs:
            self.promoted[name] = (sub, reg)
        full = self._full_trip(lowers, uppers, node, ctx)
        if full is not None:
            # interior work-groups run the footprint's full, constant trip:
            # a fully unrolled copy (constant tile offsets fold into the
            # addressing); edge groups take the general loop
            self.line(f"if (lfb_lo{n} == {full[0]} && lfb_up{n} == "
                      f"{full[1]}) {{")
            self.ind += 1
            self.line("#pragma unroll")
            self.line(f"for (lfb_ix {node.iname} = {full[0]}; {node.iname} "
                      f"<= {full[1]}; ++{node.iname}) {{")
            self.ind += 1
            self.visible.append(node.iname)
            self.walk_children(node.children, ctx)
            self.visible.pop()
            self.ind -= 1
            self.line("}")
            self.ind -= 1
            self.line("} else {")
            self.ind += 1
        if self.k.iname_tags.get(node.iname) == "unroll":
            self.line("#pragma unroll")
        self.line(f"for (lfb_ix {node.iname} = lfb_lo{n}; {node.iname} <= "
                  f"lfb_up{n}; ++{node.iname}) {{")
        self.ind += 1
        self.visible.append(node.iname)
        self.walk_children(node.children, ctx)
        self.visible.pop()
        self.ind -= 1
        self.line("}")
        if full is not None:
            self.ind -= 1
            self.line("}")
        for name, sub, reg in regs:
            del self.promoted[name]
            self.line(f"if (lfb_run{n}) {name}[{self.flat(sub)}] = {reg};")
        self.ind -= 1
        self.line("}")

    def _full_trip(self, lowers, uppers, node, ctx):
        """(lo, hi) when the loop has constant lower bounds and a constant
        upper candidate with a short trip (<= 64), a body of at most a few
        statements and no shared-tile writes (so no barriers to duplicate);
        None otherwise."""
        def const(b):
            return b.is_plain_affine() and b.as_affine().is_constant()
        if not lowers or not all(const(b) for b in lowers):
            return None
        ups = [b.as_affine().constant for b in uppers if const(b)]
        if not ups or len(ups) == len(uppers):
            return None            # nothing to specialise, or no constant
        lo = max(b.as_affine().constant for b in lowers)
        hi = min(ups)
        if not 1 <= hi - lo + 1 <= 64:
            return None
        if ctx["wg"] and self._touches(node, ctx["wg"])[0]:
            return None
        if sum(1 for _ in self._stmts(node)) > 4:
            return None
        return lo, hi

    def _bounds(self, e):
        """(in-bounds condition, failure record) of subscript *e*."""
        idx = []
        for ix in e.index:
            aff = ex.expression_to_affine(ix)
            if aff is not None:
                idx.append(f"(i64)({_aff(aff)})")
            else:
                txt, _t = self.rv(ix)
                idx.append(f"(i64)({txt})")
        names = self.arr_names
        if e.array not in names:
            names.append(e.array)
        a = names.index(e.array)
        insn = self.cur_insn if self.cur_insn is not None else -1
        if e.array in self.temp_shapes:
            shape = self.temp_shapes[e.array]
            if self.checked == "dims":
                ext = [str(n) for n in shape]
            else:  # the flat offset against the dense temporary
                size = 1
                for n in shape:
                    size *= n
                flat = self.flat(e)
                return (f"(unsigned long long)(i64)({flat}) < {size}ull",
                        f"lfb_oob(lfb_err, {insn}, {a}, -1, {len(idx)}, "
                        + ", ".join(idx + ["0"] * (5 - len(idx)))
                        + ", 0, 0, 0, 0, 0)")
        else:
            ext = [f"lfb_x_{e.array}_{d}" for d in range(len(idx))]
            self.ext_args.add(e.array)
        cond = " && ".join(f"(unsigned long long)({i}) < "
                           f"(unsigned long long)({x})"
                           for i, x in zip(idx, ext)) or "true"
        pad = ["0"] * (5 - len(idx))
        rec = (f"lfb_oob(lfb_err, {insn}, {a}, 0, {len(idx)}, "
               + ", ".join(idx + pad) + ", "
               + ", ".join([f"(i64)({x})" for x in ext] + pad) + ")")
        return cond, rec

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
                pipe = self.pipe_runs.get(id(children[i]))
                if pipe is None or pipe[1] is not None:
                    # (a work-group-level ring needs none: the barrier that
                    # ends the previous group already freed its buffers)
                    self.barrier()
                tma, other = [], False
                for c2 in children[i:j]:
                    if self._cooperative(c2, wg):
                        self.cooperative += 1
                        p = self._tma_nest(c2)
                        if p is not None:
                            tma.append((c2, p))
                            continue
                        self._emit_strided(c2, ctx)
                        other = True
                    else:
                        self.walk(c2, ctx)
                        other = True
                if tma and pipe is not None:
                    # double-buffered: prefetch the next iteration's tiles
                    # into the other buffer, then wait for this one's
                    k, loop, plans, gnext, base = pipe
                    self.line("if (lfb_tma) {")
                    self.ind += 1
                    if loop is not None:
                        nxt = polyset.AffineExpr.var(loop.iname) + 1
                        self._emit_tma_issue(
                            plans, cond=f"lfb_tid == 0 && {loop.iname} + 1 "
                                        f"<= lfb_pup{k}",
                            bar=f"{base} + (lfb_pb{k} ^ 1)",
                            buf=f"lfb_pb{k} ^ 1", subst={loop.iname: nxt})
                    else:   # NB - 1 work-groups ahead of this CTA's
                        nb = self.pipe_nbuf[plans[0].temp]
                        ahead = f"lfb_g + {nb - 1} * (lfb_ix)gridDim.x"
                        subst, pre = gnext(ahead)
                        nxt = f"(lfb_pb{k} + {nb - 1}) & {nb - 1}"
                        self._emit_tma_issue(
                            plans, cond=f"lfb_tid == 0 && {ahead} < lfb_ng",
                            bar=f"{base} + ({nxt})", buf=nxt, subst=subst,
                            pre=pre)
                    cur = f"{base} + lfb_pb{k}"
                    self.line(f"lfb_bar_wait(&lfb_bars[{cur}], "
                              f"(lfb_tph >> ({cur})) & 1u);")
                    self.line(f"lfb_tph ^= 1u << ({cur});")
                    self.ind -= 1
                elif tma:
                    # TMA when the launcher could encode every tensor map,
                    # else the same tiles fetched cooperatively
                    b = self.bar_next
                    self.bar_next += 1
                    self.line("if (lfb_tma) {")
                    self.ind += 1
                    self._emit_tma_issue([p for _c, p in tma], bar=str(b))
                    self.line(f"lfb_bar_wait(&lfb_bars[{b}], "
                              f"(lfb_tph >> {b}) & 1u);")
                    self.line(f"lfb_tph ^= 1u << {b};")
                    self.ind -= 1
                if tma:
                    self.line("} else {")
                    self.ind += 1
                    for c2, _p in tma:
                        self._emit_strided(c2, ctx)
                    if not other:   # TMA readers synchronise on the mbarrier
                        self.line("__syncthreads();")
                    self.ind -= 1
                    self.line("}")
                if other or not tma:
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

    def _const_box(self, outer, inner, b1, b2, fast):
        """((lo, extent) slow, (lo, extent) fast) when both fetch inames have
        constant lower bounds and a constant upper candidate (the footprint
        box precompute sized the temporary with, transforms.py:669-674);
        None otherwise."""
        def const(bounds):
            if not all(b.is_plain_affine() and b.as_affine().is_constant()
                       for b in bounds):
                return None
            return [b.as_affine().constant for b in bounds]
        res = {}
        for node, (lo, up) in ((outer, b1), (inner, b2)):
            los = const(lo)
            ups = [b.as_affine().constant for b in up
                   if b.is_plain_affine() and b.as_affine().is_constant()]
            if not los or not ups:
                return None
            l0, u0 = max(los), min(ups)
            if u0 < l0 or (u0 - l0 + 1) > 4096:
                return None
            res[node.iname] = (l0, u0 - l0 + 1)
        slow = outer.iname if fast == inner.iname else inner.iname
        if res[slow][1] * res[fast][1] > (1 << 20):
            return None
        return res[slow], res[fast]

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
        box = self._const_box(outer, inner, b1, b2, fast)
        self.line("{")
        self.ind += 1
        if box is not None:
            # constant footprint box (the temporary's extents): the flat
            # index splits with constant divisors, the domain clip is a test
            (ls, es), (lf, ef) = box
            self.line(f"const lfb_ix lfb_us{n} = {sup}, lfb_uf{n} = {fup};")
            # the CTA size is static (l.N extents): a fixed trip count the
            # compiler unrolls, so every work-item's loads issue together
            self.line("#pragma unroll")
            self.line(f"for (int lfb_q{n} = (int)lfb_tid; lfb_q{n} < "
                      f"{es * ef}; lfb_q{n} += {self.nthreads}) {{")
            self.ind += 1
            self.line(f"const lfb_ix {sn} = {ls} + lfb_q{n} / {ef};")
            self.line(f"const lfb_ix {fn_} = {lf} + lfb_q{n} % {ef};")
            self.line(f"if ({sn} <= lfb_us{n} && {fn_} <= lfb_uf{n}) {{")
            self.ind += 1
            self.visible += [outer.iname, inner.iname]
            self.walk_children(inner.children, ctx)
            del self.visible[-2:]
            self.ind -= 1
            self.line("}")
            self.ind -= 1
            self.line("}")
            self.ind -= 1
            self.line("}")
            return
        self.line(f"const lfb_ix lfb_s{n} = {slo}, lfb_f{n} = {flo};")
        self.line(f"const lfb_ix lfb_ns{n} = lfb_max({sup} - lfb_s{n} + 1, 0);")
        self.line(f"const lfb_ix lfb_nf{n} = lfb_max({fup} - lfb_f{n} + 1, 0);")
        self.line(f"for (lfb_ix lfb_q{n} = lfb_tid; lfb_q{n} < lfb_ns{n} * "
                  f"lfb_nf{n}; lfb_q{n} += lfb_nthreads) {{")
        self.ind += 1
        self.line(f"const lfb_ix {sn} = lfb_s{n} + lfb_q{n} / lfb_nf{n};")
        self.line(f"const lfb_ix {fn_} = lfb_f{n} + lfb_q{n} % lfb_nf{n};")
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
        if self.trace or (wg and not self.plan(wg)):
            shared = set()
        demoted = wg - shared
        self.visible = list(self.parallel)

        guards = opencl_guard_constraints(k)
        guard_text = " && ".join(
            f"({_aff(c.expr)} {'==' if c.kind == 'eq' else '>='} 0)"
            for c in guards)

        pro = []
        gnames = {}   # g axis -> iname
        block = [1, 1, 1]
        for iname in self.parallel:
            kind, axis = k.iname_tags[iname].split(".")
            comp = "xyz"[int(axis)]
            if kind == "g":
                gnames[int(axis)] = iname
                continue
            pro.append(f"const lfb_ix {iname} = (lfb_ix)threadIdx.{comp};")
            if kind == "l":
                _lo, ups = codegen.loop_bounds(k, iname, [])
                if not all(b.is_plain_affine() and b.as_affine().is_constant()
                           for b in ups):
                    raise CodegenError(
                        f"l.{axis} iname '{iname}' needs a constant extent")
                block[int(axis)] = min(b.as_affine().constant
                                       for b in ups) + 1
        pro.append("const lfb_ix lfb_tid = (lfb_ix)(threadIdx.x + blockDim.x * "
                   "(threadIdx.y + blockDim.y * threadIdx.z));")
        pro.append("const lfb_ix lfb_nthreads = (lfb_ix)(blockDim.x * blockDim.y * "
                   "blockDim.z);")

        self.nthreads = block[0] * block[1] * block[2]

        # work-groups in a grid-stride loop over a capped 1-D grid: the
        # logical g.0 x g.1 x g.2 space (extents lfb_G0..2) is walked by
        # persistent CTAs, so tiny work-groups do not leave the GPU
        # CTA-launch bound; barriers stay uniform (every thread of a CTA
        # walks the same groups), shared tiles get a barrier between groups
        if not shared:
            self.tma_plan = {}
        self.tma_ranks = set()
        self.lines = []
        self.ind = 1
        self.line("const lfb_ix lfb_ng = (lfb_ix)(lfb_G0 * lfb_G1 * lfb_G2);")
        self.line("const lfb_ix lfb_g0 = (lfb_ix)lfb_G0, lfb_g1 = (lfb_ix)lfb_G1, "
                  "lfb_g2 = (lfb_ix)lfb_G2;")
        top = max(gnames) if gnames else 0

        def gsplit(gexpr, axis):
            """Index along g.axis of linear work-group *gexpr* (< lfb_ng):
            no division for axis 0 of a 1-D space, no modulo on the last
            axis (the runtime 32/64-bit divisions are per-group cost)."""
            div = " * ".join(f"lfb_g{a}" for a in range(axis))
            q = f"(({gexpr}) / ({div}))" if div else f"({gexpr})"
            return q if axis == top else f"({q} % lfb_g{axis})"

        def gnext(gexpr):
            """Group inames of work-group index *gexpr*, as lfb_nx_*."""
            subst, pre = {}, []
            for axis, iname in sorted(gnames.items()):
                pre.append(f"const lfb_ix lfb_nx_{iname} = "
                           f"{gsplit(gexpr, axis)};")
                subst[iname] = polyset.AffineExpr.var(f"lfb_nx_{iname}")
            return subst, pre

        gpipe = None
        if shared and gnames:
            # tiles of the next work-group this CTA will walk are prefetched
            # while the current one computes (streaming kernels with one tile
            # per group are otherwise TMA-latency bound)
            root = self.tree.children if isinstance(self.tree,
                                                    codegen.Block) else []
            found = self._pipeline_run(root, {"wg": shared, "guard": None},
                                       list(gnames.values()), None)
            if found is not None:
                first, plans = found
                gpipe = (self.pipes, first, plans)
                self.pipes += 1
                self.pipe_temps |= {p.temp for p in plans}
                # ring depth: 4 tiles in flight per CTA when they are small
                # (streaming kernels: bytes in flight hide TMA latency)
                tile = sum(_buf_stride(p) * p.esize for p in plans)
                nb = 4 if tile <= 8192 else 2
                for p in plans:
                    self.pipe_nbuf[p.temp] = nb
        if gpipe is not None:
            kp, first, plans = gpipe
            nb = self.pipe_nbuf[plans[0].temp]
            gbase = self.bar_next
            self.bar_next += nb
            for d in range(nb - 1):   # prologue: this CTA's first groups
                gexpr = "(lfb_ix)blockIdx.x" + (
                    f" + {d} * (lfb_ix)gridDim.x" if d else "")
                subst, pre = gnext(gexpr)
                self._emit_tma_issue(
                    plans, cond=f"lfb_tma && lfb_tid == 0 && {gexpr} < "
                                "lfb_ng",
                    bar=str(gbase + d), buf=str(d), subst=subst, pre=pre)
            self.line("int lfb_git = 0;  /* groups walked: ring slot */")
            self.line("for (lfb_ix lfb_g = (lfb_ix)blockIdx.x; lfb_g < "
                      "lfb_ng; lfb_g += (lfb_ix)gridDim.x, ++lfb_git) {")
            self.ind += 1
            self.line(f"const int lfb_pb{kp} = lfb_git & {nb - 1};")
            for p in plans:
                self.pipe_buf[p.temp] = f"lfb_pb{kp}"
            self.pipe_runs[id(first)] = (kp, None, plans, gnext, gbase)
        else:
            self.line("for (lfb_ix lfb_g = (lfb_ix)blockIdx.x; lfb_g < "
                      "lfb_ng; lfb_g += (lfb_ix)gridDim.x) {")
            self.ind += 1
        for axis, iname in sorted(gnames.items()):
            self.line(f"const lfb_ix {iname} = {gsplit('lfb_g', axis)};")
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

        decl = []
        for name in sorted(k.temporaries):
            t = k.temporaries[name]
            ct = CT[t.dtype]
            if not t.shape:
                decl.append(f"{ct} {name} = 0;")
            else:
                size = 1
                for s in self.temp_alloc[name]:
                    size *= s
                if name in self.pipe_temps:    # multi-buffered tile
                    size = _buf_stride(self.tma_plan[name]) * \
                        (self.pipe_nbuf.get(name, 2) - 1) + size
                q = "__shared__ " if name in shared else ""
                if name in shared and name in self.tma_plan:
                    q += "__align__(1024) "   # swizzle atoms, TMA dst
                decl.append(f"{q}{ct} {name}[{size}];")

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
        prelude = PRELUDE
        if self.checked:
            prelude += CHECK_PRELUDE
            sig.append("long long *lfb_err")
            order.append("lfb_err")
            for name in sorted(self.ext_args):
                for d in range(len(self.arrays[name])):
                    sig.append(f"i64 lfb_x_{name}_{d}")
                    order.append(f"lfb_x_{name}_{d}")
        if self.trace:
            prelude += TRACE_PRELUDE
            sig += ["long long *lfb_tr", "i64 lfb_trcap"]
            order += ["lfb_tr", "lfb_trcap"]
        if self.tma_maps:
            sig.append("int lfb_tma")
            order.append("lfb_tma")
            for m in range(len(self.tma_maps)):
                sig.append(f"const __grid_constant__ lfb_tmap lfb_tm{m}")
                order.append(f"lfb_tm{m}")
            prelude += TMA_PRELUDE + "".join(
                _tma_fn(r) for r in sorted(self.tma_ranks))
            nbars = max(1, self.bar_next)
            if nbars > 32:
                raise CodegenError("more than 32 TMA barriers in one kernel")
            decl.append("__shared__ __align__(8) unsigned long long "
                        f"lfb_bars[{nbars}];")
            decl.append("unsigned lfb_tph = 0;  /* phase bit per barrier */")
            chk = " || ".join(f"(lfb_smem({t}) & 1023u)"
                              for t in sorted(self.tma_index))
            pro.append("if (lfb_tma && lfb_tid == 0) {")
            pro.append(f"  if ({chk}) __trap();  /* TMA tiles misaligned */")
            for b in range(nbars):
                pro.append(f"  lfb_bar_init(&lfb_bars[{b}]);")
            pro.append("}")
            pro.append("__syncthreads();")
        nthreads = block[0] * block[1] * block[2]
        if nthreads > 1024:
            raise CodegenError(
                f"work-group of {nthreads} work-items (l.N tags) exceeds "
                "1024 threads per CTA")
        entry = f"lfb_gen_{k.name}"
        src = "\n".join(
            [prelude,
             f'extern "C" __global__ void __launch_bounds__({nthreads})',
             f"{entry}({', '.join(sig)})", "{"]
            + ["  " + d for d in decl] + ["  " + p for p in pro]
            + body + ["}", ""])
        key = hashlib.sha256(src.encode()).hexdigest()[:16]
        return Program(src, entry, tuple(order), params, tuple(block),
                       tuple(sorted(shared)), tuple(sorted(demoted)),
                       self.cooperative, key, tuple(self.tma_maps),
                       self.checked, tuple(self.insn_ids),
                       tuple(self.arr_names), self.trace,
                       tuple(self.trace_names),
                       tuple(self.trace_vis.get(q, ())
                             for q in range(len(self.insn_ids))))


def emit_cuda(kernel, checked=None, trace=False, params=None):
    """Render *kernel* (transformed, rules expanded or not) as one CUDA
    kernel; returns a :class:`Program`.  *checked*: None, "plain" (the
    reference's interpret() checks) or "dims" (interpret_bounds_checked).
    *trace*: also record every store (make_env(trace=True)).  *params*:
    parameter values for temporaries whose extents depend on them (the
    program is then specialised to those values)."""
    return _Emitter(kernel, checked, trace, params).emit()


def temp_params(kernel):
    """Parameters the temporaries' extents depend on (sorted)."""
    k = transforms.expand_all_rules(kernel) if kernel.rules else kernel
    names = set()
    for t in k.temporaries.values():
        for s in t.shape:
            names |= set(s.variables)
    return tuple(sorted(names))


__all__ = ["Program", "TmaMap", "emit_cuda", "temp_params", "NVRTC_OPTIONS",
           "promote"]
