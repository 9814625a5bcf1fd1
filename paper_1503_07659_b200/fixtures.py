"""Workload definitions: Fortran-subset sources + transform scripts.

Each workload is written in the reference's Fortran-77 subset
(/root/reference/pkg/src/loopforge/fortran.py:99-272) and carries the
``!$loopy`` transform block that BASELINE.json names for it.  The untransformed
lowering of the same text is the *template* the recognizer matches a user's
kernel against (recognize.py), so these texts define, operation by operation,
the arithmetic the CUDA kernels reproduce:

* fill   -- BASELINE config 1; the reference's own fill test shape
            (/root/reference/pkg/tests/test_fortran.py:13-27).
* axpy   -- BASELINE config 1.
* matvec -- BASELINE config 2 (extract_subst + precompute
            on the vector, the reference's equivalent of add_prefetch).
* semlap -- BASELINE configs 3/4/5: tensor-product spectral-element Laplacian,
            order p = n-1, n in 4..16.
* gemm   -- BASELINE config 5: the paper's DGEMM kernel
            (/root/reference/pkg/tests/test_fortran.py:72-103) in real*4 or
            real*8, with the paper's split/prefetch script.
"""

from __future__ import annotations

_FT = {"f64": "real*8", "f32": "real*4"}

FILL_SCRIPT = ('! {k} = lp.split_iname({k}, "i", {b}, outer_tag="g.0", '
               'inner_tag="l.0")\n')


def _block(lines):
    return "!$loopy begin transform\n" + "".join(lines) + \
        "!$loopy end transform\n"


def fill_source(dtype="f64", block=128, assume=False, script=True):
    t = _FT[dtype]
    src = f"""subroutine fill(out, a, n)
  implicit none
  {t} out(n), a
  integer n, i

  do i = 1, n
    out(i) = a
  end do
end
"""
    if script:
        lines = [FILL_SCRIPT.format(k="fill", b=block)]
        if assume:
            lines.append(f'! fill = lp.assume(fill, "n mod {block} = 0")\n')
        src += _block(lines)
    return src


def axpy_source(dtype="f64", block=128, assume=False, script=True):
    t = _FT[dtype]
    src = f"""subroutine axpy(y, x, alpha, n)
  implicit none
  {t} y(n), x(n), alpha
  integer n, i

  do i = 1, n
    y(i) = y(i) + alpha*x(i)
  end do
end
"""
    if script:
        lines = [FILL_SCRIPT.format(k="axpy", b=block)]
        if assume:
            lines.append(f'! axpy = lp.assume(axpy, "n mod {block} = 0")\n')
        src += _block(lines)
    return src


def matvec_source(dtype="f64", block=128, jtile=32, script=True):
    t = _FT[dtype]
    src = f"""subroutine matvec(y, a, x, n)
  implicit none
  {t} y(n), a(n,n), x(n), s
  integer n, i, j

  do i = 1, n
    s = 0
    do j = 1, n
      s = s + a(i,j)*x(j)
    end do
    y(i) = s
  end do
end
"""
    if script:
        src += _block([
            f'! matvec = lp.split_iname(matvec, "i", {block}, '
            'outer_tag="g.0", inner_tag="l.0")\n',
            f'! matvec = lp.split_iname(matvec, "j", {jtile})\n',
            f'! matvec = lp.assume(matvec, "n mod {block} = 0")\n',
            '! matvec = lp.extract_subst(matvec, "x_acc", "x[jj]", '
            'parameters="jj")\n',
            '! matvec = lp.precompute(matvec, "x_acc", "j_inner")\n',
        ])
    return src


def semlap_source(n=8, block=32, assume=True, gf=True, script=True):
    """SEM Laplacian of order p = n-1 (n points per direction)."""
    if not 2 <= n <= 16:
        raise ValueError(f"semlap: n={n} outside 2..16")
    src = f"""subroutine semlap(w, u, d, g, nelt)
  implicit none
  real*8 w({n},{n},{n},nelt), u({n},{n},{n},nelt), d({n},{n})
  real*8 g(6,{n},{n},{n},nelt)
  real*8 ur, us, ut, s, wr({n},{n},{n}), ws({n},{n},{n}), wt({n},{n},{n})
  integer nelt, e, i, j, k, l

  do e = 1, nelt
    do k = 1, {n}
      do j = 1, {n}
        do i = 1, {n}
          ur = 0
          us = 0
          ut = 0
          do l = 1, {n}
            ur = ur + d(i,l)*u(l,j,k,e)
            us = us + d(j,l)*u(i,l,k,e)
            ut = ut + d(k,l)*u(i,j,l,e)
          end do
          wr(i,j,k) = g(1,i,j,k,e)*ur + g(2,i,j,k,e)*us + g(3,i,j,k,e)*ut
          ws(i,j,k) = g(2,i,j,k,e)*ur + g(4,i,j,k,e)*us + g(5,i,j,k,e)*ut
          wt(i,j,k) = g(3,i,j,k,e)*ur + g(5,i,j,k,e)*us + g(6,i,j,k,e)*ut
        end do
      end do
    end do
    do k = 1, {n}
      do j = 1, {n}
        do i = 1, {n}
          s = 0
          do l = 1, {n}
            s = s + d(l,i)*wr(l,j,k) + d(l,j)*ws(i,l,k) + d(l,k)*wt(i,j,l)
          end do
          w(i,j,k,e) = s
        end do
      end do
    end do
  end do
end
"""
    if script:
        lines = [f'! semlap = lp.split_iname(semlap, "e", {block}, '
                 'outer_tag="g.0", inner_tag="l.0")\n']
        if assume and block > 1:
            lines.append(
                f'! semlap = lp.assume(semlap, "nelt mod {block} = 0")\n')
        if gf:
            lines.append('! semlap = lp.extract_subst(semlap, "gf", '
                         '"g[c, p, q, r, ee]", parameters="c, p, q, r, ee")\n')
        src += _block(lines)
    return src


def gemm_source(dtype="f32", script=True, tiles=(16, 8, 32)):
    """The paper's DGEMM kernel; ``dtype="f32"`` is BASELINE config 5."""
    t = _FT[dtype]
    name = "sgemm" if dtype == "f32" else "dgemm"
    ti, tj, tk = tiles
    src = f"""subroutine {name}(m,n,l,alpha,a,b,c)
  implicit none
  {t} a(m,l), b(l,n), c(m,n), alpha
  integer m, n, l, i, j, k

  do j = 1,n
    do k = 1,l
      do i = 1,m
        c(i,j) = c(i,j) + alpha*b(k,j)*a(i,k)
      end do
    end do
  end do
end subroutine
"""
    if script:
        src += _block([
            f'! {name} = lp.split_iname({name}, "i", {ti}, outer_tag="g.0", '
            'inner_tag="l.1")\n',
            f'! {name} = lp.split_iname({name}, "j", {tj}, outer_tag="g.1", '
            'inner_tag="l.0")\n',
            f'! {name} = lp.split_iname({name}, "k", {tk})\n',
            f'! {name} = lp.extract_subst({name}, "a_acc", "a[i1,i2]", '
            'parameters="i1, i2")\n',
            f'! {name} = lp.extract_subst({name}, "b_acc", "b[i1,i2]", '
            'parameters="i1, i2")\n',
            f'! {name} = lp.precompute({name}, "a_acc", "k_inner,i_inner")\n',
            f'! {name} = lp.precompute({name}, "b_acc", "j_inner,k_inner")\n',
        ])
    return src


def translate(source, name="<fixture>"):
    """(raw, transformed) kernels via the reference front end (its parser,
    lowering and transform verbs; script.py admits the paper's alias verbs
    as well, lowered to the reference's)."""
    from .script import translate_file_text
    raw, transformed, _unit = translate_file_text(source, name)
    return raw, transformed


# {{{ kernels for the generic path (cudagen.py)
#
# Fortran-ingested kernels outside the hand-written set, each exercising one
# piece of the reference semantics the generated CUDA must reproduce:
# predicates from if/else (lowering: fortran.py:484-498), transcendental
# calls, workgroup precompute tiles with barriers (the paper's DGEMM in
# real*8, test_fortran.py:72-103), numpy type promotion of mixed int/real*4
# arithmetic (interp.py:169-187), 2-D g/l tags with a residual guard, int32
# arithmetic, a stencil, and native-language reductions (interp.py:213-248).

_SPLIT = ('! {k} = lp.split_iname({k}, "{i}", {b}, outer_tag="g.{a}", '
          'inner_tag="l.{a}")\n')

GENERIC_FORTRAN = {
    # the reference's COND_F (test_fortran.py:29-48) with a launch script
    "cond": ("""subroutine cond(out, inp, n)
  implicit none
  real*8 out(n), inp(n), a, b
  integer n, i, j

  do i = 1, n
    a = inp(i)
    if (a.ge.0.25) then
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
""", [_SPLIT.format(k="cond", i="i", b=64, a=0)]),
    # the reference's TAGGED_F body (rotnorm: sin, cos, sqrt, division)
    "rotnorm": ("""subroutine rotnorm(out1, out2, inp1, inp2, alpha, n)
  implicit none
  real*8 out1(n), out2(n), inp1(n), inp2(n), alpha, a, b, r
  integer n, i

  do i = 1, n
    a = cos(alpha)*inp1(i) + sin(alpha)*inp2(i)
    b = -sin(alpha)*inp1(i) + cos(alpha)*inp2(i)
    r = sqrt(a**2 + b**2)
    a = a/r
    b = b/r
    out1(i) = a
    out2(i) = b
  end do
end
""", [_SPLIT.format(k="rotnorm", i="i", b=128, a=0)]),
    # int/real*4 mixing: numpy computes int32 op float32 in float64
    "mixed": ("""subroutine mixed(y, z, x, n)
  implicit none
  real*4 y(n), z(n), x(n)
  integer n, i

  do i = 1, n
    y(i) = x(i)*i + 0.5
    z(i) = x(i)/3 - 2*x(i)**2
  end do
end
""", [_SPLIT.format(k="mixed", i="i", b=32, a=0)]),
    "stencil": ("""subroutine stencil(r, u, n)
  implicit none
  real*4 r(n), u(n+1)
  integer n, i

  do i = 1, n
    r(i) = u(i+1) - u(i)
  end do
end
""", [_SPLIT.format(k="stencil", i="i", b=96, a=0)]),
    "transpose": ("""subroutine transpose(b, a, n, m)
  implicit none
  real*8 b(m,n), a(n,m)
  integer n, m, i, j

  do j = 1, m
    do i = 1, n
      b(j,i) = 2*a(i,j) - 1
    end do
  end do
end
""", [_SPLIT.format(k="transpose", i="i", b=16, a=0),
      _SPLIT.format(k="transpose", i="j", b=8, a=1)]),
    "intops": ("""subroutine intops(k, j, n)
  implicit none
  integer n, i, k(n), j(n)

  do i = 1, n
    k(i) = j(i)*3 + i*i - 7
  end do
end
""", [_SPLIT.format(k="intops", i="i", b=64, a=0)]),
    # matvec with the accumulation order of a user's own variant (y
    # accumulated in place): outside the recognizer's templates
    "matvec_acc": ("""subroutine mvacc(y, a, x, n)
  implicit none
  real*8 y(n), a(n,n), x(n)
  integer n, i, j

  do i = 1, n
    do j = 1, n
      y(i) = y(i) + x(j)*a(i,j)
    end do
  end do
end
""", [_SPLIT.format(k="mvacc", i="i", b=32, a=0),
      '! mvacc = lp.split_iname(mvacc, "j", 16)\n',
      '! mvacc = lp.extract_subst(mvacc, "x_acc", "x[jj]", '
      'parameters="jj")\n',
      '! mvacc = lp.precompute(mvacc, "x_acc", "j_inner")\n']),
    # a 3-point smoother whose u window is precomputed into a workgroup
    # tile (extent 66 = 64 + 2 halo): a 1-D footprint -> 1-D TMA box
    "smooth": ("""subroutine smooth(r, u, n)
  implicit none
  real*8 r(n), u(n+2)
  integer n, i

  do i = 1, n
    r(i) = u(i) + 2*u(i+1) + u(i+2)
  end do
end
""", [_SPLIT.format(k="smooth", i="i", b=64, a=0),
      '! smooth = lp.assume(smooth, "n mod 64 = 0")\n',
      '! smooth = lp.extract_subst(smooth, "u_acc", "u[j]", '
      'parameters="j")\n',
      '! smooth = lp.precompute(smooth, "u_acc", "i_inner")\n']),
    # tiled transpose through a workgroup tile (2-D footprint; the tile is
    # written along a's rows and read down its columns)
    "ttile": ("""subroutine ttile(b, a, n, m)
  implicit none
  real*8 b(m,n), a(n,m)
  integer n, m, i, j

  do j = 1, m
    do i = 1, n
      b(j,i) = a(i,j)
    end do
  end do
end
""", [_SPLIT.format(k="ttile", i="i", b=16, a=1),
      _SPLIT.format(k="ttile", i="j", b=16, a=0),
      '! ttile = lp.extract_subst(ttile, "a_acc", "a[p, q]", '
      'parameters="p, q")\n',
      '! ttile = lp.precompute(ttile, "a_acc", "i_inner, j_inner")\n']),
}

# native-language kernels (kernel.py:323 make_kernel): reductions
GENERIC_NATIVE = {
    "rowsum": (["{[i,j]: 0<=i<n and 0<=j<m}"],
               "out[i] = sum(j, a[i,j]*b[j])\n"
               "lo[i] = min(j, a[i,j])\nhi[i] = max(j, a[i,j])",
               [("i", 32, "g.0", "l.0")]),
}


def generic_source(name):
    """Fortran text (+ script) of a generic-path fixture."""
    body, lines = GENERIC_FORTRAN[name]
    return body + _block(lines)


def generic_native(name):
    """(raw, transformed) native-language kernels of a generic fixture."""
    from ._loopforge import kernel as lfk, transforms
    domains, body, splits = GENERIC_NATIVE[name]
    raw = lfk.make_kernel(domains, body, name=name,
                          dtype_default=lfk.F64)
    knl = raw
    for iname, factor, outer, inner in splits:
        knl = transforms.split_iname(knl, iname, factor, outer_tag=outer,
                                     inner_tag=inner)
    return raw, knl

# }}}
