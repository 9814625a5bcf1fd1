"""The paper's transform vocabulary on top of the reference's nine verbs.

The north star names Loo.py's ``tag_inames``, ``add_prefetch``,
``assignment_to_subst`` and ``fix_parameters`` (tags ``unr`` / ``ilp``), but
the reference only has ``TRANSFORM_VERBS``
(/root/reference/pkg/src/loopforge/transforms.py:843-853), the tags ``g.N``,
``l.N``, ``unroll`` and ``sequential`` (kernel.py:23-24), and its script
runner rejects unknown verbs (fortran.py:806-808).  Each alias here lowers to
the reference's own verbs or to a plain rewrite of its immutable Kernel IR,
so the result is an ordinary reference Kernel -- the reference interpreter
(the oracle) runs exactly what the device runs:

=======================  =================================================
alias                    lowering
=======================  =================================================
``tag_inames``           set ``iname_tags`` (``unr``/``ilp`` -> ``unroll``,
                         ``for`` -> ``sequential``), ``validate_kernel``
``add_prefetch``         ``wrap_variable_access`` (extract_subst over every
                         read of the array) + ``precompute`` over the sweep
``assignment_to_subst``  ``temporary_to_subst``
``fix_parameters``       parameter -> constant in domains, shapes, strides,
                         bodies, rules and assumptions; in Fortran text it is
                         substituted *before* lowering (a symbolic order
                         makes the column-major strides non-affine,
                         fortran.py:648-657)
=======================  =================================================

:func:`translate_file_text` is the reference's front-end entry
(fortran.py:837-850) with the aliases admitted in ``!$loopy`` scripts.
"""

from __future__ import annotations

import dataclasses
import re

from ._loopforge import ex, fortran, kernel as lfk, polyset, transforms
from ._loopforge import LoopforgeError
from loopforge.errors import TransformError

_TAG_ALIASES = {"unr": "unroll", "ilp": "unroll", "ilp.unr": "unroll",
                "ilp.seq": "sequential", "for": "sequential",
                "l.auto": "sequential"}


def _tag(tag):
    return _TAG_ALIASES.get(tag, tag)


# {{{ aliases

def tag_inames(kernel, tags, force=False):
    """Loo.py's ``tag_inames``: *tags* is ``{"i": "g.0"}``, a sequence of
    ``(iname, tag)`` pairs or the text ``"i:g.0, j:l.0"``."""
    if isinstance(tags, str):
        pairs = []
        for part in tags.split(","):
            if not part.strip():
                continue
            if ":" not in part:
                raise TransformError(f"tag_inames: bad entry {part!r}; "
                                     "expected 'iname:tag'")
            name, tag = part.split(":", 1)
            pairs.append((name.strip(), tag.strip()))
    elif isinstance(tags, dict):
        pairs = list(tags.items())
    else:
        pairs = [tuple(p) for p in tags]
    new = dict(kernel.iname_tags)
    for name, tag in pairs:
        if name not in kernel.all_inames:
            raise TransformError(f"unknown iname: {name}")
        tag = _tag(tag)
        if tag is not None and tag not in lfk.VALID_TAGS \
                and not lfk.is_parallel_tag(tag):
            raise TransformError(
                f"bad iname tag {tag!r}; expected g.N, l.N, unroll, "
                "sequential (or unr / ilp)")
        old = new.get(name)
        if old is not None and old != tag and not force \
                and lfk.is_parallel_tag(old):
            raise TransformError(f"iname '{name}' is already tagged {old}")
        if tag is None:
            new.pop(name, None)
        else:
            new[name] = tag
    out = kernel.copy(iname_tags=new)
    lfk.validate_kernel(out)
    return out


def add_prefetch(kernel, var_name, sweep_inames=(), default_tag="sequential",
                 rule_name=None):
    """Loo.py's ``add_prefetch``: every read of *var_name* becomes a rule
    (``wrap_variable_access``, transforms.py:265-282), which ``precompute``
    (transforms.py:541-684) materialises over the sweep footprint; the
    temporary is ``<rule>_0``."""
    if rule_name is None:
        rule_name = kernel.fresh_name(f"{var_name}_fetch")
    k = transforms.wrap_variable_access(kernel, var_name, rule_name)
    return transforms.precompute(k, rule_name, sweep_inames,
                                 default_tag=_tag(default_tag))


def assignment_to_subst(kernel, lhs_name):
    """Loo.py's ``assignment_to_subst`` = the reference's
    ``temporary_to_subst`` (transforms.py:289)."""
    return transforms.temporary_to_subst(kernel, lhs_name)


def _fix_expr(e, values):
    return ex.substitute(e, {n: ex.IntLit(v) for n, v in values.items()})


def _fix_aff(a, values):
    return a.substitute({n: int(v) for n, v in values.items()})


def fix_parameters(kernel, **values):
    """Loo.py's ``fix_parameters``: each named parameter becomes a constant
    everywhere it appears (domains, argument shapes and strides, instruction
    bodies, rules, assumptions).  A fixed value that violates an assumption
    is a TransformError."""
    params = set(kernel.param_names)
    for name in values:
        if name not in params:
            raise TransformError(f"fix_parameters: unknown parameter "
                                 f"'{name}'")
    values = {k: int(v) for k, v in values.items()}
    nodes = []
    for node in kernel.domains.nodes:
        cs = [polyset.Constraint(c.kind, _fix_aff(c.expr, values))
              for c in node.constraints]
        nodes.append(polyset.BasicSet(
            node.set_dims, [p for p in node.params if p not in values], cs))
    domains = polyset.DomainTree(tuple(nodes), kernel.domains.parent)
    args = tuple(dataclasses.replace(
        a, shape=tuple(_fix_aff(s, values) for s in a.shape),
        strides=tuple(_fix_aff(s, values) for s in a.strides))
        for a in kernel.args)
    temps = {n: dataclasses.replace(
        t, shape=tuple(_fix_aff(s, values) for s in t.shape))
        for n, t in kernel.temporaries.items()}
    insns = tuple(dataclasses.replace(
        i, lhs=_fix_expr(i.lhs, values), rhs=_fix_expr(i.rhs, values))
        for i in kernel.instructions)
    rules = {n: dataclasses.replace(r, body=_fix_expr(r.body, values))
             for n, r in kernel.rules.items()}
    a = kernel.assumptions
    div = []
    for expr, mod in a.divisibility:
        fe = _fix_aff(expr, values)
        if not fe.coeffs:
            if fe.constant % mod:
                raise TransformError(
                    f"fix_parameters: {values} violates "
                    f"{expr.render()} mod {mod} = 0")
            continue
        div.append((fe, mod))
    pcs = []
    for c in a.param_constraints:
        fc = polyset.Constraint(c.kind, _fix_aff(c.expr, values))
        if fc.is_trivially_false():
            raise TransformError(f"fix_parameters: {values} violates an "
                                 "assumption")
        if not fc.is_trivially_true():
            pcs.append(fc)
    assumptions = polyset.Assumptions(tuple(div), tuple(pcs))
    out = kernel.copy(domains=domains, args=args, temporaries=temps,
                      instructions=insns, rules=rules,
                      assumptions=assumptions)
    lfk.validate_kernel(out)
    return out

# }}}


ALIAS_VERBS = {"tag_inames": tag_inames, "add_prefetch": add_prefetch,
               "assignment_to_subst": assignment_to_subst,
               "fix_parameters": fix_parameters}

VERBS = {**transforms.TRANSFORM_VERBS, **ALIAS_VERBS}


# {{{ script runner and front end

def _is_kernel_ref(v):
    return type(v).__name__ == "_KernelRef"


def run_transform_script(kernels, script):
    """The reference's script runner (fortran.py:798-834) -- the whole
    script validated before any transform runs, the same errors -- over the
    reference verbs plus the aliases."""
    if isinstance(script, str):
        script = fortran.parse_transform_script(script)
    kernels = dict(kernels)
    known = set(kernels)
    for st in script.statements:
        span = (None, st.line, None)
        if st.verb not in VERBS:
            raise TransformError(f"unknown transform '{st.verb}'", span=span)
        if not st.args or not _is_kernel_ref(st.args[0]):
            raise TransformError(f"transform '{st.verb}' needs a kernel as "
                                 "first argument", span=span)
        if st.args[0].name not in known:
            raise TransformError(f"unknown kernel '{st.args[0].name}'",
                                 span=span)
        bad = [a.name for a in st.args[1:] if _is_kernel_ref(a)]
        if bad:
            raise TransformError(f"unexpected identifier argument "
                                 f"'{bad[0]}'", span=span)
        known.add(st.target)
    for st in script.statements:
        try:
            kernels[st.target] = VERBS[st.verb](
                kernels[st.args[0].name], *st.args[1:], **dict(st.kwargs))
        except TypeError as err:
            raise TransformError(f"bad arguments for '{st.verb}': {err}",
                                 span=(None, st.line, None)) from err
    return kernels


_PRAGMA = re.compile(r"^\s*!\$loopy\s+(begin|end)\s+transform\s*$", re.I)


def _fix_source(source, values):
    """fix_parameters on Fortran text, before lowering: drop the parameters
    from the dummy-argument list and the integer declarations, then write
    each remaining use as its literal value (Fortran names are
    case-insensitive)."""
    out = []
    in_block = False
    names = {n.lower() for n in values}
    word = re.compile(r"\b(" + "|".join(re.escape(n) for n in values)
                      + r")\b", re.I)

    def drop_items(text):
        items = [x for x in text.split(",")
                 if x.strip().lower() not in names]
        return ",".join(items)

    for line in source.splitlines():
        if _PRAGMA.match(line):
            in_block = "begin" in line.lower()
            out.append(line)
            continue
        stripped = line.strip()
        if in_block or stripped.startswith("!") or not stripped:
            out.append(line)
            continue
        m = re.match(r"^(\s*subroutine\s+\w+\s*\()([^)]*)(\).*)$", line,
                     re.I)
        if m:
            out.append(m.group(1) + drop_items(m.group(2)) + m.group(3))
            continue
        m = re.match(r"^(\s*integer\s+)(.*)$", line, re.I)
        if m:
            rest = drop_items(m.group(2))
            if rest.strip():
                out.append(m.group(1) + rest.strip())
            continue
        out.append(word.sub(lambda mm: str(values[
            next(k for k in values if k.lower() == mm.group(1).lower())]),
            line))
    return "\n".join(out) + ("\n" if source.endswith("\n") else "")


def translate_file_text(source, source_name="<fortran>", extra_scripts=()):
    """The reference's ``translate_file_text`` (fortran.py:837-850) --
    parse, lower, run the embedded (then extra) transform scripts; returns
    (raw kernel, transformed kernel, unit) -- with the paper's alias verbs
    admitted.  ``fix_parameters`` statements of the embedded scripts are
    applied to the source text before lowering."""
    unit = fortran.parse_fortran(source, source_name)
    fixed = {}
    blocks = []
    for text, line in unit.transform_blocks:
        script = fortran.parse_transform_script(text)
        keep = []
        for st in script.statements:
            if st.verb == "fix_parameters" and not st.args[1:]:
                fixed.update(dict(st.kwargs))
            else:
                keep.append(st)
        blocks.append(fortran.TransformScript(tuple(keep)))
    if fixed:
        try:
            unit = fortran.parse_fortran(_fix_source(source, fixed),
                                         source_name)
        except LoopforgeError as err:
            raise TransformError(f"fix_parameters {fixed}: {err}") from err
    raw = fortran.lower_to_kernel(unit)
    kernels = {unit.name: raw}
    for script in blocks:
        kernels = run_transform_script(kernels, script)
    for text in extra_scripts:
        kernels = run_transform_script(kernels, text)
    return raw, kernels[unit.name], unit

# }}}


__all__ = ["tag_inames", "add_prefetch", "assignment_to_subst",
           "fix_parameters", "ALIAS_VERBS", "VERBS", "run_transform_script",
           "translate_file_text"]
