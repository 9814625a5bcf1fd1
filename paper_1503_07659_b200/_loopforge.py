"""Locate the reference front end (``loopforge``) that this executor sits behind.

The executor replaces only the *execution* step of the reference
(``loopforge.interp.interpret``, /root/reference/pkg/src/loopforge/interp.py:323).
The Fortran-subset front end, the kernel IR and the transform library are
consumed unchanged.  They are found, in order:

1. an importable ``loopforge`` (a user's own install);
2. ``<repo>/baseline/_ref`` -- the offline ``pip install --target`` of the
   reference that ``__graft_entry__.build()`` creates; it travels with the repo
   snapshot to the GPU box.

Nothing here reads ``/root/reference`` at run time.
"""

from __future__ import annotations

import importlib
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INSTALL = os.path.join(_REPO, "baseline", "_ref")


def _import():
    try:
        return importlib.import_module("loopforge")
    except ImportError:
        pass
    if os.path.isdir(os.path.join(REF_INSTALL, "loopforge")):
        if REF_INSTALL not in sys.path:
            sys.path.insert(0, REF_INSTALL)
        return importlib.import_module("loopforge")
    raise ImportError(
        "the loopforge front end is not importable; run "
        "__graft_entry__.build() (installs it into baseline/_ref) or put "
        "loopforge on PYTHONPATH")


loopforge = _import()

from loopforge import expr as ex                      # noqa: E402
from loopforge import codegen, fortran, interp, kernel, polyset, transforms  # noqa: E402,F401
from loopforge.errors import (CodegenError, InterpError, LoopforgeError,   # noqa: E402,F401
                              ScheduleError, ValidationError)

__all__ = ["loopforge", "ex", "codegen", "fortran", "interp", "kernel",
           "polyset", "transforms", "CodegenError", "InterpError",
           "LoopforgeError", "ScheduleError", "ValidationError"]
