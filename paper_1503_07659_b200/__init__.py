"""B200-native executor for Fortran-ingested, transformed loopforge kernels.

The reference (arXiv 1503.07659's Loo.py, re-created as ``loopforge``) keeps
its Fortran-subset front end and transform library; this package replaces
the execution step -- ``loopforge.interp.interpret`` -- with hand-written
sm_100a kernels behind a C ABI (include/loopforge_b200.h), and -- for kernels
outside that set -- with CUDA generated from the kernel's schedule
(cudagen.py, compiled by NVRTC for sm_100a)::

    import paper_1503_07659_b200 as lfb

    # the reference's front end (loopforge.fortran.translate_file_text), with
    # the paper's alias verbs (add_prefetch, tag_inames, ...) admitted
    raw, knl, _ = lfb.translate_file_text(source)
    env = lfb.make_device_env(knl, {"nelt": 65536}, seed=0)
    out = lfb.interpret(knl, env)                    # runs on the B200
    w = lfb.get_output(out, "w")

See DESIGN.md for the kernels and INTEGRATION.md for the ABI bindings.
"""

from .cudagen import emit_cuda
from .executor import (ENGINES, DeviceArray, DeviceEnv, Launcher,
                       env_from_buffers, flat_outputs, get_device_output,
                       get_output, interpret, interpret_bounds_checked,
                       make_device_env, make_launcher, plan_for)
from .launch import Geometry, launch_geometry
from .recognize import WORKLOADS, canonicalize, recognize
from .script import (add_prefetch, assignment_to_subst, fix_parameters,
                     tag_inames, translate_file_text)

__all__ = [
    "ENGINES", "emit_cuda", "make_launcher",
    "DeviceArray", "DeviceEnv", "Launcher", "env_from_buffers",
    "flat_outputs", "get_device_output", "get_output", "interpret",
    "interpret_bounds_checked",
    "make_device_env", "plan_for", "Geometry", "launch_geometry",
    "WORKLOADS", "canonicalize", "recognize",
    "add_prefetch", "assignment_to_subst", "fix_parameters", "tag_inames",
    "translate_file_text",
]

__version__ = "0.1.0"
