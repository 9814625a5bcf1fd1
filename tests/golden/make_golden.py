"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (where /root/reference or baseline/_ref provides loopforge):

    python tests/golden/make_golden.py

For every case: translate the fixture Fortran text with the reference front
end (``translate_file_text``, fortran.py:837), bind inputs with the
reference's ``make_env`` (interp.py:79-123: seeded arrays are
``rng.random(shape)*2-1``), execute with the reference interpreter
(``interpret``, interp.py:323) and write every flat buffer -- inputs before,
outputs after -- in the reference's own array-file format
(``write_array_file``, interp.py:426-438).  The GPU box has no
/root/reference, so these committed files are what the device parity tests
and the oracle pin against.
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
for p in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "loopforge")):
        sys.path.insert(0, p)
        break
sys.path.insert(0, REPO)

from loopforge.interp import interpret, make_env, write_array_file  # noqa
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402

# name -> (fixture generator, kwargs, params, explicit inputs, seed)
CASES = {
    "fill_f64_n300": ("fill_source", {"dtype": "f64"}, {"n": 300},
                      {"a": 1.5}, None),
    "fill_f64_assume_n256": ("fill_source", {"dtype": "f64", "assume": True},
                             {"n": 256}, {"a": -2.75}, None),
    "fill_f32_n300": ("fill_source", {"dtype": "f32"}, {"n": 300},
                      {"a": 0.1}, None),
    "axpy_f64_n300": ("axpy_source", {"dtype": "f64"}, {"n": 300},
                      {"alpha": 1.25}, 0),
    "axpy_f32_n333": ("axpy_source", {"dtype": "f32"}, {"n": 333},
                      {"alpha": -0.75}, 1),
    "matvec_f64_n128": ("matvec_source", {"dtype": "f64"}, {"n": 128},
                        {}, 2),
    "semlap_n8_b2_nelt2": ("semlap_source", {"n": 8, "block": 2},
                           {"nelt": 2}, {}, 3),
    "semlap_n4_b2_nelt4": ("semlap_source", {"n": 4, "block": 2},
                           {"nelt": 4}, {}, 4),
    "semlap_n6_b1_nelt2": ("semlap_source", {"n": 6, "block": 1},
                           {"nelt": 2}, {}, 5),
    "semlap_n5_b2_nelt2": ("semlap_source", {"n": 5, "block": 2},
                           {"nelt": 2}, {}, 6),
    "sgemm_m16_n8_l32": ("gemm_source", {"dtype": "f32"},
                         {"m": 16, "n": 8, "l": 32}, {"alpha": 1.5}, 7),
    "sgemm_m20_n12_l40": ("gemm_source", {"dtype": "f32"},
                          {"m": 20, "n": 12, "l": 40}, {"alpha": -0.5}, 8),
    # generic path (cudagen.py): kernels outside the hand-written set
    "gen_cond_n300": ("generic_source", {"name": "cond"}, {"n": 300}, {}, 11),
    "gen_rotnorm_n300": ("generic_source", {"name": "rotnorm"}, {"n": 300},
                         {"alpha": 0.3}, 12),
    "gen_mixed_n333": ("generic_source", {"name": "mixed"}, {"n": 333}, {},
                       13),
    "gen_stencil_n250": ("generic_source", {"name": "stencil"}, {"n": 250},
                         {}, 14),
    "gen_transpose_n37_m21": ("generic_source", {"name": "transpose"},
                              {"n": 37, "m": 21}, {}, 15),
    "gen_intops_n200": ("generic_source", {"name": "intops"}, {"n": 200},
                        {}, 16),
    "gen_mvacc_n64": ("generic_source", {"name": "matvec_acc"}, {"n": 64},
                      {}, 17),
    "gen_dgemm_m20_n12_l40": ("gemm_source", {"dtype": "f64"},
                              {"m": 20, "n": 12, "l": 40}, {"alpha": 0.75},
                              18),
    "gen_rowsum_n40_m17": ("generic_native", {"name": "rowsum"},
                           {"n": 40, "m": 17}, {}, 19),
    # precompute footprints fetched by TMA on the device: 1-D window with
    # halo; 2-D tile read down its columns (swizzled), ragged (m = 21) with
    # a TMA-able leading dimension (n = 40) and one that is not (n = 37:
    # 296-B rows, cooperative fallback)
    "gen_smooth_n320": ("generic_source", {"name": "smooth"}, {"n": 320},
                        {}, 20),
    "gen_ttile_n40_m21": ("generic_source", {"name": "ttile"},
                          {"n": 40, "m": 21}, {}, 21),
    "gen_ttile_n37_m21": ("generic_source", {"name": "ttile"},
                          {"n": 37, "m": 21}, {}, 22),
}

# in/out arrays: outputs that are also read (make_env never randomises
# outputs, interp.py:115, so they get values from a second stream)
INOUT = {"gemm_source": "c", "axpy_source": "y",
         ("generic_source", "matvec_acc"): "y"}


def build_case(name, spec):
    gen, kwargs, params, explicit, seed = spec
    if gen == "generic_native":
        _raw, knl = fx.generic_native(**kwargs)
    else:
        src = getattr(fx, gen)(**kwargs)
        _raw, knl = fx.translate(src, f"{name}.f")
    inputs = dict(explicit)
    inout = INOUT.get(gen) or INOUT.get((gen, kwargs.get("name")))
    if inout:
        # in/out arrays are outputs, which make_env never randomises
        # (interp.py:115): give them values from a second stream
        amap = knl.arg_map()
        shape = tuple(s.eval(params) for s in amap[inout].shape)
        inputs[inout] = np.random.default_rng(100 + seed).random(shape) * 2 - 1
    env = make_env(knl, params, inputs, seed=seed)
    t0 = time.time()
    out = interpret(knl, env)
    dt = time.time() - t0
    d = os.path.join(HERE, name)
    os.makedirs(d, exist_ok=True)
    files = {}
    for a in knl.args:
        arr_in = env.arrays[a.name].data
        write_array_file(os.path.join(d, f"{a.name}.in.bin"), arr_in, a.dtype)
        files[a.name] = {"kind": a.kind, "dtype": a.dtype,
                         "is_output": bool(a.is_output),
                         "shape": list(env.arrays[a.name].shape),
                         "strides": list(env.arrays[a.name].strides)}
        if a.is_output:
            write_array_file(os.path.join(d, f"{a.name}.out.bin"),
                             out.arrays[a.name].data, a.dtype)
    meta = {"generator": gen, "kwargs": kwargs, "params": params,
            "seed": seed, "args": files, "kernel": knl.name,
            "interpret_seconds": round(dt, 2)}
    with open(os.path.join(d, "meta.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"{name}: interpret {dt:.1f}s")


def main(names=None):
    for name, spec in CASES.items():
        if names and name not in names:
            continue
        build_case(name, spec)


if __name__ == "__main__":
    main(sys.argv[1:])
