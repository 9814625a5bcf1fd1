"""Time the direct-stiffness summation alone (tuning aid).

    python tools/dssum_probe.py [E] [n] [variants...]

E^3 elements of n points per direction; each variant (0 = default; the
kernel variant rides in bits 4+ of the ABI's mode) is timed over 20
back-to-back launches with CUDA events and checked bitwise against the
default kernel's result on the same input.
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_1503_07659_b200 import abi  # noqa: E402
from paper_1503_07659_b200.assembly import BoxMesh  # noqa: E402


def launch(w, mesh, variant):
    lib = abi.load()
    s = torch.cuda.current_stream().cuda_stream
    abi.check(lib.lfb_dssum_f64(abi.C.c_void_p(w.data_ptr()), mesh.n, mesh.ex,
                                mesh.ey, mesh.ez, 0, mesh.top, variant << 4,
                                None, None, s), "dssum")


def main():
    E = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    variants = [int(v) for v in sys.argv[3:]] or [0]
    mesh = BoxMesh(E, E, E, n)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    w0 = torch.rand(mesh.nelt * n ** 3, dtype=torch.float64, device=dev,
                    generator=g)
    ref = w0.clone()
    launch(ref, mesh, 0)
    algo = 16 * (n ** 3 - (n - 2) ** 3) * mesh.nelt
    for v in variants:
        w = w0.clone()
        launch(w, mesh, v)
        torch.cuda.synchronize()
        ok = torch.equal(w, ref)
        for _ in range(3):
            launch(w, mesh, v)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            launch(w, mesh, v)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"E": E, "n": n, "variant": v, "ms": round(ms, 4),
                          "algo_GBs": round(algo / ms / 1e6, 1),
                          "sector_floor_GBs": round(
                              2 * 8 * n ** 3 * mesh.nelt / ms / 1e6, 1),
                          "bitwise_vs_default": bool(ok)}), flush=True)


if __name__ == "__main__":
    main()
