"""Time SEM kernel variants per order (tuning aid, not the driver's bench).

    python tools/sem_sweep.py 4:0,20,21 5:0,20 ...   [--bytes 2]  (GiB/order)

For each (n, variant): nelt = bytes / (64 n^3) rounded to 32, CUDA-event
time of back-to-back launches (inputs >> L2), GDOF/s and the HBM fraction,
plus a bitwise check of the first/last 64 elements against the oracle.
"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    gib = 2.0
    if "--bytes" in sys.argv:
        gib = float(sys.argv[sys.argv.index("--bytes") + 1])
        args = [a for a in args if a != sys.argv[sys.argv.index("--bytes") + 1]]
    peak, _ = bench._peaks()
    dev = torch.device("cuda", 0)
    for spec in args:
        n_s, vs = spec.split(":")
        n = int(n_s)
        nelt = int(gib * (1 << 30) / (64 * n ** 3)) // 32 * 32
        _r, knl = fx.translate(fx.semlap_source(n))
        u, d, g, w = bench.sem_buffers(n, nelt, dev, n)
        env = lfb.env_from_buffers(knl, {"nelt": nelt},
                                   {"u": u, "d": d, "g": g, "w": w})
        for v in vs.split(","):
            v = int(v)
            row = {"n": n, "variant": v, "nelt": nelt}
            try:
                L = lfb.Launcher(knl, env, variant=v)
                for _ in range(3):
                    L.launch()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                reps = 10
                e0.record()
                for _ in range(reps):
                    L.launch()
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                row["ms"] = round(ms, 4)
                row["gdofs"] = round(nelt * n ** 3 / (ms * 1e-3) / 1e9, 2)
                row["hbm_frac"] = round(64 * n ** 3 * nelt / (ms * 1e-3)
                                        / 1e9 / peak, 4)
                np3 = n ** 3
                ok = True
                dh = d.cpu().numpy()
                for lo in (0, nelt - 64):
                    uh = u[lo * np3:(lo + 64) * np3].cpu().numpy()
                    gh = g[6 * lo * np3:6 * (lo + 64) * np3].cpu().numpy()
                    ref = oracle.semlap(np.zeros_like(uh), uh, dh, gh, n, 64)
                    ok &= w[lo * np3:(lo + 64) * np3].cpu().numpy() \
                        .tobytes() == ref.tobytes()
                row["bitwise"] = bool(ok)
            except Exception as exc:  # report and go on
                row["error"] = str(exc)[:200]
            print(json.dumps(row), flush=True)
        del u, d, g, w, env
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
