"""SEM operator back to back for ~3 s while nvidia-smi samples SM clock,
power and throttle reasons every 10 ms: is a kernel power-capped when
sustained?   python tools/sem_clock.py n variant [nelt]"""
import json
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402


def main():
    n, variant = int(sys.argv[1]), int(sys.argv[2])
    nelt = int(sys.argv[3]) if len(sys.argv) > 3 else (1 << 21) * 512 // n ** 3
    dev = torch.device("cuda", 0)
    _r, knl = fx.translate(fx.semlap_source(n))
    u, d, g, w = bench.sem_buffers(n, nelt, dev, n)
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    L = lfb.Launcher(knl, env, variant=variant)
    for _ in range(3):
        L.launch()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    L.launch()
    e1.record()
    torch.cuda.synchronize()
    one = e0.elapsed_time(e1)
    reps = max(10, int(3000 / one))
    smi = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,power.draw,"
         "clocks_throttle_reasons.active", "--format=csv,noheader,nounits",
         "-lms", "10"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0.record()
    for _ in range(reps):
        L.launch()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    ms = e0.elapsed_time(e1) / reps
    samples = [r.split(", ") for r in out if r.strip()]
    mid = samples[30:-10] if len(samples) > 50 else samples
    clk = sorted(float(s[0]) for s in mid)
    pw = sorted(float(s[1]) for s in mid)
    print(json.dumps({"n": n, "variant": variant, "nelt": nelt,
                      "first_launch_ms": one, "sustained_ms": ms,
                      "gdofs": nelt * n ** 3 / (ms * 1e-3) / 1e9,
                      "hbm_gbs": 64 * n ** 3 * nelt / (ms * 1e-3) / 1e9,
                      "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                      "sm_mhz_min": clk[0] if clk else None,
                      "power_median": pw[len(pw) // 2] if pw else None,
                      "reasons": sorted({s[2] for s in samples}),
                      "samples": len(samples)}), flush=True)


if __name__ == "__main__":
    main()
