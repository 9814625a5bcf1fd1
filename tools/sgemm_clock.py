"""sgemm 8192^3 back to back for ~3 s while nvidia-smi samples the SM
clock and power every 10 ms (is the tcgen05 3xTF32 kernel clock-limited?).
Prints per-launch time, the implied TFLOP/s and the clock/power samples
taken while the kernels ran."""
import json
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402


def main():
    m = n = l = 8192
    variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(0)
    _r, kg = fx.translate(fx.gemm_source("f32"))
    a = torch.rand(m * l, dtype=torch.float32, device=dev, generator=gen)
    b = torch.rand(l * n, dtype=torch.float32, device=dev, generator=gen)
    c = torch.rand(m * n, dtype=torch.float32, device=dev, generator=gen)
    env = lfb.env_from_buffers(kg, {"m": m, "n": n, "l": l},
                               {"a": a, "b": b, "c": c}, {"alpha": 1.5})
    L = lfb.Launcher(kg, env, variant=variant)
    for _ in range(3):
        L.launch()
    torch.cuda.synchronize()
    smi = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "10"],
        stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = 700
    e0.record()
    for _ in range(reps):
        L.launch()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    ms = e0.elapsed_time(e1) / reps
    samples = [r.split(", ") for r in out if r.strip()]
    clk = sorted(float(s[0]) for s in samples[30:-10]) if len(samples) > 50 else []
    pw = sorted(float(s[1]) for s in samples[30:-10]) if len(samples) > 50 else []
    print(json.dumps({"variant": variant, "ms": ms,
                      "tflops": 2.0 * m * n * l / (ms * 1e-3) / 1e12,
                      "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                      "sm_mhz_min": clk[0] if clk else None,
                      "power_median": pw[len(pw) // 2] if pw else None,
                      "reasons": sorted({s[2] for s in samples})[:5],
                      "samples": len(samples)}))


if __name__ == "__main__":
    main()
