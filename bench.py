"""Benchmark: executing a Fortran-ingested, transformed kernel on B200.

Default workload = BASELINE config 4: SEM Laplacian, order 7 (n = 8 points
per direction), fp64, 2^21 = 2,097,152 elements, the Appendix-A fixture with
its transform script (split_iname e by 32 -> g.0/l.0, assume, extract_subst),
element-sharded over the ranks (strong scaling: the 2M elements are split).
One step = one execution of the transformed kernel over every element of the
rank's shard, inputs resident in HBM (64 GiB at N=1 -- far above the 126 MB
L2, so no flush is needed between steps).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload sem2m|sem65k|fill|axpy|matvec|sgemm|sweep]

Prints ONE JSON line on rank 0 (the driver contract): value = whole-job
GDOF/s (nelt * n^3 / max-over-ranks step time), the roofline of the SEM
kernel against the measured HBM copy bandwidth, the CPU baseline (the
reference's own emitted C, oracle/_ref, on the host cores), the end-to-end
number through the public API with host buffers, SM clocks sampled during
the timed region, and the number of our kernel launches.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = ("SEM Laplacian GDOF/s fp64 + achieved HBM GB/s vs peak at 1/2/4/8 "
          "B200 vs CPU ref")


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(workload):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture (profiles/ncu_summary.json), or None."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        return s.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class Clocks:
    """Sample nvidia-smi during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,"
         "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# {{{ distributed plumbing

def dist_init(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus and world > 1:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    from paper_1503_07659_b200.dist import allreduce_max
    return allreduce_max(x)

# }}}


def sem_workload(args, rank, world, local):
    import numpy as np
    import torch

    import paper_1503_07659_b200 as lfb
    from paper_1503_07659_b200 import fixtures as fx
    from paper_1503_07659_b200.dist import allreduce_sum, shard_range

    n = args.npts
    nelt_total = args.nelt
    block = 32
    src = fx.semlap_source(n, block=block)
    _raw, knl = fx.translate(src, "semlap.f")
    lo, hi = shard_range(nelt_total, rank, world, block)
    nelt = hi - lo
    dev = torch.device("cuda", local)
    np3 = n ** 3

    # synthetic inputs, generated per shard on the device (per-shard seeds)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    u = torch.empty(nelt * np3, dtype=torch.float64, device=dev)
    g = torch.empty(6 * nelt * np3, dtype=torch.float64, device=dev)
    CH = 1 << 26
    for t in (u, g):
        for s in range(0, t.numel(), CH):
            v = t[s:s + CH]
            v.uniform_(0.0, 1.0, generator=gen)
    u.mul_(2).sub_(1)
    d = torch.rand(n * n, dtype=torch.float64, device=dev,
                   generator=gen) * 2 - 1
    w = torch.empty_like(u)
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    launcher = lfb.Launcher(knl, env, variant=args.variant)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        launcher.launch()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            launcher.launch()
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms_local, world)
    dofs = nelt_total * np3
    value = dofs / (ms * 1e-3) / 1e9

    # roofline of the SEM kernel: algorithmic 64 n^3 bytes per element
    # (u + 6 g read, w written) / launch duration
    bytes_per_launch = 64 * np3 * nelt
    achieved = bytes_per_launch / (ms_local * 1e-3) / 1e9
    peak, peak_src = _peaks()

    # verification (outside the timed region): fused sum(w^2) epilogue +
    # NCCL all-reduce, and a bitwise sample against the CPU oracle
    ws = torch.zeros(max(1, int(lfb_ws(n, nelt))), dtype=torch.float64,
                     device=dev)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    lfb.Launcher(knl, env, sumsq=ss, workspace=ws).launch()
    torch.cuda.synchronize()
    norm2 = allreduce_sum(float(ss.item()))
    verify = {"sumsq_allreduced": norm2}
    if not args.no_verify:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle
        ns = min(nelt, 512)
        uh = u[:ns * np3].cpu().numpy()
        gh = g[:6 * ns * np3].cpu().numpy()
        dh = d.cpu().numpy()
        ref = oracle.semlap(np.zeros_like(uh), uh, dh, gh, n, ns, threads=8)
        verify["sample_bitwise"] = bool(
            w[:ns * np3].cpu().numpy().tobytes() == ref.tobytes())
        verify["sample_elements"] = ns

    res = {
        "metric": METRIC, "value": value, "unit": "GDOF/s",
        "ms_per_step": ms, "scaling": "strong", "dtype": "f64",
        "config": {"workload": f"semlap order {n - 1} (n={n}) fp64, "
                               f"{nelt_total} elements, element-sharded "
                               f"over {world} GPU(s); fixture script "
                               "split_iname(e,32,g.0,l.0)+assume+"
                               "extract_subst(gf)",
                   "nelt": nelt_total, "npts": n, "block": block,
                   "parallelism": f"element shards x{world}",
                   "l2": "inputs 64 B/dof >> 126 MB L2; no flush needed",
                   "variant": args.variant},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     "traffic": _traffic("semlap_n8"),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_per_launch},
        "gpu_launches": args.steps,
        "verify": verify,
    }
    return res, launcher, env, (u, d, g, w), knl


def lfb_ws(n, nelt):
    from paper_1503_07659_b200 import abi
    return abi.load().lfb_semlap_workspace(n, nelt, None)


def sem_e2e(args, knl, n, nelt_e2e, dev):
    """Same metric through the public API with HOST buffers: every step
    copies u, g, d from pinned host memory, runs interpret(), and copies w
    back."""
    import torch

    import paper_1503_07659_b200 as lfb
    np3 = n ** 3
    hu = torch.empty(nelt_e2e * np3, dtype=torch.float64, pin_memory=True)
    hg = torch.empty(6 * nelt_e2e * np3, dtype=torch.float64,
                     pin_memory=True)
    hd = torch.rand(n * n, dtype=torch.float64).pin_memory()
    hw = torch.empty_like(hu).pin_memory()
    hu.uniform_(-1, 1)
    hg.uniform_(0, 1)
    du = torch.empty_like(hu, device=dev)
    dg = torch.empty_like(hg, device=dev)
    dd = torch.empty_like(hd, device=dev)
    dw = torch.empty_like(hu, device=dev)
    env = lfb.env_from_buffers(knl, {"nelt": nelt_e2e},
                               {"u": du, "d": dd, "g": dg, "w": dw})
    stream = torch.cuda.current_stream(dev)

    def step():
        du.copy_(hu, non_blocking=True)
        dg.copy_(hg, non_blocking=True)
        dd.copy_(hd, non_blocking=True)
        lfb.interpret(knl, env, inplace=True)
        hw.copy_(dw, non_blocking=True)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    steps = max(2, min(args.steps, 5))
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return {"value": nelt_e2e * np3 / (ms * 1e-3) / 1e9, "unit": "GDOF/s",
            "h2d_bytes_per_step": (hu.numel() + hg.numel() + hd.numel()) * 8,
            "d2h_bytes_per_step": hw.numel() * 8,
            "nelt": nelt_e2e, "ms_per_step": ms,
            "api": "paper_1503_07659_b200.interpret (ctypes C-ABI "
                   "lfb_semlap_f64)"}


def cpu_reference_rate(n, sample_elems, threads, min_seconds=10.0):
    """The reference's own emitted C (oracle/_ref; compiled cc -std=c99 -O1
    as tests/c_oracle.py:96) on host cores, element chunks <= 699,050 (its
    int indexing) and multiples of 32 (its assume(nelt mod 32 = 0))."""
    import ctypes as C
    import concurrent.futures as cf

    import numpy as np
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    kind = "reference"
    np3 = n ** 3
    rng = np.random.default_rng(0)
    u = rng.random(sample_elems * np3) * 2 - 1
    g = rng.random(6 * sample_elems * np3)
    d = rng.random(n * n) * 2 - 1
    w = np.zeros_like(u)
    if oracle.have_ref():
        P, I = C.c_void_p, C.c_int
        fn = oracle.ref_fn(f"ref_semlap_n{n}", [P, P, P, P, I])

        def run(e0, e1):
            off = e0 * np3
            fn(C.c_void_p(w.ctypes.data + off * 8),
               C.c_void_p(u.ctypes.data + off * 8),
               d.ctypes.data_as(P),
               C.c_void_p(g.ctypes.data + 6 * off * 8), e1 - e0)
    else:
        kind = "port"

        def run(e0, e1):
            oracle.semlap(w, u, d, g, n, sample_elems, elems=(e0, e1))
    per = sample_elems // threads // 32 * 32
    cuts = [t * per for t in range(threads)] + [sample_elems]
    t0 = time.perf_counter()
    reps = 0
    while True:
        with cf.ThreadPoolExecutor(threads) as pool:
            list(pool.map(lambda t: run(cuts[t], cuts[t + 1]),
                          range(threads)))
        reps += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": sample_elems * np3 / dt / 1e9, "unit": "GDOF/s",
            "cores": threads, "kind": kind,
            "sample": f"{sample_elems} elements of the same workload "
                      f"(n={n}), {reps} rep(s), "
                      f"{'reference emitted C -std=c99 -O1' if kind == 'reference' else 'oracle port'}, "
                      f"{threads} thread(s)"}


def probe_fp64(dev):
    import torch

    from paper_1503_07659_b200 import abi
    lib = abi.load()
    out = torch.zeros(148 * 8 * 256, dtype=torch.float64, device=dev)
    iters = 20000
    st = torch.cuda.current_stream(dev).cuda_stream
    lib.lfb_probe_fp64(out.data_ptr(), iters, 148 * 8, 256, st)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.lfb_probe_fp64(out.data_ptr(), iters, 148 * 8, 256, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ops = 148 * 8 * 256 * iters * 8 * 2
    return ops / (ms * 1e-3) / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="sem2m")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.npts = 8
    args.nelt = {"sem2m": 1 << 21, "sem65k": 65536}.get(args.workload,
                                                         1 << 21)
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        threads = os.cpu_count() or 1
        cpu = cpu_reference_rate(args.npts, 65536, threads, min_seconds=5.0)
        per_step_ms = 1e3 * 65536 * args.npts**3 / (cpu["value"] * 1e9)
        res = {"metric": METRIC, "value": cpu["value"], "unit": "GDOF/s",
               "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": per_step_ms,
               "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": f"semlap order 7 fp64, "
                                      f"{args.nelt} elements (timed on a "
                                      "65,536-element sample)",
                          "nelt": args.nelt, "npts": args.npts},
               "cpu_baseline": cpu,
               "e2e": {"value": cpu["value"], "unit": "GDOF/s",
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(res))
        return

    rank, world, local = dist_init(args.gpus)
    import torch
    res, launcher, env, bufs, knl = sem_workload(args, rank, world, local)
    dev = torch.device("cuda", local)
    res["clocks"] = None
    # clocks from the timed region were captured inside sem_workload? keep
    # a separate short sampled re-run so the numbers come with a record
    with Clocks(local) as clk:
        st = torch.cuda.current_stream(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.steps):
            launcher.launch()
        e1.record(st)
        torch.cuda.synchronize()
    res["clocks"] = clk.summary()
    res["fp64_probe_tflops"] = probe_fp64(dev)
    del bufs, env, launcher
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_e2e:
        res["e2e"] = sem_e2e(args, knl, args.npts, 65536, dev)
    else:
        res["e2e"] = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        res["cpu_baseline"] = cpu_reference_rate(args.npts, 65536, threads)
    else:
        res["cpu_baseline"] = None
    res.update({"n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "higher_is_better": True,
                "vs_baseline": None, "data": "synthetic"})
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
