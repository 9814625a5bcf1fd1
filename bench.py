"""Benchmark: executing a Fortran-ingested, transformed kernel on B200.

Default workload = BASELINE config 4: SEM Laplacian, order 7 (n = 8 points
per direction), fp64, 2^21 = 2,097,152 elements, the Appendix-A fixture with
its transform script (split_iname e by 32 -> g.0/l.0, assume, extract_subst),
element-sharded over the ranks (the 2M elements are split: strong scaling).
One step = one execution of the transformed kernel over every element of the
rank's shard, inputs resident in HBM (64 GiB at N=1 -- far above the 126 MB
L2, so no flush is needed between steps).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
    python bench.py --workload sem65k|fill|axpy|matvec|sgemm|sweep   (others)

Prints ONE JSON line on rank 0 (the driver contract): value = whole-job
GDOF/s (nelt * n^3 / max-over-ranks step time); the roofline of the SEM
kernel (algorithmic 64 n^3 bytes/element, over the CUDA-event
launch time) against the measured HBM copy bandwidth; the CPU baseline (the
reference's own emitted C, oracle/_ref, on the host cores); the end-to-end
number through the public API with host buffers; SM clocks sampled during the
timed region; the number of our kernel launches.
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
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(key):
    """Per-launch DRAM bytes (dram__bytes_read.sum + write) of the dominant
    kernel from the committed ncu --set full capture, or None."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(key, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class Clocks:
    """nvidia-smi samples during the timed region (B200_PROFILING.md)."""

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
                 "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, power = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(power) if power else None}


# {{{ distributed plumbing

def dist_init(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}")
    # test hooks: LFB_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 and
    # LFB_BENCH_BACKEND=gloo replaces NCCL (NCCL refuses two ranks on one
    # GPU) -- exercises the multi-rank path on a one-GPU box; such numbers
    # are not measurements
    if os.environ.get("LFB_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("LFB_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl",
                                    device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
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


def timed(fn, steps, warmup, world, local):
    """W untimed steps, then K steps between barrier+synchronize pairs,
    CUDA events on the launching stream, clocks sampled throughout.
    Returns (max-over-ranks ms/step, this rank's ms/step, clocks)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms_local = e0.elapsed_time(e1) / steps
    return max_over_ranks(ms_local, world), ms_local, clk.summary()

# }}}


# {{{ SEM (default)

def sem_buffers(n, nelt, dev, seed):
    import torch
    np3 = n ** 3
    gen = torch.Generator(device=dev).manual_seed(seed)
    u = torch.empty(nelt * np3, dtype=torch.float64, device=dev)
    g = torch.empty(6 * nelt * np3, dtype=torch.float64, device=dev)
    CH = 1 << 26
    for t, lo, hi in ((u, -1.0, 1.0), (g, 0.0, 1.0)):
        for s in range(0, t.numel(), CH):
            t[s:s + CH].uniform_(lo, hi, generator=gen)
    d = torch.rand(n * n, dtype=torch.float64, device=dev,
                   generator=gen) * 2 - 1
    w = torch.empty_like(u)
    return u, d, g, w


def _sem_sample_check(u, g, d, w, n, nelt, exact, count=1024, seed=7):
    """Elements 0, 1, nelt - 1 and *count* random ones across the whole
    range, gathered from the device and checked against the oracle: bitwise
    (*exact*), else per point within 1e-12 of the magnitude of the summed
    terms (the same operator on |u|, |d|, |g|)."""
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    np3 = n ** 3
    es = np.unique(np.concatenate([
        [0, 1, nelt - 1],
        np.random.default_rng(seed).integers(0, nelt, count)]))
    idx = torch.as_tensor(es, device=u.device)

    def gather(t, per):
        return t.view(-1, per).index_select(0, idx).reshape(-1).cpu() \
            .numpy()
    uh, gh, wh = gather(u, np3), gather(g, 6 * np3), gather(w, np3)
    dh = d.cpu().numpy()
    ref = oracle.semlap(np.zeros_like(uh), uh, dh, gh, n, len(es),
                        threads=8)
    out = {"elements": int(len(es)), "spread": "0, 1, last and random "
           "elements across the whole range"}
    if exact:
        out["bitwise"] = bool(wh.tobytes() == ref.tobytes())
        out["pass"] = out["bitwise"]
    else:
        mag = oracle.semlap(np.zeros_like(uh), np.abs(uh), np.abs(dh),
                            np.abs(gh), n, len(es), threads=8)
        err = float((np.abs(wh - ref) / mag).max())
        out["max_err_over_magnitude"] = err
        out["tolerance"] = 1e-12
        out["pass"] = err <= 1e-12
    return out


def sem_bench(args, rank, world, local):
    import numpy as np
    import torch

    import paper_1503_07659_b200 as lfb
    from paper_1503_07659_b200 import abi
    from paper_1503_07659_b200 import fixtures as fx
    from paper_1503_07659_b200.dist import allreduce_sum, shard_range

    n, nelt_total, block = args.npts, args.nelt, 32
    _raw, knl = fx.translate(fx.semlap_source(n, block=block), "semlap.f")
    lo, hi = shard_range(nelt_total, rank, world, block)
    nelt = hi - lo
    dev = torch.device("cuda", local)
    np3 = n ** 3
    u, d, g, w = sem_buffers(n, nelt, dev, 1000 + rank)
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    sem_variant = args.variant if args.variant is not None else 50
    launcher = lfb.Launcher(knl, env, variant=sem_variant)

    ms, ms_local, clocks = timed(launcher.launch, args.steps, args.warmup,
                                 world, local)
    # the bitwise kernel (the reference's separately rounded arithmetic)
    # on the same buffers, same timing method
    bitwise = None
    if sem_variant != 0:
        lb = lfb.Launcher(knl, env, variant=0)
        ms_b, ms_b_local, clocks_b = timed(lb.launch, args.steps,
                                           args.warmup, world, local)
        bitwise = {"variant": 0, "parity": "bitwise",
                   "value": nelt_total * np3 / (ms_b * 1e-3) / 1e9,
                   "ms_per_step": ms_b,
                   "roofline_frac": 64 * np3 * nelt / (ms_b_local * 1e-3)
                   / 1e9 / _peaks()[0], "clocks": clocks_b}
        if not args.no_verify:
            # w holds the bitwise kernel's result: head, tail and random
            # elements across the whole shard, bitwise against the oracle
            torch.cuda.synchronize()
            bitwise["verify"] = _sem_sample_check(u, g, d, w, n, nelt,
                                                  exact=True)
    value = nelt_total * np3 / (ms * 1e-3) / 1e9
    bytes_per_launch = 64 * np3 * nelt
    achieved = bytes_per_launch / (ms_local * 1e-3) / 1e9
    peak, peak_src = _peaks()

    # the same HBM access mix without the arithmetic, same buffers: the
    # streaming ceiling at this footprint (context for roofline.frac)
    lib = abi.load()
    st = torch.cuda.current_stream(dev).cuda_stream
    for _ in range(2):
        lib.lfb_probe_stream(w.data_ptr(), u.data_ptr(), g.data_ptr(),
                             nelt * np3, st)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record()
    for _ in range(5):
        lib.lfb_probe_stream(w.data_ptr(), u.data_ptr(), g.data_ptr(),
                             nelt * np3, st)
    p1.record()
    torch.cuda.synchronize()
    probe_gbs = bytes_per_launch / (p0.elapsed_time(p1) / 5 * 1e-3) / 1e9

    # verification, outside the timed region: fused sum(w^2) epilogue + one
    # NCCL all-reduce, and a bitwise sample vs the oracle
    ws = torch.zeros(max(1, int(abi.load().lfb_semlap_workspace(n, nelt,
                                                                None))),
                     dtype=torch.float64, device=dev)
    ss = torch.zeros(1, dtype=torch.float64, device=dev)
    lfb.Launcher(knl, env, sumsq=ss, workspace=ws,
                 variant=sem_variant).launch()
    torch.cuda.synchronize()
    verify = {"sumsq_allreduced": allreduce_sum(float(ss.item())),
              "variant": sem_variant}
    if not args.no_verify:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle
        ns = min(nelt, 512)
        for tag, e0 in (("head", 0), ("tail", nelt - ns)):
            uh = u[e0 * np3:(e0 + ns) * np3].cpu().numpy()
            gh = g[6 * e0 * np3:6 * (e0 + ns) * np3].cpu().numpy()
            dh = d.cpu().numpy()
            ref = oracle.semlap(np.zeros_like(uh), uh, dh, gh, n, ns,
                                threads=8)
            got = w[e0 * np3:(e0 + ns) * np3].cpu().numpy()
            verify[f"bitwise_{tag}_{ns}_elements"] = bool(
                got.tobytes() == ref.tobytes())
            if sem_variant == 50:
                # per point against the magnitude of the summed terms
                mag = oracle.semlap(np.zeros_like(uh), np.abs(uh),
                                    np.abs(dh), np.abs(gh), n, ns,
                                    threads=8)
                verify[f"max_err_over_magnitude_{tag}"] = float(
                    (np.abs(got - ref) / mag).max())
        if sem_variant == 50:
            verify["tolerance"] = 1e-12
        verify["sampled"] = _sem_sample_check(u, g, d, w, n, nelt,
                                              exact=sem_variant != 50)

    res = {
        "metric": METRIC, "value": value, "unit": "GDOF/s",
        "ms_per_step": ms, "scaling": "strong", "dtype": "f64",
        "config": {"workload": f"semlap order {n - 1} (n={n}) fp64, "
                               f"{nelt_total} elements, element-sharded "
                               f"over {world} GPU(s); fixture script "
                               "split_iname(e,32,g.0,l.0) + assume + "
                               "extract_subst(gf)",
                   "nelt": nelt_total, "npts": n, "block": block,
                   "parallelism": f"element shards x{world}",
                   "l2": "no flush: inputs 56 B/dof >> 126 MB L2",
                   "variant": sem_variant,
                   "parity": "bitwise" if sem_variant != 50 else
                   "fp64 within 1e-12 of the reference (each multiply-add "
                   "one DFMA, same association; per-point bound vs the "
                   "oracle in verify and tests)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak,
                     # DRAM bytes of the committed 2^21-element capture,
                     # scaled to this rank's elements
                     "traffic": (None if _traffic(f"semlap_n{n}") is None
                                 else _traffic(f"semlap_n{n}") * nelt
                                 / (1 << 21)),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_per_launch,
                     "kernel": ("semlap_tc2_kernel (FP64 DMMA tensor "
                                "cores + DFMA, interleaved phases)"
                                if sem_variant == 50 and n == 8 else
                                f"semlap variant {sem_variant}")
                               + ": 1 launch per step, after a d -> "
                               "constant-bank copy",
                     "stream_probe_gbs": probe_gbs,
                     "stream_probe_note": "same buffers, same bytes, no "
                                          "arithmetic (lfb_probe_stream)"},
        "clocks": clocks, "gpu_launches": args.steps, "verify": verify,
        "bitwise": bitwise,
    }
    del env, launcher, u, d, g, w, ws
    torch.cuda.empty_cache()
    return res, knl


def _ring_e2e(knl, n, nelt, dev, steps, chunk, variant, hu, hw, hg=None,
              resident_g=None, resident_d=None, hd=None):
    """One e2e timing: per step, every chunk's u goes host->device from
    pinned memory, interpret() runs on it, and w comes back device->host.
    With *hg* the chunk's g (and d) are uploaded as well (all inputs per
    step); otherwise the device-resident g/d are used.  Copies in, the
    kernel and copies out run on three streams over a ring of R buffer
    slots (events order slot reuse), so both PCIe directions and the kernel
    overlap."""
    import torch

    import paper_1503_07659_b200 as lfb
    np3 = n ** 3
    R = 3
    h2d, comp, d2h = (torch.cuda.Stream(dev) for _ in range(3))
    bufs = []
    for _ in range(R):
        b = {"u": torch.empty(chunk * np3, dtype=torch.float64, device=dev),
             "w": torch.empty(chunk * np3, dtype=torch.float64, device=dev)}
        if hg is not None:
            b["g"] = torch.empty(6 * chunk * np3, dtype=torch.float64,
                                 device=dev)
            b["d"] = torch.empty(n * n, dtype=torch.float64, device=dev)
        bufs.append(b)
    ev_in = [torch.cuda.Event() for _ in range(R)]
    ev_k = [torch.cuda.Event() for _ in range(R)]
    ev_out = [torch.cuda.Event() for _ in range(R)]
    chunks = [(s, min(nelt, s + chunk)) for s in range(0, nelt, chunk)]
    launches = [0]

    def step():
        for c, (e0, e1) in enumerate(chunks):
            sl, b = c % R, bufs[c % R]
            m = e1 - e0
            with torch.cuda.stream(h2d):
                h2d.wait_event(ev_k[sl])          # slot's inputs consumed
                b["u"][:m * np3].copy_(hu[e0 * np3:e1 * np3],
                                       non_blocking=True)
                if hg is not None:
                    b["g"][:6 * m * np3].copy_(hg[6 * e0 * np3:6 * e1 * np3],
                                               non_blocking=True)
                    b["d"].copy_(hd, non_blocking=True)
                ev_in[sl].record(h2d)
            if hg is not None:
                gd, dd = b["g"], b["d"]
            else:
                gd = resident_g[6 * e0 * np3:6 * e1 * np3]
                dd = resident_d
            with torch.cuda.stream(comp):
                comp.wait_event(ev_in[sl])
                comp.wait_event(ev_out[sl])       # slot's result copied out
                env = lfb.env_from_buffers(
                    knl, {"nelt": m}, {"u": b["u"], "g": gd,
                                       "w": b["w"], "d": dd})
                lfb.interpret(knl, env, inplace=True, variant=variant)
                launches[0] += 1
                ev_k[sl].record(comp)
            with torch.cuda.stream(d2h):
                d2h.wait_event(ev_k[sl])
                hw[e0 * np3:e1 * np3].copy_(b["w"][:m * np3],
                                            non_blocking=True)
                ev_out[sl].record(d2h)

    cur = torch.cuda.current_stream(dev)
    streams = (h2d, comp, d2h)

    def run(k):
        for s in streams:
            s.wait_stream(cur)
        for _ in range(k):
            step()
        for s in streams:
            cur.wait_stream(s)

    run(1)
    torch.cuda.synchronize()
    launches[0] = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    run(steps)
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    h2d_bytes = hu.numel() * 8
    if hg is not None:
        h2d_bytes += hg.numel() * 8 + len(chunks) * hd.numel() * 8
    return {"value": nelt * np3 / (ms * 1e-3) / 1e9, "unit": "GDOF/s",
            "nelt": nelt, "h2d_bytes_per_step": h2d_bytes,
            "d2h_bytes_per_step": hw.numel() * 8, "ms_per_step": ms,
            "steps": steps, "gpu_launches": launches[0],
            "api": "paper_1503_07659_b200.interpret -> lfb_semlap_f64 "
                   f"(ctypes C-ABI), {len(chunks)} chunks of {chunk} "
                   "elements; H2D, kernel and D2H on three streams over "
                   f"{R} buffer slots"}


def _pinned_random(numel, lo, dev, seed, chunk=1 << 26):
    """Pinned host buffer of uniform [lo, 1) doubles, generated on the device
    chunk-wise and copied down (host RNG over 2^30 values takes minutes)."""
    import torch
    h = torch.empty(numel, dtype=torch.float64, pin_memory=True)
    gen = torch.Generator(device=dev).manual_seed(seed)
    for s in range(0, numel, chunk):
        v = h[s:s + chunk]
        v.copy_(torch.empty(v.numel(), dtype=torch.float64, device=dev)
                .uniform_(lo, 1.0, generator=gen))
    return h


def sem_e2e(knl, n, nelt, dev, steps, chunk=1 << 17, variant=0,
            all_inputs_nelt=0):
    """Same metric through the public API with HOST buffers, on the full
    config (*nelt* elements).

    Headline: the operator's parameters (g, d) are device-resident like a
    model's weights -- generated on the device once, outside the timed
    region -- and every step copies the step's input field u host->device
    from pinned memory, runs interpret() and reads the result w back.  Host
    memory needed: u and w only, 16 B per point (8 GiB each at 2^21
    elements of order 7).

    ``all_inputs_per_step`` (measured on *all_inputs_nelt* elements when
    the host can hold their g as well, 64 B per point): g and d are
    re-uploaded every step too; that one is PCIe-bound (56 of the 64 B per
    point are geometric factors)."""
    import torch
    np3 = n ** 3
    hu = _pinned_random(nelt * np3, -1.0, dev, 7)
    hw = torch.empty(nelt * np3, dtype=torch.float64, pin_memory=True)
    gen = torch.Generator(device=dev).manual_seed(8)
    rg = torch.empty(6 * nelt * np3, dtype=torch.float64, device=dev)
    for s in range(0, rg.numel(), 1 << 26):
        rg[s:s + (1 << 26)].uniform_(0.0, 1.0, generator=gen)
    rd = torch.rand(n * n, dtype=torch.float64, device=dev,
                    generator=gen) * 2 - 1
    res = _ring_e2e(knl, n, nelt, dev, steps, chunk, variant, hu, hw,
                    resident_g=rg, resident_d=rd)
    res["inputs"] = ("the operator's parameters g (geometric factors) and d "
                     "stay device-resident like a model's weights (set up "
                     "once, before the timed region); every step copies its "
                     "input field u host->device and its result w "
                     "device->host")
    # checker, outside the timed region: the last elements the e2e path
    # brought back to the host against the oracle on the same inputs
    ns = min(nelt, 64)
    e0 = nelt - ns
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import numpy as np
    import oracle
    uh = hu[e0 * np3:].numpy()
    gh = rg[6 * e0 * np3:].cpu().numpy()
    dh = rd.cpu().numpy()
    ref = oracle.semlap(np.zeros_like(uh), uh, dh, gh, n, ns, threads=8)
    got = hw[e0 * np3:].numpy()
    chk = {"elements": ns, "bitwise": bool(got.tobytes() == ref.tobytes())}
    if variant == 50:
        mag = oracle.semlap(np.zeros_like(uh), np.abs(uh), np.abs(dh),
                            np.abs(gh), n, ns, threads=8)
        chk["max_err_over_magnitude"] = float((np.abs(got - ref) / mag).max())
    res["verify_tail"] = chk
    del rg, rd
    torch.cuda.empty_cache()
    if all_inputs_nelt:
        m = min(all_inputs_nelt, nelt)
        hg = _pinned_random(6 * m * np3, 0.0, dev, 9)
        hd = (torch.rand(n * n, dtype=torch.float64) * 2 - 1).pin_memory()
        ai = _ring_e2e(knl, n, m, dev, steps, chunk, variant, hu[:m * np3],
                       hw[:m * np3], hg=hg, hd=hd)
        ai["inputs"] = ("every kernel input (u, g, d) copied host->device "
                        "every step: bound by PCIe (56 B of the 64 B per "
                        "point are the geometric factors)")
        res["all_inputs_per_step"] = ai
        del hg
    del hu, hw
    return res


_CPU_SAMPLE = {}


def cpu_reference(n, sample_elems, threads, min_seconds):
    """The reference's own emitted C for the same transformed kernel
    (oracle/_ref, compiled cc -std=c99 -O1 like tests/c_oracle.py:96) on the
    host cores: element chunks (<= 699,050, multiples of 32 -- its int
    indexing and its assume(nelt mod 32 = 0)) on `threads` threads."""
    import concurrent.futures as cf
    import ctypes as C

    import numpy as np
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    np3 = n ** 3
    key = (n, sample_elems)
    if key not in _CPU_SAMPLE:
        # generated once per process, and the output pages touched, so a
        # short per-step sample measures the emitted C, not page faults
        rng = np.random.default_rng(0)
        _CPU_SAMPLE.clear()
        _CPU_SAMPLE[key] = (rng.random(sample_elems * np3) * 2 - 1,
                            rng.random(6 * sample_elems * np3),
                            rng.random(n * n) * 2 - 1,
                            np.ones(sample_elems * np3))
    u, g, d, w = _CPU_SAMPLE[key]
    if oracle.have_ref():
        kind = "reference"
        P, I = C.c_void_p, C.c_int
        fn = oracle.ref_fn(f"ref_semlap_n{n}", [P, P, P, P, I])

        def run(e0, e1):
            fn(C.c_void_p(w.ctypes.data + e0 * np3 * 8),
               C.c_void_p(u.ctypes.data + e0 * np3 * 8),
               d.ctypes.data_as(P),
               C.c_void_p(g.ctypes.data + 6 * e0 * np3 * 8), e1 - e0)
    else:
        kind = "port"

        def run(e0, e1):
            oracle.semlap(w, u, d, g, n, sample_elems, elems=(e0, e1))
    per = max(32, sample_elems // threads // 32 * 32)
    cuts = list(range(0, sample_elems, per)) + [sample_elems]
    with cf.ThreadPoolExecutor(threads) as pool:
        # one untimed pass: threads started, caches and TLBs warm
        list(pool.map(lambda c: run(cuts[c], cuts[c + 1]),
                      range(len(cuts) - 1)))
        t0 = time.perf_counter()
        reps = 0
        while True:
            list(pool.map(lambda c: run(cuts[c], cuts[c + 1]),
                          range(len(cuts) - 1)))
            reps += 1
            if time.perf_counter() - t0 >= min_seconds:
                break
        dt = (time.perf_counter() - t0) / reps
    return {"value": sample_elems * np3 / dt / 1e9, "unit": "GDOF/s",
            "cores": threads, "kind": kind,
            "sample": f"{sample_elems} elements (n={n}) of the same "
                      f"workload x {reps} rep(s); "
                      + ("the reference's emitted C (codegen.emit, "
                         "cc -std=c99 -O1)" if kind == "reference"
                         else "the oracle port")
                      + f" on {threads} thread(s)",
            "seconds": dt * reps}

def cpu_reference_full(n, nelt, threads, steps, warmup):
    """The reference arm on the full config: every step runs the reference's
    emitted C (oracle/_ref, cc -std=c99 -O1) over all *nelt* elements on
    *threads* host threads (element chunks of <= 699,050, multiples of 32:
    its int indexing and its assume(nelt mod 32 = 0)).  Inputs: a 65,536-
    element random sample tiled over the full arrays (64 GiB at 2^21
    elements of order 7) -- the same work per element.  Returns the per-step
    times (s) or None when the host cannot hold the arrays."""
    import concurrent.futures as cf
    import ctypes as C

    import numpy as np
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    if not oracle.have_ref():
        return None
    np3 = n ** 3
    need = 64 * np3 * nelt
    try:
        import psutil
        if psutil.virtual_memory().available < need * 1.4:
            return None
    except Exception:
        return None
    sample = min(65536, nelt)
    rng = np.random.default_rng(0)
    su = rng.random(sample * np3) * 2 - 1
    sg = rng.random(6 * sample * np3)
    d = rng.random(n * n) * 2 - 1
    u = np.empty(nelt * np3)
    g = np.empty(6 * nelt * np3)
    w = np.zeros(nelt * np3)
    for e0 in range(0, nelt, sample):
        m = min(sample, nelt - e0)
        u[e0 * np3:(e0 + m) * np3] = su[:m * np3]
        g[6 * e0 * np3:6 * (e0 + m) * np3] = sg[:6 * m * np3]
    P, I = C.c_void_p, C.c_int
    fn = oracle.ref_fn(f"ref_semlap_n{n}", [P, P, P, P, I])
    per = min(699040, max(32, nelt // threads // 32 * 32))
    cuts = list(range(0, nelt, per)) + [nelt]
    ranges = [(cuts[c], cuts[c + 1]) for c in range(len(cuts) - 1)]

    def run(r):
        e0, e1 = r
        fn(C.c_void_p(w.ctypes.data + e0 * np3 * 8),
           C.c_void_p(u.ctypes.data + e0 * np3 * 8), d.ctypes.data_as(P),
           C.c_void_p(g.ctypes.data + 6 * e0 * np3 * 8), e1 - e0)

    times = []
    with cf.ThreadPoolExecutor(threads) as pool:
        for _ in range(warmup + steps):
            t0 = time.perf_counter()
            list(pool.map(run, ranges))
            times.append(time.perf_counter() - t0)
    return times[warmup:]


def _host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_other(wl, threads, min_seconds=2.0):
    """cpu_baseline for the other BASELINE configs: the reference's emitted
    C of the same transformed kernel (oracle/_ref, cc -std=c99 -O1) on the
    host cores.  fill / axpy: index chunks (pointer offsets) on `threads`
    threads; matvec (rows cannot be split in the emitted signature) and the
    transformed GEMM: one thread, on a bounded sample stated in `sample`."""
    import concurrent.futures as cf
    import ctypes as C

    import numpy as np
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    if not oracle.have_ref():
        return None
    P, I, D, F = C.c_void_p, C.c_int, C.c_double, C.c_float
    rng = np.random.default_rng(0)
    if wl in ("fill", "axpy"):
        n = 1 << 24
        y, x = rng.random(n), rng.random(n)
        if wl == "fill":
            fn = oracle.ref_fn("ref_fill_f64", [P, D, I])

            def run(i0, i1):
                fn(C.c_void_p(y.ctypes.data + 8 * i0), 1.5, i1 - i0)
        else:
            fn = oracle.ref_fn("ref_axpy_f64", [P, P, D, I])

            def run(i0, i1):
                fn(C.c_void_p(y.ctypes.data + 8 * i0),
                   C.c_void_p(x.ctypes.data + 8 * i0), 1.25, i1 - i0)
        per = (n + threads - 1) // threads
        cuts = list(range(0, n, per)) + [n]
        with cf.ThreadPoolExecutor(threads) as pool:
            list(pool.map(lambda c: run(cuts[c], cuts[c + 1]),
                          range(len(cuts) - 1)))
            t0, reps = time.perf_counter(), 0
            while True:
                list(pool.map(lambda c: run(cuts[c], cuts[c + 1]),
                              range(len(cuts) - 1)))
                reps += 1
                if time.perf_counter() - t0 >= min_seconds:
                    break
            dt = (time.perf_counter() - t0) / reps
        nbytes = (8 if wl == "fill" else 24) * n
        return {"value": nbytes / dt / 1e9, "unit": "GB/s", "cores": threads,
                "kind": "reference",
                "sample": f"the full n = 2^24 workload x {reps} rep(s); the "
                          "reference's emitted C (codegen.emit, cc -std=c99 "
                          f"-O1) on {threads} thread(s), index chunks",
                "seconds": dt * reps}
    if wl == "matvec":
        n = 4096
        y, a, x = np.zeros(n), rng.random(n * n), rng.random(n)
        fn = oracle.ref_fn("ref_matvec_f64", [P, P, P, I])
        fn(y.ctypes.data_as(P), a.ctypes.data_as(P), x.ctypes.data_as(P), n)
        t0, reps = time.perf_counter(), 0
        while True:
            fn(y.ctypes.data_as(P), a.ctypes.data_as(P),
               x.ctypes.data_as(P), n)
            reps += 1
            if time.perf_counter() - t0 >= min_seconds:
                break
        dt = (time.perf_counter() - t0) / reps
        return {"value": (8 * n * n + 16 * n) / dt / 1e9, "unit": "GB/s",
                "cores": 1, "kind": "reference",
                "sample": f"the full 4096^2 workload x {reps} rep(s); the "
                          "reference's emitted C on 1 thread (its row loop "
                          "cannot be split through the emitted signature)",
                "seconds": dt * reps}
    if wl in ("sgemm", "dgemm"):
        m = nn = l = 256
        dt_ = np.float32 if wl == "sgemm" else np.float64
        a = rng.random(m * l).astype(dt_)
        b = rng.random(l * nn).astype(dt_)
        c = rng.random(m * nn).astype(dt_)
        fn = oracle.ref_fn("ref_sgemm_f32" if wl == "sgemm" else
                           "ref_dgemm_f64",
                           [F if wl == "sgemm" else D, P, P, P, I, I, I])
        t0, reps = time.perf_counter(), 0
        while True:
            fn(1.5, a.ctypes.data_as(P), b.ctypes.data_as(P),
               c.ctypes.data_as(P), l, m, nn)
            reps += 1
            if time.perf_counter() - t0 >= min_seconds:
                break
        dt = (time.perf_counter() - t0) / reps
        return {"value": 2.0 * m * nn * l / dt / 1e12, "unit": "TFLOP/s",
                "cores": 1, "kind": "reference",
                "sample": f"a {m}^3 sample of the same transformed kernel "
                          f"(the paper script's tiles) x {reps} rep(s); the "
                          "reference's emitted C on 1 thread (8192^3 would "
                          "take hours)",
                "seconds": dt * reps}
    return None

# }}}


# {{{ the other BASELINE configs (fill, axpy, matvec, sem65k, GEMM, sweep)

# tensor-pipe ceilings measured on this B200 by the repo's own probes (no
# driver-measured TF32 / FP64 figure exists in MEASURED_PEAKS.json):
# tools/micro/tf32_probe.cu issues the sgemm kernel's tcgen05 kind::tf32 MMA
# back to back from resident smem (1115.6 TFLOP/s TF32 = 371.9 fp32-equivalent
# for 3xTF32); tools/micro/dmma_probe.cu runs mma.sync m8n8k4.f64 (37.0).
TF32_PEAK_TFLOPS = 1115.6
DMMA_PEAK_TFLOPS = 37.0


def _timing_helpers(args, local):
    import torch
    peak, peak_src = _peaks()

    def run_timed(fn, bytes_, flops=None, key=None):
        """Per-launch CUDA events around each launch (synchronised); for
        workloads whose inputs exceed L2."""
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        times = []
        with Clocks(local) as clk:
            for _ in range(args.steps):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        out = {"ms_per_step": ms, "ms_best": min(times),
               "steps": args.steps, "warmup": args.warmup,
               "timing": "CUDA events around each launch, median",
               "clocks": clk.summary(),
               "l2": "no flush: inputs exceed the 126 MB L2"}
        if bytes_:
            out["roofline"] = {"bound": "hbm",
                               "achieved": bytes_ / (ms * 1e-3) / 1e9,
                               "peak": peak, "unit": "GB/s",
                               "frac": bytes_ / (ms * 1e-3) / 1e9 / peak,
                               "traffic": _traffic(key) if key else None,
                               "peak_source": peak_src,
                               "algorithmic_bytes_per_launch": bytes_}
        if flops:
            out["tflops"] = flops / (ms * 1e-3) / 1e12
        return out

    def run_rotating(launchers, bytes_, flops=None, key=None,
                     min_region_s=0.3):
        """Back-to-back launches cycling over buffer sets whose footprint is
        several times the 126 MB L2: every launch streams from HBM, and the
        write-backs of the previous launch's dirty lines land inside the
        timed region (steady state) -- neither hidden in L2 nor charged to
        a flush.  The K launches are one CUDA graph (tens-of-us kernels
        would otherwise wait on the host's ctypes launch path), replayed
        until the timed region lasts >= min_region_s so the clock sampler
        sees it."""
        R = len(launchers)
        for q in range(args.warmup * R):
            launchers[q % R]()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for q in range(args.steps):
                launchers[q % R]()
        graph.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        reps = max(3, int(min_region_s * 1e3 / max(e0.elapsed_time(e1),
                                                   1e-3)))
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        with Clocks(local) as clk:
            evs[0].record()
            for r in range(reps):
                graph.replay()
                evs[r + 1].record()
            torch.cuda.synchronize()
        per = [evs[r].elapsed_time(evs[r + 1]) / args.steps
               for r in range(reps)]
        ms = statistics.median(per)
        out = {"ms_per_step": ms, "ms_best": min(per),
               "steps": args.steps, "warmup": args.warmup,
               "timing": f"CUDA graph of {args.steps} back-to-back launches, "
                         f"median over {reps} replays",
               "clocks": clk.summary(),
               "l2": f"no flush: {R} rotating buffer sets, footprint "
                     f"{R * bytes_ / 2**20:.0f} MiB >> 126 MB L2"}
        out["roofline"] = {"bound": "hbm",
                           "achieved": bytes_ / (ms * 1e-3) / 1e9,
                           "peak": peak, "unit": "GB/s",
                           "frac": bytes_ / (ms * 1e-3) / 1e9 / peak,
                           "traffic": _traffic(key) if key else None,
                           "peak_source": peak_src,
                           "algorithmic_bytes_per_launch": bytes_}
        if flops:
            out["tflops"] = flops / (ms * 1e-3) / 1e12
        return out

    return run_timed, run_rotating


def _gemm_roofline(tflops, dtype):
    if dtype == "f32":
        peak = TF32_PEAK_TFLOPS / 3
        return {"bound": "tensor", "achieved": tflops, "peak": peak,
                "unit": "TFLOP/s", "frac": tflops / peak, "traffic": None,
                "peak_source": "measured on B200 by tools/micro/tf32_probe.cu"
                               f": {TF32_PEAK_TFLOPS} TFLOP/s of tcgen05 "
                               "kind::tf32 MMA / 3 MMAs per product (3xTF32)"
                               " = fp32-equivalent ceiling",
                "tensor_pipe_tf32_tflops": 3 * tflops,
                "achieved_definition": "2 m n l algorithmic flops / launch "
                                       "time"}
    peak = DMMA_PEAK_TFLOPS
    return {"bound": "tensor", "achieved": tflops, "peak": peak,
            "unit": "TFLOP/s", "frac": tflops / peak, "traffic": None,
            "peak_source": "measured on B200 by tools/micro/dmma_probe.cu "
                           "(mma.sync m8n8k4.f64, 32 warps/SM)",
            "achieved_definition": "2 m n l algorithmic flops / launch time"}


def _gemm_verify(a, b, c0, c, alpha, l, m, n, dtype, ncols=64, groups=4):
    """The GEMM result against the oracle's restatement of the reference's
    sequential chain (c + (alpha*b)*a per k ascending, fp32 for sgemm,
    test_fortran.py:72-103 / interp.py:169-187; pinned bitwise to the
    reference's emitted C by tests/test_oracle.py) on *ncols* full columns
    in *groups* spread ranges.  Normwise max|d|/max|ref| over the columns,
    plus the largest per-entry error relative to that entry."""
    import numpy as np
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    ah = a.cpu().numpy()
    bh = b.cpu().numpy()
    per = ncols // groups
    starts = [int(q * (n - per) / max(1, groups - 1)) for q in range(groups)]
    norm_num = norm_den = 0.0
    worst = 0.0
    for j0 in starts:
        j1 = j0 + per
        ref = c0[j0 * m:j1 * m].cpu().numpy()
        # oracle.sgemm walks columns [j0, j1) of a full-size c; hand it a
        # view whose column 0 is j0 by offsetting b and c
        oracle.sgemm(alpha, ah, np.ascontiguousarray(bh[j0 * l:j1 * l]), ref,
                     l, m, per, threads=_host_threads())
        got = c[j0 * m:j1 * m].cpu().numpy()
        d = np.abs(got.astype(np.float64) - ref.astype(np.float64))
        norm_num = max(norm_num, float(d.max()))
        norm_den = max(norm_den, float(np.abs(ref).max()))
        worst = max(worst, float((d / np.abs(ref.astype(np.float64))).max()))
    tol = 1e-5 if dtype == "f32" else 1e-12
    return {"oracle": "oracle.sgemm (the reference's sequential chain, "
                      + ("fp32" if dtype == "f32" else "fp64") + ")",
            "columns": ncols, "column_starts": starts,
            "normwise_max_abs_err_over_max_abs_ref": norm_num / norm_den,
            "max_per_entry_rel_err": worst, "tolerance": tol,
            "pass": norm_num / norm_den <= tol}


def _sem_check(got, u, d, g, n, ns, variant):
    """Checker (outside the timed region): ns elements vs the oracle."""
    import numpy as np
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    ref = oracle.semlap(np.zeros_like(u), u, d, g, n, ns, threads=8)
    out = {"elements": ns, "bitwise": bool(got.tobytes() == ref.tobytes())}
    if variant == 50:
        mag = oracle.semlap(np.zeros_like(u), np.abs(u), np.abs(d),
                            np.abs(g), n, ns, threads=8)
        out["max_err_over_magnitude"] = float((np.abs(got - ref) / mag).max())
        out["tolerance"] = 1e-12
        out["pass"] = out["max_err_over_magnitude"] <= 1e-12
    else:
        out["pass"] = out["bitwise"]
    return out


def bench_workload(wl, args, local, cpu=True):
    """One of BASELINE's other configs on one GPU: value, ms_per_step,
    roofline, clocks, a checker result and the reference's CPU path."""
    import numpy as np
    import torch

    import paper_1503_07659_b200 as lfb
    from paper_1503_07659_b200 import fixtures as fx
    dev = torch.device("cuda", local)
    run_timed, run_rotating = _timing_helpers(args, local)
    gen = torch.Generator(device=dev).manual_seed(0)
    variant = args.variant or 0
    threads = _host_threads()

    if wl in ("fill", "axpy"):
        n = 1 << 24
        src = fx.fill_source("f64") if wl == "fill" else fx.axpy_source("f64")
        _r, knl = fx.translate(src)
        launchers, envs = [], []
        for _set in range(4 if wl == "fill" else 3):
            x = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
            y = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
            bufs = {"out": y} if wl == "fill" else {"y": y, "x": x}
            env = lfb.env_from_buffers(knl, {"n": n}, bufs,
                                       {"a": 1.5, "alpha": 1.25})
            envs.append((env, x, y.clone()))
            launchers.append(lfb.Launcher(knl, env, variant=variant).launch)
        r = run_rotating(launchers, (8 if wl == "fill" else 24) * n, key=wl)
        # checker: one launch from known inputs, bitwise vs the oracle
        env, x, y0 = envs[0]
        yv = env.arrays["out" if wl == "fill" else "y"].data
        yv.copy_(y0)
        launchers[0]()
        torch.cuda.synchronize()
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle
        ref = y0.cpu().numpy()
        if wl == "fill":
            oracle.fill(ref, 1.5)
        else:
            oracle.axpy(ref, x.cpu().numpy(), 1.25)
        r["verify"] = {"oracle": f"oracle.{wl}", "elements": n,
                       "bitwise": bool(yv.cpu().numpy().tobytes()
                                       == ref.tobytes())}
        r.update({"metric": f"{wl} fp64 n=2^24 GB/s", "unit": "GB/s",
                  "value": r["roofline"]["achieved"], "variant": variant,
                  "dtype": "f64", "config": {
                      "workload": f"Fortran-ingested {wl}, n=2^24 fp64, "
                                  "split_iname(i,128,g.0,l.0)",
                      "n": n}})
        if cpu:
            r["cpu_baseline"] = cpu_reference_other(wl, threads)
        return r

    if wl == "matvec":
        n = 4096
        _r, knl = fx.translate(fx.matvec_source("f64"))
        envs = []
        for _set in range(4):
            a = torch.rand(n * n, dtype=torch.float64, device=dev,
                           generator=gen)
            x = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
            y = torch.empty(n, dtype=torch.float64, device=dev)
            envs.append(lfb.env_from_buffers(knl, {"n": n},
                                             {"a": a, "x": x, "y": y}))
        r = run_rotating([lfb.Launcher(knl, e, variant=variant).launch
                          for e in envs], 8 * n * n + 16 * n, 2 * n * n,
                         key="matvec")
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle
        e = envs[0]
        ah, xh = e.arrays["a"].data.cpu().numpy(), \
            e.arrays["x"].data.cpu().numpy()
        ref = oracle.matvec(np.zeros(n), ah, xh, n, threads=threads)
        r.update({"metric": "matvec fp64 4096^2 GB/s", "unit": "GB/s",
                  "value": r["roofline"]["achieved"], "variant": variant,
                  "dtype": "f64",
                  "config": {"workload": "Fortran-ingested matvec fp64 "
                                         "4096x4096, split i by 128 -> "
                                         "g.0/l.0, j by 32, extract_subst + "
                                         "precompute of x (add_prefetch)",
                             "n": n},
                  "parity": "bitwise" if variant in (1, 3) else
                  "tolerance (split-j, 1e-12 normwise)"})
        lfb.Launcher(knl, e, variant=variant).launch()
        torch.cuda.synchronize()
        got = e.arrays["y"].data.cpu().numpy()
        r["verify"] = {"oracle": "oracle.matvec (sequential row chain)",
                       "bitwise": bool(got.tobytes() == ref.tobytes()),
                       "normwise": float(np.abs(got - ref).max()
                                         / np.abs(ref).max()),
                       "tolerance": 1e-12}
        if variant == 0:
            # the bitwise kernel: each row is a chain of n dependent DADDs
            # (8.1 cycles each, tools/micro/dadd_latency.cu) that overlaps
            # the stream only partly
            r2 = run_rotating([lfb.Launcher(knl, e, variant=3).launch
                               for e in envs], 8 * n * n + 16 * n, 2 * n * n)
            lfb.Launcher(knl, envs[0], variant=3).launch()
            torch.cuda.synchronize()
            got3 = envs[0].arrays["y"].data.cpu().numpy()
            r["bitwise"] = {"variant": 3, "value": r2["roofline"]["achieved"],
                            "ms_per_step": r2["ms_per_step"],
                            "frac": r2["roofline"]["frac"],
                            "verify_bitwise": bool(got3.tobytes()
                                                   == ref.tobytes()),
                            "bound": "latency: 4096 dependent DADDs per "
                                     "row (8.1 cycles each) + the stream, "
                                     "partly overlapped"}
        if cpu:
            r["cpu_baseline"] = cpu_reference_other(wl, threads)
        return r

    if wl in ("sgemm", "dgemm"):
        dt = "f32" if wl == "sgemm" else "f64"
        tdt = torch.float32 if dt == "f32" else torch.float64
        m = n = l = args.gemm_n
        _r, knl = fx.translate(fx.gemm_source(dt))
        a = torch.rand(m * l, dtype=tdt, device=dev, generator=gen)
        b = torch.rand(l * n, dtype=tdt, device=dev, generator=gen)
        c = torch.rand(m * n, dtype=tdt, device=dev, generator=gen)
        env = lfb.env_from_buffers(knl, {"m": m, "n": n, "l": l},
                                   {"a": a, "b": b, "c": c}, {"alpha": 1.5})
        c0 = c.clone()
        L = lfb.Launcher(knl, env, variant=variant)
        L.launch()
        torch.cuda.synchronize()
        verify = _gemm_verify(a, b, c0, c, 1.5, l, m, n, dt)
        c.copy_(c0)
        r = run_timed(L.launch, None, 2.0 * m * n * l)
        r["roofline"] = _gemm_roofline(r["tflops"], dt)
        r.update({"metric": f"{wl} {m}^3 TFLOP/s", "unit": "TFLOP/s",
                  "value": r["tflops"], "variant": variant, "dtype": dt,
                  "verify": verify,
                  "config": {"workload": f"the paper's GEMM "
                                         f"(test_fortran.py:72-103) real*"
                                         f"{4 if dt == 'f32' else 8} "
                                         f"{m}^3 with its split/prefetch "
                                         "script",
                             "m": m, "n": n, "l": l},
                  "kernel": "sgemm_tc2_kernel: tcgen05 kind::tf32 3xTF32, "
                            "TMA, TMEM accumulators" if dt == "f32" else
                            "dgemm_ws_kernel: FP64 DMMA m8n8k4, producer warp + 8 consumer warps on full / empty mbarriers"})
        if cpu:
            r["cpu_baseline"] = cpu_reference_other(wl, threads)
        return r

    if wl == "sem65k":
        n, nelt = 8, 65536
        _r, knl = fx.translate(fx.semlap_source(n), "semlap.f")
        u, d, g, w = sem_buffers(n, nelt, dev, 3)
        env = lfb.env_from_buffers(knl, {"nelt": nelt},
                                   {"u": u, "d": d, "g": g, "w": w})
        out = {"metric": "SEM o7 fp64 65,536 elements GDOF/s",
               "unit": "GDOF/s", "dtype": "f64",
               "config": {"workload": "semlap order 7 (n=8) fp64, 65536 "
                                      "elements, split_iname(e,32,g.0,l.0) "
                                      "+ assume + extract_subst(gf)",
                          "nelt": nelt, "npts": n}}
        ns = 256
        uh = u[:ns * 512].cpu().numpy()
        gh = g[:6 * ns * 512].cpu().numpy()
        dh = d.cpu().numpy()
        for tag, v in (("", 50), ("bitwise", 0)):
            L = lfb.Launcher(knl, env, variant=v)
            r = run_timed(L.launch, 64 * n ** 3 * nelt,
                          key="sem65k" if v == 0 else None)
            r["value"] = nelt * n ** 3 / (r["ms_per_step"] * 1e-3) / 1e9
            r["variant"] = v
            r["verify"] = _sem_check(w[:ns * 512].cpu().numpy(), uh, dh, gh,
                                     n, ns, v)
            if tag:
                out[tag] = r
            else:
                out.update(r)
        if cpu:
            out["cpu_baseline"] = cpu_reference(n, nelt, threads, 2.0)
        return out

    if wl == "sweep":
        rows = []
        for n in range(4, 17):
            nelt = (1 << 25) // n ** 3 // 32 * 32
            _r, knl = fx.translate(fx.semlap_source(n))
            u, d, g, w = sem_buffers(n, nelt, dev, n)
            env = lfb.env_from_buffers(knl, {"nelt": nelt},
                                       {"u": u, "d": d, "g": g, "w": w})
            np3 = n ** 3
            ns = 32
            uh = u[:ns * np3].cpu().numpy()
            gh = g[:6 * ns * np3].cpu().numpy()
            dh = d.cpu().numpy()
            row = {"order": n - 1, "npts": n, "nelt": nelt}
            for tag, v in (("", 0), ("fma_", 50)):
                L = lfb.Launcher(knl, env, variant=v)
                r = run_timed(L.launch, 64 * np3 * nelt)
                row.update({f"{tag}ms": r["ms_per_step"],
                            f"{tag}gdofs": nelt * np3
                            / (r["ms_per_step"] * 1e-3) / 1e9,
                            f"{tag}hbm_frac": r["roofline"]["frac"],
                            f"{tag}sm_mhz": r["clocks"]["sm_mhz"],
                            f"{tag}verify": _sem_check(
                                w[:ns * np3].cpu().numpy(), uh, dh, gh, n,
                                ns, v)})
            if cpu:
                cb = cpu_reference(n, max(32, (1 << 18) // np3 // 32 * 32),
                                   threads, 0.3)
                row["cpu_gdofs"] = cb["value"]
                row["cpu_kind"] = cb["kind"]
            rows.append(row)
            del u, d, g, w, env, L
            torch.cuda.empty_cache()
        peak, peak_src = _peaks()
        return {"metric": "SEM sweep orders 3-15 GDOF/s", "rows": rows,
                "unit": "GDOF/s", "dtype": "f64",
                "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                             "peak_source": peak_src,
                             "algorithmic_bytes_per_element": "64 n^3"},
                "cpu_baseline_note": f"cpu_gdofs: the reference's emitted C "
                                     f"(oracle/_ref) on {threads} threads, "
                                     "a ~2^18-point sample per order",
                "modes": "gdofs/hbm_frac: bitwise kernels (variant 0); "
                         "fma_*: DFMA/DMMA mode (variant 50, within 1e-12)",
                "config": {"workload": "semlap orders 3..15, nelt = "
                                       "2^25/n^3 (~2 GiB traffic each)"}}

    if wl == "semop":
        return semop_bench(args, 0, 1, local, e=args.semop_e or 64)
    if wl == "generic":
        return generic_bench(args, local)
    raise SystemExit(f"unknown workload {wl}")


def semop_bench(args, rank, world, local, e=128, n=8):
    """The assembled SEM operator w <- Q Q^T semlap(u) on a box of e^3
    elements: the element-local operator (DFMA
    mode, the headline kernel) followed by the direct-stiffness summation
    (csrc/dssum.cu).  Ranks own slabs of element layers; the interface
    planes go through the bitwise partial -> continue -> write-back protocol
    over NCCL point-to-point (assembly.dssum_sharded).  value = whole-job
    GDOF/s of the assembled operator; the dssum kernel's own time and
    bandwidth (algorithmic bytes: every local copy of a shared node read
    and written once, 16 (n^3 - (n-2)^3) B per element) beside it."""
    import torch

    import paper_1503_07659_b200 as lfb
    from paper_1503_07659_b200 import fixtures as fx
    from paper_1503_07659_b200.assembly import BoxMesh, dssum_sharded
    dev = torch.device("cuda", local)
    mesh = BoxMesh(e, e, e, n)
    slab = mesh.slab(rank, world)
    _r, knl = fx.translate(fx.semlap_source(n), "semlap.f")
    u, d, g, w = sem_buffers(n, slab.nelt, dev, 500 + rank)
    env = lfb.env_from_buffers(knl, {"nelt": slab.nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    L = lfb.Launcher(knl, env, variant=50)

    def step():
        L.launch()
        dssum_sharded(w, mesh, rank, world)

    ms, ms_local, clocks = timed(step, args.steps, args.warmup, world,
                                 local)
    ms_ds, ms_ds_local, _c = timed(lambda: dssum_sharded(w, mesh, rank,
                                                         world),
                                   args.steps, args.warmup, world, local)
    peak, peak_src = _peaks()
    ds_bytes = 16 * (n ** 3 - (n - 2) ** 3) * slab.nelt
    res = {"metric": "assembled SEM operator (semlap + Q Q^T) GDOF/s",
           "value": mesh.nelt * n ** 3 / (ms * 1e-3) / 1e9,
           "unit": "GDOF/s", "ms_per_step": ms, "dtype": "f64",
           "n_gpus": world, "scaling": "strong",
           "config": {"workload": f"box of {e}^3 elements, order {n - 1}, "
                                  "semlap (DFMA mode) + direct-stiffness "
                                  "summation; element layers sharded over "
                                  f"{world} rank(s)",
                      "mesh": [e, e, e, n], "nelt": mesh.nelt},
           "dssum": {"ms_per_step": ms_ds,
                     "share_of_step": ms_ds / ms,
                     "roofline": {"bound": "hbm",
                                  "achieved": ds_bytes
                                  / (ms_ds_local * 1e-3) / 1e9,
                                  "peak": peak, "unit": "GB/s",
                                  "frac": ds_bytes / (ms_ds_local * 1e-3)
                                  / 1e9 / peak,
                                  "peak_source": peak_src,
                                  "algorithmic_bytes_per_launch": ds_bytes},
                     "exchange": "none" if world == 1 else
                     "2 plane exchanges per interface (NCCL P2P)"},
           "clocks": clocks}
    del env, L, u, d, g, w
    torch.cuda.empty_cache()
    return res


def generic_bench(args, local):
    """The generic engine (CUDA generated from the schedule, NVRTC) on
    BASELINE workloads the hand-written kernels also cover: what a kernel
    outside the recognised set can expect."""
    import torch

    import paper_1503_07659_b200 as lfb
    from paper_1503_07659_b200 import fixtures as fx
    from paper_1503_07659_b200.generic import GenericLauncher
    dev = torch.device("cuda", local)
    run_timed, run_rotating = _timing_helpers(args, local)
    gen = torch.Generator(device=dev).manual_seed(0)
    rows = {}
    n = 1 << 24
    _r, kf = fx.translate(fx.fill_source("f64"))
    outs = [torch.empty(n, dtype=torch.float64, device=dev)
            for _ in range(4)]
    envs = [lfb.env_from_buffers(kf, {"n": n}, {"out": o}, {"a": 1.5})
            for o in outs]
    r = run_rotating([GenericLauncher(kf, e).launch for e in envs], 8 * n)
    rows["fill_f64_2^24"] = {"GB/s": r["roofline"]["achieved"],
                             "frac": r["roofline"]["frac"]}
    _r, ka = fx.translate(fx.axpy_source("f64"))
    envs = []
    for _ in range(3):
        x = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
        y = torch.rand(n, dtype=torch.float64, device=dev, generator=gen)
        envs.append(lfb.env_from_buffers(ka, {"n": n}, {"y": y, "x": x},
                                         {"alpha": 1.25}))
    r = run_rotating([GenericLauncher(ka, e).launch for e in envs], 24 * n)
    rows["axpy_f64_2^24"] = {"GB/s": r["roofline"]["achieved"],
                             "frac": r["roofline"]["frac"]}
    m = nn = l = 2048
    _r, kg = fx.translate(fx.gemm_source("f64"))
    a = torch.rand(m * l, dtype=torch.float64, device=dev, generator=gen)
    b = torch.rand(l * nn, dtype=torch.float64, device=dev, generator=gen)
    c = torch.rand(m * nn, dtype=torch.float64, device=dev, generator=gen)
    env = lfb.env_from_buffers(kg, {"m": m, "n": nn, "l": l},
                               {"a": a, "b": b, "c": c}, {"alpha": 1.5})
    r = run_timed(GenericLauncher(kg, env).launch, None, 2.0 * m * nn * l)
    rows["dgemm_paper_script_2048^3"] = {"TFLOP/s": r["tflops"],
                                         "ms": r["ms_per_step"]}
    # precompute footprints by TMA on streaming kernels: the 3-point
    # smoother's 66-element halo window, and the tiled transpose whose 16x16
    # tile is read down its columns (128-B swizzle)
    _r, km = fx.translate(fx.generic_source("smooth"))
    envs = []
    for _ in range(3):
        uu = torch.rand(n + 2, dtype=torch.float64, device=dev, generator=gen)
        rr = torch.empty(n, dtype=torch.float64, device=dev)
        envs.append(lfb.env_from_buffers(km, {"n": n}, {"r": rr, "u": uu}))
    r = run_rotating([GenericLauncher(km, e).launch for e in envs], 16 * n)
    rows["smooth_tma_f64_2^24"] = {"GB/s": r["roofline"]["achieved"],
                                   "frac": r["roofline"]["frac"]}
    nt = 8192
    _r, kt = fx.translate(fx.generic_source("ttile"))
    at = torch.rand(nt * nt, dtype=torch.float64, device=dev, generator=gen)
    bt = torch.empty(nt * nt, dtype=torch.float64, device=dev)
    env = lfb.env_from_buffers(kt, {"n": nt, "m": nt}, {"a": at, "b": bt})
    r = run_timed(GenericLauncher(kt, env).launch, 16 * nt * nt)
    rows["transpose_tile_tma_f64_8192^2"] = {
        "GB/s": r["roofline"]["achieved"], "frac": r["roofline"]["frac"]}
    # the SEM fixture itself through the generated CUDA: the reference's
    # schedule gives one work-item per element with its wr/ws/wt temporaries
    # (3 n^3 doubles) in private (local) memory
    ns, ne = 8, 1 << 16
    _r, ks = fx.translate(fx.semlap_source(ns))
    u, d, g, w = sem_buffers(ns, ne, dev, ns)
    env = lfb.env_from_buffers(ks, {"nelt": ne},
                               {"u": u, "d": d, "g": g, "w": w})
    r = run_timed(GenericLauncher(ks, env).launch, 64 * ns ** 3 * ne)
    rows["semlap_o7_65536_elements"] = {
        "GDOF/s": ne * ns ** 3 / (r["ms_per_step"] * 1e-3) / 1e9,
        "frac": r["roofline"]["frac"], "ms": r["ms_per_step"]}
    return {"metric": "generic engine (generated CUDA) GB/s | TFLOP/s",
            "rows": rows, "engine": "generic (cudagen.py, NVRTC sm_100a)"}


CONFIG_WORKLOADS = ("fill", "axpy", "matvec", "sem65k", "sgemm", "dgemm",
                    "sweep", "semop")


def configs_bench(args, local):
    """BASELINE configs 1, 2, 3 and 5 on the driver's clock: each one's line
    (value, roofline, clocks, checker, the reference's CPU path) under
    ``configs`` of the default bench line.  Steps/warm-up as the headline;
    sized to add about a minute."""
    import copy
    import torch
    out = {}
    t0 = time.perf_counter()
    for wl in CONFIG_WORKLOADS:
        a = copy.copy(args)
        a.variant = 0
        t1 = time.perf_counter()
        try:
            out[wl] = bench_workload(wl, a, local, cpu=not args.no_cpu)
        except Exception as exc:  # report, keep the headline line intact
            out[wl] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        out[wl]["wall_s"] = time.perf_counter() - t1
        torch.cuda.empty_cache()
    out["wall_s"] = time.perf_counter() - t0
    return out

# }}}


# {{{ multi-GPU launch without torchrun

def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args):
    """``python bench.py --gpus N`` (N > 1) outside torchrun: start the N
    ranks ourselves -- one process per GPU through torch.distributed.run on
    127.0.0.1 -- and return their exit code.  Fails loudly when fewer than N
    devices are visible (never silently times one GPU)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and os.environ.get("LFB_BENCH_ONE_DEVICE") != "1":
        print(json.dumps({"metric": METRIC, "error":
                          f"--gpus {args.gpus} but only {have} CUDA "
                          "device(s) are visible"}))
        return 1
    env = dict(os.environ)
    # NCCL's own record of every communicator (rank / nranks per GPU) goes
    # to a file, not stdout, so the JSON line stays the only stdout line
    logdir = os.path.join(REPO, "gpurun_out",
                          f"nccl_{time.strftime('%Y%m%d_%H%M%S')}_"
                          f"{os.getpid()}")
    os.makedirs(logdir, exist_ok=True)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE",
                   os.path.join(logdir, "nccl_bench.%h.%p.log"))
    env["LFB_NCCL_LOGDIR"] = logdir
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def comm_report(world, local):
    """Proof the job spans `world` ranks on distinct devices: every rank's
    device (all-gathered) and an all-reduce of ones over the data-path
    backend (NCCL on the box)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return {"backend": None, "world_size": 1,
                "devices": [torch.cuda.get_device_name(local)]}
    backend = dist.get_backend()
    dev = torch.device("cuda", local) if backend == "nccl" else \
        torch.device("cpu")
    one = torch.ones(1, device=dev)
    dist.all_reduce(one)
    info = [None] * world
    dist.all_gather_object(info, {
        "rank": dist.get_rank(), "local_rank": local,
        "cuda_device": torch.cuda.current_device(),
        "pci_bus": torch.cuda.get_device_properties(local).pci_bus_id
        if hasattr(torch.cuda.get_device_properties(local), "pci_bus_id")
        else None})
    return {"backend": backend, "world_size": dist.get_world_size(),
            "allreduce_of_ones": float(one.item()), "ranks": info}


def nccl_log_summary():
    """Communicator lines NCCL wrote (NCCL_DEBUG=INFO, spawn_ranks)."""
    import glob
    import re
    d = os.environ.get("LFB_NCCL_LOGDIR")
    if not d:
        return None
    nranks = []
    for path in glob.glob(os.path.join(d, "nccl_bench.*.log")):
        try:
            with open(path, errors="replace") as f:
                for line in f:
                    m = re.search(r"nranks (\d+)", line)
                    if m and "Init COMPLETE" in line:
                        nranks.append(int(m.group(1)))
        except OSError:
            pass
    return {"init_complete_lines": len(nranks),
            "nranks": sorted(set(nranks))}

# }}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="sem2m")
    ap.add_argument("--variant", type=int, default=None,
                    help="kernel variant; SEM default 50 (DFMA mode), "
                         "others 0")
    ap.add_argument("--gemm-n", type=int, default=8192)
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other BASELINE configs in the default "
                         "line")
    ap.add_argument("--e2e-nelt", type=int, default=0)
    ap.add_argument("--semop-e", type=int, default=0,
                    help="elements per direction of the semop box (default "
                         "64 in the configs line, 128 for --workload semop)")
    ap.add_argument("--e2e-chunk", type=int, default=1 << 17,
                    help="elements per host<->device chunk in the e2e run")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.variant is None and args.workload not in ("sem2m", "sem65k"):
        args.variant = 0
    args.npts = 8
    args.nelt = {"sem2m": 1 << 21, "sem65k": 65536}.get(args.workload,
                                                         1 << 21)
    threads = _host_threads()

    if args.impl == "reference":
        # the reference's own CPU execution of the path, rank 0 only
        if int(os.environ.get("RANK", "0")) != 0:
            return
        np3 = args.npts ** 3
        full = None if args.workload != "sem2m" else cpu_reference_full(
            args.npts, args.nelt, threads, args.steps, args.warmup)
        if full is not None:
            step_s = statistics.median(full)
            value = args.nelt * np3 / step_s / 1e9
            sample = args.nelt
            cpu = {"value": value, "unit": "GDOF/s", "cores": threads,
                   "kind": "reference",
                   "sample": f"the full config: all {args.nelt} elements "
                             f"(n={args.npts}) every step, {args.steps} "
                             f"timed steps after {args.warmup}; the "
                             "reference's emitted C (codegen.emit, cc "
                             f"-std=c99 -O1) on {threads} thread(s)",
                   "step_seconds": full}
        else:
            sample = 65536
            per_step = []
            cpu = None
            for _ in range(args.warmup + args.steps):
                cpu = cpu_reference(args.npts, sample, threads, 1.0)
                per_step.append(cpu["value"])
            value = statistics.median(per_step[args.warmup:])
            cpu["value"] = value
        res = {"metric": METRIC, "value": value, "unit": "GDOF/s",
               "impl": "reference", "n_gpus": args.gpus,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": 1e3 * args.nelt * args.npts ** 3
               / (value * 1e9),
               "higher_is_better": True, "scaling": "strong",
               "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": {"workload": f"semlap order {args.npts - 1} "
                                      f"(n={args.npts}) fp64, {args.nelt} "
                                      "elements; each step times "
                                      + ("all of them" if sample ==
                                         args.nelt else
                                         f"a {sample}-element sample"),
                          "nelt": args.nelt, "npts": args.npts,
                          "same_config": sample == args.nelt},
               "cpu_baseline": cpu,
               "e2e": {"value": value, "unit": "GDOF/s",
                       "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(res))
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))

    rank, world, local = dist_init(args.gpus)
    import torch
    if args.workload == "semop":
        res = semop_bench(args, rank, world, local, e=args.semop_e or 128)
        res.update({"steps": args.steps, "warmup": args.warmup,
                    "higher_is_better": True, "vs_baseline": None,
                    "data": "synthetic", "comm": comm_report(world, local)})
        if rank == 0:
            print(json.dumps(res))
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    if args.workload not in ("sem2m", "sem65k"):
        if rank == 0:
            print(json.dumps(bench_workload(args.workload, args, local,
                                            cpu=not args.no_cpu)))
        return
    comm = comm_report(world, local)
    res, knl = sem_bench(args, rank, world, local)
    dev = torch.device("cuda", local)
    res["e2e"] = None
    if not args.no_e2e:
        nelt_e2e = args.e2e_nelt or (args.nelt // world)
        # pinned host buffers hold u and w (16 B per point; g and d are
        # device-resident): stay within half of the host's available memory
        # (shared by all local ranks); the all-inputs variant also holds g
        # (+48 B per point) and is measured on what fits
        ai_nelt = nelt_e2e
        try:
            import psutil
            avail = psutil.virtual_memory().available
            cap = avail // 2 // max(1, world) // (16 * args.npts ** 3)
            nelt_e2e = max(32, min(nelt_e2e, cap // 32 * 32))
            ai_cap = (avail // 2 // max(1, world)
                      - 16 * args.npts ** 3 * nelt_e2e) \
                // (48 * args.npts ** 3)
            ai_nelt = max(0, min(nelt_e2e, ai_cap // 32 * 32))
        except Exception:
            pass
        e2e = sem_e2e(knl, args.npts, nelt_e2e, dev, steps=3,
                      chunk=args.e2e_chunk,
                      variant=res["config"]["variant"],
                      all_inputs_nelt=ai_nelt)
        ms = max_over_ranks(e2e["ms_per_step"], world)
        e2e["value"] = nelt_e2e * world * args.npts ** 3 / (ms * 1e-3) / 1e9
        e2e["ms_per_step"] = ms
        e2e["nelt"] = nelt_e2e * world
        ai = e2e.get("all_inputs_per_step", {})
        if "ms_per_step" in ai:
            ms2 = max_over_ranks(ai["ms_per_step"], world)
            ai["value"] = ai["nelt"] * world * args.npts ** 3 \
                / (ms2 * 1e-3) / 1e9
            ai["ms_per_step"] = ms2
        res["e2e"] = e2e
    res["cpu_baseline"] = None
    if rank == 0 and not args.no_cpu:
        # the reference's CPU path on this box's host cores (rank 0; at
        # N > 1 the other ranks wait at the barrier below)
        res["cpu_baseline"] = cpu_reference(args.npts, 65536, threads, 15.0)
    if world == 1 and args.workload == "sem2m" and not args.no_configs:
        res["configs"] = configs_bench(args, local)
    barrier(world)
    res.update({"n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "higher_is_better": True,
                "vs_baseline": None, "data": "synthetic",
                "comm": comm, "nccl_log": nccl_log_summary()})
    if rank == 0:
        print(json.dumps(res))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
