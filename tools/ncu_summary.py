"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py <report.ncu-rep> <key> [--round r01]
        -> profiles/<round>_<key>.md  (key metrics, stall mix, top SASS)
        -> profiles/ncu_summary.json[key] (dram bytes per launch, duration)
    python tools/ncu_summary.py --launches <launches.csv> <key> [--round r01]
        -> profiles/<round>_<key>_launches.md (per-kernel share of the step)
"""

from __future__ import annotations

import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum",
]


def _csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep):
    rows = _csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        m = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
        out.append(m)
    return out


def _num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def _bytes(val, unit):
    x = _num(val)
    if x is None:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "Tbyte": 1e12}.get(unit, 1)
    return x * scale


def source_hot(rep, top=15):
    rows = _csv(["-i", rep, "--page", "source", "--csv", "--print-source",
                 "sass"])
    start = 2 if rows and rows[0] and rows[0][0].startswith("Kernel") else 1
    hdr = rows[start - 1]
    try:
        ia = hdr.index("Source")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        ie = hdr.index("Instructions Executed")
    except ValueError:
        return [], []
    data = []
    for r in rows[start:]:
        if len(r) > max(ia, ss, ie):
            data.append((int(_num(r[ss]) or 0), int(_num(r[ie]) or 0),
                         r[ia].strip()))
    tot = sum(d[0] for d in data) or 1
    byop = collections.Counter()
    for s, _n, src in data:
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else "?"
        byop[op] += s
    ops = [(op, 100.0 * s / tot) for op, s in byop.most_common(12)]
    hot = [(100.0 * s / tot, src) for s, _n, src in
           sorted(data, reverse=True)[:top]]
    return ops, hot


def summarise(rep, key, rnd):
    ms = raw_metrics(rep)
    lines = [f"# {rnd} ncu --set full: {key}", "",
             f"report: `{os.path.basename(rep)}` (gpurun_out, not committed)",
             ""]
    summary = {}
    for idx, m in enumerate(ms):
        name = m.get("Kernel Name", ("?", ""))[0]
        lines.append(f"## launch {idx}: `{name[:160]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            if k in m:
                lines.append(f"| {k} | {m[k][0]} | {m[k][1]} |")
        stalls = sorted(((h, _num(v[0]) or 0) for h, v in m.items()
                         if h.startswith("smsp__average_warps_issue_stalled")
                         and h.endswith("per_issue_active.ratio")),
                        key=lambda x: -x[1])
        lines.append("")
        lines.append("stall reasons (warps per issue-active cycle):")
        lines.append("")
        for h, v in stalls[:10]:
            if v > 0.01:
                nm = h.replace("smsp__average_warps_issue_stalled_", "") \
                    .replace("_per_issue_active.ratio", "")
                lines.append(f"- {nm}: {v:.3f}")
        lines.append("")
        rd = _bytes(*m.get("dram__bytes_read.sum", ("", "")))
        wr = _bytes(*m.get("dram__bytes_write.sum", ("", "")))
        dv, du = m.get("gpu__time_duration.sum", ("", ""))
        dur = _num(dv)
        if dur is not None:
            dur *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                    "msecond": 1e3, "s": 1e6, "second": 1e6}.get(
                        du.strip(), 1.0)
        if idx == 0:
            summary = {"dram_bytes_per_launch": (rd or 0) + (wr or 0),
                       "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "duration_us_under_ncu": dur, "kernel": name,
                       "report": os.path.basename(rep), "round": rnd}
    ops, hot = source_hot(rep)
    if ops:
        lines.append("stall samples by SASS opcode (launch 0):")
        lines.append("")
        for op, pct in ops:
            lines.append(f"- {op}: {pct:.1f}%")
        lines.append("")
        lines.append("hottest SASS lines:")
        lines.append("")
        lines.append("```")
        for pct, src in hot:
            lines.append(f"{pct:5.1f}%  {src}")
        lines.append("```")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"{rnd}_{key}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    path = os.path.join(PROF, "ncu_summary.json")
    allsum = json.load(open(path)) if os.path.exists(path) else {}
    allsum[key] = summary
    with open(path, "w") as f:
        json.dump(allsum, f, indent=1, sort_keys=True)
    return summary


def launches(csv_path, key, rnd):
    rows = list(csv.reader(open(csv_path)))
    # skip ncu's preamble lines
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, im, iv, iu = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        v = _num(r[iv])
        if v is None:
            continue
        if r[iu] in ("msecond", "ms"):
            v *= 1e3
        elif r[iu] in ("nsecond", "ns"):
            v *= 1e-3
        per[r[ik]][r[im]].append(v)
    tot = sum(sum(m.get("gpu__time_duration.sum", [])) for m in per.values())
    lines = [f"# {rnd} launch list: {key}", "",
             "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum --clock-control none` over the bench "
             "command (cold-cache, serialised: compare shares, not absolute "
             "times)", "",
             "| kernel | launches | total us | share | mean us |",
             "|---|---|---|---|---|"]
    for k, m in sorted(per.items(),
                       key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum",
                                                     []))):
        t = m.get("gpu__time_duration.sum", [])
        if not t:
            continue
        lines.append(f"| `{k[:90]}` | {len(t)} | {sum(t):.1f} | "
                     f"{100 * sum(t) / tot:.1f}% | {sum(t) / len(t):.1f} |")
    with open(os.path.join(PROF, f"{rnd}_{key}_launches.md"), "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    args = sys.argv[1:]
    rnd = "r01"
    if "--round" in args:
        i = args.index("--round")
        rnd = args[i + 1]
        del args[i:i + 2]
    if args[0] == "--launches":
        launches(args[1], args[2], rnd)
    else:
        print(json.dumps(summarise(args[0], args[1], rnd), indent=1))
