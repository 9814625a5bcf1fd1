"""Experiment: back-to-back vs isolated SEM launches, with/without the
nvidia-smi sampler (is the 2M-element gap power/clock or measurement?)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1503_07659_b200 as lfb
from paper_1503_07659_b200 import fixtures as fx
n, nelt = 8, 1 << 21
dev = torch.device("cuda", 0)
_r, knl = fx.translate(fx.semlap_source(n))
u, d, g, w = bench.sem_buffers(n, nelt, dev, 1)
env = lfb.env_from_buffers(knl, {"nelt": nelt}, {"u": u, "d": d, "g": g, "w": w})
L = lfb.Launcher(knl, env, variant=int(os.environ.get("V", "0")))
for _ in range(3): L.launch()
torch.cuda.synchronize()
def ev(): return torch.cuda.Event(enable_timing=True)
res = {}
# isolated launches with idle gaps
iso = []
for gap in (0.0, 0.05, 0.2):
    ts = []
    for _ in range(5):
        time.sleep(gap); a, b = ev(), ev(); a.record(); L.launch(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    res[f"isolated_gap{gap}"] = ts
# back to back, no sampler
a, b = ev(), ev(); a.record()
for _ in range(10): L.launch()
b.record(); torch.cuda.synchronize(); res["b2b10"] = a.elapsed_time(b) / 10
a, b = ev(), ev(); a.record()
for _ in range(40): L.launch()
b.record(); torch.cuda.synchronize(); res["b2b40"] = a.elapsed_time(b) / 40
# per-launch events in a back-to-back chain
evs = [ev() for _ in range(21)]
evs[0].record()
for k in range(20):
    L.launch(); evs[k + 1].record()
torch.cuda.synchronize()
res["chain"] = [round(evs[k].elapsed_time(evs[k + 1]), 3) for k in range(20)]
with bench.Clocks(0) as clk:
    a, b = ev(), ev(); a.record()
    for _ in range(40): L.launch()
    b.record(); torch.cuda.synchronize()
res["b2b40_sampled"] = a.elapsed_time(b) / 40
res["clocks"] = clk.summary()
res["clock_lines"] = clk.lines[:40]
print(json.dumps(res, indent=1))
