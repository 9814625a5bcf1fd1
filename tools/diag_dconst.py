"""Diagnose constant-bank d slot ordering (graph replays vs eager launches)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import torch
import oracle
import paper_1503_07659_b200 as lfb
from paper_1503_07659_b200 import fixtures as fx

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 50
nelt = 8192 if n <= 8 else 2048
_raw, knl = fx.translate(fx.semlap_source(n))


def inputs(seed):
    gen = torch.Generator(device=dev).manual_seed(seed)
    u = torch.rand(nelt * n**3, dtype=torch.float64, device=dev, generator=gen) * 2 - 1
    g = torch.rand(6 * nelt * n**3, dtype=torch.float64, device=dev, generator=gen)
    d = torch.rand(n * n, dtype=torch.float64, device=dev, generator=gen) * 2 - 1
    return u, d, g


def run(mode, reps=6):
    cur = torch.cuda.current_stream(dev)
    cases = []
    for c in range(4):
        u, d, g = inputs(300 + c)
        w = torch.full_like(u, float("nan"))
        env = lfb.env_from_buffers(knl, {"nelt": nelt}, {"u": u, "d": d, "g": g, "w": w})
        cases.append((env, u, d, g, w))
    s_graph, s_eager, s_graph2 = (torch.cuda.Stream(dev) for _ in range(3))
    graphs = []
    if mode in ("mixed", "graphs"):
        for c, s in ((0, s_graph), (2, s_graph2)):
            L = lfb.Launcher(knl, cases[c][0], variant=variant)
            L.launch()
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                L.launch()
            graphs.append((gr, s))
    for s in (s_graph, s_eager, s_graph2):
        s.wait_stream(cur)
    if mode == "mixed":
        eager = [lfb.Launcher(knl, cases[c][0], variant=variant) for c in (1, 3)]
    elif mode == "eager":
        eager = [lfb.Launcher(knl, cases[c][0], variant=variant) for c in range(4)]
    else:
        eager = []
    for rep in range(reps):
        if mode == "eager":
            for q, L in enumerate(eager):
                s = (s_graph, s_eager)[q % 2]
                with torch.cuda.stream(s):
                    L.launch(stream=s.cuda_stream)
            continue
        for q, (gr, s) in enumerate(graphs):
            with torch.cuda.stream(s):
                gr.replay()
            if mode == "mixed":
                with torch.cuda.stream(s_eager):
                    eager[q].launch(stream=s_eager.cuda_stream)
    torch.cuda.synchronize()
    bad = []
    used = {"mixed": [0, 1, 2, 3], "graphs": [0, 2], "eager": [0, 1, 2, 3]}[mode]
    for c in used:
        env, u, d, g, w = cases[c]
        uh, dh, gh = u.cpu().numpy(), d.cpu().numpy(), g.cpu().numpy()
        ref = oracle.semlap(np.zeros(nelt * n ** 3), uh, dh, gh, n, nelt, threads=8)
        mag = oracle.semlap(np.zeros(nelt * n ** 3), np.abs(uh), np.abs(dh), np.abs(gh), n, nelt, threads=8)
        got = w.cpu().numpy()
        okp = np.abs(got - ref) <= 1e-12 * mag
        if not okp.all():
            badel = np.unique(np.nonzero(~okp)[0] // n**3)
            bad.append((c, len(badel), int(badel.min()), int(badel.max())))
    return bad


for mode in ("eager", "graphs", "mixed"):
    for t in range(3):
        print(mode, t, run(mode), flush=True)
