"""Constant-bank d slot ordering under graph replay + eager launches, from a
cold process (the first launches of an order happen inside a capture)."""
import os
import sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [REPO, os.path.join(REPO, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
import oracle  # noqa: E402
import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 50
warm_first = len(sys.argv) > 3 and sys.argv[3] == "warm"
nelt = 1 << 16 if n <= 8 else 8192
_raw, knl = fx.translate(fx.semlap_source(n))


def inputs(seed):
    gen = torch.Generator(device=dev).manual_seed(seed)
    u = torch.rand(nelt * n**3, dtype=torch.float64, device=dev,
                   generator=gen) * 2 - 1
    g = torch.rand(6 * nelt * n**3, dtype=torch.float64, device=dev,
                   generator=gen)
    d = torch.rand(n * n, dtype=torch.float64, device=dev,
                   generator=gen) * 2 - 1
    return u, d, g


cur = torch.cuda.current_stream(dev)
cases = []
for c in range(4):
    u, d, g = inputs(300 + c)
    w = torch.full_like(u, float("nan"))
    env = lfb.env_from_buffers(knl, {"nelt": nelt},
                               {"u": u, "d": d, "g": g, "w": w})
    cases.append((env, u, d, g, w))
if warm_first:
    for env, *_r in cases:
        lfb.Launcher(knl, env, variant=variant).launch()
    torch.cuda.synchronize()
s_graph, s_eager, s_graph2 = (torch.cuda.Stream(dev) for _ in range(3))
graphs = []
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
eager = [lfb.Launcher(knl, cases[c][0], variant=variant) for c in (1, 3)]
for rep in range(20):
    for q, (gr, s) in enumerate(graphs):
        with torch.cuda.stream(s):
            gr.replay()
        with torch.cuda.stream(s_eager):
            eager[q].launch(stream=s_eager.cuda_stream)
torch.cuda.synchronize()
bad = []
for c in range(4):
    env, u, d, g, w = cases[c]
    ns = 256
    uh = u[-ns * n**3:].cpu().numpy()
    gh = g[-6 * ns * n**3:].cpu().numpy()
    dh = d.cpu().numpy()
    ref = oracle.semlap(np.zeros(ns * n ** 3), uh, dh, gh, n, ns, threads=8)
    mag = oracle.semlap(np.zeros(ns * n ** 3), np.abs(uh), np.abs(dh),
                        np.abs(gh), n, ns, threads=8)
    got = w[-ns * n**3:].cpu().numpy()
    ok = (np.abs(got - ref) <= 1e-12 * mag) if variant else got == ref
    if not ok.all():
        bad.append((c, int((~ok).sum())))
print(f"n={n} variant={variant} warm_first={warm_first}: bad={bad}")
