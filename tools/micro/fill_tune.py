"""fill: CTAs per SM for the bulk-store kernel (tuning aid)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1503_07659_b200 import abi
lib = abi.load()
dev = torch.device("cuda", 0)
n = 1 << 24
outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(4)]
res = {}
for variant, per_sm in ((0, 1), (0, 2), (0, 4), (0, 8), (1, 0)):
    geom = abi.make_launch(None, variant=variant, ctas_per_sm=per_sm)
    st = torch.cuda.current_stream().cuda_stream
    def launch(o):
        rc = lib.lfb_fill_f64(o.data_ptr(), 1.5, n, abi.C.byref(geom), torch.cuda.current_stream().cuda_stream)
        assert rc == 0
    for _ in range(8):
        launch(outs[_ % 4])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for q in range(40):
            launch(outs[q % 4])
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 40
    res[f"v{variant}_ctas{per_sm}"] = round(8 * n / (ms * 1e-3) / 1e9, 1)
    assert bool((outs[0] == 1.5).all())
print(json.dumps(res))
