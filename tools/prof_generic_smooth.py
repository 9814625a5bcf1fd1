"""One launch of the generated smoother (TMA ring) for ncu."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402
from paper_1503_07659_b200.generic import GenericLauncher  # noqa: E402
dev = torch.device("cuda", 0)
n = 1 << 24
_r, km = fx.translate(fx.generic_source("smooth"))
u = torch.rand(n + 2, dtype=torch.float64, device=dev)
r = torch.empty(n, dtype=torch.float64, device=dev)
L = GenericLauncher(km, lfb.env_from_buffers(km, {"n": n}, {"r": r, "u": u}))
for _ in range(4):
    L.launch()
torch.cuda.synchronize()
