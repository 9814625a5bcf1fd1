"""One launch of the generated fill (f64, 2^24, split 128) for ncu."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402
from paper_1503_07659_b200.generic import GenericLauncher  # noqa: E402
dev = torch.device("cuda", 0)
n = 1 << 24
_r, kf = fx.translate(fx.fill_source("f64"))
out = torch.empty(n, dtype=torch.float64, device=dev)
L = GenericLauncher(kf, lfb.env_from_buffers(kf, {"n": n}, {"out": out},
                                             {"a": 1.5}))
for _ in range(4):
    L.launch()
torch.cuda.synchronize()
