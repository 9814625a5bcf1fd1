"""One SEM launch for an ncu capture: python tools/prof_sem.py N VARIANT
(sweep sizes: nelt = 2 GiB / (64 n^3); 2 warm-up launches first)."""
import os
import sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402
import bench  # noqa: E402
import paper_1503_07659_b200 as lfb  # noqa: E402
from paper_1503_07659_b200 import fixtures as fx  # noqa: E402

n, v = int(sys.argv[1]), int(sys.argv[2])
nelt = (1 << 31) // (64 * n ** 3) // 32 * 32
dev = torch.device("cuda", 0)
_r, knl = fx.translate(fx.semlap_source(n))
u, d, g, w = bench.sem_buffers(n, nelt, dev, n)
env = lfb.env_from_buffers(knl, {"nelt": nelt},
                           {"u": u, "d": d, "g": g, "w": w})
L = lfb.Launcher(knl, env, variant=v)
for _ in range(3):
    L.launch()
torch.cuda.synchronize()
