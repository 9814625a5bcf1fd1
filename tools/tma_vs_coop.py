import sys, torch
sys.path.insert(0, '.')
import paper_1503_07659_b200 as lfb
from paper_1503_07659_b200 import fixtures as fx
from paper_1503_07659_b200 import generic
dev = torch.device("cuda", 0)
def timeit(f, reps=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
orig = generic.GenericLauncher.tensor_maps
for name, src, params, bufs, byts in [
    ("smooth", fx.generic_source("smooth"), {"n": 1 << 24}, lambda: {"r": torch.empty(1 << 24, dtype=torch.float64, device=dev), "u": torch.rand((1 << 24) + 2, dtype=torch.float64, device=dev)}, 16 * (1 << 24)),
    ("ttile", fx.generic_source("ttile"), {"n": 8192, "m": 8192}, lambda: {"a": torch.rand(8192 * 8192, dtype=torch.float64, device=dev), "b": torch.empty(8192 * 8192, dtype=torch.float64, device=dev)}, 16 * 8192 * 8192),
    ("dgemm", fx.gemm_source("f64"), {"m": 2048, "n": 2048, "l": 2048}, lambda: {"a": torch.rand(2048*2048, dtype=torch.float64, device=dev), "b": torch.rand(2048*2048, dtype=torch.float64, device=dev), "c": torch.rand(2048*2048, dtype=torch.float64, device=dev)}, None)]:
    _r, knl = fx.translate(src)
    env = lfb.env_from_buffers(knl, params, bufs(), {"alpha": 1.5})
    for mode in ("tma", "coop"):
        if mode == "coop":
            generic.GenericLauncher.tensor_maps = lambda self, env: (orig(self, env)[0], False)
        else:
            generic.GenericLauncher.tensor_maps = orig
        L = generic.GenericLauncher(knl, env)
        ms = timeit(L.launch)
        if byts: print(name, mode, round(ms, 3), "ms", round(byts / ms / 1e6, 1), "GB/s")
        else: print(name, mode, round(ms, 3), "ms", round(2 * 2048**3 / ms / 1e9, 2), "TFLOP/s")
