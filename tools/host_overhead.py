import time, torch, sys
sys.path.insert(0, '.')
import paper_1503_07659_b200 as lfb
from paper_1503_07659_b200 import fixtures as fx
dev = torch.device("cuda", 0)
for name, src, params in [("semlap", fx.semlap_source(8), {"nelt": 64}), ("fill", fx.fill_source("f64"), {"n": 4096}),
                          ("dgemm-generic", fx.gemm_source("f64"), {"m": 64, "n": 64, "l": 64})]:
    _r, knl = fx.translate(src)
    env = lfb.make_device_env(knl, params, seed=0, device=dev)
    eng = "generic" if "generic" in name else "auto"
    for _ in range(20): lfb.interpret(knl, env, inplace=True, engine=eng)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); N = 500
    for _ in range(N): lfb.interpret(knl, env, inplace=True, engine=eng)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    L = lfb.make_launcher(knl, env, engine=eng)
    t2 = time.perf_counter()
    for _ in range(N): L.launch()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(name, "interpret us/call", round((t1-t0)/N*1e6,1), "prepared launcher us/call", round((t3-t2)/N*1e6,1))
