import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2505_21404_b200 import kernels as K
for k in (40, 64, 96, 128, 160, 192, 256):
    g = torch.Generator(device="cuda").manual_seed(k)
    X = torch.randn(k, 512, dtype=torch.float64, device="cuda", generator=g)
    d = torch.logspace(0, -14, 512, dtype=torch.float64, device="cuda")
    G = (X * d) @ X.T
    K.syev_jacobi(G, k); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): w, V, sw = K.syev_jacobi(G, k)
    b.record(); torch.cuda.synchronize()
    print(k, round(a.elapsed_time(b) / 3, 3), "ms", int(sw.item()), "sweeps", flush=True)
