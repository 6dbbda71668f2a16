"""J^T y / J x bandwidth over a materialised J (m x n FP64): python tools/gemv_bench.py m n."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21404_b200 import kernels as K  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2800
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12737
J = torch.randn(m, K.pad_ld(n), dtype=torch.float64, device="cuda")
y = torch.randn(m, dtype=torch.float64, device="cuda")
x = torch.randn(n, dtype=torch.float64, device="cuda")
ref = J[:, :n].T @ y
got = K.gemv_t(J, y, n)
assert torch.allclose(got, ref, rtol=1e-12, atol=1e-12), (got - ref).abs().max()


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


nb = 8.0 * m * n + 8.0 * (m + n)
out = torch.empty(n, dtype=torch.float64, device="cuda")
outm = torch.empty(m, dtype=torch.float64, device="cuda")
tt = timed(lambda: K.gemv_t(J, y, n, out=out))
tn = timed(lambda: K.gemv_n(J, x, n, out=outm))
print(f"m={m} n={n}  J^T y {tt*1e6:.1f} us "
      f"{nb/tt/1e9:.0f} GB/s   J x {tn*1e6:.1f} us {nb/tn/1e9:.0f} GB/s")
