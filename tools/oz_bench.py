"""Emulated-FP64 (Ozaki int8 tcgen05) GEMM vs the FP64 DMMA GEMM: CUDA-event
timing of C = A B^T at Gram-like shapes (K = 512 hidden width)."""

import sys

import torch

sys.path.insert(0, ".")
from paper_2505_21404_b200 import kernels as K  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for (M, N, Kd) in [(8192, 8192, 512), (25088, 4096, 512), (16384, 16384, 1024)]:
    A = torch.randn(M, Kd, dtype=torch.float64, device="cuda")
    B = torch.randn(N, Kd, dtype=torch.float64, device="cuda")
    C = torch.empty(M, N, dtype=torch.float64, device="cuda")
    fl = 2.0 * M * N * Kd
    t_d = timeit(lambda: K.gemm_nt(A, B, C))
    line = f"M={M} N={N} K={Kd}: DMMA {t_d:.3f} ms {fl / t_d / 1e9:.1f} TF"
    for s in (8, 7, 6):
        t_o = timeit(lambda: K.oz_gemm_nt(A, B, C, slices=s))
        ops = fl * s * (s + 1) / 2
        line += f" | oz{s} {t_o:.3f} ms {fl / t_o / 1e9:.1f} TF-eq ({ops / t_o / 1e9:.0f} int8 TOPS)"
    print(line, flush=True)
