"""Micro-benchmarks of the individual kernels + the FP64 peak denominators.

python tools/kernel_bench.py [--quick]   (on a B200; prints one JSON line per item)
"""

import argparse
import json
import time

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_21404_b200 import kernels as Kn


def timed(fn, iters=10, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    dev = "cuda"
    out = []
    # cuBLAS DGEMM peak (the FP64 tensor denominator)
    for N in (4096, 8192):
        A = torch.randn(N, N, dtype=torch.float64, device=dev)
        B = torch.randn(N, N, dtype=torch.float64, device=dev)
        t = timed(lambda: A @ B, iters=5)
        out.append({"item": f"cublas_dgemm_{N}", "ms": t * 1e3, "tflops": 2 * N**3 / t / 1e12})
        Ad = torch.zeros(N, N, dtype=torch.float64, device=dev); Ad.copy_(A)
        t = timed(lambda: Kn.gemm_nt(A, B), iters=5)
        out.append({"item": f"dngd_gemm_nt_{N}", "ms": t * 1e3, "tflops": 2 * N**3 / t / 1e12})
        del A, B, Ad
    # SYRK shapes of the configs
    for m, n in [(1020, 1185), (2800, 12737), (4000, 200000), (4000, 791553)]:
        if a.quick and n > 200000:
            continue
        J = torch.randn(m, Kn.pad_ld(n), dtype=torch.float64, device=dev)
        K = torch.empty(m, m, dtype=torch.float64, device=dev)
        t = timed(lambda: Kn.syrk(J, n, K), iters=5)
        out.append({"item": f"syrk_{m}x{n}", "ms": t * 1e3, "tflops": m * (m + 1) * n / t / 1e12})
        y = torch.randn(m, dtype=torch.float64, device=dev)
        g = torch.randn(n, dtype=torch.float64, device=dev)
        t = timed(lambda: Kn.gemv_t(J, y, n, g, -1.0))
        out.append({"item": f"gemv_t_{m}x{n}", "ms": t * 1e3, "gbs": 8 * m * n / t / 1e9})
        t = timed(lambda: Kn.gemv_n(J, g, n))
        out.append({"item": f"gemv_n_{m}x{n}", "ms": t * 1e3, "gbs": 8 * m * n / t / 1e9})
        del J
    for m in (1020, 2800, 4000, 8000):
        A = torch.randn(m, m + 16, dtype=torch.float64, device=dev)
        Km = (A @ A.T) / m
        fac = Kn.CholeskyFactor(m, dev)
        t = timed(lambda: fac.factor(Km, 1e-3), iters=5)
        out.append({"item": f"potrf_{m}", "ms": t * 1e3, "tflops": m**3 / 3 / t / 1e12,
                    "info": int(fac.info.item())})
        t = timed(lambda: torch.linalg.cholesky(Km), iters=5)
        out.append({"item": f"cusolver_potrf_{m}", "ms": t * 1e3, "tflops": m**3 / 3 / t / 1e12})
        b = torch.randn(m, dtype=torch.float64, device=dev)
        t = timed(lambda: fac.solve_(b))
        out.append({"item": f"potrs_{m}", "ms": t * 1e3, "gbs": 8 * m * m / t / 1e9})
    for o in out:
        print(json.dumps(o), flush=True)


if __name__ == "__main__":
    main()
