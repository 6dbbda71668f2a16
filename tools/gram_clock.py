"""SM clock and power while the emulated Gram runs back to back at config 3 (NVML, 5 ms),
per DNGD_GOZ_DBG mode: tells a clock-limited kernel from an issue-limited one."""
import os
import sys
import threading
import time

import numpy as np
import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_21404_b200 as P  # noqa: E402
from paper_2505_21404_b200 import kernels as K  # noqa: E402

prob = P.make_problem("poisson5d_sin")
spec = P.MlpSpec((5, 512, 512, 512, 512, 1))
rmap = P.PinnResidualMap(prob, spec, prob.sample((3500, 500), np.random.default_rng(0)))
theta = P.xavier_normal_params(spec)
d = rmap._device()
rmap.residuals_act_t(theta)
ws = rmap._act_workspace()
Kt = torch.zeros(rmap.m, rmap.m, dtype=torch.float64, device="cuda")
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for dbg in sys.argv[1:] or ["0"]:
    os.environ["DNGD_GOZ_DBG"] = dbg
    K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], Kt, ws, slices=int(os.environ.get("GOZ_S", "6")))
    torch.cuda.synchronize()
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
            time.sleep(0.005)

    th = threading.Thread(target=sample)
    th.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 40
    for _ in range(n):
        K.gram_factored_act(d["mlp"], d["arr"], d["nclass"], Kt, ws, slices=int(os.environ.get("GOZ_S", "6")))
    b.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    cl = np.array([s[0] for s in samples[len(samples) // 5:]])
    pw = np.array([s[1] for s in samples[len(samples) // 5:]])
    print(f"dbg {dbg}: {a.elapsed_time(b) / n:.2f} ms  sm clock median {np.median(cl):.0f} MHz "
          f"(min {cl.min():.0f})  power median {np.median(pw):.0f} W", flush=True)
