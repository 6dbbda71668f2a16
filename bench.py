"""D-NGD step benchmark (BASELINE.json metric: "D-NGD steps/s; Gram+Cholesky FP64
TFLOP/s and matvec GB/s vs peak, 1/2/4/8 GPU").

Workload at N=1 (default --config 3, the configuration the metric is quoted on:
"parameter-sharded over 1/2/4/8 GPUs"): 5-D Poisson -Delta u = f on [0,1]^5,
u* = sum_i sin(pi x_i), 3500 interior + 500 boundary points (m = 4000), MLP
5 -> 512x4 -> 1 tanh (n = 791,553), Xavier-normal init, FP64, dense dual Gram +
Cholesky, GN + geodesic correction, 31-point line search.  One "step" = one full
outer iteration of the reference loop (optimizer.py:212-262): residuals, damping,
Gram, Cholesky (+ retries), GN solve, f_vv, GA solve, line search, parameter
update -- with fresh collocation points every step.

  value : steps/s with every step's collocation points already resident in HBM
  e2e   : steps/s through the public API (dngd_run) with host-side sampling,
          host->device upload of the points/data and device->host reads of the
          per-step scalars inside the timed region
  --impl reference : the CPU oracle (oracle/dngd_oracle.py, a numpy port of the
          reference algorithm) on all host cores, same workload
  --gpus N (N > 1, outside torchrun): relaunches itself under torch.distributed.run
          with N ranks on this node

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                       [--config 1..7]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from dataclasses import replace

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs (1-based)
    1: dict(problem="poisson2d", widths=(2, 32, 32, 1), counts=(900, 120), lam_cap=1e-8,
            dense_threshold=4000, name="cfg1_poisson2d_2-32-32-1_m1020"),
    2: dict(problem="heat1d", widths=(2, 64, 64, 64, 64, 1), counts=(2000, 400, 400), lam_cap=1e-3,
            dense_threshold=4000, name="cfg2_heat1d_2-64x4-1_m2800"),
    3: dict(problem="poisson5d_sin", widths=(5, 512, 512, 512, 512, 1), counts=(3500, 500),
            lam_cap=1e-5, dense_threshold=4001, name="cfg3_poisson5d_5-512x4-1_m4000",
            multi_gpu="tiles"),
    4: dict(problem="poisson5d_sin", widths=(5, 1792, 1792, 1792, 1792, 1792, 1),
            counts=(7000, 1000), lam_cap=1e-5, dense_threshold=8001,
            name="cfg4_poisson5d_5-1792x5-1_m8000_n12.86M", multi_gpu="tiles"),
    5: dict(problem="poisson2d", widths=(2, 256, 256, 256, 256, 1), counts=(30000, 2000),
            lam_cap=1e-5, dense_threshold=4000, nystrom_rank=512, cg_max_iters=200,
            name="cfg5_poisson2d_2-256x4-1_m32000_pcg"),
    # not a BASELINE config: the reference's own configs/allen_cahn.json problem
    # (periodic embedding + cubic reaction) at its default collocation counts
    6: dict(problem="allen_cahn", widths=(3, 32, 32, 32, 1), counts=(1125, 225), lam_cap=1e-5,
            dense_threshold=4000, name="ref_allen_cahn_3-32x3-1_m1350"),
    # not a BASELINE config: the paper's STDE case -- 100000-D
    # Poisson on the ball, [100000, 128x4, 1] (n = 12.85M), m = 100, k = 8 directions
    7: dict(problem="poisson_ball_stde", problem_kw=dict(dim=100000, index_set_size=8),
            widths=(100000, 128, 128, 128, 128, 1), counts=(100,), lam_cap=1e3,
            dense_threshold=4000, name="paper_stde_100000-128x4-1_m100_n12.85M",
            no_cpu="numpy oracle would hold a 10 GB Jacobian plus per-sample einsum "
                   "temporaries of the same size; not run on the host"),
}
METRIC = "D-NGD steps/s"
UNIT = "steps/s"


def _env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(
        os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML from a
    background thread every 5 ms (the timed region of a default run is ~0.1 s, too
    short for nvidia-smi's 100 ms loop), nvidia-smi -lms as the fallback."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.thread = None
        self.samples = []
        self.reasons = set()
        self.smax = None

    def _nvml_loop(self, nv, h):
        import time
        while not self._stop:
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for nm, bit in self.BITS.items():
                    if mask & bit:
                        self.reasons.add(nm)
            except Exception:
                return
            time.sleep(0.005)

    def start(self):
        try:
            import threading

            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self._stop = False
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self._stop = True
            self.thread.join(timeout=2)
            sm = self.samples
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.smax,
                    "reasons": sorted(self.reasons), "samples": len(sm), "source": "nvml 5 ms"}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi 100 ms"}


# ------------------------------------------------------------------ our arm


def _fp64_peak():
    """Measured FP64 tensor peak on this GPU: cuBLAS DGEMM 8192^3 (MEASURED_PEAKS.json has
    no FP64 figure).  Best of 3 after warm-up."""
    import torch

    N = 8192
    A = torch.randn(N, N, dtype=torch.float64, device="cuda")
    B = torch.randn(N, N, dtype=torch.float64, device="cuda")
    for _ in range(2):
        A @ B
    best = 0.0
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        A @ B
        e.record()
        torch.cuda.synchronize()
        best = max(best, 2 * N**3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    del A, B
    torch.cuda.empty_cache()
    return best


def _hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


def _count_our_kernels(fn):
    """Number of libdngd_b200 kernels one call of fn launches (CUPTI via torch.profiler)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    n = 0
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA and "dngd::" in ev.name:
            n += 1
    return n


# tcgen05 kind::i8 dense MMA rate of the Ozaki kernels' own issue pattern (one MMA
# per digit slice, N = 64 (S - t), operands resident in shared memory, all 148 SMs;
# tools/micro/umma_wide.cu, profiles/r02b/int8_mma_*.txt): 920 cycles per 7-digit
# K-chunk (896 ideal).  With random operand bytes over 1.4 s of back-to-back MMAs the
# board's power limit holds the chip at 3715 TOPS -- the SUSTAINED peak, the
# denominator for a kernel timed inside a long step (B200_PROFILING: burst figure
# for a kernel timed alone, sustained for one inside a step).  The burst rate (2 ms,
# near-constant operands) is 4446 TOPS.
INT8_PEAK_TOPS = 3715.0
INT8_BURST_TOPS = 4446.0
INT8_PEAK_SOURCE = ("sustained tcgen05.mma kind::i8 rate of the Ozaki chunk pattern with random "
                    "operands, power-limited steady state (tools/micro/umma_wide.cu 30000 1 40: "
                    "3715 TOPS; burst with near-constant operands 4446 TOPS)")


def _emulated_gram(rmap):
    """(issued int8 ops, useful int8 ops, slices) of one emulated factored-Gram launch,
    or None when the Gram runs on the FP64 DMMA kernel (kernels.gram_emulation_slices)."""
    from paper_2505_21404_b200 import kernels as K

    mlp = rmap._device()["mlp"]
    S = K.gram_emulation_slices(mlp)
    if not S:
        return None
    widths = [mlp.widths[k] for k in range(mlp.nlayers + 1)]
    L = mlp.nlayers
    kp = lambda k: (k + 31) // 32 * 32  # noqa: E731
    chunks = sum(kp(widths[0] if k == 0 else widths[k]) // 32 for k in range(L))
    chunks += sum(kp(widths[k + 1]) // 32 for k in range(L - 1))
    cls = [(c.count, rmap._nch(c)) for c in rmap.collocation.classes]
    tiles = 0
    for a in range(len(cls)):
        for b in range(a + 1):
            ppa, ppb = 64 // cls[a][1], 64 // cls[b][1]
            TI = -(-cls[a][0] // (2 * ppa))
            TJ = -(-cls[b][0] // ppb)
            tiles += TI * (TI + 1) if a == b else TI * TJ
    per_chunk = S * (S + 1) // 2 * 2.0 * 128 * 64 * 32
    ops = tiles * chunks * per_chunk
    useful = S * (S + 1) // 2 * rmap.factored_gram_flops()
    return ops, useful, S


def _profiled_traffic(workload, kernel):
    """DRAM bytes per launch of the roofline kernel from the committed ncu capture
    (profiles/<round>/traffic.json), or None when this kernel/workload has none."""
    import glob

    best = None
    for path in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                              "profiles", "r*", "traffic.json"))):
        try:
            with open(path) as f:
                table = json.load(f)
        except (OSError, ValueError):
            continue
        for name, ent in table.get(workload, {}).items():
            if name.split("<")[0] in kernel:
                best = ent.get("bytes")
    return best


def _hbm_stages(rmap, theta, hbm_peak, reps=10):
    """The HBM-bound stages of the dense path WITH J materialised, at the bench
    workload (north star: Jacobian writes and J/J^T matvecs vs the HBM roofline;
    the product path at configs 2-7 never forms J, so these are measured here
    separately, outside the timed region).  Algorithmic bytes:
    assembly 8mn written (its activation reads are not counted), J^T y and J x
    8mn + 8(m+n).  J > L2 at config 2 (285 MB vs 126 MB), so each launch streams
    J from HBM.  CUDA events on the launching stream, mean of `reps` launches."""
    import torch

    from paper_2505_21404_b200 import kernels as K

    m, n = rmap.m, rmap.n
    if 8.0 * m * K.pad_ld(n) > 40e9:
        return None
    th = rmap._theta_t(theta)
    d = rmap._device()
    dev = d["device"]
    J = torch.empty((m, K.pad_ld(n)), dtype=torch.float64, device=dev)
    r = torch.empty(m, dtype=torch.float64, device=dev)
    y = torch.randn(m, dtype=torch.float64, device=dev)
    x = torch.randn(n, dtype=torch.float64, device=dev)
    out_n = torch.empty(n, dtype=torch.float64, device=dev)
    out_m = torch.empty(m, dtype=torch.float64, device=dev)
    ws = rmap._act_workspace()

    def timed(fn):
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

    t_asm = timed(lambda: K.assemble(d["mlp"], th, d["arr"], d["nclass"], r, J, 0, n, ws))
    t_jt = timed(lambda: K.gemv_t(J, y, n, out=out_n))
    t_j = timed(lambda: K.gemv_n(J, x, n, out=out_m))
    mv = 8.0 * m * n + 8.0 * (m + n)

    def ent(kern, nbytes, t):
        gbs = nbytes / t / 1e9
        return {"kernel": kern, "bytes": nbytes, "us": t * 1e6, "gbs": gbs,
                "frac_of_hbm_peak": gbs / hbm_peak}

    rmap._cache = None  # the probe's J is not the loop's
    return {"J_assembly": ent("dngd_assemble (activation pass + k_jwrite)", 8.0 * m * n, t_asm),
            "JT_y": ent("dngd_gemv_t (k_gemv_t + reduce)", mv, t_jt),
            "J_x": ent("dngd_gemv_n (k_gemv_n_row)", mv, t_j),
            "note": "dense path with J materialised (m x n FP64, ldJ padded to 16); the J-free "
                    "product path does not run these"}


def run_ours(args, cfg):
    import torch

    import paper_2505_21404_b200 as P
    from paper_2505_21404_b200 import kernels as K
    from paper_2505_21404_b200 import timing
    from paper_2505_21404_b200.optimizer import device_line_search, lm_damping

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.sharded:
        return run_sharded(args, cfg)

    problem = P.make_problem(cfg["problem"], **cfg.get("problem_kw", {}))
    spec = P.MlpSpec(cfg["widths"], seed=0)
    config = P.OptimizerConfig(max_iters=args.warmup + args.steps, lam_cap=cfg["lam_cap"],
                               dense_threshold=cfg["dense_threshold"],
                               nystrom_rank=cfg.get("nystrom_rank", 64),
                               cg_max_iters=cfg.get("cg_max_iters", 500))
    fp64_peak = 35.47 if args.profile else _fp64_peak()
    hbm_peak, hbm_src = _hbm_peak()

    # -------- device-resident run: all collocation sets uploaded before timing
    # (N > 1 runs through run_sharded)
    tiles = sharded = False
    comm = None
    rng = np.random.default_rng(1000 if world > 1 else 1000 + rank)
    total = args.warmup + args.steps + 2  # +2: the pipelined loop's ramp (see below)
    maps = []
    base = None
    for _ in range(total):
        colloc = P.sample_collocation(problem, cfg["counts"], rng)
        if base is None:
            mp = P.PinnResidualMap(problem, spec, colloc)
        else:
            mp = base.rebind(colloc)
        maps.append(mp)
        base = mp
    for mp in maps:
        mp._device()  # upload points and data now
    shared_J = None
    theta = P.xavier_normal_params(spec)
    theta = P.ParameterVector(theta.tensor, theta.layout)

    def one_step(rmap, theta):
        nonlocal shared_J
        from paper_2505_21404_b200.optimizer import LineSearchResult, _dispatch_step, _select
        from paper_2505_21404_b200.solver import dense_iteration

        dense = rmap.m < config.dense_threshold
        jfree = dense and rmap.jfree()
        if dense:
            # the product's dense iteration (optimizer._dngd_loop): damping on the
            # device, one host read-back per step
            if not jfree:
                rmap._J = shared_J
            step, losses, anyd, loss, r = dense_iteration(
                rmap, theta, config.use_ga, config.line_search_points, config.lam_cap)
            if not jfree:
                shared_J = rmap._J
            if step is not None:
                delta = step.delta.tensor
                etas = 2.0 ** -np.arange(config.line_search_points, dtype=np.float64)
                ls = (_select(losses, etas, loss, config.line_search_points) if anyd
                      else LineSearchResult(1.0, loss, False, 0, False))
            else:  # factorisation failed: eager path with the retry ladder
                lam = lm_damping(loss, config.lam_cap)
                g = None if jfree else K.gemv_t(rmap.jacobian_t(theta), r, rmap.n)
                step = _dispatch_step(rmap, theta, g, lam, config, rng)
                delta = step.delta.tensor
                ls = device_line_search(rmap, theta, delta, loss, config.line_search_points)
        else:  # Nystrom-PCG configuration
            pcg_jfree = rmap.jfree_pcg()
            if pcg_jfree:  # J-free PCG (solver.pcg_step with g=None)
                r, J = rmap.residuals_act_t(theta), None
            else:
                rmap._J = shared_J
                r, J = rmap.linearize_t(theta)
                shared_J = rmap._J
            loss = 0.5 * float(K.dot(r, r).item())
            lam = lm_damping(loss, config.lam_cap)
            g = None
            if not pcg_jfree:
                with timing.stage("gemv"):
                    g = K.gemv_t(J, r, rmap.n)
            step = _dispatch_step(rmap, theta, g, lam, config, rng)
            delta = step.delta.tensor
            ls = device_line_search(rmap, theta, delta, loss, config.line_search_points)
        if ls.rejected:
            return theta, step
        return P.ParameterVector(K.axpby(ls.eta, delta, 1.0, theta.tensor), theta.layout), step

    # the product's pipelined loop (optimizer._pipelined_loop: step i+1 queued before
    # step i's results are read, selection and update on the device) where it applies
    from paper_2505_21404_b200.optimizer import TrainTrace, _dngd_loop, _pipeline_ok

    pipelined = (not sharded and not tiles and sum(cfg["counts"]) < cfg["dense_threshold"]
                 and _pipeline_ok(maps[0], config))

    def run_loop(first, count, theta, on_step=None):
        sub = maps[first:first + count]
        tr = TrainTrace(problem=problem.name, method="dngd", seed=0)
        _dngd_loop(tr, lambda it: sub[min(it, count) - 1], theta, replace(config, max_iters=count),
                   rng, None, on_step)
        if tr.aborted:
            raise SystemExit(f"bench loop aborted: {tr.abort_reason}")
        return tr.final_theta

    if pipelined:
        theta = run_loop(0, args.warmup, theta)
    else:
        for i in range(args.warmup):
            theta, _ = one_step(maps[i], theta)
    if args.profile:
        launches = 0
    elif pipelined:  # per iteration of the loop: (3 iterations - 1 iteration) / 2
        launches = (_count_our_kernels(lambda: run_loop(args.warmup, 3, theta))
                    - _count_our_kernels(lambda: run_loop(args.warmup, 1, theta))) // 2
    else:
        launches = _count_our_kernels(lambda: one_step(maps[args.warmup], theta))
    for mp in maps:
        mp._cache = None  # the counting step must not pre-assemble a timed step's Jacobian
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if pipelined:
        # steady state of the pipelined loop: on_step(i) runs when iteration i+1 is
        # already queued, so events recorded there bracket iterations 3 .. K+2 of a
        # K+2 iteration run (device time of exactly K iterations, no ramp)
        tm = timing.StageTimer()

        def mark(it, th, step, ls):
            if it == 1:
                s.record()
            if it == 2:
                timing.set_active(tm)  # fetches of iterations 3 .. K+2
            if it == args.steps + 1:
                e.record()

        mark.needs_theta = False  # no per-iteration copy of theta for a timing callback

        try:
            theta = run_loop(args.warmup, args.steps + 2, theta, mark)
        finally:
            timing.set_active(None)
        torch.cuda.synchronize()
        stages, counts = tm.summary_ms()
    else:
        with timing.collect() as tm:
            s.record()
            for i in range(args.steps):
                theta, last = one_step(maps[args.warmup + i], theta)
            e.record()
            torch.cuda.synchronize()
            stages, counts = tm.summary_ms()
    dev_s = s.elapsed_time(e) * 1e-3
    if dist:
        t = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
    clk = clocks.stop()

    # -------- end to end through the public API (dngd_run): host sampling + H2D + D2H
    e2e = {}
    bytes_in = []

    orig_device = P.PinnResidualMap._device

    def counting_device(self):
        fresh = self._dev is None
        d = orig_device(self)
        if fresh:
            bytes_in.append(sum(t.numel() * t.element_size() for t in d["keep"]))
        return d

    if not args.profile:
        P.PinnResidualMap._device = counting_device
    marks = {}

    lag = 1 if pipelined else 0  # pipelined: iteration i+1 is queued when on_step(i) runs

    def on_step(it, th, step, ls):
        if it == args.warmup - lag:
            torch.cuda.synchronize()
            marks["t0"] = time.perf_counter()
        if it == args.warmup + args.steps - lag:
            torch.cuda.synchronize()
            marks["t1"] = time.perf_counter()

    on_step.needs_theta = False

    tr = None
    try:
        if not args.profile:
            tr = P.dngd_run(problem, spec, config, seed=rank, counts=cfg["counts"],
                            init="xavier_normal", track_rel_l2=False, on_step=on_step)
    finally:
        P.PinnResidualMap._device = orig_device
    if "t0" in marks and "t1" in marks:
        e2e_s = marks["t1"] - marks["t0"]
        if dist:
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        h2d = (int(np.median(bytes_in)) if bytes_in else 0) * world  # every rank uploads the points
        # per step the host reads: loss (8 B), |v|, |a| (16 B), Cholesky info (4 B),
        # 31 line-search losses (248 B), the delta-nonzero flag (1 B)
        d2h = (8 + 16 + 4 + 8 * config.line_search_points + 1) * world
        if pipelined:  # packed results + device selection, one pinned buffer per step
            d2h = 8 * (10 + config.line_search_points) * world
        e2e = {"value": args.steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "aborted": tr.aborted}

    # PCG configurations: CG iterations per step of the end-to-end run (the device
    # loop's count, read once per step)
    cg_per_step = None
    if tr is not None:
        its = [r.cg_iterations for r in tr.rows[1:] if getattr(r, "cg_iterations", None) is not None]
        if its and max(its) > 0:  # (dense steps record 0)
            cg_per_step = float(np.mean(its))

    # -------- roofline of the dominant kernel
    m = sum(cfg["counts"])
    n = spec.param_count()
    ms_per_step = dev_s / args.steps * 1e3
    stage_ms = {k: v / args.steps for k, v in stages.items()}
    syrk_avg = stages.get("syrk", 0.0) / max(counts.get("syrk", 1), 1) * 1e-3
    potrf_avg = stages.get("potrf", 0.0) / max(counts.get("potrf", 1), 1) * 1e-3
    roof = None
    if syrk_avg > 0:
        flops = m * (m + 1) * n
        ach = flops / syrk_avg / 1e12
        roof = {"kernel": "dngd::k_gemm_nt<128,128> (SYRK K=JJ^T, lower tiles, split-K)",
                "bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": ach / fp64_peak, "traffic": None,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 DMMA)",
                "algorithmic": f"m(m+1)n = {flops:.3e} FLOP per launch"}
    gram_avg = stages.get("gram", 0.0) / max(counts.get("gram", 1), 1) * 1e-3
    gk_avg = stages.get("gram_kernel", 0.0) / max(counts.get("gram_kernel", 1), 1) * 1e-3
    if gk_avg > 0 and (roof is None or gk_avg > syrk_avg):
        # the Gram kernel alone (its own CUDA events; the activation pass that feeds
        # it is the separate "activations" stage), on USEFUL FLOPs: packed channel
        # rows, exact K-dims, lower triangle of point pairs -- nothing padded counted
        flops = maps[0].factored_gram_flops()
        flops_x = maps[0].factored_gram_flops(executed=True)
        ach = flops / gk_avg / 1e12
        emu = _emulated_gram(maps[0])
        if emu is not None:
            ops, useful_ops, slices = emu
            roof = {"kernel": f"dngd::k_gram_oz<{slices}> (factored Gram, emulated FP64: "
                              f"{slices} int8 Ozaki digits per activation row, tcgen05 kind::i8)",
                    "bound": "tensor", "achieved": ops / gk_avg / 1e12, "peak": INT8_PEAK_TOPS,
                    "unit": "TOPS (int8)", "frac": ops / gk_avg / 1e12 / INT8_PEAK_TOPS,
                    "traffic": None,
                    "peak_source": INT8_PEAK_SOURCE,
                    "algorithmic": f"{ops:.4e} int8 ops issued per launch = S(S+1)/2 digit "
                                   "products x 2 x 128 x 64 x 32 per K-chunk x chunks x tiles "
                                   f"({useful_ops:.4e} on useful rows = {slices * (slices + 1) // 2}"
                                   f" x the {flops:.4e} useful FP64 FLOP)",
                    "useful_frac": useful_ops / gk_avg / 1e12 / INT8_PEAK_TOPS,
                    "kernel_ms": gk_avg * 1e3,
                    "fp64_equivalent_tflops": ach,
                    "fp64_equivalent_frac_of_dmma_peak": ach / fp64_peak,
                    "burst_peak_tops": INT8_BURST_TOPS,
                    "frac_of_burst_peak": ops / gk_avg / 1e12 / INT8_BURST_TOPS}
        else:
            roof = None
    if gk_avg > 0 and roof is None:
        roof = {"kernel": "dngd::k_gram_factored (K = sum_k S (G^H_k o G^Z_k) S^T, J-free)",
                "bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": ach / fp64_peak, "traffic": None,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 DMMA)",
                "algorithmic": f"factored Gram {flops:.4e} useful FLOP per launch (2 x point-pair "
                               "channel blocks of the lower triangle x sum_k (w_k + w_k+1)); "
                               f"{flops_x:.4e} issued (64-row tiles, 16-column K chunks)",
                "kernel_ms": gk_avg * 1e3,
                "issued_tflops": flops_x / gk_avg / 1e12,
                "jjt_equivalent_tflops": m * (m + 1) * n / gk_avg / 1e12}
    vjp_avg = stages.get("vjp", 0.0) / max(counts.get("vjp", 1), 1) * 1e-3
    if gram_avg > 0 and maps[0].wide_input() and vjp_avg > 0:
        # wide raw input (STDE): the Gram is formed analytically (X X^T + hidden
        # SYRK); the heaviest kernel is J^T w's input block, FP64 FMA over every
        # parameter (B200's nominal FP64 vector and DMMA peaks are the same)
        flops = 2.0 * m * n
        ach = flops / vjp_avg / 1e12
        roof = {"kernel": "dngd::k_jt_input_wide (+ hidden-layer split-K GEMMs): J^T w, J-free",
                "bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": ach / fp64_peak, "traffic": None,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 DMMA)",
                "algorithmic": f"2 m n = {flops:.3e} FLOP per J^T w"}
    ls_avg = stages.get("line_search", 0.0) / max(counts.get("line_search", 1), 1) * 1e-3
    if roof is None and ls_avg > 0:
        # Nystrom-PCG configuration (no Gram): the 31-candidate line search is the
        # largest tensor-core stage -- batched hidden-layer GEMMs over all channel rows
        w = list(cfg["widths"])
        rows = sum(c * maps[0]._nch(cl) for c, cl in zip(cfg["counts"], maps[0].collocation.classes))
        flops = 31 * 2.0 * rows * sum(w[k] * w[k + 1] for k in range(1, len(w) - 2))
        ach = flops / ls_avg / 1e12
        ls_S = int(os.environ.get("DNGD_GEMM_SLICES", "6" if max(w[1:-1]) >= 128 else "0"))
        emulated = ls_S in (6, 7)
        if emulated:  # int8 engine (pinn.cu oz_ls_slices): S(S+1)/2 digit products
            nprod = ls_S * (ls_S + 1) // 2
            ops = nprod * flops
            roof = {"kernel": f"dngd::k_oz_gemm<{ls_S},2> (31-candidate line-search forward, emulated "
                              "FP64, batched; stage time includes k_chan_slice / k_tanh_head)",
                    "bound": "tensor", "achieved": ops / ls_avg / 1e12, "peak": INT8_PEAK_TOPS,
                    "unit": "TOPS (int8)", "frac": ops / ls_avg / 1e12 / INT8_PEAK_TOPS,
                    "traffic": None, "peak_source": INT8_PEAK_SOURCE,
                    "algorithmic": f"{nprod} x 31 x 2 R sum_k w_k w_k+1 = {ops:.3e} useful int8 ops per "
                                   f"line search ({flops:.3e} FP64 FLOP; hidden layers, R = channel rows)",
                    "fp64_equivalent_tflops": ach,
                    "fp64_equivalent_frac_of_dmma_peak": ach / fp64_peak}
        else:
            roof = {"kernel": "dngd::k_gemm_nt<128,128> (31-candidate line-search forward, batched)",
                    "bound": "tensor", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s",
                    "frac": ach / fp64_peak, "traffic": None,
                    "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 DMMA)",
                    "algorithmic": f"31 x 2 R sum_k w_k w_k+1 = {flops:.3e} FLOP per line search "
                                   "(hidden layers; R = channel rows)"}
    if roof is not None:
        roof["traffic"] = _profiled_traffic(cfg["name"], roof["kernel"])
    gram_chol = None
    g_avg = syrk_avg if syrk_avg > 0 else (gk_avg if gk_avg > 0 else gram_avg)
    if g_avg > 0 and potrf_avg > 0:
        # J J^T-equivalent rate of the Gram + Cholesky stage (north-star definition)
        gf = (m * (m + 1) * n + m**3 / 3) / (g_avg + potrf_avg) / 1e12
        gram_chol = {"tflops": gf, "frac_of_fp64_peak": gf / fp64_peak,
                     "gram_ms": g_avg * 1e3, "potrf_ms": potrf_avg * 1e3,
                     "useful_tflops": ((maps[0].factored_gram_flops() if gk_avg > 0 else m * (m + 1) * n)
                                       + m**3 / 3) / (g_avg + potrf_avg) / 1e12,
                     "useful_frac_of_fp64_peak": None,
                     "gram_path": "syrk" if syrk_avg > 0 else (
                         "wide-input (hidden SYRK + analytic input block)"
                         if maps[0].wide_input() else "factored"),
                     "definition": "(m(m+1)n + m^3/3) / (t_gram + t_potrf), SURVEY 8(d); on the "
                                   "factored path this is a J J^T-equivalent rate (the kernel "
                                   "performs fewer FLOPs), so it can exceed the FP64 peak"}
    if gram_chol is not None:
        gram_chol["useful_frac_of_fp64_peak"] = gram_chol["useful_tflops"] / fp64_peak
    jfree = (syrk_avg == 0 and gram_avg > 0) or (
        m >= cfg["dense_threshold"] and not sharded and maps[0].jfree_pcg())
    gemv_bytes = None if jfree else 8 * m * n
    if jfree and m >= cfg["dense_threshold"]:
        l2_note = ("per-step working set exceeds L2: the per-point activations, the m x l "
                   "Nystrom columns and the 31-candidate line-search activations are "
                   "rewritten every step (J-free PCG: J is never formed)")
    elif jfree:
        l2_note = ("per-step working set exceeds L2: K + its factor (%.0f MB) and the "
                   "31-candidate line-search activations are rewritten every step (J-free: "
                   "J is never formed)" % (16 * m * m / 1e6))
    else:
        l2_note = "per-step working set exceeds L2 (J = %.0f MB rewritten every step)" % (
            8 * m * n / 1e6)
    line = {
        "metric": METRIC,
        "value": args.steps / dev_s,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded collocation sampling; Xavier-normal random init)",
        "config": {"workload": cfg["name"], "m": m, "n": n, "widths": list(cfg["widths"]),
                   "solver": "dense Cholesky + geodesic acceleration" if m < cfg["dense_threshold"]
                   else "Nystrom-PCG", "lam_cap": cfg["lam_cap"], "line_search_points": 31,
                   "parallelism": (f"tile-sharded factored Gram over {world} GPUs (NCCL "
                                   "all-reduce of K, rest replicated)") if tiles else
                   (f"column-sharded J over {world} GPUs (NCCL all-reduce of K)"
                    if world > 1 else "single GPU"),
                   "l2": l2_note},
        "roofline": roof,
        "gram_cholesky": gram_chol,
        "stages_ms_per_step": stage_ms,
        "gemv_bytes_per_launch": gemv_bytes,
        "hbm_stages": (_hbm_stages(maps[0], theta, hbm_peak)
                       if (not sharded and not args.profile) else None),
        "hbm_peak_gbs": hbm_peak,
        "hbm_peak_source": hbm_src,
        "fp64_peak_tflops": fp64_peak,
        "e2e": e2e or None,
        "gpu_launches": launches * args.steps,
        "clocks": clk,
        "final_loss": float(0.5 * float(maps[-1].residuals_t(theta).norm().item() ** 2)),
        "cg_iterations_per_step": cg_per_step,
    }
    if rank == 0 and not args.no_cpu_baseline and not args.profile:
        line["cpu_baseline"] = (cpu_baseline(cfg, max_seconds=args.cpu_seconds)
                                if not cfg.get("no_cpu") else
                                {"value": None, "unavailable": cfg["no_cpu"]})
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_sharded(args, cfg):
    """N > 1 ranks (one per GPU, NCCL): the column-sharded D-NGD loop of sharded.py.
    Configs 3-4 ("tiles"): J-free, each rank computes 1/N of the factored Gram's
    tiles and its own J_p^T w rows, K all-reduced; configs 1, 2, 5 ("columns"):
    each rank assembles J_p, K_p = J_p J_p^T (dense) or one m-vector all-reduce per
    CG product (PCG).  Every rank draws the same collocation points; value = steps
    / max-over-ranks device time of K steps (all ranks advance one shared step)."""
    import torch
    import torch.distributed as dist

    import paper_2505_21404_b200 as P
    from paper_2505_21404_b200 import timing
    from paper_2505_21404_b200.optimizer import TrainTrace
    from paper_2505_21404_b200.sharded import Comm, make_ops, sharded_dngd_run, sharded_loop

    rank, world, local = _env_rank()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if "MASTER_PORT" not in os.environ:
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            os.environ["MASTER_PORT"] = str(sk.getsockname()[1])
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank,
                            world_size=world)
    comm = Comm()
    problem = P.make_problem(cfg["problem"], **cfg.get("problem_kw", {}))
    spec = P.MlpSpec(cfg["widths"], seed=0)
    layout = cfg.get("multi_gpu", "columns")
    config = P.OptimizerConfig(max_iters=args.steps + 1, lam_cap=cfg["lam_cap"],
                               dense_threshold=cfg["dense_threshold"],
                               nystrom_rank=cfg.get("nystrom_rank", 64),
                               cg_max_iters=cfg.get("cg_max_iters", 500),
                               deterministic_timing=True)
    fp64_peak = 35.47 if args.profile else _fp64_peak()
    hbm_peak, hbm_src = _hbm_peak()
    theta = P.xavier_normal_params(spec)
    theta = P.ParameterVector(theta.tensor, theta.layout)
    rng = np.random.default_rng(1000)  # the same draws on every rank
    total = args.warmup + args.steps + 1
    ops_list = []
    for _ in range(total):
        ops = make_ops(layout, problem, spec, P.sample_collocation(problem, cfg["counts"], rng),
                       theta, comm, prev=ops_list[-1] if ops_list else None)
        ops.rmap._device()  # upload points and data now
        ops_list.append(ops)

    def run(first, count, theta, on_step=None):
        sub = ops_list[first:first + count]
        tr = TrainTrace(problem=problem.name, method="dngd-sharded", seed=0)
        sharded_loop(tr, lambda it: sub[min(it, count) - 1], theta,
                     replace(config, max_iters=count), comm, np.random.default_rng(7), layout,
                     on_step)
        if tr.aborted:
            raise SystemExit(f"sharded bench loop aborted: {tr.abort_reason}\n{tr.abort_traceback}")
        return tr.final_theta

    theta = run(0, args.warmup, theta)
    clocks = ClockSampler(local)
    torch.cuda.synchronize()
    dist.barrier()
    clocks.start()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def mark(it, th, step, ls):  # steps 2 .. K+1 of a K+1 step run: K whole steps
        if it == 1:
            s.record()
        if it == args.steps + 1:
            e.record()

    mark.needs_theta = False
    with timing.collect() as tm:
        theta = run(args.warmup, args.steps + 1, theta, mark)
        torch.cuda.synchronize()
        stages, counts = tm.summary_ms()
    dist.barrier()
    dev_s = s.elapsed_time(e) * 1e-3
    t = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s = float(t.item())
    clk = clocks.stop()
    # per-stage ms per step (this rank; stage timers include the collectives)
    stage_ms = {k: v / (args.steps + 1) for k, v in stages.items()}

    # -------- end to end: sharded_dngd_run (host sampling + uploads + per-step reads)
    marks = {}

    def on_step(it, th, step, ls):
        if it == args.warmup:
            torch.cuda.synchronize()
            marks["t0"] = time.perf_counter()
        if it == args.warmup + args.steps:
            torch.cuda.synchronize()
            marks["t1"] = time.perf_counter()

    on_step.needs_theta = False
    e2e = None
    if not args.profile:
        tr = sharded_dngd_run(problem, spec, replace(config, max_iters=args.warmup + args.steps),
                              seed=0, comm=comm, counts=cfg["counts"], init="xavier_normal",
                              on_step=on_step, layout=layout)
        if "t0" in marks and "t1" in marks:
            e2e_s = marks["t1"] - marks["t0"]
            t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
            m = sum(cfg["counts"])
            h2d = 8 * m * (problem.raw_dim + 1) * world  # points + data, every rank
            e2e = {"value": args.steps / e2e_s, "unit": UNIT,
                   "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": (8 * (config.line_search_points + 4)) * world,
                   "aborted": tr.aborted}
    m = sum(cfg["counts"])
    n = spec.param_count()
    roof = None
    ops0 = ops_list[0]
    gk = stages.get("gram_kernel", 0.0) / max(counts.get("gram_kernel", 1), 1) * 1e-3
    sy = stages.get("syrk", 0.0) / max(counts.get("syrk", 1), 1) * 1e-3
    emu = _emulated_gram(ops0.rmap) if gk > 0 else None
    if gk > 0 and emu is not None:
        ops, useful_ops, slices = emu
        ops, useful_ops = ops / world, useful_ops / world
        roof = {"kernel": f"dngd::k_gram_oz<{slices}> (this rank's 1/N of the tiles; emulated FP64)",
                "bound": "tensor", "achieved": ops / gk / 1e12, "peak": INT8_PEAK_TOPS,
                "unit": "TOPS (int8)", "frac": ops / gk / 1e12 / INT8_PEAK_TOPS, "traffic": None,
                "peak_source": INT8_PEAK_SOURCE,
                "algorithmic": f"{ops:.4e} int8 ops issued per rank per launch "
                               f"({useful_ops:.4e} on useful rows)"}
    elif gk > 0:
        flops = ops0.rmap.factored_gram_flops() / world
        roof = {"kernel": "dngd::k_gram_factored (this rank's 1/N of the tiles)",
                "bound": "tensor", "achieved": flops / gk / 1e12, "peak": fp64_peak,
                "unit": "TFLOP/s", "frac": flops / gk / 1e12 / fp64_peak, "traffic": None,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 DMMA)",
                "algorithmic": f"factored Gram {flops:.4e} useful FLOP per rank per launch"}
    elif sy > 0:
        flops = m * (m + 1) * ops0.rmap.ncols
        roof = {"kernel": "dngd::k_gemm_nt<128,128> (SYRK K_p = J_p J_p^T)", "bound": "tensor",
                "achieved": flops / sy / 1e12, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": flops / sy / 1e12 / fp64_peak, "traffic": None,
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 DMMA)",
                "algorithmic": f"m(m+1)n_p = {flops:.3e} FLOP per rank per launch"}
    line = {
        "metric": METRIC, "value": args.steps / dev_s, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded collocation sampling; Xavier-normal random init)",
        "config": {"workload": cfg["name"], "m": m, "n": n, "widths": list(cfg["widths"]),
                   "solver": "dense Cholesky + geodesic acceleration"
                   if m < cfg["dense_threshold"] else "Nystrom-PCG",
                   "lam_cap": cfg["lam_cap"], "line_search_points": 31,
                   "parallelism": f"{layout}-sharded J over {world} GPUs (NCCL: all-reduce of K "
                                  "or of the CG m-vector, all-gathers of v, f_vv, delta, losses)",
                   "l2": "per-step working set exceeds L2"},
        "roofline": roof, "stages_ms_per_step_rank0": stage_ms, "e2e": e2e,
        "hbm_peak_gbs": hbm_peak, "hbm_peak_source": hbm_src, "fp64_peak_tflops": fp64_peak,
        "gpu_launches": None, "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


# ------------------------------------------------------------------ CPU oracle arm


def _oracle_problem(name):
    from oracle import dngd_oracle as O

    return {"poisson2d": O.OraclePoisson2d(), "heat1d": O.OracleHeat1d(),
            "poisson5d_sin": O.OraclePoissonSin(5), "allen_cahn": O.OracleAllenCahn()}[name]


def cpu_baseline(cfg, max_seconds=25.0, warmup=1):
    """The numpy oracle (a port of the reference algorithm) on this host's cores:
    full D-NGD steps of the same workload (fresh collocation, J, Gram, Cholesky,
    GN + GA solves, 31-candidate line search, update), bounded to ~max_seconds of
    CPU work.  Where J would be large (config 3: 25 GB) the oracle forms it one
    layer block at a time (dense_dual_solve_streamed: K = sum_k J_k J_k^T) and
    evaluates the line-search candidates on all host threads."""
    from oracle import dngd_oracle as O

    cores = O._threads()
    problem = _oracle_problem(cfg["problem"])
    lc = O.LoopConfig(lam_cap=cfg["lam_cap"], dense_threshold=cfg["dense_threshold"],
                      nystrom_rank=cfg.get("nystrom_rank", 64),
                      cg_max_iters=cfg.get("cg_max_iters", 500), max_iters=1)
    m = sum(cfg["counts"])
    n = O.param_count(cfg["widths"])
    streamed = 8.0 * m * n > 2e9
    big = 8.0 * m * n > 1e10
    if big:
        warmup = 0  # one step is tens of seconds: no untimed warm-up step
    # the streamed oracle holds one layer block J_k (m x (w_k + 1) w_{k+1}) at a time
    w = cfg["widths"]
    block = max(8.0 * m * (w[k] + 1) * w[k + 1] for k in range(len(w) - 1))
    try:
        import psutil

        avail = float(psutil.virtual_memory().available)
    except Exception:  # noqa: BLE001
        avail = float("inf")
    if block > 0.5 * avail:
        return {"value": None, "unit": UNIT, "cores": cores, "kind": "port",
                "unavailable": f"one oracle step needs a {block / 1e9:.0f} GB layer block of J "
                               f"(host memory available: {avail / 1e9:.0f} GB)",
                "sample": "none"}
    times = []
    t_start = time.perf_counter()
    rng = np.random.default_rng(0)
    theta = O.xavier_normal_init(cfg["widths"], 0)
    steps_done = 0
    while True:
        classes = problem.sample(cfg["counts"], rng)
        t0 = time.perf_counter()
        if streamed and m < lc.dense_threshold:
            r, _ = O.jacobian_blocks(theta, cfg["widths"], classes)
            cur = 0.5 * float(r @ r)
            lam = O.lm_damping(cur, lc.lam_cap)
            step = O.dense_dual_solve_streamed(theta, cfg["widths"], classes, lam, True)
        else:
            r, J = O.linearize(theta, cfg["widths"], classes)
            g = J.T @ r
            cur = 0.5 * float(r @ r)
            lam = O.lm_damping(cur, lc.lam_cap)
            if m < lc.dense_threshold:
                step = O.dense_dual_solve(
                    J, g, lam, True,
                    lambda v: O.second_directional(theta, cfg["widths"], classes, v))
            else:
                step = O.pcg_step(J, g, lam, lc.nystrom_rank, lc.cg_tol, lc.cg_max_iters, rng)
            del J
        ls = O.line_search(lambda c: O.loss_many(c, cfg["widths"], classes, parallel=True),
                           theta, step.delta, cur, lc.line_search_points)
        if not ls.rejected:
            theta = theta + ls.eta * step.delta
        dt = time.perf_counter() - t0
        steps_done += 1
        if steps_done > warmup:
            times.append(dt)
        if time.perf_counter() - t_start > max_seconds and times:
            break
    v = len(times) / sum(times)
    how = ("J one layer block at a time (K = sum_k J_k J_k^T, dsyrk)" if streamed
           else "J materialised")
    return {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(times)} full oracle D-NGD step(s) of {cfg['name']} after {warmup} "
                      f"warm-up ({how}; numpy/OpenBLAS on {cores} host threads, line-search "
                      f"candidates in parallel)"}


def run_reference(args, cfg):
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    budget = float(os.environ.get("DNGD_REF_SECONDS", "150"))
    res = cpu_baseline(cfg, max_seconds=budget, warmup=min(args.warmup, 1))
    if res["value"] is None:
        print(json.dumps({"impl": "reference", "unavailable": res["unavailable"],
                          "config": {"workload": cfg["name"]}}), flush=True)
        return
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / res["value"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded collocation sampling; Xavier-normal random init)",
        "config": {"workload": cfg["name"], "m": sum(cfg["counts"]),
                   "widths": list(cfg["widths"])},
        "impl": "reference",
        "cpu_baseline": res,
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _relaunch_distributed(n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: start N ranks (one per GPU) under
    torch.distributed.run on this node and return its exit status."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=25.0)
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU (sharded) loop even at one rank (checks that path)")
    ap.add_argument("--profile", action="store_true",
                    help="timed steps only (no peak probe / e2e / CPU arm): for ncu launch lists")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 1)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch_distributed(args.gpus))
    rank, world, _ = _env_rank()
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; measuring {world} rank(s)",
              file=sys.stderr)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
