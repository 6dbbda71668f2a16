"""Helpers shared by the GPU parity tests (test infrastructure)."""

import ctypes

import numpy as np
import torch

from paper_2505_21404_b200 import _lib, kernels


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device="cuda")


def class_descs(classes):
    """oracle OpClass list -> (ctypes ClassDesc array, keep-alive device tensors)."""
    arr = (_lib.ClassDesc * len(classes))()
    keep = []
    for k, c in enumerate(classes):
        d = arr[k]
        pts = dev(c.points)
        f = dev(c.f)
        keep += [pts, f]
        d.count = c.count
        d.ngrad = len(c.grad_dims)
        d.nlap = len(c.lap_dims)
        for g, gd in enumerate(c.grad_dims):
            d.grad_dims[g] = gd
            d.cg[g] = c.cg[g]
        for l, ld in enumerate(c.lap_dims):
            d.lap_grad[l] = c.grad_dims.index(ld)
        d.cu, d.cl, d.weight = c.cu, c.cl, c.weight
        d.points = pts.data_ptr()
        d.f = f.data_ptr()
        d.c3 = getattr(c, "c3", 0.0)
        if getattr(c, "inputs", None) is not None:
            inp = dev(c.inputs)
            keep.append(inp)
            d.inputs = inp.data_ptr()
        if getattr(c, "pgrad", None) is not None:
            gi = torch.as_tensor(np.ascontiguousarray(c.pgrad, dtype=np.int32), device="cuda")
            keep.append(gi)
            d.grad_idx = gi.data_ptr()
        if getattr(c, "pcoef", None) is not None:
            co = dev(c.pcoef)
            keep.append(co)
            d.coefs = co.data_ptr()
    return arr, keep


class ThreadComm:
    """Collectives between ranks that are THREADS of one process on one GPU (test
    infrastructure): host barriers plus device copies, each rank on its own stream,
    fixed rank-order summation.  No kernel ever waits on another rank's kernel --
    the ranks only meet at host barriers -- so this checks the orchestration and
    the per-rank numerics of the sharded step, not its multi-GPU performance."""

    class Shared:
        def __init__(self, world):
            import threading

            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared, rank):
        self.s = shared
        self.rank = rank
        self.world = shared.world

    def _publish(self, t):
        self.s.slots[self.rank] = t.clone()
        torch.cuda.current_stream().synchronize()
        self.s.barrier.wait()

    def _release(self):
        torch.cuda.current_stream().synchronize()
        self.s.barrier.wait()

    def allreduce_sum_(self, t):
        self._publish(t)
        acc = self.s.slots[0].clone()
        for p in range(1, self.world):
            acc += self.s.slots[p]
        t.copy_(acc)
        self._release()
        return t

    def allgather_cat(self, t_local, sizes):
        self._publish(t_local)
        out = torch.cat([self.s.slots[p][: sizes[p]] for p in range(self.world)])
        self._release()
        return out


def run_ranks(world, fn):
    """fn(comm) on `world` threads (each on its own CUDA stream); returns the results."""
    import threading

    from paper_2505_21404_b200._state import thread_stream

    shared = ThreadComm.Shared(world)
    out, errs = [None] * world, []

    def work(rank):
        try:
            with thread_stream():
                out[rank] = fn(ThreadComm(shared, rank))
                torch.cuda.current_stream().synchronize()
        except Exception:
            import traceback

            errs.append(traceback.format_exc())
            shared.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, "\n".join(errs)
    return out
