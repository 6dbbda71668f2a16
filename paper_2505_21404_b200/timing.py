"""Per-stage CUDA-event timers (off by default; bench.py turns them on).

Events are recorded on the current stream around each stage of the step, so
stage times are device times of the kernels that stage launched.
"""

from __future__ import annotations

import contextlib

_ACTIVE = None


class StageTimer:
    def __init__(self):
        self.pairs = []  # (name, start_event, end_event)

    def summary_ms(self) -> dict:
        import torch

        torch.cuda.synchronize()
        out = {}
        counts = {}
        for name, s, e in self.pairs:
            out[name] = out.get(name, 0.0) + s.elapsed_time(e)
            counts[name] = counts.get(name, 0) + 1
        return out, counts


@contextlib.contextmanager
def stage(name: str):
    t = _ACTIVE
    if t is None:
        yield
        return
    import torch

    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    try:
        yield
    finally:
        e.record()
        t.pairs.append((name, s, e))


@contextlib.contextmanager
def collect():
    global _ACTIVE
    prev = _ACTIVE
    _ACTIVE = StageTimer()
    try:
        yield _ACTIVE
    finally:
        _ACTIVE = prev
