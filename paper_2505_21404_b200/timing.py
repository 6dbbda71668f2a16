"""Per-stage CUDA-event timers (off by default; bench.py turns them on).

Events are recorded on the current stream around each stage of the step, so
stage times are device times of the kernels that stage launched.
"""

from __future__ import annotations

import contextlib

from ._state import tls


def active():
    """This thread's collecting StageTimer (None = stage timing off)."""
    return tls().timer


def set_active(timer) -> None:
    tls().timer = timer


class StageTimer:
    def __init__(self):
        self.pairs = []  # (name, start_event, end_event)
        self.done = []  # (name, ms) already read (stages replayed inside a CUDA graph)

    def summary_ms(self) -> dict:
        import torch

        torch.cuda.synchronize()
        out = {}
        counts = {}
        for name, s, e in self.pairs:
            out[name] = out.get(name, 0.0) + s.elapsed_time(e)
            counts[name] = counts.get(name, 0) + 1
        for name, ms in self.done:
            out[name] = out.get(name, 0.0) + ms
            counts[name] = counts.get(name, 0) + 1
        return out, counts


@contextlib.contextmanager
def capture_into(sink: list):
    """Stage events recorded during graph capture go to `sink` as external event
    nodes (they fire on every replay); add_captured() reads them after a replay."""
    st = tls()
    prev = st.capture
    st.capture = sink
    try:
        yield
    finally:
        st.capture = prev


def add_captured(pairs):
    t = tls().timer
    if t is None:
        return
    for name, s, e in pairs:
        t.done.append((name, s.elapsed_time(e)))


@contextlib.contextmanager
def stage(name: str):
    st = tls()
    t, cap = st.timer, st.capture
    if t is None and cap is None:
        yield
        return
    import torch

    if cap is not None:
        s = torch.cuda.Event(enable_timing=True, external=True)
        e = torch.cuda.Event(enable_timing=True, external=True)
        s.record()
        try:
            yield
        finally:
            e.record()
            cap.append((name, s, e))
        return
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
    st = tls()
    prev = st.timer
    st.timer = StageTimer()
    try:
        yield st.timer
    finally:
        st.timer = prev
