"""Per-thread host state of the Python layer (reentrancy).

The reference service fans seeds out over threads (service.py:125-128), so
nothing here is module-global: every thread gets its own workspaces, Gram and
factor buffers, captured CUDA graphs, activation bookkeeping and stage timers,
next to its own C-ABI context (_lib.ctx) -- and, off the main thread, its own
CUDA stream (thread_stream)."""

from __future__ import annotations

import contextlib
import threading

_tls = threading.local()


class ThreadState:
    def __init__(self):
        self.ws = {}  # kernels.workspace tables: tag -> Workspace
        self.ws_stack = []  # private tables of a CUDA graph being built
        self.gram_buf = {}  # solver._gram_buffer
        self.owned = []  # solver: buffer tables owned by a graph under construction
        self.factor_cache = {}  # solver._Factor
        self.graph_cache = {}  # solver._DenseGraph
        self.etas = {}  # line-search step sizes on the device
        self.act_state = {}  # residuals: which (theta, map) the activation workspace holds
        self.timer = None  # timing.StageTimer collecting this thread's stages
        self.capture = None  # timing: sink for stage events while capturing a graph
        self.stream = None  # the thread's own CUDA stream (non-main threads)
        self._capture_stream = None

    def capture_stream(self):
        """Stream for this thread's CUDA-graph captures (torch's default capture
        stream is one per process: two threads capturing at once would share it)."""
        if self._capture_stream is None:
            import torch

            self._capture_stream = torch.cuda.Stream()
        return self._capture_stream


def tls() -> ThreadState:
    s = getattr(_tls, "s", None)
    if s is None:
        s = _tls.s = ThreadState()
    return s


@contextlib.contextmanager
def graph_capture(graph, pool=None):
    """Capture CUDA work into `graph` on this thread's capture stream.

    torch.cuda.graph's context manager synchronises the whole device and empties
    the allocator cache on entry -- both break a capture running on another
    thread -- so the capture is begun directly, in thread-local error mode (only
    this thread's unsafe calls are refused), after the capture stream has waited
    for the caller's stream; the caller's stream then waits for the capture
    stream (graph warm-up work must be ordered, replays run on the caller's stream)."""
    import torch

    st = tls()
    cap = st.capture_stream()
    cur = torch.cuda.current_stream()
    cap.wait_stream(cur)
    with torch.cuda.stream(cap):
        graph.capture_begin(pool=pool, capture_error_mode="thread_local")
        try:
            yield graph
        finally:
            graph.capture_end()
    cur.wait_stream(cap)


@contextlib.contextmanager
def thread_stream():
    """Run the body on this thread's own CUDA stream when called off the main thread
    on the default stream (two threads on the legacy stream would serialise and
    could not capture graphs independently); the caller's stream then waits for
    the work, so results are ordered for it as if run in place."""
    import torch

    if threading.current_thread() is threading.main_thread():
        yield
        return
    cur = torch.cuda.current_stream()
    if cur != torch.cuda.default_stream():
        yield
        return
    st = tls()
    if st.stream is None:
        st.stream = torch.cuda.Stream()
    st.stream.wait_stream(cur)
    try:
        with torch.cuda.stream(st.stream):
            yield
    finally:
        cur.wait_stream(st.stream)
