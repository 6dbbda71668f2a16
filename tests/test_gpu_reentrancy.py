"""Reentrancy: the reference service runs seeds concurrently on
threads (service.py:125-128).  Two dngd_run calls on two threads must give the
same traces, bit for bit, as the same calls run one after the other -- every
workspace, Gram / factor buffer, captured CUDA graph, activation record and
C-ABI context is per thread, and each thread runs on its own stream."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2505_21404_b200 as P
    return P


CASES = [
    # dense, pipelined CUDA-graph loop (factored Gram, J-free)
    ("heat1d", (2, 24, 24, 1), (120, 30, 30), dict(lam_cap=1e-3)),
    # dense, materialised J + SYRK
    ("poisson2d", (2, 16, 16, 1), (90, 30), dict(lam_cap=1e-3)),
    # Nystrom-PCG
    ("poisson2d", (2, 16, 16, 1), (90, 30), dict(lam_cap=1e-3, dense_threshold=10,
                                                  nystrom_rank=16, cg_max_iters=100)),
]


def _run(P, case, seed):
    pname, widths, counts, cfg = case
    config = P.OptimizerConfig(max_iters=6, deterministic_timing=True, **cfg)
    tr = P.dngd_run(P.make_problem(pname), P.MlpSpec(widths), config, seed, counts=counts,
                    init="xavier_normal")
    torch.cuda.current_stream().synchronize()  # not a device-wide sync: others may be capturing
    return ([(r.loss, r.rel_l2, r.eta, r.lam, r.cg_iterations) for r in tr.rows],
            tr.final_theta.data.copy(),
            (tr.abort_reason + "\n" + (tr.abort_traceback or "")) if tr.aborted else None)


@pytest.mark.parametrize("case", range(len(CASES)))
def test_concurrent_seeds_match_sequential(P, case):
    seeds = (3, 4, 5)
    seq = {s: _run(P, CASES[case], s) for s in seeds}
    out, errs = {}, []

    def work(s):
        try:
            out[s] = _run(P, CASES[case], s)
        except Exception:  # surfaced below
            import traceback

            errs.append(traceback.format_exc())

    threads = [threading.Thread(target=work, args=(s,)) for s in seeds]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for s in seeds:
        if s in out and out[s][2] is not None:
            print(out[s][2])
    for e in errs:
        print(e)
    assert not errs, errs
    for s in seeds:
        assert seq[s][2] is None and out[s][2] is None, (seq[s][2], out[s][2])
        assert out[s][0] == seq[s][0]  # every row, bit for bit
        np.testing.assert_array_equal(out[s][1], seq[s][1])


def test_thread_state_is_private(P):
    from paper_2505_21404_b200 import _lib
    from paper_2505_21404_b200._state import tls

    mine = tls()
    seen = {}

    def work():
        seen["state"] = tls()
        seen["ctx"] = _lib.ctx().value

    t = threading.Thread(target=work)
    t.start()
    t.join()
    assert seen["state"] is not mine
    assert seen["ctx"] != _lib.ctx().value
