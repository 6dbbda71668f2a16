"""GPU checks of the column-sharded path on one device (no cross-rank waiting):
per-shard assembly + SYRK sums to the full Gram, and the world-1 sharded step
equals dense_dual_solve."""

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


def test_shard_grams_sum_to_full_gram(P):
    from paper_2505_21404_b200 import kernels as K
    from paper_2505_21404_b200.sharded import column_ranges
    prob = P.make_problem("heat1d")
    spec = P.MlpSpec((2, 64, 64, 64, 64, 1))
    colloc = prob.sample((300, 60, 60), np.random.default_rng(0))
    theta = P.xavier_normal_params(spec)
    full = P.assemble_gramian(P.PinnResidualMap(prob, spec, colloc), theta).K
    for world in (2, 3, 8):
        acc = None
        for c0, c1 in column_ranges(spec.param_count(), world):
            mp = P.PinnResidualMap(prob, spec, colloc, col_range=(c0, c1))
            _, J = mp.linearize_t(theta)
            Kp = K.syrk(J, mp.ncols)
            acc = Kp.clone() if acc is None else acc + Kp
        rel = np.linalg.norm(acc.cpu().numpy() - full) / np.linalg.norm(full)
        assert rel <= 1e-13, (world, rel)


def test_world1_sharded_step_equals_dense_solve(P):
    from paper_2505_21404_b200.sharded import (CudaShardOps, LocalComm, column_ranges,
                                               sharded_dense_step)
    prob = P.make_problem("heat1d")
    spec = P.MlpSpec((2, 32, 32, 32, 1))
    colloc = prob.sample((200, 40, 40), np.random.default_rng(1))
    theta = P.xavier_normal_params(spec)
    ranges = column_ranges(spec.param_count(), 1)
    rmap = P.PinnResidualMap(prob, spec, colloc, col_range=ranges[0])
    res = sharded_dense_step(CudaShardOps(rmap, theta, ranges), LocalComm(), 1e-3, True)
    ref_map = P.PinnResidualMap(prob, spec, colloc)
    _, g = ref_map.residuals_and_gradient(theta)
    ref = P.dense_dual_solve(ref_map, theta, g, lam=1e-3, use_ga=True)
    d = res["delta"].cpu().numpy()
    assert np.linalg.norm(d - ref.delta.data) / np.linalg.norm(ref.delta.data) <= 1e-9
    assert res["lambda_used"] == ref.lambda_used
