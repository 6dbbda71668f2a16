"""GPU parity of the PINN residual-map kernels (assembly, f_vv, loss_many)."""

import numpy as np
import pytest

from oracle import dngd_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CASES = [
    ("poisson2d", O.OraclePoisson2d(), (2, 32, 32, 1), (90, 30)),
    ("heat1d", O.OracleHeat1d(), (2, 64, 64, 64, 64, 1), (60, 20, 20)),
    ("poisson5d", O.OraclePoissonSin(5), (5, 32, 32, 32, 32, 1), (40, 12)),
    ("poisson5d_wide", O.OraclePoissonSin(5), (5, 128, 96, 1), (20, 10)),
    # emulated GEMMs through the fused line-search maps (k_chan_slice, k_tanh_head)
    ("poisson5d_deep_wide", O.OraclePoissonSin(5), (5, 128, 128, 128, 1), (20, 8)),
    # nch = 12 > 8: the unfused emulated line search (k_tanh_fwd + slicing, k_head)
    ("poisson10d_wide", O.OraclePoissonSin(10), (10, 128, 128, 1), (24, 8)),
    # reference Allen-Cahn: periodic input embedding + cubic reaction term
    ("allen_cahn", O.OracleAllenCahn(), (3, 32, 32, 32, 1), (60, 20)),
    ("allen_cahn_wide", O.OracleAllenCahn(), (3, 160, 96, 1), (30, 10)),
    # reference PoissonBallStde: per-point derivative subsets + per-point coefficients
    ("stde", O.OraclePoissonBallStde(10, 3), (10, 16, 16, 1), (40,)),
    ("stde_wide", O.OraclePoissonBallStde(10, 6), (10, 160, 96, 1), (24,)),
]

# large input dimension: x W0 runs as a split-K tensor-core GEMM (input_gemm) and
# J's input block through k_jwrite_in; 150 points = a full and a ragged 128-row tile
BIG_DIN = [
    ("stde_din600", O.OraclePoissonBallStde(600, 4), (600, 64, 32, 1), (150,)),
    ("stde_din1000_wide", O.OraclePoissonBallStde(1000, 3), (1000, 160, 1), (40,)),
    # odd din below the GEMM threshold: loop input layer and the k_xx_dot Gram
    ("stde_din25", O.OraclePoissonBallStde(25, 4), (25, 32, 32, 1), (70,)),
]

# edge sizes: one point per class, a ragged 65-row class next to a 1-point class,
# classes that fill whole 64-row G-tiles exactly
EDGE = [
    ("single_points", O.OracleHeat1d(), (2, 8, 8, 1), (1, 1, 1)),
    ("ragged_65_1", O.OraclePoisson2d(), (2, 16, 16, 1), (65, 1)),
    ("full_tiles", O.OraclePoisson2d(), (2, 16, 1), (64, 64)),
]


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_2505_21404_b200 import kernels
    return kernels


def _setup(K, problem, widths, counts, seed):
    from tests.gpu_util import class_descs, dev
    rng = np.random.default_rng(seed)
    classes = problem.sample(counts, rng)
    theta = O.xavier_normal_init(widths, seed)
    arr, keep = class_descs(classes)
    mlp = K.mlp_desc(widths)
    nb = K.pinn_workspace_bytes(mlp, arr, len(classes), 31)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    return classes, theta, arr, keep, mlp, ws, dev(theta)


@pytest.mark.parametrize("name,problem,widths,counts", CASES + BIG_DIN + EDGE)
def test_assemble_matches_oracle(K, name, problem, widths, counts):
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 3)
    r_ref, J_ref = O.linearize(theta, widths, classes)
    m, n = J_ref.shape
    r = torch.empty(m, dtype=torch.float64, device="cuda")
    J = torch.full((m, K.pad_ld(n)), np.nan, dtype=torch.float64, device="cuda")
    K.assemble(mlp, th, arr, len(classes), r, J, 0, n, ws)
    torch.cuda.synchronize()
    assert _rel(r.cpu().numpy(), r_ref) <= 1e-12
    Jg = J[:, :n].cpu().numpy()
    assert np.all(np.isfinite(Jg))
    assert _rel(Jg, J_ref) <= 1e-12
    # column-sharded assembly (multi-GPU layout): an odd and an even split
    for c0, c1 in [(0, n // 3), (n // 3 + 1, n), (2, n - 3)]:
        c0 -= c0 % 2
        Js = torch.full((m, K.pad_ld(c1 - c0)), np.nan, dtype=torch.float64, device="cuda")
        K.assemble(mlp, th, arr, len(classes), r, Js, c0, c1, ws)
        assert np.array_equal(Js[:, : c1 - c0].cpu().numpy(), Jg[:, c0:c1])


@pytest.mark.parametrize("name,problem,widths,counts", CASES + BIG_DIN + EDGE)
def test_fvv_matches_oracle(K, name, problem, widths, counts):
    from tests.gpu_util import dev
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 4)
    v = np.random.default_rng(9).normal(size=theta.size)
    ref = O.second_directional(theta, widths, classes, v)
    out = torch.empty(ref.size, dtype=torch.float64, device="cuda")
    K.fvv(mlp, th, dev(v), arr, len(classes), out, ws)
    assert _rel(out.cpu().numpy(), ref) <= 1e-11


@pytest.mark.parametrize("name,problem,widths,counts", CASES + BIG_DIN + EDGE)
def test_loss_many_matches_oracle(K, name, problem, widths, counts):
    from tests.gpu_util import dev
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 5)
    delta = 0.3 * np.random.default_rng(10).normal(size=theta.size)
    etas = 2.0 ** -np.arange(31, dtype=np.float64)
    cands = theta[None, :] + etas[:, None] * delta[None, :]
    ref = O.loss_many(cands, widths, classes)
    out = torch.empty(31, dtype=torch.float64, device="cuda")
    K.loss_many(mlp, th, dev(delta), dev(etas), 31, arr, len(classes), out, ws)
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=1e-12)
    # explicit candidate stack
    out2 = torch.empty(31, dtype=torch.float64, device="cuda")
    K.loss_many(mlp, dev(cands), None, None, 31, arr, len(classes), out2, ws)
    np.testing.assert_allclose(out2.cpu().numpy(), ref, rtol=1e-12)


@pytest.mark.parametrize("name,problem,widths,counts", CASES + BIG_DIN + EDGE + [
    ("poisson2d_cfg1", O.OraclePoisson2d(), (2, 32, 32, 1), (900, 120)),
    ("heat1d_cfg2", O.OracleHeat1d(), (2, 64, 64, 64, 64, 1), (500, 100, 100)),
])
def test_gram_factored_matches_jjt(K, name, problem, widths, counts):
    """Factored Gram (no J) == oracle J J^T to 1e-12 (north-star Gram tolerance)."""
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 6)
    r_ref, J_ref = O.linearize(theta, widths, classes)
    K_ref = O.gram(J_ref)
    m = J_ref.shape[0]
    r = torch.empty(m, dtype=torch.float64, device="cuda")
    Kd = torch.full((m, m), np.nan, dtype=torch.float64, device="cuda")
    K.gram_factored(mlp, th, arr, len(classes), r, Kd, ws)
    Kg = Kd.cpu().numpy()
    assert np.all(np.isfinite(Kg))
    assert np.array_equal(Kg, Kg.T)
    assert _rel(Kg, K_ref) <= 1e-12
    assert _rel(r.cpu().numpy(), r_ref) <= 1e-12


@pytest.mark.parametrize("name,problem,widths,counts", CASES + BIG_DIN + EDGE)
def test_jt_factored_matches_oracle(K, name, problem, widths, counts):
    """J^T w from the activations (no J) == oracle J^T w (tiled and wide paths)."""
    from tests.gpu_util import dev
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 7)
    r_ref, J_ref = O.linearize(theta, widths, classes)
    m, n = J_ref.shape
    w = np.random.default_rng(11).normal(size=m)
    r = torch.empty(m, dtype=torch.float64, device="cuda")
    K.activations(mlp, th, arr, len(classes), r, ws)
    scratch = torch.empty(K.jt_workspace_bytes(mlp, arr, len(classes)), dtype=torch.uint8,
                          device="cuda")
    out = torch.full((n,), np.nan, dtype=torch.float64, device="cuda")
    K.jt_factored(mlp, arr, len(classes), dev(w), -0.5, out, ws, scratch)
    assert _rel(out.cpu().numpy(), -0.5 * (J_ref.T @ w)) <= 1e-12
    assert _rel(r.cpu().numpy(), r_ref) <= 1e-12


@pytest.mark.parametrize("nparts", [2, 3, 8])
def test_gram_factored_parts_sum_to_full(K, nparts):
    """Tile-sharded Gram (multi-GPU layout): the parts written by each rank are
    disjoint and sum to the full K, bit for bit."""
    problem, widths, counts = O.OracleHeat1d(), (2, 32, 32, 1), (300, 60, 60)
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 12)
    m = sum(c.count for c in classes)
    r = torch.empty(m, dtype=torch.float64, device="cuda")
    full = torch.empty((m, m), dtype=torch.float64, device="cuda")
    K.gram_factored(mlp, th, arr, len(classes), r, full, ws)
    acc = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    cover = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    for p in range(nparts):
        part = torch.zeros((m, m), dtype=torch.float64, device="cuda")
        sentinel = torch.full((m, m), np.nan, dtype=torch.float64, device="cuda")
        K.gram_factored(mlp, th, arr, len(classes), r, part, ws, p, nparts)
        K.gram_factored(mlp, th, arr, len(classes), r, sentinel, ws, p, nparts)
        cover += (~torch.isnan(sentinel)).to(torch.int32)
        acc += part
    assert int(cover.min()) == 1 and int(cover.max()) == 1  # every entry written exactly once
    assert torch.equal(acc, full)


@pytest.mark.parametrize("name,problem,widths,counts", CASES + BIG_DIN + EDGE)
def test_jvp_factored_matches_oracle(K, name, problem, widths, counts):
    """J v from first-order forward t-jets (no J) == oracle J v."""
    from tests.gpu_util import dev
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 8)
    _, J_ref = O.linearize(theta, widths, classes)
    v = np.random.default_rng(13).normal(size=theta.size)
    out = torch.full((J_ref.shape[0],), np.nan, dtype=torch.float64, device="cuda")
    K.jvp_factored(mlp, th, dev(v), arr, len(classes), out, ws)
    assert _rel(out.cpu().numpy(), J_ref @ v) <= 1e-12


@pytest.mark.parametrize("name,problem,widths,counts", BIG_DIN[:2])
def test_act_reuse_of_input_products(K, name, problem, widths, counts):
    """f_vv and the line-search losses reusing x W0(theta) from the activation pass at
    theta are bit-identical to the self-contained calls (and match the oracle)."""
    from tests.gpu_util import dev
    classes, theta, arr, keep, mlp, ws, th = _setup(K, problem, widths, counts, 14)
    m = sum(c.count for c in classes)
    act = torch.empty_like(ws)
    r = torch.empty(m, dtype=torch.float64, device="cuda")
    K.activations(mlp, th, arr, len(classes), r, act)
    v = dev(np.random.default_rng(15).normal(size=theta.size))
    a = torch.empty(m, dtype=torch.float64, device="cuda")
    b = torch.empty(m, dtype=torch.float64, device="cuda")
    K.fvv(mlp, th, v, arr, len(classes), a, ws)
    K.fvv(mlp, th, v, arr, len(classes), b, ws, act)
    assert torch.equal(a, b)
    etas = dev(2.0 ** -np.arange(31, dtype=np.float64))
    la = torch.empty(31, dtype=torch.float64, device="cuda")
    lb = torch.empty(31, dtype=torch.float64, device="cuda")
    K.loss_many(mlp, th, v, etas, 31, arr, len(classes), la, ws)
    K.loss_many(mlp, th, v, etas, 31, arr, len(classes), lb, ws, act)
    assert torch.equal(la, lb)
    cands = theta[None, :] + (2.0 ** -np.arange(31))[:, None] * v.cpu().numpy()[None, :]
    np.testing.assert_allclose(lb.cpu().numpy(), O.loss_many(cands, widths, classes), rtol=1e-12)
