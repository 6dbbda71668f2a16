"""GPU parity of the individual CUDA kernels against the numpy oracle.

Run on a B200 (pytest -m gpu).  Every product call goes through the C ABI.
"""

import numpy as np
import pytest
import scipy.linalg

from oracle import dngd_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def K():
    from paper_2505_21404_b200 import kernels
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    return kernels


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("m,n", [(1, 5), (37, 1185), (200, 333), (300, 4099), (1020, 1185), (520, 12737)])
def test_syrk_matches_oracle(K, m, n):
    from tests.gpu_util import dev
    rng = np.random.default_rng(m + n)
    Jh = rng.normal(size=(m, n))
    ld = K.pad_ld(n)
    J = torch.zeros((m, ld), dtype=torch.float64, device="cuda")
    J[:, :n] = dev(Jh)
    Kd = K.syrk(J, n).cpu().numpy()
    Kref = O.gram(Jh)
    assert _rel(Kd, Kref) <= 1e-13  # north star: Gram rel err <= 1e-12
    assert np.array_equal(Kd, Kd.T)
    # determinism: bitwise identical on repeat
    assert np.array_equal(K.syrk(J, n).cpu().numpy(), Kd)


@pytest.mark.parametrize("M,N,Kd,lower", [(100, 64, 64, False), (257, 32, 64, False),
                                            (300, 300, 70, True), (1000, 250, 33, False)])
def test_gemm_nt(K, M, N, Kd, lower):
    from tests.gpu_util import dev
    rng = np.random.default_rng(M * N)
    A = rng.normal(size=(M, Kd))
    B = rng.normal(size=(N, Kd))
    C0 = rng.normal(size=(M, N))
    lda = K.pad_ld(Kd, 2)
    Ad = torch.zeros((M, lda), dtype=torch.float64, device="cuda"); Ad[:, :Kd] = dev(A)
    Bd = torch.zeros((N, lda), dtype=torch.float64, device="cuda"); Bd[:, :Kd] = dev(B)
    Cd = torch.zeros((M, K.pad_ld(N, 2)), dtype=torch.float64, device="cuda")
    Cd[:, :N] = dev(C0)
    K.gemm_nt(Ad, Bd, Cd[:, :N], K=Kd, alpha=-1.5, beta=0.5, lower=lower)
    ref = -1.5 * A @ B.T + 0.5 * C0
    got = Cd[:, :N].cpu().numpy()
    if lower:
        mask = np.tril(np.ones((M, N), bool))
        assert _rel(got[mask], ref[mask]) <= 1e-13
        assert np.array_equal(got[~mask], C0[~mask])
    else:
        assert _rel(got, ref) <= 1e-13


@pytest.mark.parametrize("m", [5, 64, 100, 129, 161, 1020, 2800])
def test_potrf_potrs(K, m):
    from tests.gpu_util import dev
    rng = np.random.default_rng(m)
    A = rng.normal(size=(m, m + 7))
    Km = A @ A.T / m
    lam = 1e-3
    Kd = dev(Km)
    fac = K.CholeskyFactor(m, Kd.device)
    fac.factor(Kd, lam)
    assert int(fac.info.item()) == 0
    Lref = np.linalg.cholesky(Km + lam * np.eye(m))
    Lg = np.tril(fac.L[:, :m].cpu().numpy())
    assert _rel(Lg, Lref) <= 1e-12
    b = rng.normal(size=m)
    bd = dev(b)
    fac.solve_(bd)
    y = scipy.linalg.cho_solve((Lref, True), b)
    assert _rel(bd.cpu().numpy(), y) <= 1e-10
    res = (Km + lam * np.eye(m)) @ bd.cpu().numpy() - b
    assert np.linalg.norm(res) / (np.linalg.norm(Km) * np.linalg.norm(y) + np.linalg.norm(b)) <= 1e-14


@pytest.mark.parametrize("m", [4864, 8000])
def test_potrf_panels_in_waves(K, m):
    """Panels wider than one wave of CTAs (m > 64 + 148 x 32): every CTA must read
    the unfactored diagonal block before CTA 0 writes L_pp in place (config 4's
    m = 8000 factored garbage below row 4768 before the per-panel arrival count)."""
    A = torch.randn(m, m, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(m))
    Km = A @ A.T / m + torch.eye(m, dtype=torch.float64, device="cuda")
    fac = K.CholeskyFactor(m, Km.device)
    fac.factor(Km, 0.0)
    assert int(fac.info.item()) == 0
    Lref = torch.linalg.cholesky(Km)
    L = torch.tril(fac.L[:, :m])
    assert float(torch.linalg.norm(L - Lref) / torch.linalg.norm(Lref)) <= 1e-13
    b = torch.randn(m, dtype=torch.float64, device="cuda")
    x = b.clone()
    fac.solve_(x)
    assert float(torch.linalg.norm(Km @ x - b) / torch.linalg.norm(b)) <= 1e-12


def test_potrf_reports_failing_column(K):
    from tests.gpu_util import dev
    m = 130
    Km = np.eye(m)
    Km[70, 70] = -5.0
    fac = K.CholeskyFactor(m, "cuda")
    fac.factor(dev(Km), 1e-3)
    assert int(fac.info.item()) == 71


@pytest.mark.parametrize("m,n", [(3, 10), (1020, 1185), (2800, 12737), (64, 100000)])
def test_gemv(K, m, n):
    from tests.gpu_util import dev
    rng = np.random.default_rng(n)
    Jh = rng.normal(size=(m, n))
    J = torch.zeros((m, K.pad_ld(n)), dtype=torch.float64, device="cuda")
    J[:, :n] = dev(Jh)
    y, g, x = rng.normal(size=m), rng.normal(size=n), rng.normal(size=n)
    out = K.gemv_t(J, dev(y), n, dev(g), scale=-0.25).cpu().numpy()
    assert _rel(out, -0.25 * (Jh.T @ y + g)) <= 1e-13
    add = rng.normal(size=m)
    out = K.gemv_n(J, dev(x), n, alpha=2.0, add=dev(add), beta=0.5).cpu().numpy()
    assert _rel(out, 2.0 * Jh @ x + 0.5 * add) <= 1e-13


def test_nonfinite_report_names_class_and_point():
    """dngd_nonfinite_report: the first non-finite entry's class and point
    (residuals.py:125-136 -> errors.py:14-20 NonFiniteError(class_id, point_index))."""
    import numpy as np

    import paper_2505_21404_b200 as P
    from paper_2505_21404_b200 import kernels as K

    x = torch.zeros(50, dtype=torch.float64, device="cuda")
    assert K.nonfinite_report(x, [30, 50]) is None
    x[41] = float("inf")
    x[37] = float("nan")
    assert K.nonfinite_report(x, [30, 50]) == (1, 7)
    prob = P.make_problem("poisson2d")
    colloc = prob.sample((20, 8), np.random.default_rng(0))
    colloc.classes[1].points[5, 0] = np.nan
    rmap = P.PinnResidualMap(prob, P.MlpSpec((2, 8, 1)), colloc)
    theta = P.xavier_normal_params(P.MlpSpec((2, 8, 1)))
    with pytest.raises(P.NonFiniteError) as ei:
        rmap.residual_batch(theta)
    assert ei.value.class_id == "boundary" and ei.value.point_index == 5
