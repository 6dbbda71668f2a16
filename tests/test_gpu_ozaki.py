"""Emulated-FP64 GEMM on the int8 tensor cores (ozaki.cu, dngd_oz_gemm_nt)
against the FP64 product: the Ozaki slices must reproduce A B^T to FP64-level
accuracy (tolerance written per slice count below)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def K():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    from paper_2505_21404_b200 import kernels as K
    return K


def _ref(A, B):
    # exact-ish reference: long double accumulation on the host
    return (A.astype(np.longdouble) @ B.astype(np.longdouble).T).astype(np.float64)


@pytest.mark.parametrize("M,N,Kd", [(128, 64, 32), (300, 200, 512), (1, 7, 5), (257, 130, 1000)])
@pytest.mark.parametrize("slices", [7, 6])
def test_oz_gemm_matches_fp64(K, M, N, Kd, slices):
    rng = np.random.default_rng(M * 7 + N + Kd)
    A = rng.standard_normal((M, Kd)) * np.exp(rng.uniform(-3, 3, size=(M, 1)))
    B = rng.standard_normal((N, Kd)) * np.exp(rng.uniform(-3, 3, size=(N, 1)))
    At = torch.as_tensor(A, device="cuda")
    Bt = torch.as_tensor(B, device="cuda")
    C = K.oz_gemm_nt(At, Bt, slices=slices).cpu().numpy()
    R = _ref(A, B)
    # normwise per entry: |C - R| <= tol * |a_i| |b_j|
    bound = np.outer(np.linalg.norm(A, axis=1), np.linalg.norm(B, axis=1))
    err = np.max(np.abs(C - R) / bound)
    tol = {7: 1e-15, 6: 1e-13}[slices]
    print(f"M={M} N={N} K={Kd} S={slices}: max normwise err {err:.2e}")
    assert err <= tol
    # and against the FP64 tensor-core GEMM of the library
    if Kd % 2:
        return  # the FP64 TMA GEMM needs an even leading dimension
    D = K.gemm_nt(At, Bt).cpu().numpy()
    assert np.max(np.abs(C - D) / bound) <= tol + 1e-15


def test_oz_gemm_nonfinite_row(K):
    A = torch.ones((130, 40), dtype=torch.float64, device="cuda")
    B = torch.ones((70, 40), dtype=torch.float64, device="cuda")
    A[3, 5] = float("nan")
    C = K.oz_gemm_nt(A, B).cpu().numpy()
    assert np.isnan(C[3]).all()
    assert np.isfinite(np.delete(C, 3, axis=0)).all()
    assert np.allclose(np.delete(C, 3, axis=0), 40.0, rtol=0, atol=1e-13)


def test_oz_gemm_zero_rows(K):
    A = torch.zeros((128, 64), dtype=torch.float64, device="cuda")
    B = torch.randn((64, 64), dtype=torch.float64, device="cuda")
    C = K.oz_gemm_nt(A, B).cpu().numpy()
    assert (C == 0).all()


# ---------------------------------------------------------------- factored Gram
from oracle import dngd_oracle as O  # noqa: E402

GRAM_CASES = [
    ("poisson2d", O.OraclePoisson2d(), (2, 32, 32, 1), (90, 30)),
    ("heat1d", O.OracleHeat1d(), (2, 64, 64, 64, 64, 1), (60, 20, 20)),
    ("poisson5d", O.OraclePoissonSin(5), (5, 32, 32, 32, 32, 1), (40, 12)),
    ("poisson5d_wide", O.OraclePoissonSin(5), (5, 128, 96, 1), (20, 10)),
    ("allen_cahn_wide", O.OraclePoissonSin(5), (5, 160, 96, 1), (30, 10)),
    ("allen_cahn", O.OracleAllenCahn(), (3, 32, 32, 32, 1), (60, 20)),
    ("stde", O.OraclePoissonBallStde(10, 3), (10, 16, 16, 1), (40,)),
    ("single_points", O.OracleHeat1d(), (2, 8, 8, 1), (1, 1, 1)),
    ("ragged_65_1", O.OraclePoisson2d(), (2, 16, 16, 1), (65, 1)),
    # nch = 7 interior (18 points per 128-row tile) at the config-3 structure
    ("cfg3_structure", O.OraclePoissonSin(5), (5, 256, 256, 1), (200, 60)),
]


def _act_setup(K, problem, widths, counts, seed):
    from tests.gpu_util import class_descs, dev
    rng = np.random.default_rng(seed)
    classes = problem.sample(counts, rng)
    theta = O.xavier_normal_init(widths, seed)
    arr, keep = class_descs(classes)
    mlp = K.mlp_desc(widths)
    nb = K.pinn_workspace_bytes(mlp, arr, len(classes), 31)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    m = sum(c.count for c in classes)
    r = torch.empty(m, dtype=torch.float64, device="cuda")
    K.activations(mlp, dev(theta), arr, len(classes), r, ws)
    return classes, theta, arr, keep, mlp, ws, m


@pytest.mark.parametrize("name,problem,widths,counts", GRAM_CASES)
@pytest.mark.parametrize("slices", [7, 6])
def test_gram_emulated_matches_oracle(K, name, problem, widths, counts, slices):
    """Emulated-FP64 factored Gram (int8 tcgen05) == oracle J J^T to 1e-12 (the
    north-star Gram tolerance) and to the FP64 DMMA kernel at the FP64 rounding level."""
    classes, theta, arr, keep, mlp, ws, m = _act_setup(K, problem, widths, counts, 21)
    _, J_ref = O.linearize(theta, widths, classes)
    K_ref = O.gram(J_ref)
    Ke = torch.full((m, m), np.nan, dtype=torch.float64, device="cuda")
    K.gram_factored_act(mlp, arr, len(classes), Ke, ws, slices=slices)
    Kd = torch.full((m, m), np.nan, dtype=torch.float64, device="cuda")
    K.gram_factored_act(mlp, arr, len(classes), Kd, ws, slices=0)
    Kg, Kdm = Ke.cpu().numpy(), Kd.cpu().numpy()
    assert np.all(np.isfinite(Kg))
    assert np.array_equal(Kg, Kg.T)
    rel = np.linalg.norm(Kg - K_ref) / np.linalg.norm(K_ref)
    rel_d = np.linalg.norm(Kg - Kdm) / np.linalg.norm(Kdm)
    print(f"{name} S={slices}: vs oracle {rel:.2e}, vs DMMA {rel_d:.2e}")
    assert rel <= 1e-12
    assert rel_d <= {7: 2e-15, 6: 1e-13}[slices]
    # deterministic: a second launch is bit-identical
    Ke2 = torch.empty_like(Ke)
    K.gram_factored_act(mlp, arr, len(classes), Ke2, ws, slices=slices)
    assert torch.equal(Ke, Ke2)


@pytest.mark.parametrize("nparts", [2, 3, 8])
def test_gram_emulated_parts_sum_to_full(K, nparts):
    """Tile-sharded emulated Gram: parts disjoint, every entry written once, sum
    bit-equal to the full K."""
    classes, theta, arr, keep, mlp, ws, m = _act_setup(K, O.OraclePoissonSin(5), (5, 128, 128, 1),
                                                       (150, 40), 13)
    full = torch.empty((m, m), dtype=torch.float64, device="cuda")
    K.gram_factored_act(mlp, arr, len(classes), full, ws, slices=6)
    acc = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    cover = torch.zeros((m, m), dtype=torch.int32, device="cuda")
    for p in range(nparts):
        part = torch.zeros((m, m), dtype=torch.float64, device="cuda")
        sentinel = torch.full((m, m), np.nan, dtype=torch.float64, device="cuda")
        K.gram_factored_act(mlp, arr, len(classes), part, ws, p, nparts, slices=6)
        K.gram_factored_act(mlp, arr, len(classes), sentinel, ws, p, nparts, slices=6)
        cover += (~torch.isnan(sentinel)).to(torch.int32)
        acc += part
    assert int(cover.min()) == 1 and int(cover.max()) == 1
    assert torch.equal(acc, full)


def test_gram_emulated_rejects_8_slices(K):
    """8 digits would need 235 KB of shared memory in the Gram kernel: refused loudly."""
    from paper_2505_21404_b200.errors import DngdError
    classes, theta, arr, keep, mlp, ws, m = _act_setup(K, O.OraclePoisson2d(), (2, 32, 32, 1),
                                                       (20, 8), 3)
    Ke = torch.empty((m, m), dtype=torch.float64, device="cuda")
    with pytest.raises(DngdError):
        K.gram_factored_act(mlp, arr, len(classes), Ke, ws, slices=8)


COLS_CASES = [
    ("heat1d_w128", O.OracleHeat1d(), (2, 128, 128, 128, 1), (150, 40, 40)),
    ("cfg3_structure", O.OraclePoissonSin(5), (5, 256, 256, 1), (120, 40)),
    ("cfg5_structure", O.OraclePoisson2d(), (2, 256, 256, 256, 1), (400, 60)),
]


@pytest.mark.parametrize("name,problem,widths,counts", COLS_CASES)
def test_gram_cols_emulated_matches_full_gram(K, name, problem, widths, counts):
    """Nystrom sketch columns K[:, I] on the int8 engine (gram_oz.cuh rect mode:
    full activations as row tiles, gathered landmark activations as column tiles)
    against the emulated full Gram's columns and the oracle's J J_I^T."""
    classes, theta, arr, keep, mlp, ws, m = _act_setup(K, problem, widths, counts, 3)
    rng = np.random.default_rng(5)
    ell = min(m - 1, 97)
    landmarks = np.sort(rng.choice(m, size=ell, replace=False)).astype(np.int64)
    Kf = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    K.gram_factored_act(mlp, arr, len(classes), Kf, ws, slices=6)
    Kc = torch.full((m, ell + ell % 2), float("nan"), dtype=torch.float64, device="cuda")
    K.gram_factored_cols(mlp, arr, len(classes), landmarks, Kc, ws)
    torch.cuda.synchronize()
    kc = Kc[:, :ell].cpu().numpy()
    kf = Kf.cpu().numpy()[:, landmarks]
    assert np.isfinite(kc).all()
    assert np.linalg.norm(kc - kf) / np.linalg.norm(kf) <= 1e-14
    r, J = O.linearize(theta, widths, classes)
    ko = J @ J[landmarks].T
    assert np.linalg.norm(kc - ko) / np.linalg.norm(ko) <= 1e-12
