"""CPU-only tests: the C-ABI library loads and exports the header's symbols, and
the host logic (config schema, damping, line search, sampling, problem operators)
matches the reference semantics.  No kernel is launched here."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import dngd_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "dngd_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dngd_\w+)\(", text, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    from paper_2505_21404_b200 import _build, _lib

    if not os.path.exists(_lib.LIB_PATH):
        _build.build_library()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = _header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.dngd_version() == 1


def test_ctypes_struct_layout_matches_header():
    from paper_2505_21404_b200 import _lib

    # int64 count, 2 ints, 12 ints, 12 ints, 12 doubles, 3 doubles, 2 pointers
    assert ctypes.sizeof(_lib.ClassDesc) == 8 + 8 + 48 + 48 + 96 + 24 + 16 + 16 + 16
    assert ctypes.sizeof(_lib.MlpDesc) == 4 * 10


def test_optimizer_config_validation():
    from paper_2505_21404_b200 import ConfigError, OptimizerConfig

    OptimizerConfig(max_iters=3)
    with pytest.raises(ConfigError):
        OptimizerConfig()
    with pytest.raises(ConfigError):
        OptimizerConfig(max_iters=3, wall_seconds=1.0)
    with pytest.raises(ConfigError):
        OptimizerConfig(max_iters=3, lam_cap=0.0)
    with pytest.raises(ConfigError):
        OptimizerConfig(max_iters=3, dense_threshold=0)
    with pytest.raises(ConfigError):
        OptimizerConfig(max_iters=3, nystrom_rank=0)


def test_damping_table():
    from paper_2505_21404_b200 import DomainError, lm_damping

    assert lm_damping(0.3, 1e-5) == 1e-5
    assert lm_damping(1e-7, 1e-5) == 1e-7
    assert lm_damping(0.0, 1e-5) == 1e-12
    with pytest.raises(DomainError):
        lm_damping(-1.0, 1e-5)


def test_line_search_semantics():
    from paper_2505_21404_b200 import line_search

    res = line_search(lambda c: (c[:, 0] - 1.0) ** 2 + 0.3, np.zeros(1), np.ones(1), 10.0)
    assert res.eta == 1.0 and not res.rejected and not res.degraded
    assert line_search(lambda c: c[:, 0], np.zeros(1), np.ones(1), 0.0).eta == 2.0**-30
    assert line_search(lambda c: np.full(c.shape[0], 7.0), np.zeros(1), np.ones(1), 8.0).eta == 1.0
    res = line_search(lambda c: 5.0 + c[:, 0], np.zeros(1), np.ones(1), 1.0)
    assert res.degraded and not res.rejected
    res = line_search(lambda c: np.full(c.shape[0], np.nan), np.zeros(1), np.ones(1), 1.0)
    assert res.rejected and res.eta is None

    def lm(c):
        out = c[:, 0].copy()
        out[out < 0.25] = np.inf
        return out

    assert line_search(lm, np.zeros(1), np.ones(1), 1.0).eta == 0.25
    seen = []
    line_search(lambda c: seen.append(c.shape[0]) or np.arange(c.shape[0], dtype=float),
                np.zeros(2), np.ones(2), 0.0)
    assert seen == [31]


@pytest.mark.parametrize("name,oracle,counts", [
    ("poisson2d", O.OraclePoisson2d(), (50, 20)),
    ("heat1d", O.OracleHeat1d(), (50, 20, 20)),
    ("poisson5d_sin", O.OraclePoissonSin(5), (40, 10)),
])
def test_sampling_and_operators_match_oracle(name, oracle, counts):
    """Host sampling consumes the Generator exactly like the oracle/reference, and the
    class operators and data terms describe the same residuals."""
    from paper_2505_21404_b200 import make_problem

    prob = make_problem(name)
    a = prob.sample(counts, np.random.default_rng(7))
    b = oracle.sample(counts, np.random.default_rng(7))
    assert [c.class_id for c in a.classes] == [c.class_id for c in b]
    for ca, cb in zip(a.classes, b):
        assert np.array_equal(ca.points, cb.points)
        assert ca.weight == cb.weight
        op = prob.class_operator(ca.class_id)
        assert (op.cu, tuple(op.grad_dims), tuple(op.cg), tuple(op.lap_dims), op.cl) == (
            cb.cu, tuple(cb.grad_dims), tuple(cb.cg), tuple(cb.lap_dims), cb.cl)
        np.testing.assert_array_equal(prob.class_data(ca), cb.f)


def test_reference_problems_exact_solutions_annihilate_residuals():
    """test_problems.py:40-66 style: u* zeroes every class residual (FD derivatives)."""
    from paper_2505_21404_b200 import make_problem

    rng = np.random.default_rng(0)
    for name in ("poisson2d", "poisson10d", "heat2d", "heat1d", "poisson5d_sin"):
        prob = make_problem(name)
        coll = prob.sample(None, rng)
        for cls in coll.classes:
            p = cls.points[:50]
            op = prob.class_operator(cls.class_id)
            f = prob.class_data(cls)[:50]
            h = 1e-4
            u = prob.exact_solution(p)
            val = op.cu * u - f
            for j, cg in zip(op.grad_dims, op.cg):
                e = np.zeros(p.shape[1]); e[j] = h
                val = val + cg * (prob.exact_solution(p + e) - prob.exact_solution(p - e)) / (2 * h)
            for j in op.lap_dims:
                e = np.zeros(p.shape[1]); e[j] = h
                val = val + op.cl * (prob.exact_solution(p + e) - 2 * u
                                     + prob.exact_solution(p - e)) / h**2
            scale = max(1.0, float(np.max(np.abs(f))))
            assert np.max(np.abs(val)) <= 2e-5 * scale, (name, cls.class_id)


def test_param_layout_and_counts():
    from paper_2505_21404_b200 import MlpSpec, init_params, xavier_normal_params

    for widths, n in [((2, 32, 32, 1), 1185), ((2, 64, 64, 64, 64, 1), 12737),
                      ((5, 512, 512, 512, 512, 1), 791553), ((2, 256, 256, 256, 256, 1), 198401),
                      ((5, 1792, 1792, 1792, 1792, 1792, 1), 12864769)]:
        assert MlpSpec(widths).param_count() == n
    spec = MlpSpec((2, 8, 1), seed=3)
    assert np.array_equal(xavier_normal_params(spec).data, O.xavier_normal_init((2, 8, 1), 3))
    assert np.array_equal(init_params(spec).data, O.glorot_uniform_init((2, 8, 1), 3))


def test_unknown_problems_fail_loudly():
    from paper_2505_21404_b200 import DomainError, make_problem

    for name in ("not_a_problem", "poisson3d"):
        with pytest.raises(DomainError):
            make_problem(name)
    with pytest.raises(DomainError):
        make_problem("poisson_ball_stde", dim=10, index_set_size=20)


def test_stde_plugin_matches_oracle():
    """Host side of PoissonBallStde (problems.py:331-402): sampling order, per-point
    derivative subsets and coefficients, estimator data term, exact solution."""
    from paper_2505_21404_b200 import make_problem

    prob = make_problem("poisson_ball_stde", dim=10, index_set_size=3)
    oprob = O.OraclePoissonBallStde(10, 3)
    colloc = prob.sample((25,), np.random.default_rng(7))
    (oc,) = oprob.sample((25,), np.random.default_rng(7))
    (cls,) = colloc.classes
    assert np.array_equal(cls.points, oc.points)
    op = prob.class_operator(cls.class_id)
    assert np.array_equal(prob.point_grad_dims(cls), oc.pgrad)
    np.testing.assert_allclose(prob.point_coefs(cls, op), oc.pcoef, rtol=0, atol=0)
    np.testing.assert_allclose(prob.class_data(cls), oc.f, rtol=1e-14, atol=1e-14)
    pts = prob.eval_points(50)
    np.testing.assert_allclose(prob.exact_solution(pts), oprob.exact(pts), rtol=1e-14)


def test_allen_cahn_plugin_matches_oracle():
    """Host side of the Allen-Cahn plugin (problems.py:286-328): sampling order,
    operator coefficients, data term and the periodic-embedding input channels."""
    from paper_2505_21404_b200 import make_problem

    prob = make_problem("allen_cahn")
    assert prob.input_dim == 3 and not prob.has_exact
    colloc = prob.sample((40, 12), np.random.default_rng(5))
    oclasses = O.OracleAllenCahn().sample((40, 12), np.random.default_rng(5))
    for cls, oc in zip(colloc.classes, oclasses):
        assert np.array_equal(cls.points, oc.points)
        op = prob.class_operator(cls.class_id)
        assert (op.cu, op.c3, op.cl, op.grad_dims, op.cg, op.lap_dims) == (
            oc.cu, oc.c3, oc.cl, oc.grad_dims, oc.cg, oc.lap_dims)
        np.testing.assert_allclose(prob.class_data(cls), oc.f, rtol=0, atol=0)
        np.testing.assert_allclose(prob.input_channels(cls, op), oc.inputs, rtol=0, atol=1e-15)


def test_class_counts_must_be_positive():
    """problems.py:143-145: empty (or negative) classes are a DomainError, like the
    reference, for every sampler."""
    from paper_2505_21404_b200 import DomainError, make_problem

    for name, counts in [("poisson2d", (10, 0)), ("heat1d", (5, 0, 3)), ("allen_cahn", (0, 4)),
                         ("poisson2d", (10, -1))]:
        with pytest.raises(DomainError):
            make_problem(name).sample(counts, np.random.default_rng(0))


def test_stde_index_draw_matches_reference_argsort():
    """PoissonBallStde.sample picks the k smallest of each row's uniforms with
    argpartition; the reference (problems.py:363) uses argsort()[:, :k] on the
    same draws -- identical indices, identical RNG stream afterwards."""
    import numpy as np

    import paper_2505_21404_b200 as P

    pr = P.make_problem("poisson_ball_stde", dim=300, index_set_size=8)
    rng_a, rng_b = np.random.default_rng(7), np.random.default_rng(7)
    got = pr.sample((50,), rng_a).classes[0].aux["stde_idx"]
    from paper_2505_21404_b200.problems import _ball_interior
    _ball_interior(rng_b, 50, 300)
    want = rng_b.random((50, 300)).argsort(axis=1)[:, :8]
    assert np.array_equal(np.asarray(got), want)
    assert rng_a.random() == rng_b.random()


def test_output_transform_and_host_jets():
    """OutputTransform validation (model.py:181-197) and the host 2-jets that give
    ic_shift its L q0 data term, against central differences."""
    from paper_2505_21404_b200.errors import DomainError
    from paper_2505_21404_b200.model import OutputTransform, point_columns

    with pytest.raises(DomainError):
        OutputTransform("sideways")
    with pytest.raises(DomainError):
        OutputTransform("ic_shift")
    p = np.random.default_rng(0).uniform(size=(7, 2))

    def q(c):
        return np.sin(2 * np.pi * c[1]) * np.exp(-c[0]) + c[1] ** 3 / (1 + c[1]) - np.tanh(c[0] * c[1])

    h = 1e-4
    for d in (0, 1):
        jet = q(point_columns(p, d))
        e = np.zeros(2)
        e[d] = h
        f = lambda x: q([x[:, 0], x[:, 1]])
        np.testing.assert_allclose(jet.v, f(p), rtol=1e-15)
        np.testing.assert_allclose(jet.d1, (f(p + e) - f(p - e)) / (2 * h), atol=1e-6)
        np.testing.assert_allclose(jet.d2, (f(p + e) - 2 * f(p) + f(p - e)) / h**2, atol=1e-4)


def test_ic_shift_parts_match_oracle_classes():
    """The two device problems of an ic_shift map (residuals._IcShiftPart) state the
    same operators and data as the oracle's ic_shift_class restatement."""
    from oracle import dngd_oracle as O
    from paper_2505_21404_b200 import Heat, MlpSpec, OutputTransform, PinnResidualMap
    from paper_2505_21404_b200.errors import DomainError

    prob = Heat(1)
    prob.transform = OutputTransform("ic_shift", q0=lambda c: np.sin(2.0 * np.pi * c[1]))
    colloc = prob.sample({"interior": 30, "boundary": 12}, np.random.default_rng(2))
    rmap = PinnResidualMap(prob, MlpSpec((2, 8, 1)), colloc)
    ocls = O.OracleHeatIcShift().classes(*[c.points for c in colloc.classes])
    for part, shifted in ((rmap.A, False), (rmap.B, True)):
        for c, oc in zip(part.collocation.classes, ocls):
            oc = oc.shift if shifted else oc
            op = part.problem.class_operator(c.class_id)
            assert (op.cu, tuple(op.grad_dims), tuple(op.cg), tuple(op.lap_dims), op.cl) == \
                (oc.cu, tuple(oc.grad_dims), tuple(oc.cg), tuple(oc.lap_dims), oc.cl)
            np.testing.assert_array_equal(c.points, oc.points)
            np.testing.assert_allclose(part.problem.class_data(c), oc.f, rtol=1e-13, atol=1e-13)
    from paper_2505_21404_b200 import AllenCahn

    ac = AllenCahn()
    ac.transform = OutputTransform("ic_shift", q0=lambda c: c[1])
    with pytest.raises(DomainError, match="linear"):
        PinnResidualMap(ac, MlpSpec((3, 8, 1)), ac.sample(None, np.random.default_rng(0))).A \
            .problem.class_operator("interior")
