"""The reference-object adapter (paper_2505_21404_b200.compat) on the REAL
reference package, CPU only: reference problems, collocation sets, specs,
parameter vectors and residual maps are adapted to the device map types, and the
adapted definitions (class operators + host data, evaluated by the numpy oracle)
reproduce the reference's own residuals.  Skipped where /root/reference is absent
(the GPU box); tests/test_gpu_compat.py runs the adapted steps on the device."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not present")


@pytest.fixture(scope="module")
def dngd():
    sys.path.insert(0, REF)
    try:
        import dngd  # noqa: F401
        import dngd.optimizer  # noqa: F401
        import dngd.solver  # noqa: F401
        yield sys.modules["dngd"]
    finally:
        sys.path.remove(REF)


def _oracle_classes(problem, colloc):
    """The adapted problem's device operators as oracle OpClasses (test helper)."""
    from oracle import dngd_oracle as O

    out = []
    for cls in colloc.classes:
        op = problem.class_operator(cls.class_id)
        inputs = problem.input_channels(cls, op) if hasattr(problem, "input_channels") else None
        out.append(O.OpClass(cls.class_id, cls.points, cls.weight, op.cu, tuple(op.grad_dims),
                             tuple(op.cg), tuple(op.lap_dims), op.cl,
                             np.asarray(problem.class_data(cls), dtype=np.float64),
                             getattr(op, "c3", 0.0), inputs))
    return out


@pytest.mark.parametrize("name,counts,widths", [
    ("poisson2d", (60, 20), (2, 12, 12, 1)),
    ("poisson10d", (40, 20), (10, 8, 1)),
    ("heat2d", (50, 30), (3, 10, 10, 1)),
    ("heat10d", (40, 20), (11, 8, 1)),
    ("allen_cahn", (50, 20), None),
])
def test_adapted_reference_map_reproduces_reference_residuals(dngd, name, counts, widths):
    from oracle import dngd_oracle as O
    from paper_2505_21404_b200 import compat

    ref_problem = dngd.problems.make_problem(name)
    widths = widths or ref_problem.default_widths
    rng = np.random.default_rng(3)
    colloc = dngd.problems.sample_collocation(ref_problem, counts, rng)
    spec = dngd.model.MlpSpec(widths, seed=2)
    ref_map = dngd.residuals.PinnResidualMap(ref_problem, spec, colloc)
    theta = dngd.model.init_params(spec) if hasattr(dngd.model, "init_params") else None
    ref_r = ref_map.residual_batch(theta).values

    ours = compat.map_from_reference(ref_map)
    assert type(ours).__name__ == "PinnResidualMap"
    assert ours.m == ref_map.m and ours.n == ref_map.n
    assert [(c, a, b) for c, a, b in ours.partition()] == list(ref_map.partition())
    th = compat.params_from_reference(theta, ours.layout)
    np.testing.assert_array_equal(th.data, theta.data)
    r = O.residuals(th.data, ours.spec.layer_widths, _oracle_classes(ours.problem, ours.collocation))
    np.testing.assert_allclose(r, ref_r, rtol=1e-12, atol=1e-14 * np.abs(ref_r).max())


def test_stde_problem_seed_and_linear_maps(dngd):
    from paper_2505_21404_b200 import compat

    p = compat.problem_from_reference(dngd.problems.PoissonBallStde(20, 4))
    assert p.dim == 20 and p.k == 4
    A = np.arange(12.0).reshape(3, 4)
    lm = compat.map_from_reference(dngd.residuals.LinearResidualMap(A, np.ones(3)))
    np.testing.assert_array_equal(lm.A, A)


def test_unknown_problem_is_refused(dngd):
    from paper_2505_21404_b200 import compat
    from paper_2505_21404_b200.errors import DomainError

    class MyProblem(dngd.problems.PdeProblem):
        pass

    with pytest.raises(DomainError, match="ClassOperator"):
        compat.problem_from_reference(MyProblem())


def test_install_routes_reference_steps(dngd):
    """install() swaps solver.dense_dual_solve / pcg_step and the names the
    reference optimizer imported (optimizer.py:20) for the adapters; uninstall
    restores them.  (The adapted steps run in tests/test_gpu_compat.py.)"""
    from paper_2505_21404_b200 import compat

    before = (dngd.solver.dense_dual_solve, dngd.optimizer.dense_dual_solve,
              dngd.solver.pcg_step, dngd.optimizer.pcg_step)
    orig = compat.install(dngd)
    try:
        assert dngd.optimizer.dense_dual_solve is dngd.solver.dense_dual_solve
        assert dngd.solver.dense_dual_solve is not before[0]
        assert dngd.optimizer.pcg_step is dngd.solver.pcg_step is not before[2]
    finally:
        compat.uninstall(dngd, orig)
    assert (dngd.solver.dense_dual_solve, dngd.optimizer.dense_dual_solve,
            dngd.solver.pcg_step, dngd.optimizer.pcg_step) == before


def test_ic_shift_reference_problem_reproduces_reference_residuals(dngd):
    """A reference Heat(1) with OutputTransform("ic_shift", q0) written against the
    reference's ops module (model.py:181-277): the adapter yields the two-map
    IcShiftResidualMap, the reference q0 evaluates on host jets, and the two parts'
    operators + data reproduce the reference residuals (oracle evaluation)."""
    from oracle import dngd_oracle as O
    from paper_2505_21404_b200 import compat

    ops = dngd.ops

    class HeatIc(dngd.problems.Heat):
        def __init__(self):
            super().__init__(1)
            self.transform = dngd.model.OutputTransform(
                "ic_shift", q0=lambda c: ops.mul(ops.sin(ops.mul(np.pi, c[1])),
                                                 ops.exp(ops.mul(0.5, c[1]))))

    ref_problem = HeatIc()
    colloc = dngd.problems.sample_collocation(ref_problem, (50, 30), np.random.default_rng(5))
    spec = dngd.model.MlpSpec((2, 10, 10, 1), seed=4)
    ref_map = dngd.residuals.PinnResidualMap(ref_problem, spec, colloc)
    theta = dngd.model.init_params(spec)
    ref_r = ref_map.residual_batch(theta).values

    ours = compat.map_from_reference(ref_map)
    assert type(ours).__name__ == "IcShiftResidualMap"
    a = _oracle_classes(ours.A.problem, ours.A.collocation)
    b = _oracle_classes(ours.B.problem, ours.B.collocation)
    for ca, cb in zip(a, b):
        ca.shift = cb
    r = O.residuals(np.asarray(theta.data), (2, 10, 10, 1), a)
    np.testing.assert_allclose(r, ref_r, rtol=1e-12, atol=1e-13 * np.abs(ref_r).max())
