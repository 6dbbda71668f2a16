"""Reference-typed inputs on the device (the reference package is not on the GPU
box, so its public types are mirrored here by attribute, citing params.py:13-100,
model.py:23-46, residuals.py:34-104 and 422-454, solver.py:40-49): the adapted
steps equal the native ones, and install() makes a reference-shaped module tree's
_dispatch_step get reference-typed StepResults back."""

import types
from dataclasses import dataclass, field

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


# ---- attribute mirrors of the reference's public types ------------------------------


@dataclass
class RefEntry:
    name: str
    shape: tuple
    offset: int


class RefLayout:
    def __init__(self, entries):
        self.entries, off = [], 0
        for name, shape in entries:
            self.entries.append(RefEntry(name, tuple(shape), off))
            off += int(np.prod(shape))
        self.size = off


class ParameterVector:  # params.py:75-100: (data, layout)
    def __init__(self, data, layout):
        self.data, self.layout = np.asarray(data, dtype=np.float64), layout


@dataclass(frozen=True)
class MlpSpec:  # model.py:23
    layer_widths: tuple
    seed: int = 0


@dataclass
class CollocationClass:  # residuals.py:34
    class_id: str
    points: np.ndarray
    weight: float
    aux: dict = field(default_factory=dict)

    @property
    def count(self):
        return self.points.shape[0]


class CollocationSet:  # residuals.py:59
    def __init__(self, classes):
        self.classes = list(classes)


class Poisson2d:  # problems.py:149 (the adapter dispatches on the class name)
    pass


class PinnResidualMap:  # residuals.py:422
    def __init__(self, problem, spec, collocation):
        self.problem, self.spec, self.collocation = problem, spec, collocation


@dataclass
class StepResult:  # solver.py:40
    delta: object
    lambda_used: float
    cg_iterations: int = 0
    eta: float | None = None
    ga_ratio: float | None = None
    warning: str | None = None


def _reference_inputs(P, counts=(90, 30), widths=(2, 16, 16, 1)):
    native_problem = P.make_problem("poisson2d")
    colloc = native_problem.sample(counts, np.random.default_rng(4))
    ref_colloc = CollocationSet([CollocationClass(c.class_id, c.points, c.weight)
                                 for c in colloc.classes])
    spec = P.MlpSpec(widths)
    layout = spec.layout()
    ref_layout = RefLayout([(e.name, e.shape) for e in layout.entries])
    theta = P.xavier_normal_params(spec)
    ref_map = PinnResidualMap(Poisson2d(), MlpSpec(widths), ref_colloc)
    native_map = P.PinnResidualMap(native_problem, spec, colloc)
    return ref_map, ParameterVector(theta.data, ref_layout), native_map, theta


def test_reference_typed_dense_and_pcg_steps(P):
    from paper_2505_21404_b200 import compat

    ref_map, ref_theta, native_map, theta = _reference_inputs(P)
    _, g = native_map.residuals_and_gradient(theta)
    a = compat.dense_dual_solve(ref_map, ref_theta, g, lam=1e-3, use_ga=True)
    b = P.dense_dual_solve(native_map, theta, g, lam=1e-3, use_ga=True)
    np.testing.assert_array_equal(a.delta.data, b.delta.data)
    assert a.lambda_used == b.lambda_used and a.ga_ratio == b.ga_ratio
    pa = compat.pcg_step(ref_map, ref_theta, g, lam=1e-3, landmark_count=16, tol=1e-10,
                         max_iters=100, rng=np.random.default_rng(9))
    pb = P.pcg_step(native_map, theta, g, lam=1e-3, landmark_count=16, tol=1e-10,
                    max_iters=100, rng=np.random.default_rng(9))
    np.testing.assert_array_equal(pa.delta.data, pb.delta.data)
    assert pa.cg_iterations == pb.cg_iterations


def test_install_returns_reference_typed_steps(P):
    from paper_2505_21404_b200 import compat

    ref_map, ref_theta, native_map, theta = _reference_inputs(P)
    solver = types.SimpleNamespace(StepResult=StepResult, dense_dual_solve=None, pcg_step=None)
    optimizer = types.SimpleNamespace(dense_dual_solve=None, pcg_step=None)
    dngd = types.SimpleNamespace(solver=solver, optimizer=optimizer)
    orig = compat.install(dngd)
    _, g = native_map.residuals_and_gradient(theta)
    step = dngd.optimizer.dense_dual_solve(ref_map, ref_theta, g, lam=1e-3, use_ga=True)
    assert isinstance(step, StepResult) and isinstance(step.delta, ParameterVector)
    assert step.delta.layout is ref_theta.layout
    ref = P.dense_dual_solve(native_map, theta, g, lam=1e-3, use_ga=True)
    np.testing.assert_array_equal(step.delta.data, ref.delta.data)
    step = dngd.solver.pcg_step(ref_map, ref_theta, g, lam=1e-3, landmark_count=16,
                                rng=np.random.default_rng(1))
    assert isinstance(step, StepResult) and step.cg_iterations >= 1
    compat.uninstall(dngd, orig)
    assert dngd.solver.dense_dual_solve is None
