"""Drop-in adapter for objects of the reference package `dngd`.

The step API here keeps the reference names and signatures; this module makes it
accept the reference's own objects as well, so an existing `dngd` install can
route its dense and PCG steps to the B200 path:

  reference object (file:line)                      adapted to
  ------------------------------------------------  ------------------------------------------
  params.ParameterVector(data, layout) (params.py:75)  ParameterVector on the same layout
  model.MlpSpec(layer_widths, seed) (model.py:23)      MlpSpec
  residuals.CollocationSet / CollocationClass          CollocationSet / CollocationClass
     (residuals.py:34-104)                               (class id, points, weight, aux)
  problems.Poisson2d / Poisson10d / Heat(d) /          the same problem with device class
     AllenCahn / PoissonBallStde (problems.py:149-398)   operators (problems.py here)
  residuals.PinnResidualMap / RegressionResidualMap /  PinnResidualMap / RegressionResidualMap /
     LinearResidualMap (residuals.py:325-454)            LinearResidualMap on the device

The adapter reads only public attributes of those objects (names cited above);
it never imports the reference.  `install(dngd)` swaps the step functions of a
reference module tree for wrappers that adapt the arguments, run the step here,
and hand back a reference-typed StepResult -- what `_dispatch_step`
(optimizer.py:172-184) consumes.  Problems without a device operator (a
user-written `class_residual` over the reference's AD algebra) raise DomainError:
state them as problems.ClassOperator classes instead.
"""

from __future__ import annotations

import numpy as np

from .errors import DimensionError, DomainError

_CACHE_ATTR = "_b200_adapted"


def is_native(obj) -> bool:
    return type(obj).__module__.startswith(__package__)


def spec_from_reference(spec):
    from .model import MlpSpec

    if is_native(spec):
        return spec
    return MlpSpec(tuple(int(w) for w in spec.layer_widths), int(getattr(spec, "seed", 0)))


def collocation_from_reference(colloc):
    from .residuals import CollocationClass, CollocationSet

    if is_native(colloc):
        return colloc
    return CollocationSet([CollocationClass(c.class_id, np.asarray(c.points, dtype=np.float64),
                                            float(c.weight), dict(getattr(c, "aux", {}) or {}))
                           for c in colloc.classes])


def problem_from_reference(problem):
    """The device twin of a reference problem instance (by class and parameters)."""
    from . import problems as PR

    if is_native(problem) or hasattr(problem, "class_operator"):
        return problem
    twin = _twin(problem)
    tr = getattr(problem, "transform", None)
    if tr is not None and getattr(tr, "kind", "identity") == "ic_shift":
        # the reference's q0 is written against its ops module, which falls through to
        # numpy operators for non-box values: it evaluates unchanged on HostJet columns
        from .model import OutputTransform

        twin.transform = OutputTransform("ic_shift", q0=tr.q0)
    return twin


def _twin(problem):
    from . import problems as PR

    kind = type(problem).__name__
    if kind == "Poisson2d":
        return PR.Poisson2d()
    if kind == "Poisson10d":
        return PR.Poisson10d()
    heat = [b for b in type(problem).__mro__ if b.__name__ == "Heat"]
    if heat and type(problem).class_residual is heat[0].class_residual:
        return PR.Heat(int(problem.d))  # Heat or a subclass with Heat's residuals
    if kind == "AllenCahn":
        return PR.AllenCahn()
    if kind == "PoissonBallStde":
        return PR.PoissonBallStde(int(problem.dim), int(problem.k),
                                  coeff_seed=_stde_seed(problem))
    raise DomainError(
        f"reference problem {kind!r} has no device operator: state its residual classes as "
        "paper_2505_21404_b200.problems.ClassOperator (class_operator / class_data)")


def _stde_seed(problem):
    """PoissonBallStde draws its coefficients from default_rng(coeff_seed)
    (problems.py:346-355); recover the seed by matching the stored draw."""
    coeffs = np.asarray(problem.coeffs)
    for seed in (1234, 0, 1, 42):
        if np.array_equal(np.random.default_rng(seed).normal(size=coeffs.size), coeffs):
            return seed
    raise DomainError("PoissonBallStde with a custom coefficient draw is not supported")


def map_from_reference(rmap):
    """The device residual map for a reference residual map (cached on the object)."""
    from .residuals import LinearResidualMap, PinnResidualMap, RegressionResidualMap

    if is_native(rmap):
        return rmap
    cached = getattr(rmap, _CACHE_ATTR, None)
    if cached is not None and cached[0] is rmap.collocation:
        return cached[1]
    kind = type(rmap).__name__
    if kind == "LinearResidualMap":
        out = LinearResidualMap(np.asarray(rmap.A), np.asarray(rmap.c))
    elif kind == "RegressionResidualMap":
        cls = rmap.collocation.classes[0]
        out = RegressionResidualMap(spec_from_reference(rmap.spec), np.asarray(cls.points),
                                    np.asarray(cls.aux["targets"]), float(cls.weight))
    elif kind == "PinnResidualMap" or hasattr(rmap, "problem"):
        out = PinnResidualMap(problem_from_reference(rmap.problem),
                              spec_from_reference(rmap.spec),
                              collocation_from_reference(rmap.collocation))
    else:
        raise DomainError(f"no device counterpart for residual map {kind!r}")
    try:
        setattr(rmap, _CACHE_ATTR, (rmap.collocation, out))
    except (AttributeError, TypeError):
        pass
    return out


def params_from_reference(theta, layout):
    """A reference ParameterVector (or a flat array) on this map's layout."""
    from .params import ParameterVector

    if isinstance(theta, ParameterVector):
        return theta
    data = getattr(theta, "data", theta)
    ref_layout = getattr(theta, "layout", None)
    if ref_layout is not None:
        ref_entries = [(e.name, tuple(e.shape)) for e in ref_layout.entries]
        ours = [(e.name, tuple(e.shape)) for e in layout.entries]
        if ref_entries != ours:
            raise DimensionError("parameter layout does not match the residual map's layout")
    return ParameterVector(np.asarray(data, dtype=np.float64), layout)


def vector_from_reference(v):
    """ResidualBatch / ParameterVector of either package -> numpy (or tensor) data."""
    if v is None:
        return None
    if hasattr(v, "tensor") and is_native(v):
        return v.tensor
    if hasattr(v, "values"):
        return np.asarray(v.values, dtype=np.float64)
    if hasattr(v, "data") and hasattr(v, "layout"):
        return np.asarray(v.data, dtype=np.float64)
    return v


def step_to_reference(step, ref_solver, ref_theta):
    """Our StepResult -> the reference's StepResult with a reference ParameterVector."""
    ref_pv = type(ref_theta)
    return ref_solver.StepResult(delta=ref_pv(step.delta.data, ref_theta.layout),
                                 lambda_used=step.lambda_used,
                                 cg_iterations=step.cg_iterations, eta=step.eta,
                                 ga_ratio=step.ga_ratio, warning=step.warning)


def _adapt(residual_map, theta, g, points):
    rmap = map_from_reference(residual_map)
    if points is not None:
        rmap = rmap.rebind(collocation_from_reference(points))
    th = params_from_reference(theta, rmap.layout)
    return rmap, th, vector_from_reference(g)


def dense_dual_solve(residual_map, theta, g, points=None, lam: float = 1e-3, use_ga: bool = True):
    """solver.dense_dual_solve (solver.py:176-219) on reference-typed or native inputs;
    returns this package's StepResult."""
    from . import solver

    rmap, th, gv = _adapt(residual_map, theta, g, points)
    return solver.dense_dual_solve(rmap, th, gv, lam=lam, use_ga=use_ga)


def pcg_step(residual_map, theta, g, points=None, lam: float = 1e-3, landmark_count: int = 64,
             tol: float = 1e-10, max_iters: int = 500, rng=None, precond=None):
    """solver.pcg_step (solver.py:290-366) on reference-typed or native inputs.  A
    reference NystromPreconditioner (U, lam_hat, lam, landmarks) is carried over."""
    from . import solver

    rmap, th, gv = _adapt(residual_map, theta, g, points)
    if precond is not None and not is_native(precond):
        precond = solver.NystromPreconditioner(np.asarray(precond.U), np.asarray(precond.lam_hat),
                                               float(precond.lam), np.asarray(precond.landmarks))
    return solver.pcg_step(rmap, th, gv, lam=lam, landmark_count=landmark_count, tol=tol,
                           max_iters=max_iters, rng=rng, precond=precond)


def install(dngd):
    """Route a reference module tree's dense and PCG steps to the B200 path.

    `dngd` is the imported reference package; its solver.dense_dual_solve /
    pcg_step and the names the optimizer imported from it (optimizer.py:20) are
    replaced by wrappers returning reference-typed StepResults.  Returns the
    originals (pass them to uninstall)."""
    ref_solver, ref_opt = dngd.solver, dngd.optimizer
    originals = {"solver": (ref_solver.dense_dual_solve, ref_solver.pcg_step),
                 "optimizer": (ref_opt.dense_dual_solve, ref_opt.pcg_step)}

    def dense(residual_map, theta, g, points=None, lam=1e-3, use_ga=True):
        step = dense_dual_solve(residual_map, theta, g, points, lam, use_ga)
        return step_to_reference(step, ref_solver, theta)

    def pcg(residual_map, theta, g, points=None, lam=1e-3, landmark_count=64, tol=1e-10,
            max_iters=500, rng=None, precond=None):
        step = pcg_step(residual_map, theta, g, points, lam, landmark_count, tol, max_iters, rng,
                        precond)
        return step_to_reference(step, ref_solver, theta)

    ref_solver.dense_dual_solve = ref_opt.dense_dual_solve = dense
    ref_solver.pcg_step = ref_opt.pcg_step = pcg
    return originals


def uninstall(dngd, originals):
    dngd.solver.dense_dual_solve, dngd.solver.pcg_step = originals["solver"]
    dngd.optimizer.dense_dual_solve, dngd.optimizer.pcg_step = originals["optimizer"]
