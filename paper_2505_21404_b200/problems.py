"""PDE problem plugins: sampling, class operators and host-side data terms.

Same plugin surface as the reference PdeProblem (problems.py:107-146):
`sample(counts, rng)`, `resolve_counts`, `exact_solution`, `eval_points`,
`default_counts`, `default_widths`, `default_lam_cap`, `name`.  Instead of a
`class_residual(net, cls)` written against the AD algebra, each problem
states every residual class as a differential operator

    r = w * (cu*u + c3*u^3 + sum_g cg[g] d_{grad_dims[g]} u + cl * sum_{j in lap_dims} d_jj u - f(x))

(`class_operator`) plus its data term f (`class_data`, evaluated on the host
with the reference's numpy expressions), and optionally an input embedding
(`input_channels`: the network-input channels phi(x), d_j phi, sum d_jj phi of
model.py:133-175); the device kernels (pinn.cu) evaluate u and its derivative
channels.  This covers all of the reference's deterministic problems --
Poisson2d, Poisson10d, Heat(d), Allen-Cahn (periodic embedding + cubic
reaction) -- and the BASELINE configs' heat1d (G2) and sine-Poisson (G3).
STDE subsampling (PoissonBallStde) is out of scope and raises DomainError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DomainError
from .model import OutputTransform
from .residuals import BOUNDARY, INITIAL, INTERIOR, CollocationClass, CollocationSet


@dataclass(frozen=True)
class ClassOperator:
    cu: float = 0.0
    grad_dims: tuple = ()
    cg: tuple = ()
    lap_dims: tuple = ()
    cl: float = 0.0
    c3: float = 0.0  # coefficient of u^3 (Allen-Cahn reaction)


VALUE = ClassOperator(cu=1.0)  # r = u - g


# -- samplers (reference problems.py:39-79) -----------------------------------------


def _box_interior(rng, n, lows, highs):
    lows, highs = np.asarray(lows, dtype=float), np.asarray(highs, dtype=float)
    return lows + rng.uniform(size=(n, lows.size)) * (highs - lows)


def _box_faces(rng, n, lows, highs):
    lows, highs = np.asarray(lows, dtype=float), np.asarray(highs, dtype=float)
    d = lows.size
    x = _box_interior(rng, n, lows, highs)
    face = rng.integers(0, 2 * d, size=n)
    j, side = face // 2, face % 2
    x[np.arange(n), j] = np.where(side == 0, lows[j], highs[j])
    return x


def _parabolic_boundary(rng, n, d):
    piece = rng.integers(0, 2 * d + 1, size=n)
    t = np.where(piece == 0, 0.0, rng.uniform(size=n))
    x = rng.uniform(size=(n, d))
    rows = np.flatnonzero(piece > 0)
    j = (piece[rows] - 1) // 2
    x[rows, j] = ((piece[rows] - 1) % 2).astype(np.float64)
    return np.column_stack([t, x])


def _ball_interior(rng, n, d):
    """Uniform points in the open unit ball (problems.py:74-79)."""
    z = rng.normal(size=(n, d))
    z /= np.linalg.norm(z, axis=1, keepdims=True)
    radius = rng.uniform(size=(n, 1)) ** (1.0 / d)
    return z * radius


def _halton(num: int, lows, highs) -> np.ndarray:
    from scipy.stats import qmc

    lows, highs = np.asarray(lows, dtype=float), np.asarray(highs, dtype=float)
    unit = qmc.Halton(d=lows.size, scramble=False).random(num)
    return lows + unit * (highs - lows)


def _pairwise_sum(terms):
    """Balanced summation tree, same order as the reference (problems.py:88-95)."""
    while len(terms) > 1:
        terms = [terms[i] + terms[i + 1] if i + 1 < len(terms) else terms[i]
                 for i in range(0, len(terms), 2)]
    return terms[0]


def _cls(class_id, points, aux=None):
    return CollocationClass(class_id, points, 1.0 / np.sqrt(points.shape[0]), aux or {})


# -- problem surface ------------------------------------------------------------------------


class PdeProblem:
    name: str
    raw_dim: int
    transform = OutputTransform("identity")  # model.py:181-197; ic_shift -> IcShiftResidualMap
    default_counts: dict
    default_widths: tuple
    default_lam_cap: float = 1e-5
    has_exact: bool = True

    @property
    def input_dim(self) -> int:
        """Network input width: raw_dim, or the embedding's output width."""
        return self.raw_dim

    def input_channels(self, cls: CollocationClass, op: ClassOperator):
        """(N, nch, input_dim) embedded input channels, or None for the identity
        embedding (model.py:133-146)."""
        return None

    def sample(self, counts, rng) -> CollocationSet:
        raise NotImplementedError

    def class_operator(self, class_id: str) -> ClassOperator:
        raise NotImplementedError

    def class_data(self, cls: CollocationClass) -> np.ndarray:
        raise NotImplementedError

    def exact_solution(self, pts: np.ndarray) -> np.ndarray:
        raise DomainError(f"problem {self.name} has no closed-form solution")

    def eval_points(self, num: int = 10_000) -> np.ndarray:
        raise NotImplementedError

    def resolve_counts(self, counts) -> dict:
        """Reference problems.py:132-146."""
        merged = dict(self.default_counts)
        if counts is not None and not isinstance(counts, dict):
            counts = dict(zip(merged, counts))
        if counts:
            unknown = set(counts) - set(merged)
            if unknown:
                raise DomainError(f"problem {self.name} has no classes {sorted(unknown)}")
            merged.update(counts)
        bad = {k: v for k, v in merged.items() if int(v) < 1}
        if bad:
            raise DomainError(f"class counts must be >= 1, got {bad}")
        return {k: int(v) for k, v in merged.items()}


class Poisson2d(PdeProblem):
    """-Lap u = 2 pi^2 sin(pi x) sin(pi y) on (0,1)^2, u = 0 on the faces (problems.py:149-190)."""

    name = "poisson2d"
    raw_dim = 2
    default_counts = {INTERIOR: 480, BOUNDARY: 120}
    default_widths = (2, 32, 32, 1)

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        return CollocationSet([
            _cls(INTERIOR, _box_interior(rng, c[INTERIOR], [0, 0], [1, 1])),
            _cls(BOUNDARY, _box_faces(rng, c[BOUNDARY], [0, 0], [1, 1])),
        ])

    def class_operator(self, class_id):
        if class_id == INTERIOR:
            return ClassOperator(grad_dims=(0, 1), cg=(0.0, 0.0), lap_dims=(0, 1), cl=-1.0)
        return VALUE

    def class_data(self, cls):
        p = cls.points
        if cls.class_id == INTERIOR:
            return 2.0 * np.pi**2 * np.sin(np.pi * p[:, 0]) * np.sin(np.pi * p[:, 1])
        return np.zeros(p.shape[0])

    def exact_solution(self, pts):
        return np.sin(np.pi * pts[:, 0]) * np.sin(np.pi * pts[:, 1])

    def eval_points(self, num=10_000):
        return _halton(num, [0, 0], [1, 1])


class PoissonSin(PdeProblem):
    """BASELINE configs 3-4: -Lap u = pi^2 sum sin(pi x_i) on (0,1)^d, u* = sum sin(pi x_i)."""

    default_lam_cap = 1e-5

    def __init__(self, dim: int = 5):
        self.dim = int(dim)
        self.name = f"poisson{self.dim}d_sin"
        self.raw_dim = self.dim
        self.default_counts = {INTERIOR: 3500, BOUNDARY: 500}
        self.default_widths = (self.dim, 512, 512, 512, 512, 1)

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        d = self.dim
        return CollocationSet([
            _cls(INTERIOR, _box_interior(rng, c[INTERIOR], np.zeros(d), np.ones(d))),
            _cls(BOUNDARY, _box_faces(rng, c[BOUNDARY], np.zeros(d), np.ones(d))),
        ])

    def class_operator(self, class_id):
        if class_id == INTERIOR:
            dims = tuple(range(self.dim))
            return ClassOperator(grad_dims=dims, cg=(0.0,) * self.dim, lap_dims=dims, cl=-1.0)
        return VALUE

    def class_data(self, cls):
        p = cls.points
        if cls.class_id == INTERIOR:
            return np.pi**2 * np.sum(np.sin(np.pi * p), axis=1)
        return self.exact_solution(p)

    def exact_solution(self, pts):
        return np.sum(np.sin(np.pi * pts), axis=1)

    def eval_points(self, num=10_000):
        return _halton(num, np.zeros(self.dim), np.ones(self.dim))


class Poisson10d(PdeProblem):
    """-Lap u = 0 on (0,1)^10, u = sum x_{2k-1} x_{2k} on the faces (problems.py:193-228)."""

    name = "poisson10d"
    raw_dim = 10
    default_counts = {INTERIOR: 400, BOUNDARY: 200}
    default_widths = (10, 32, 32, 1)

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        lows, highs = np.zeros(10), np.ones(10)
        return CollocationSet([
            _cls(INTERIOR, _box_interior(rng, c[INTERIOR], lows, highs)),
            _cls(BOUNDARY, _box_faces(rng, c[BOUNDARY], lows, highs)),
        ])

    def class_operator(self, class_id):
        if class_id == INTERIOR:
            dims = tuple(range(10))
            return ClassOperator(grad_dims=dims, cg=(0.0,) * 10, lap_dims=dims, cl=-1.0)
        return VALUE

    def class_data(self, cls):
        if cls.class_id == INTERIOR:
            return np.zeros(cls.count)
        return self.exact_solution(cls.points)

    def exact_solution(self, pts):
        return _pairwise_sum([pts[:, 2 * k] * pts[:, 2 * k + 1] for k in range(5)])

    def eval_points(self, num=10_000):
        return _halton(num, np.zeros(10), np.ones(10))


class Heat(PdeProblem):
    """u_t = kappa Lap u, kappa = 1/4, parabolic-boundary class (problems.py:231-285)."""

    kappa = 0.25
    default_lam_cap = 1e-3

    def __init__(self, spatial_dim: int):
        self.d = int(spatial_dim)
        self.name = f"heat{self.d}d"
        self.raw_dim = 1 + self.d
        if self.d == 2:
            self.default_counts = {INTERIOR: 320, BOUNDARY: 160}
            self.default_widths = (3, 24, 24, 1)
        else:
            self.default_counts = {INTERIOR: 400, BOUNDARY: 210}
            self.default_widths = (self.raw_dim, 32, 32, 1)

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        d = self.d
        interior = np.column_stack([
            rng.uniform(size=c[INTERIOR]),
            _box_interior(rng, c[INTERIOR], np.zeros(d), np.ones(d)),
        ])
        boundary = _parabolic_boundary(rng, c[BOUNDARY], d)
        return CollocationSet([_cls(INTERIOR, interior), _cls(BOUNDARY, boundary)])

    def class_operator(self, class_id):
        if class_id == INTERIOR:
            dims = tuple(range(self.raw_dim))
            cg = (1.0,) + (0.0,) * self.d
            return ClassOperator(grad_dims=dims, cg=cg, lap_dims=dims[1:], cl=-self.kappa)
        return VALUE

    def class_data(self, cls):
        if cls.class_id == INTERIOR:
            return np.zeros(cls.count)
        return self.exact_solution(cls.points)

    def exact_solution(self, pts):
        decay = np.exp(-4.0 * np.pi**2 * self.kappa * pts[:, 0])
        modes = _pairwise_sum([np.sin(2.0 * np.pi * pts[:, 1 + j]) for j in range(self.d)])
        return decay * modes

    def eval_points(self, num=10_000):
        return _halton(num, np.zeros(self.raw_dim), np.ones(self.raw_dim))


class Heat1d(PdeProblem):
    """BASELINE config 2: u_t = 0.1 u_xx on (0,1)x(0,1), coordinates (t, x),
    u* = exp(-0.1 pi^2 t) sin(pi x); classes interior / boundary (x in {0,1}) / initial (t=0)."""

    name = "heat1d"
    raw_dim = 2
    kappa = 0.1
    default_counts = {INTERIOR: 2000, BOUNDARY: 400, INITIAL: 400}
    default_widths = (2, 64, 64, 64, 64, 1)
    default_lam_cap = 1e-3

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        pi = _box_interior(rng, c[INTERIOR], [0, 0], [1, 1])
        tb = rng.uniform(size=c[BOUNDARY])
        xb = rng.integers(0, 2, size=c[BOUNDARY]).astype(np.float64)
        x0 = rng.uniform(size=c[INITIAL])
        return CollocationSet([
            _cls(INTERIOR, pi),
            _cls(BOUNDARY, np.column_stack([tb, xb])),
            _cls(INITIAL, np.column_stack([np.zeros(c[INITIAL]), x0])),
        ])

    def class_operator(self, class_id):
        if class_id == INTERIOR:
            return ClassOperator(grad_dims=(0, 1), cg=(1.0, 0.0), lap_dims=(1,), cl=-self.kappa)
        return VALUE

    def class_data(self, cls):
        if cls.class_id == INTERIOR:
            return np.zeros(cls.count)
        return self.exact_solution(cls.points)

    def exact_solution(self, pts):
        return np.exp(-self.kappa * np.pi**2 * pts[:, 0]) * np.sin(np.pi * pts[:, 1])

    def eval_points(self, num=10_000):
        return _halton(num, [0, 0], [1, 1])


def periodic_channels(points: np.ndarray, omega: float, op: ClassOperator) -> np.ndarray:
    """PeriodicEmbedding1d (model.py:148-175): (t, x) -> [t, sin wx, cos wx] and its
    directional derivatives, as network-input channels in the device's channel
    order: value, d_j per grad dim, sum_{j in lap} d_jj."""
    t, x = points[:, 0], points[:, 1]
    s, c = np.sin(omega * x), np.cos(omega * x)
    zero = np.zeros_like(t)
    chans = [np.stack([t, s, c], axis=1)]
    for j in op.grad_dims:
        if j == 0:
            chans.append(np.stack([np.ones_like(t), zero, zero], axis=1))
        else:
            chans.append(np.stack([zero, omega * c, -omega * s], axis=1))
    if op.lap_dims:
        lap = np.zeros((points.shape[0], 3))
        for j in op.lap_dims:
            if j == 1:
                lap += np.stack([zero, -omega * omega * s, -omega * omega * c], axis=1)
        chans.append(lap)
    return np.ascontiguousarray(np.stack(chans, axis=1))


class AllenCahn(PdeProblem):
    """u_t - 1e-4 u_xx + 5u^3 - 5u = 0 on (0,1) x (-1,1), periodic in x (period 2)
    through the sin/cos input embedding; u(0, x) = x^2 cos(pi x) (problems.py:286-328).
    Classes interior / initial; no closed-form solution."""

    name = "allen_cahn"
    raw_dim = 2
    default_counts = {INTERIOR: 1125, INITIAL: 225}
    default_widths = (3, 32, 32, 32, 1)
    has_exact = False
    diffusivity = 1e-4
    omega = np.pi  # 2 pi / period

    @property
    def input_dim(self) -> int:
        return 3

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        interior = np.column_stack(
            [rng.uniform(size=c[INTERIOR]), rng.uniform(-1.0, 1.0, size=c[INTERIOR])])
        initial = np.column_stack(
            [np.zeros(c[INITIAL]), rng.uniform(-1.0, 1.0, size=c[INITIAL])])
        return CollocationSet([_cls(INTERIOR, interior), _cls(INITIAL, initial)])

    def class_operator(self, class_id):
        if class_id == INTERIOR:
            return ClassOperator(cu=-5.0, grad_dims=(0, 1), cg=(1.0, 0.0), lap_dims=(1,),
                                 cl=-self.diffusivity, c3=5.0)
        return VALUE

    def class_data(self, cls):
        if cls.class_id == INTERIOR:
            return np.zeros(cls.count)
        x = cls.points[:, 1]
        return x**2 * np.cos(np.pi * x)

    def input_channels(self, cls, op):
        return periodic_channels(cls.points, self.omega, op)

    def eval_points(self, num=10_000):
        return _halton(num, [0.0, -1.0], [1.0, 1.0])


class PoissonBallStde(PdeProblem):
    """-Lap u = f on the unit ball in R^d, u = (1 - |x|^2) phi exactly zero on the
    sphere (dirichlet_ball transform, model.py:181-199), Laplacians of the network
    and of the exact solution estimated on one random k-subset of directions per
    point (problems.py:331-402):
        r = -(d/k) sum_{j in S} (d_jj u - d_jj u_ex),
        d_jj[(1 - |x|^2) phi] = (1 - |x|^2) d_jj phi - 4 x_j d_j phi - 2 phi,
    i.e. device channels (phi, d_j phi for j in S, sum_S d_jj phi) with per-point
    derivative dims S and coefficients (2d, 4 (d/k) x_j, -(d/k)(1 - |x|^2))."""

    name = "poisson_ball_stde"
    transform = OutputTransform("dirichlet_ball")  # stated as per-point coefficients below
    default_lam_cap = 1e3
    has_exact = True

    def __init__(self, dim: int = 100, index_set_size: int = 8, coeff_seed: int = 1234):
        self.dim = int(dim)
        self.k = int(index_set_size)
        if not 1 <= self.k <= self.dim:
            raise DomainError(f"index set size {self.k} outside [1, {self.dim}]")
        if self.k > 12:
            raise DomainError("index set size above 12 exceeds the device channel limit")
        self.raw_dim = self.dim
        self.default_counts = {INTERIOR: 128}
        self.default_widths = (self.dim, 64, 64, 1)
        self.coeffs = np.random.default_rng(coeff_seed).normal(size=self.dim - 1)

    def sample(self, counts, rng):
        c = self.resolve_counts(counts)
        n = c[INTERIOR]
        pts = _ball_interior(rng, n, self.dim)
        # same draws and result as the reference's argsort(axis=1)[:, :k] (the k
        # smallest of n distinct uniforms, ascending) in O(dim) per row
        u = rng.random((n, self.dim))
        part = np.argpartition(u, self.k - 1, axis=1)[:, : self.k]
        order = np.argsort(np.take_along_axis(u, part, axis=1), axis=1)
        idx = np.take_along_axis(part, order, axis=1)
        return CollocationSet([_cls(INTERIOR, pts, {"stde_idx": idx})])

    def class_operator(self, class_id):
        dims = tuple(range(self.k))  # placeholders: the dims are per point
        return ClassOperator(grad_dims=dims, cg=(0.0,) * self.k, lap_dims=dims, cl=0.0)

    def point_grad_dims(self, cls):
        return np.asarray(cls.aux["stde_idx"], dtype=np.int32)

    def point_coefs(self, cls, op):
        d, k = self.dim, self.k
        x = cls.points
        idx = np.asarray(cls.aux["stde_idx"])
        rows = np.arange(x.shape[0])
        co = np.empty((x.shape[0], k + 2))
        co[:, 0] = 2.0 * d
        for g in range(k):
            co[:, 1 + g] = 4.0 * (d / k) * x[rows, idx[:, g]]
        co[:, k + 1] = -(d / k) * (1.0 - np.sum(x * x, axis=1))
        return co

    def _F(self, x):
        c = self.coeffs
        return np.sum(c * (np.sin(x[:, :-1] + np.cos(x[:, 1:])) + x[:, 1:] * np.cos(x[:, :-1])),
                      axis=1)

    def _exact_dd(self, x, j, F=None, s=None):
        """d^2/dx_j^2 of the exact solution, per point direction j (product rule).
        F = _F(x) and s = 1 - |x|^2 may be passed in (they do not depend on j)."""
        c, d = self.coeffs, self.dim
        rows = np.arange(x.shape[0])
        xj = x[rows, j]
        if F is None:
            F = self._F(x)
        m1 = j < d - 1
        jj = np.where(m1, j, 0)
        xn = x[rows, np.minimum(j + 1, d - 1)]
        a = xj + np.cos(xn)
        dF = np.where(m1, c[jj] * (np.cos(a) - xn * np.sin(xj)), 0.0)
        ddF = np.where(m1, c[jj] * (-np.sin(a) - xn * np.cos(xj)), 0.0)
        m2 = j > 0
        jm = np.where(m2, j - 1, 0)
        xp = x[rows, np.maximum(j - 1, 0)]
        b = xp + np.cos(xj)
        dF = dF + np.where(m2, c[jm] * (-np.cos(b) * np.sin(xj) + np.cos(xp)), 0.0)
        ddF = ddF + np.where(m2, c[jm] * (-np.sin(b) * np.sin(xj) ** 2 - np.cos(b) * np.cos(xj)),
                             0.0)
        if s is None:
            s = 1.0 - np.sum(x * x, axis=1)
        return s * ddF - 4.0 * xj * dF - 2.0 * F

    def class_data(self, cls):
        idx = np.asarray(cls.aux["stde_idx"])
        x = cls.points
        F, s = self._F(x), 1.0 - np.sum(x * x, axis=1)  # shared by the k directions
        lap_ex = sum(self._exact_dd(x, idx[:, g], F, s) for g in range(self.k))
        return -(self.dim / self.k) * lap_ex

    def value_factor(self, pts):
        """u = (1 - |x|^2) phi on evaluation points."""
        return 1.0 - np.sum(pts * pts, axis=1)

    def exact_solution(self, pts):
        return (1.0 - np.sum(pts * pts, axis=1)) * self._F(pts)

    def eval_points(self, num=10_000):
        return _ball_interior(np.random.default_rng(0), num, self.dim)


PROBLEMS = {
    "poisson2d": Poisson2d,
    "poisson10d": Poisson10d,
    "heat2d": lambda: Heat(2),
    "heat10d": lambda: Heat(10),
    "heat1d": Heat1d,
    "poisson5d_sin": lambda: PoissonSin(5),
    "allen_cahn": AllenCahn,
    "poisson_ball_stde": PoissonBallStde,
}

UNSUPPORTED: set = set()


def make_problem(name: str, **kwargs) -> PdeProblem:
    if name in UNSUPPORTED:
        raise DomainError(
            f"problem {name!r} needs STDE subsampling, which the device residual map does "
            "not implement in this build"
        )
    if name not in PROBLEMS:
        raise DomainError(f"unknown problem {name!r}; available: {sorted(PROBLEMS)}")
    return PROBLEMS[name](**kwargs)


def sample_collocation(problem: PdeProblem, counts, rng) -> CollocationSet:
    """Reference problems.py:419-423."""
    if isinstance(rng, (int, np.integer)):
        rng = np.random.default_rng(rng)
    return problem.sample(counts, rng)


def build_map(problem: PdeProblem, spec, collocation: CollocationSet):
    from .residuals import PinnResidualMap

    return PinnResidualMap(problem, spec, collocation)


def eval_residuals(problem, spec, theta, points: CollocationSet):
    from .residuals import PinnResidualMap

    return PinnResidualMap(problem, spec, points).residual_batch(theta)
