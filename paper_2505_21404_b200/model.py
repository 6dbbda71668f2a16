"""Tanh MLP specification, layout and initialisers (reference model.py:22-67).

The network itself is evaluated only on the device (pinn.cu); this module
holds the host-side description: widths, flat layout W0 (in x out, row
major), b0, W1, b1, ..., and the seeded initialisers.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DomainError
from .params import ParameterLayout, ParameterVector


@dataclass(frozen=True)
class MlpSpec:
    """Layer widths input -> hidden... -> output; tanh on hidden layers (model.py:22-54)."""

    layer_widths: tuple[int, ...]
    seed: int = 0

    def __post_init__(self):
        if len(self.layer_widths) < 2:
            raise DomainError("an MLP needs at least input and output widths")
        if any(w < 1 for w in self.layer_widths):
            raise DomainError(f"layer widths must be >= 1, got {self.layer_widths}")
        object.__setattr__(self, "layer_widths", tuple(int(w) for w in self.layer_widths))

    @property
    def input_dim(self) -> int:
        return self.layer_widths[0]

    @property
    def output_dim(self) -> int:
        return self.layer_widths[-1]

    def param_count(self) -> int:
        w = self.layer_widths
        return sum((w[k] + 1) * w[k + 1] for k in range(len(w) - 1))

    def layout(self) -> ParameterLayout:
        entries = []
        w = self.layer_widths
        for k in range(len(w) - 1):
            entries.append((f"W{k}", (w[k], w[k + 1])))
            entries.append((f"b{k}", (w[k + 1],)))
        return ParameterLayout(entries)

    def layer_offsets(self) -> list[int]:
        offs, off = [], 0
        w = self.layer_widths
        for k in range(len(w) - 1):
            offs.append(off)
            off += (w[k] + 1) * w[k + 1]
        return offs


def init_params(spec: MlpSpec) -> ParameterVector:
    """Uniform Glorot weights, zero biases -- the reference default (model.py:57-67)."""
    rng = np.random.default_rng(spec.seed)
    arrays = []
    w = spec.layer_widths
    for k in range(len(w) - 1):
        scale = np.sqrt(6.0 / (w[k] + w[k + 1]))
        arrays.append(rng.uniform(-scale, scale, size=(w[k], w[k + 1])))
        arrays.append(np.zeros(w[k + 1]))
    return ParameterVector.from_arrays(arrays, spec.layout())


def xavier_normal_params(spec: MlpSpec) -> ParameterVector:
    """Xavier-normal N(0, 2/(fan_in+fan_out)) weights, zero biases (BASELINE configs).

    Same generator discipline as init_params: default_rng(spec.seed), layers in layout order.
    """
    rng = np.random.default_rng(spec.seed)
    arrays = []
    w = spec.layer_widths
    for k in range(len(w) - 1):
        std = np.sqrt(2.0 / (w[k] + w[k + 1]))
        arrays.append(rng.normal(0.0, std, size=(w[k], w[k + 1])))
        arrays.append(np.zeros(w[k + 1]))
    return ParameterVector.from_arrays(arrays, spec.layout())


INITIALIZERS = {"glorot_uniform": init_params, "xavier_normal": xavier_normal_params}


# -- output transforms (reference model.py:181-277) ----------------------------------------


@dataclass(frozen=True)
class OutputTransform:
    """Hard-constraint wrappers on the raw network output phi (model.py:181-197).

    identity:       u = phi
    dirichlet_ball: u = (1 - |x|^2) phi (PoissonBallStde states it as per-point
                    channel coefficients, problems.py)
    ic_shift:       u(t, x) = phi(t, x) - phi(0, x) + q0(x), exact at t = 0; evaluated
                    as two device residual maps (residuals.IcShiftResidualMap)

    `q0` is a callable on per-coordinate columns written with numpy ufuncs
    (np.sin, np.exp, ...) and arithmetic, so it evaluates on plain columns and on
    `HostJet` columns alike (the reference's algebra-generic q0).
    """

    kind: str = "identity"
    q0: object = field(default=None, compare=False)

    def __post_init__(self):
        if self.kind not in ("identity", "dirichlet_ball", "ic_shift"):
            raise DomainError(f"unknown output transform kind: {self.kind}")
        if self.kind == "ic_shift" and self.q0 is None:
            raise DomainError("ic_shift transform needs the initial function q0")


class HostJet:
    """2-jet (value, d1, d2) along one coordinate direction, numpy arrays -- the host
    evaluation of the data terms' derivatives (L q0 for ic_shift; reference Jet2,
    jets.py).  Supports + - * / ** and the ufuncs sin, cos, exp, tanh, negative."""

    __slots__ = ("v", "d1", "d2")
    __array_priority__ = 1000

    def __init__(self, v, d1, d2):
        self.v, self.d1, self.d2 = v, d1, d2

    @staticmethod
    def lift(x):
        if isinstance(x, HostJet):
            return x
        z = np.zeros_like(np.asarray(x, dtype=np.float64))
        return HostJet(np.asarray(x, dtype=np.float64), z, z)

    def __add__(self, o):
        o = HostJet.lift(o)
        return HostJet(self.v + o.v, self.d1 + o.d1, self.d2 + o.d2)

    __radd__ = __add__

    def __neg__(self):
        return HostJet(-self.v, -self.d1, -self.d2)

    def __sub__(self, o):
        return self + (-HostJet.lift(o))

    def __rsub__(self, o):
        return HostJet.lift(o) + (-self)

    def __mul__(self, o):
        o = HostJet.lift(o)
        return HostJet(self.v * o.v, self.d1 * o.v + self.v * o.d1,
                       self.d2 * o.v + 2.0 * self.d1 * o.d1 + self.v * o.d2)

    __rmul__ = __mul__

    def _chain(self, f0, f1, f2):
        return HostJet(f0, f1 * self.d1, f1 * self.d2 + f2 * self.d1 * self.d1)

    def reciprocal(self):
        r = 1.0 / self.v
        return self._chain(r, -r * r, 2.0 * r * r * r)

    def __truediv__(self, o):
        return self * HostJet.lift(o).reciprocal()

    def __rtruediv__(self, o):
        return HostJet.lift(o) * self.reciprocal()

    def __pow__(self, p: int):
        p = int(p)
        out = HostJet.lift(np.ones_like(self.v))
        for _ in range(p):
            out = out * self
        return out

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        if method != "__call__" or len(inputs) not in (1, 2) or kwargs:
            return NotImplemented
        if len(inputs) == 2:
            a, b = (HostJet.lift(x) for x in inputs)
            ops = {np.add: a.__add__, np.subtract: a.__sub__, np.multiply: a.__mul__,
                   np.true_divide: a.__truediv__}
            if ufunc not in ops:
                return NotImplemented
            return ops[ufunc](b)
        x = self.v
        if ufunc is np.sin:
            return self._chain(np.sin(x), np.cos(x), -np.sin(x))
        if ufunc is np.cos:
            return self._chain(np.cos(x), -np.sin(x), -np.cos(x))
        if ufunc is np.exp:
            e = np.exp(x)
            return self._chain(e, e, e)
        if ufunc is np.tanh:
            t = np.tanh(x)
            s = 1.0 - t * t
            return self._chain(t, s, -2.0 * t * s)
        if ufunc is np.negative:
            return -self
        return NotImplemented


def point_columns(pts: np.ndarray, direction=None) -> list:
    """Per-coordinate columns (model.py:200-211): plain numpy columns, or HostJet
    2-jets along the unit coordinate `direction`."""
    d = pts.shape[1]
    if direction is None:
        return [pts[:, i] for i in range(d)]
    zero = np.zeros(pts.shape[0])
    one = np.ones(pts.shape[0])
    return [HostJet(pts[:, i], one if i == int(direction) else zero, zero) for i in range(d)]


def jet_value(x, n: int) -> HostJet:
    """A q0 result as a HostJet over n points (constants and plain arrays lift)."""
    if isinstance(x, HostJet):
        return x
    return HostJet.lift(np.broadcast_to(np.asarray(x, dtype=np.float64), (n,)).copy())
