"""Tanh MLP specification, layout and initialisers (reference model.py:22-67).

The network itself is evaluated only on the device (pinn.cu); this module
holds the host-side description: widths, flat layout W0 (in x out, row
major), b0, W1, b1, ..., and the seeded initialisers.
"""

from __future__ import annotations

from dataclasses import dataclass

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
