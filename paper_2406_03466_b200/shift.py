"""Parameter-shift machinery, mirroring the reference's `qvirt.gradients`
(pkg/src/qvirt/gradients.py:17-60).

`shifted_circuits` yields the same (k, tag, circuit) sequence -- k-major, '+'
before '-', angle theta[k] + sign*pi/2 computed with the same IEEE double
addition -- but the circuits are rows of one shared angle table bound lazily
to the template, so a 28-qubit x 8-layer batch (2688 circuits x 1588 gates)
costs one numpy table instead of 4.27M Gate objects.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Iterator, Sequence

import numpy as np

from .ir import Circuit, bind_rows

SHIFT = math.pi / 2

# '+' precedes '-' for every parameter (fixes the batch layout)
SHIFT_TAGS = ((1.0, "+"), (-1.0, "-"))


@dataclass(frozen=True)
class GradientReport:
    """One gradient evaluation: the vector, its cost, its pool wall time."""

    gradient: tuple[float, ...]
    n_circuit_executions: int
    wall_time_s: float


def shift_table(theta: Sequence[float]) -> np.ndarray:
    """[2P, P] parameter rows: row 2k+s is theta with theta[k] += sign_s * SHIFT."""
    base = np.asarray([float(v) for v in theta], dtype=np.float64)
    count = base.shape[0]
    rows = np.repeat(base[None, :], 2 * count, axis=0)
    ks = np.arange(count)
    for s, (sign, _) in enumerate(SHIFT_TAGS):
        rows[2 * ks + s, ks] = base + sign * SHIFT   # same double add as `shifted[k] += sign * SHIFT`
    return rows


def shifted_batch(template: Circuit, theta: Sequence[float], names: Sequence[str] | None = None) -> list[Circuit]:
    """All 2P shifted circuits, lazily bound to one shared angle table."""
    values = [float(v) for v in theta]
    if len(values) != len(template.params):
        raise ValueError(f"expected {len(template.params)} angles, got {len(values)}")
    table = shift_table(values)
    if names is None:
        names = [template.name] * table.shape[0]
    return bind_rows(template, table, names)


def shifted_circuits(template: Circuit, theta: Sequence[float]) -> Iterator[tuple[int, str, Circuit]]:
    """Yield (k, tag, bound circuit) for theta[k] +- pi/2, k-major, '+' first."""
    batch = shifted_batch(template, theta)
    for i, circuit in enumerate(batch):
        k, s = divmod(i, 2)
        yield k, SHIFT_TAGS[s][1], circuit


def central_difference(loss, theta: Sequence[float], h: float = 1e-4) -> list[float]:
    """(loss(theta + h e_k) - loss(theta - h e_k)) / 2h; the estimator shift
    results are validated against (gradients.py:49-60)."""
    base = [float(v) for v in theta]
    grad = []
    for k in range(len(base)):
        up, down = list(base), list(base)
        up[k] += h
        down[k] -= h
        grad.append((loss(up) - loss(down)) / (2.0 * h))
    return grad
