"""Gate-level circuit IR, mirroring the reference's `qvirt.circuits`
(pkg/src/qvirt/circuits.py:27-166): the same names, argument meaning and
validation errors, so code written against the reference runs unchanged.

B200-first difference: binding is lazy.  `bind(template, theta)` and the
parameter-shift generator return circuits that carry (template lowering,
angle row) and only build `Gate` objects if someone reads `.gates`.  The
executor lowers such batches straight to one topology plus an angle table
(no per-gate Python work), which is what removes the reference's 28.8 s
circuit-construction cost at 28 qubits x 8 layers.

Conventions are the reference's: angles in radians; qubit 0 is the most
significant bit of an amplitude index; bitstring character i is qubit i.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum
from typing import TYPE_CHECKING, Optional, Sequence

import numpy as np

if TYPE_CHECKING:  # pragma: no cover
    from .observables import Observable, PauliTerm

ParameterVector = Sequence[float]


class GateKind(Enum):
    """Gate set of the reference (circuits.py:27-33) plus RX and CZ."""

    H = "h"
    X = "x"
    CNOT = "cnot"
    RY = "ry"
    RZ = "rz"
    MEASURE_ALL = "measure_all"
    RX = "rx"   # extension (north star: RY/RZ/RX/CNOT/CZ fusion)
    CZ = "cz"   # extension


# C-ABI gate codes (include/qvb200.h QV_GATE_*)
KIND_CODE = {
    GateKind.H: 0, GateKind.X: 1, GateKind.CNOT: 2, GateKind.RY: 3,
    GateKind.RZ: 4, GateKind.MEASURE_ALL: 5, GateKind.RX: 6, GateKind.CZ: 7,
}
CODE_BY_VALUE = {k.value: c for k, c in KIND_CODE.items()}

_ARITY = {GateKind.H: 1, GateKind.X: 1, GateKind.RY: 1, GateKind.RZ: 1, GateKind.RX: 1,
          GateKind.CNOT: 2, GateKind.CZ: 2, GateKind.MEASURE_ALL: 0}
_ANGLED = frozenset({GateKind.RY, GateKind.RZ, GateKind.RX})


@dataclass(frozen=True)
class Gate:
    """One instruction: kind, target qubits, angle (float radians or a
    parameter name).  Validation follows circuits.py:71-96."""

    kind: GateKind
    targets: tuple[int, ...] = ()
    angle: float | str | None = None

    def __post_init__(self) -> None:
        targets = tuple(int(q) for q in self.targets)
        object.__setattr__(self, "targets", targets)
        arity = _ARITY[self.kind]
        if len(targets) != arity:
            raise ValueError(f"{self.kind.value} takes {arity} target(s), got {targets}")
        if min(targets, default=0) < 0:
            raise ValueError(f"negative qubit index in {targets}")
        if len(set(targets)) < len(targets):
            raise ValueError(f"repeated qubit index in {targets}")
        if self.kind in _ANGLED:
            if self.angle is None:
                raise ValueError(f"{self.kind.value} requires an angle")
            if not isinstance(self.angle, str):
                value = float(self.angle)
                if not math.isfinite(value):
                    raise ValueError(f"non-finite angle {value}")
                object.__setattr__(self, "angle", value)
        elif self.angle is not None:
            raise ValueError(f"{self.kind.value} takes no angle")

    @property
    def is_parameterized(self) -> bool:
        return isinstance(self.angle, str)

    def touches(self, qubit: int) -> bool:
        return self.kind is GateKind.MEASURE_ALL or qubit in self.targets


def h(qubit: int) -> Gate:
    return Gate(GateKind.H, (qubit,))


def x(qubit: int) -> Gate:
    return Gate(GateKind.X, (qubit,))


def cnot(control: int, target: int) -> Gate:
    return Gate(GateKind.CNOT, (control, target))


def cz(a: int, b: int) -> Gate:
    return Gate(GateKind.CZ, (a, b))


def ry(qubit: int, angle: float | str) -> Gate:
    return Gate(GateKind.RY, (qubit,), angle)


def rz(qubit: int, angle: float | str) -> Gate:
    return Gate(GateKind.RZ, (qubit,), angle)


def rx(qubit: int, angle: float | str) -> Gate:
    return Gate(GateKind.RX, (qubit,), angle)


def measure_all() -> Gate:
    return Gate(GateKind.MEASURE_ALL)


class Lowering:
    """Structure-of-arrays form of a gate list: the topology (kinds, qubits)
    plus, per gate, either a literal angle or the index of the parameter that
    supplies it.  Shared by every circuit bound from the same template."""

    __slots__ = ("n_qubits", "kinds", "q0", "q1", "param_index", "literal", "n_params", "gates", "_key")

    def __init__(self, n_qubits: int, gates: Sequence[Gate], params: Sequence[str]):
        slot = {p: i for i, p in enumerate(params)}
        count = len(gates)
        self.n_qubits = n_qubits
        self.kinds = np.empty(count, dtype=np.uint8)
        self.q0 = np.zeros(count, dtype=np.int32)
        self.q1 = np.full(count, -1, dtype=np.int32)
        self.param_index = np.full(count, -1, dtype=np.int64)
        self.literal = np.zeros(count, dtype=np.float64)
        for i, g in enumerate(gates):
            self.kinds[i] = KIND_CODE[g.kind]
            if g.targets:
                self.q0[i] = g.targets[0]
            if len(g.targets) > 1:
                self.q1[i] = g.targets[1]
            if isinstance(g.angle, str):
                self.param_index[i] = slot[g.angle]
            elif g.angle is not None:
                self.literal[i] = g.angle
        self.n_params = len(params)
        self.gates = tuple(gates)
        self._key = None

    def key(self) -> bytes:
        if self._key is None:
            self._key = (np.int64(self.n_qubits).tobytes() + self.kinds.tobytes()
                         + self.q0.tobytes() + self.q1.tobytes())
        return self._key

    def gate_angles(self, values: np.ndarray) -> np.ndarray:
        """Per-gate angles for parameter rows `values` ([..., n_params])."""
        values = np.asarray(values, dtype=np.float64)
        idx = np.where(self.param_index >= 0, self.param_index, 0)
        out = values[..., idx]
        return np.where(self.param_index >= 0, out, self.literal)


class BoundRows:
    """A table of parameter rows bound to one template lowering (a whole
    parameter-shift batch shares one of these)."""

    __slots__ = ("lowering", "values")

    def __init__(self, lowering: Lowering, values: np.ndarray):
        self.lowering = lowering
        self.values = values   # [rows, n_params] float64


class Circuit:
    """Immutable gate sequence on `n_qubits` qubits (reference circuits.py:112-153).

    `params` declares free parameter names in binding order; `observable`
    optionally names the quantity an executor should return.
    """

    __slots__ = ("n_qubits", "name", "params", "observable", "_gates", "_rows", "_row", "_lowering")

    def __init__(self, n_qubits: int, gates: Sequence[Gate] = (), name: str = "circuit",
                 params: Sequence[str] = (), observable: "PauliTerm | Observable | None" = None,
                 *, _rows: Optional[BoundRows] = None, _row: int = 0):
        object.__setattr__(self, "n_qubits", int(n_qubits))
        object.__setattr__(self, "name", name)
        object.__setattr__(self, "params", tuple(params))
        object.__setattr__(self, "observable", observable)
        object.__setattr__(self, "_rows", _rows)
        object.__setattr__(self, "_row", _row)
        object.__setattr__(self, "_lowering", None)
        if _rows is not None:
            object.__setattr__(self, "_gates", None)
            if self.n_qubits < 1:
                raise ValueError(f"n_qubits must be positive, got {self.n_qubits}")
            if not name:
                raise ValueError("circuit name must be nonempty")
            return
        object.__setattr__(self, "_gates", tuple(gates))
        if self.n_qubits < 1:
            raise ValueError(f"n_qubits must be positive, got {self.n_qubits}")
        if not name:
            raise ValueError("circuit name must be nonempty")
        if len(set(self.params)) != len(self.params):
            raise ValueError("duplicate parameter names")
        declared = set(self.params)
        for g in self._gates:
            for q in g.targets:
                if q >= self.n_qubits:
                    raise ValueError(f"gate {g.kind.value} targets qubit {q} on {self.n_qubits} qubits")
            if isinstance(g.angle, str) and g.angle not in declared:
                raise ValueError(f"unbound parameter {g.angle!r}")

    def __setattr__(self, key, value):
        raise AttributeError("Circuit is immutable")

    def __repr__(self) -> str:
        return f"Circuit(n_qubits={self.n_qubits}, name={self.name!r}, gates={len(self.gates)})"

    @property
    def gates(self) -> tuple[Gate, ...]:
        if self._gates is None:   # materialise a lazily bound circuit
            lw = self._rows.lowering
            angles = lw.gate_angles(self._rows.values[self._row])
            gates = tuple(
                Gate(g.kind, g.targets, float(angles[i])) if isinstance(g.angle, str) else g
                for i, g in enumerate(lw.gates)
            )
            object.__setattr__(self, "_gates", gates)
        return self._gates

    @property
    def is_parameterized(self) -> bool:
        if self._rows is not None:
            return False
        return any(g.is_parameterized for g in self._gates)

    def _copy(self, **changes) -> "Circuit":
        fields = {"name": self.name, "observable": self.observable}
        fields.update(changes)
        if self._rows is not None:
            return Circuit(self.n_qubits, (), fields["name"], (), fields["observable"], _rows=self._rows, _row=self._row)
        return Circuit(self.n_qubits, self._gates, fields["name"], self.params, fields["observable"])

    def with_name(self, name: str) -> "Circuit":
        return self._copy(name=name)

    def with_observable(self, observable) -> "Circuit":
        return self._copy(observable=observable)

    def lowering(self) -> Lowering:
        """Topology + angle sources of this circuit's (template) gate list."""
        if self._rows is not None:
            return self._rows.lowering
        if self._lowering is None:
            object.__setattr__(self, "_lowering", Lowering(self.n_qubits, self._gates, self.params))
        return self._lowering

    def bound_rows(self) -> tuple[Optional[BoundRows], int]:
        return self._rows, self._row


def bind(circuit: Circuit, theta: ParameterVector) -> Circuit:
    """Substitute parameter values positionally (reference circuits.py:156-166)."""
    values = [float(v) for v in theta]
    if len(values) != len(circuit.params):
        raise ValueError(f"expected {len(circuit.params)} parameter values, got {len(values)}")
    for v in values:
        if not math.isfinite(v):
            raise ValueError(f"non-finite angle {v}")
    rows = BoundRows(circuit.lowering(), np.asarray([values], dtype=np.float64).reshape(1, len(values)))
    return Circuit(circuit.n_qubits, (), circuit.name, (), circuit.observable, _rows=rows, _row=0)


def bind_rows(circuit: Circuit, values: np.ndarray, names: Sequence[str]) -> list[Circuit]:
    """Bind many parameter rows at once; row i becomes a circuit named names[i]."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    if values.ndim != 2 or values.shape[1] != len(circuit.params):
        raise ValueError(f"expected rows of {len(circuit.params)} parameter values")
    if not np.all(np.isfinite(values)):
        raise ValueError("non-finite angle")
    rows = BoundRows(circuit.lowering(), values)
    return [Circuit(circuit.n_qubits, (), nm, (), circuit.observable, _rows=rows, _row=i)
            for i, nm in enumerate(names)]
