"""The accelerator plugin: `B200Backend.execute(buffer, circuits, config)`.

Drop-in for the reference's `StatevectorBackend` (pkg/src/qvirt/backend.py:189-227)
behind the `Accelerator` protocol (:182-186): one `ChildResult` per circuit in
input order; with an observable the exact expectation (coefficient and
constant applied as in :94-101), without one the exact outcome distribution
(:122-137).  Errors name the failing circuit with `ExecutionError` (:36-41)
and leave earlier children in the buffer, as the reference's serial loop does.

Everything numerical runs in libqvb200.so on a B200 (native.py).  There is no
CPU execution path: without the library or a GPU, construction raises.

Distribution results.  Exact-mode distributions at large n are 2^n-entry
dicts in the reference (1.67 s per circuit at 20 qubits, infeasible at 28).
Constructed with `support=` (a target distribution or its bitstrings), the
backend instead returns the normalised probabilities on that support plus
one off-support key carrying the remaining mass.  Jensen-Shannon divergence
against a target with that support is unchanged by the lumping
(JS(P,Q) = sum_{b in supp P}[...] + (ln 2 / 2)(1 - sum_{b in supp P} q_b)),
so the reference's `ddcl_gradient` (ddcl.py:197-226) computes the same
gradient from these children.
"""

from __future__ import annotations

import itertools
import math
import threading
from operator import attrgetter, itemgetter
from dataclasses import dataclass
from typing import Callable, Iterable, Mapping, Protocol, Sequence

import numpy as np

from . import native
from .ir import CODE_BY_VALUE, Circuit, bind, h, measure_all
from .observables import Observable, PauliTerm, term_masks
from .results import ChildResult, ResultBuffer

MODES = ("expectation", "counts")
MAX_FULL_DISTRIBUTION_QUBITS = 24


class ExecutionError(RuntimeError):
    """A circuit failed during batch execution; the batch is abandoned."""

    def __init__(self, circuit_name: str, message: str):
        super().__init__(f"circuit {circuit_name!r}: {message}")
        self.circuit_name = circuit_name


@dataclass(frozen=True)
class ExecutionConfig:
    """How a backend runs one batch (reference backend.py:160-179)."""

    mode: str = "expectation"
    shots: int = 8192
    seed: int = 0
    first_global_index: int = 0

    def __post_init__(self) -> None:
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.shots < 1:
            raise ValueError(f"shots must be positive, got {self.shots}")
        if self.first_global_index < 0:
            raise ValueError("first_global_index must be nonnegative")


class Accelerator(Protocol):
    def execute(self, buffer: ResultBuffer, circuits: Sequence[Circuit], config: ExecutionConfig) -> None:
        ...


# ---------------------------------------------------------------------------
# lowering: Circuit objects -> C-ABI gate arrays

_KIND_OF = attrgetter("kind")
_TARGETS_OF = attrgetter("targets")
_ANGLE_OF = attrgetter("angle")


class _ForeignTopology:
    """Gate arrays of one reference-shaped gate list (duck-typed: .gates with
    .kind.value / .targets / .angle, e.g. a `qvirt.Circuit`), reused for every
    later circuit with the same kinds and targets (a parameter-shift batch is
    2 N_theta bindings of one template, gradients.py:33-46).  The per-circuit
    work is three C-level passes over the gate tuple (kinds, targets, and the
    angles of the rotation gates) instead of a Python loop per gate."""

    def __init__(self, gates):
        self.kind_list = list(map(_KIND_OF, gates))
        self.target_list = list(map(_TARGETS_OF, gates))
        count = len(gates)
        self.kinds = np.fromiter((CODE_BY_VALUE[k.value] for k in self.kind_list), np.uint8, count)
        self.q0 = np.fromiter((t[0] if t else 0 for t in self.target_list), np.int32, count)
        self.q1 = np.fromiter((t[1] if len(t) > 1 else -1 for t in self.target_list), np.int32, count)
        angles = list(map(_ANGLE_OF, gates))
        self.rot = np.fromiter((i for i, a in enumerate(angles) if a is not None), np.int64)
        self.pick = itemgetter(*self.rot.tolist()) if self.rot.size > 1 else None

    def matches(self, gates) -> bool:
        return (len(gates) == len(self.kind_list) and list(map(_KIND_OF, gates)) == self.kind_list
                and list(map(_TARGETS_OF, gates)) == self.target_list)

    def angles(self, gates) -> np.ndarray:
        ang = np.zeros(len(self.kind_list), np.float64)
        if self.rot.size == 0:
            return ang
        chosen = self.pick(gates) if self.pick is not None else (gates[int(self.rot[0])],)
        try:
            ang[self.rot] = np.fromiter(map(_ANGLE_OF, chosen), np.float64, self.rot.size)
        except (TypeError, ValueError):
            bad = next(a for a in map(_ANGLE_OF, chosen) if not isinstance(a, (int, float)))
            raise ValueError(f"unbound parameter {bad!r}; bind before executing") from None
        return ang


def _foreign_arrays(circuit, topo: _ForeignTopology | None = None):
    """(kinds, q0, q1, angles) of a reference-shaped circuit, and the
    topology they came from (reused when `topo` matches)."""
    gates = tuple(circuit.gates)
    if topo is None or not topo.matches(gates):
        topo = _ForeignTopology(gates)
    return (topo.kinds, topo.q0, topo.q1, topo.angles(gates)), topo


def lower_batch(circuits: Sequence) -> native.LoweredBatch:
    """One topology + angle table when every circuit was bound from the same
    template (the parameter-shift case: no per-gate Python work), otherwise
    concatenated per-circuit gate lists."""
    first = circuits[0]
    rows0 = first.bound_rows()[0] if isinstance(first, Circuit) else None
    if rows0 is not None:
        lw = rows0.lowering
        if all(isinstance(c, Circuit) and c._rows is not None and c._rows.lowering is lw for c in circuits):
            tables = {}
            for i, c in enumerate(circuits):
                tables.setdefault(id(c._rows), (c._rows, []))[1].append(i)
            if len(tables) == 1:
                values = rows0.values[np.fromiter((c._row for c in circuits), np.int64, len(circuits))]
            else:
                values = np.stack([c._rows.values[c._row] for c in circuits])
            angles = lw.gate_angles(values)
            return native.LoweredBatch(len(circuits), True, lw.kinds.shape[0], None, lw.kinds, lw.q0, lw.q1, angles)
    parts = []
    topo = None
    for c in circuits:
        if isinstance(c, Circuit) and not c.is_parameterized:
            if c._rows is not None:
                lw = c._rows.lowering
                parts.append((lw.kinds, lw.q0, lw.q1, lw.gate_angles(c._rows.values[c._row])))
            else:
                lw = c.lowering()
                parts.append((lw.kinds, lw.q0, lw.q1, lw.literal))
        else:
            arrays, topo = _foreign_arrays(c, topo)
            parts.append(arrays)
    counts = np.fromiter((p[0].shape[0] for p in parts), np.int64, len(parts))
    offsets = np.zeros(len(parts) + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    cat = lambda j, dt: np.concatenate([p[j] for p in parts]).astype(dt, copy=False) if offsets[-1] else np.zeros(0, dt)
    return native.LoweredBatch(len(parts), False, 0, offsets, cat(0, np.uint8), cat(1, np.int32),
                               cat(2, np.int32), cat(3, np.float64))


def _gate_count(circuits: Sequence) -> int:
    total = 0
    for c in circuits:
        if isinstance(c, Circuit) and c._rows is not None:
            total += int(c._rows.lowering.kinds.shape[0])
        else:
            total += len(c.gates)
    return total


def support_indices(support, n_qubits: int) -> np.ndarray:
    """Sorted unique amplitude indices of a support given as a target
    distribution (bitstring keys), bitstrings, or integer indices."""
    items = list(support.keys()) if isinstance(support, Mapping) else list(support)
    if items and all(isinstance(item, str) for item in items):
        # every key must be n bits wide: a joined length check alone would let
        # keys of mixed widths ('0', '111' for n = 2) parse into a wrong support
        bad = next((it for it in items if len(it) != n_qubits), None)
        if bad is not None:
            raise ValueError(f"bad support bitstring {bad!r} for {n_qubits} qubits")
        # vectorised parse: one uint8 row per bitstring, most significant bit first
        try:
            raw = np.frombuffer("".join(items).encode("ascii"), dtype=np.uint8)
        except UnicodeEncodeError:
            raw = None
        if raw is None or raw.size != len(items) * n_qubits or n_qubits > 64:
            bad = next((it for it in items if len(it) != n_qubits), items[0])
            raise ValueError(f"bad support bitstring {bad!r} for {n_qubits} qubits")
        bits = raw.reshape(len(items), n_qubits) - np.uint8(48)
        if np.any(bits > 1):
            bad = items[int(np.nonzero(np.any(bits > 1, axis=1))[0][0])]
            raise ValueError(f"bad support bitstring {bad!r} for {n_qubits} qubits")
        weights = np.left_shift(np.uint64(1), np.arange(n_qubits - 1, -1, -1, dtype=np.uint64))
        arr = np.unique((bits.astype(np.uint64) * weights).sum(axis=1, dtype=np.uint64))
        return arr
    idx = []
    for item in items:
        if isinstance(item, str):
            if len(item) != n_qubits or set(item) - {"0", "1"}:
                raise ValueError(f"bad support bitstring {item!r} for {n_qubits} qubits")
            idx.append(int(item, 2))
        else:
            idx.append(int(item))
    arr = np.unique(np.asarray(idx, dtype=np.uint64))
    if arr.size and int(arr[-1]) >> n_qubits:
        raise ValueError("support index beyond the register")
    return arr


def _first_gap(sorted_idx: np.ndarray, n_qubits: int) -> int | None:
    """Smallest index not in the support (the remainder key), or None."""
    if sorted_idx.size == 0:
        return 0
    ar = np.arange(sorted_idx.size, dtype=np.uint64)
    miss = np.nonzero(sorted_idx != ar)[0]
    gap = int(miss[0]) if miss.size else int(sorted_idx.size)
    return gap if gap < (1 << n_qubits) else None


_device_cursor = itertools.count()
_device_lock = threading.Lock()


def _next_device() -> int:
    count = native.device_count()
    if count < 1:
        raise native.NativeUnavailable("no CUDA device visible to libqvb200.so")
    with _device_lock:
        return next(_device_cursor) % count


class B200Backend:
    """State-vector executor on one B200.

    Instances are cheap; each worker thread of the virtual-QPU pool gets its
    own (reference backend.py:189-201).  Instances on the same device share
    one native engine, whose calls serialise.  Without `device`, devices are
    assigned round-robin across the visible GPUs at construction.
    """

    def __init__(self, device: int | None = None, precision: str = "complex128",
                 support: Mapping[str, float] | Iterable | None = None):
        self.device = _next_device() if device is None else int(device)
        self.precision = precision
        self._engine = native.engine(self.device, precision)
        self._support_spec = support
        self._support_cache: dict[int, np.ndarray] = {}
        self.gate_counter = 0
        self.last_stats: dict[str, float] = {}

    # -- Accelerator -------------------------------------------------------
    def execute(self, buffer: ResultBuffer, circuits: Sequence[Circuit], config: ExecutionConfig) -> None:
        n = buffer.n_qubits
        counts = config.mode == "counts"
        stop, reason = len(circuits), ""
        for i, c in enumerate(circuits):
            reason = self._precheck(c, n, children=not counts) or (self._counts_precheck(c, n) if counts else "")
            if reason:
                stop = i
                break
        ok = circuits[:stop]
        if ok:
            children = self._counts_children(ok, n, config) if config.mode == "counts" else self._children(ok, n)
            if hasattr(buffer, "extend_children"):
                buffer.extend_children(children)
            else:   # a reference `qvirt.ResultBuffer`
                for child in children:
                    buffer.append_child(child)
        if stop < len(circuits):
            raise ExecutionError(circuits[stop].name, reason)

    # -- B200 fast paths (no ChildResult objects) --------------------------
    def expectation_values(self, circuits: Sequence[Circuit], n_qubits: int) -> np.ndarray:
        """Exact expectation of each circuit's observable (coefficients and
        constant applied), float64 [len(circuits)]."""
        self._check_all(circuits, n_qubits)
        return self._expectations(circuits, n_qubits)

    def js_losses(self, circuits: Sequence[Circuit], n_qubits: int, target: Mapping[str, float]) -> np.ndarray:
        """JS(target || p_c) for each circuit's exact distribution (ddcl.py:37-61),
        computed on the device; float64 [len(circuits)]."""
        self._check_all(circuits, n_qubits)
        keys = sorted(target)
        sup = support_indices(keys, n_qubits)
        order = np.argsort(np.asarray([int(k, 2) for k in keys], dtype=np.uint64), kind="stable")
        p = np.asarray([float(target[k]) for k in keys], dtype=np.float64)[order]
        lowered = lower_batch(circuits)
        out = self._run(lowered, n_qubits, native.QV_OUT_JS, circuits, support=sup, target=p)
        self.gate_counter += _gate_count(circuits)
        return out

    def pauli_values(self, circuits: Sequence[Circuit], n_qubits: int, term_offsets: np.ndarray,
                     xmask: np.ndarray, ymask: np.ndarray, zmask: np.ndarray) -> np.ndarray:
        """Raw <P_t> of Pauli strings given as masks (bit n-1-q for qubit q),
        terms term_offsets[c]..term_offsets[c+1] on circuit c: float64
        [term_offsets[-1]].  The circuits' own observables are ignored."""
        self._check_all(circuits, n_qubits)
        out = self._run(lower_batch(circuits), n_qubits, native.QV_OUT_PAULI, circuits,
                        terms=(np.ascontiguousarray(term_offsets, np.int64), np.ascontiguousarray(xmask, np.uint64),
                               np.ascontiguousarray(ymask, np.uint64), np.ascontiguousarray(zmask, np.uint64)))
        self.gate_counter += _gate_count(circuits)
        return out

    def support_probabilities(self, circuits: Sequence[Circuit], n_qubits: int, support) -> np.ndarray:
        """Exact Born probabilities p_c(b) = |<b|psi_c>|^2 / <psi_c|psi_c> of each
        circuit on the basis states `support` (bit strings or indices, taken in
        ascending index order; see `support_indices`): float64
        [len(circuits), len(support)].  Only the support's light cone is swept."""
        self._check_all(circuits, n_qubits)
        sup = support_indices(support, n_qubits)
        flat = self._run(lower_batch(circuits), n_qubits, native.QV_OUT_SUPPORT, circuits, support=sup)
        self.gate_counter += _gate_count(circuits)
        return flat.reshape(len(circuits), sup.size + 1)[:, : sup.size]

    def js_losses_targets(self, circuits: Sequence[Circuit], n_qubits: int, support, targets: np.ndarray) -> np.ndarray:
        """JS(targets[c] || P_c) for each circuit against its OWN target row
        (config 3's forward batch: one target per data point), float64
        [len(circuits)].  `targets` is [len(circuits), len(support)] in the
        support's ascending index order; the losses are formed on the device
        from the support + remainder identity (ddcl.py:37-61), so only one
        scalar per circuit comes back."""
        self._check_all(circuits, n_qubits)
        sup = support_indices(support, n_qubits)
        t = np.ascontiguousarray(targets, dtype=np.float64)
        if t.shape != (len(circuits), sup.size):
            raise ValueError(f"expected targets of shape ({len(circuits)}, {sup.size}), got {t.shape}")
        out = self._run(lower_batch(circuits), n_qubits, native.QV_OUT_JS, circuits, support=sup, target=t,
                        flags=native.QV_RES_TARGET_ROWS)
        self.gate_counter += _gate_count(circuits)
        return out[: len(circuits)]

    def js_losses_rows(self, template: Circuit, values: np.ndarray, target: Mapping[str, float],
                       name_of: Callable[[int], str] | None = None) -> np.ndarray:
        """`js_losses` of the template bound to each parameter row of `values`
        ([rows, n_params]): one uniform lowered batch, no per-row circuit
        objects (the parameter-shift tables of the gradient drivers)."""
        values = np.ascontiguousarray(values, dtype=np.float64)
        lw = template.lowering()
        if values.ndim != 2 or values.shape[1] != lw.n_params:
            raise ValueError(f"expected rows of {lw.n_params} parameter values")
        if not np.all(np.isfinite(values)):
            raise ValueError("non-finite angle")
        n = template.n_qubits
        lowered = native.LoweredBatch(values.shape[0], True, lw.kinds.shape[0], None, lw.kinds, lw.q0, lw.q1,
                                      lw.gate_angles(values))
        keys = sorted(target)
        sup = support_indices(keys, n)
        order = np.argsort(np.asarray([int(k, 2) for k in keys], dtype=np.uint64), kind="stable")
        p = np.asarray([float(target[k]) for k in keys], dtype=np.float64)[order]
        try:
            out = self._engine.execute(n, lowered, native.QV_OUT_JS, support=sup, target=p)
        except native.NativeError as err:
            name = name_of(err.circuit) if name_of else f"{template.name}[row {err.circuit}]"
            raise ExecutionError(name, str(err)) from err
        self.last_stats = dict(self._engine.last_stats)
        self.gate_counter += values.shape[0] * int(lw.kinds.shape[0])
        return out

    def shift_js_losses(self, template: Circuit, theta: Sequence[float], target: Mapping[str, float],
                        params: Sequence[int]) -> np.ndarray:
        """JS losses of the circuits with theta[k] + pi/2 and theta[k] - pi/2,
        for each k in `params`: [2 * len(params)], '+' then '-' per parameter.

        Uses R(t +- pi/2) = R(t)(I -+ iP)/sqrt2: the unshifted output Psi0 plus
        ONE extra state per parameter (P inserted at the parameter's gate)
        replace the two shifted circuits (qv_shift_js).  Exact up to FP64
        rounding; each parameter must feed exactly one rotation gate, and the
        register must span several tiles (otherwise use `js_losses`)."""
        n = template.n_qubits
        lw = template.lowering()
        gate_of = np.full(lw.n_params, -1, np.int64)
        for g, k in enumerate(lw.param_index.tolist()):
            if k >= 0:
                if gate_of[k] >= 0:
                    raise ValueError(f"parameter {k} feeds several gates; shift pairs need one gate per parameter")
                gate_of[k] = g
        ks = np.asarray(params, dtype=np.int64)
        if np.any(gate_of[ks] < 0):
            raise ValueError("a shifted parameter feeds no gate")
        base = lower_batch([bind(template, theta)])
        keys = sorted(target)
        sup = support_indices(keys, n)
        p = np.asarray([float(target[k]) for k in keys], dtype=np.float64)
        name = template.name
        try:
            out = self._engine.shift_js(n, base, gate_of[ks], sup, p)
        except native.NativeError as err:
            raise ExecutionError(name, str(err)) from err
        self.last_stats = dict(self._engine.last_stats)
        self.gate_counter += 2 * len(ks) * int(lw.kinds.shape[0])
        return out

    def tile_qubits(self) -> int:
        """Widest register simulated inside one CTA's shared memory."""
        return 12

    # -- internals -----------------------------------------------------------
    def _precheck(self, c, n: int, children: bool = True) -> str:
        if c.n_qubits != n:
            return f"circuit has {c.n_qubits} qubits, buffer {n}"
        if c.is_parameterized:
            bad = next(g.angle for g in c.gates if isinstance(g.angle, str))
            return f"unbound parameter {bad!r}; bind before executing"
        obs = c.observable
        if obs is not None and obs.min_qubits > n:
            return f"term on qubit {obs.min_qubits - 1} exceeds {n} qubits"
        if children and obs is None and self._support_spec is None and n > MAX_FULL_DISTRIBUTION_QUBITS:
            return (f"a full {n}-qubit distribution has 2^{n} entries; construct the backend "
                    "with support= to receive the target support plus the remainder")
        return ""

    @staticmethod
    def _counts_precheck(c, n: int) -> str:
        """Counts-mode rules of reference backend.py:220-223, pauli.py:147-162."""
        obs = c.observable
        if n > MAX_FULL_DISTRIBUTION_QUBITS:
            return f"counts mode samples a 2^{n} distribution; limited to {MAX_FULL_DISTRIBUTION_QUBITS} qubits"
        if obs is None:
            return ""
        if hasattr(obs, "terms"):
            return "counts mode measures one Pauli term per circuit"
        if any(letter == "Y" for _, letter in obs.factors):
            return "no basis-change gates for Y factors"
        return ""

    def _counts_children(self, circuits, n, config: ExecutionConfig) -> list[ChildResult]:
        """Sample `config.shots` outcomes per circuit on the device with the
        reference's sampler: seed = config.seed + first_global_index + offset
        (backend.py:203, :226), PCG64 doubles, inverse CDF (backend.py:140-157).
        Circuits with a Pauli term are first rotated into its basis (H on each
        X factor; pauli.py:147-162)."""
        from types import SimpleNamespace

        mask64 = (1 << 64) - 1
        states = np.zeros((len(circuits), 4), dtype=np.uint64)
        for off in range(len(circuits)):
            st = np.random.PCG64(config.seed + config.first_global_index + off).state["state"]
            s, inc = int(st["state"]), int(st["inc"])
            states[off] = (s >> 64, s & mask64, inc >> 64, inc & mask64)
        runs = []
        for c in circuits:
            gates = tuple(c.gates)
            if c.observable is not None:
                gates = gates + tuple(h(q) for q, letter in c.observable.factors if letter == "X") + (measure_all(),)
            runs.append(SimpleNamespace(gates=gates, name=c.name, n_qubits=n, observable=None))
        lowered = lower_batch(runs)
        shots = int(config.shots)
        out = self._run(lowered, n, native.QV_OUT_COUNTS, circuits, shots=shots, rng_state=states)
        rows = out.reshape(len(circuits), 2 * shots + 1)
        fmt = f"0{n}b"
        children = []
        for c, row in zip(circuits, rows):
            m = int(row[0])
            idx = row[1:1 + 2 * m:2].astype(np.int64)
            cnt = row[2:2 + 2 * m:2].astype(np.int64)
            counts = {format(int(i), fmt): int(k) for i, k in zip(idx, cnt)}
            children.append(ChildResult(name=c.name, counts=counts, shots=shots))
        self.gate_counter += sum(len(r.gates) for r in runs)
        return children

    def _check_all(self, circuits, n):
        for c in circuits:
            reason = self._precheck(c, n, children=False)
            if reason:
                raise ExecutionError(c.name, reason)

    def _run(self, lowered, n, kind, circuits, **kw) -> np.ndarray:
        try:
            out = self._engine.execute(n, lowered, kind, **kw)
        except native.NativeError as err:
            name = circuits[err.circuit].name if 0 <= err.circuit < len(circuits) else circuits[0].name
            raise ExecutionError(name, str(err)) from err
        self.last_stats = dict(self._engine.last_stats)
        return out

    def _expectations(self, circuits, n) -> np.ndarray:
        offsets = [0]
        xs, ys, zs, coeffs, consts = [], [], [], [], []
        for c in circuits:
            obs = c.observable
            single = not hasattr(obs, "terms")   # a PauliTerm (ours or the reference's)
            for t in ((obs,) if single else obs.terms):
                xm, ym, zm = term_masks(t, n)
                xs.append(xm)
                ys.append(ym)
                zs.append(zm)
                coeffs.append(t.coefficient)
            offsets.append(len(xs))
            consts.append(None if single else obs.constant)
        lowered = lower_batch(circuits)
        vals = self._run(lowered, n, native.QV_OUT_PAULI, circuits,
                         terms=(np.asarray(offsets, np.int64), np.asarray(xs, np.uint64),
                                np.asarray(ys, np.uint64), np.asarray(zs, np.uint64)))
        out = np.empty(len(circuits), np.float64)
        for i, const in enumerate(consts):
            a, b = offsets[i], offsets[i + 1]
            if const is None:   # PauliTerm: coefficient * <P>
                out[i] = coeffs[a] * vals[a]
            else:               # Observable: constant + sum_i c_i <P_i>, in term order
                total = const
                for j in range(a, b):
                    total += coeffs[j] * vals[j]
                out[i] = total
        self.gate_counter += _gate_count(circuits)
        return out

    def _support_for(self, n: int) -> np.ndarray:
        if n not in self._support_cache:
            self._support_cache[n] = support_indices(self._support_spec, n)
        return self._support_cache[n]

    def _distributions(self, circuits, n) -> list[dict[str, float]]:
        lowered = lower_batch(circuits)
        fmt = f"0{n}b"
        dists = []
        if self._support_spec is None:
            flat = self._run(lowered, n, native.QV_OUT_FULL, circuits).reshape(len(circuits), 1 << n)
            for row in flat:
                nz = np.nonzero(row > 0.0)[0]
                dists.append({format(int(i), fmt): float(row[i]) for i in nz})
        else:
            sup = self._support_for(n)
            flat = self._run(lowered, n, native.QV_OUT_SUPPORT, circuits, support=sup)
            flat = flat.reshape(len(circuits), sup.shape[0] + 1)
            gap = _first_gap(sup, n)
            keys = [format(int(i), fmt) for i in sup]
            for row in flat:
                probs = row[:-1]
                d = {keys[j]: float(probs[j]) for j in np.nonzero(probs > 0.0)[0]}
                rest = 1.0 - math.fsum(probs)
                if gap is not None and rest > 0.0:
                    d[format(gap, fmt)] = rest
                dists.append(d)
        self.gate_counter += _gate_count(circuits)
        return dists

    def _children(self, circuits, n) -> list[ChildResult]:
        exp_idx = [i for i, c in enumerate(circuits) if c.observable is not None]
        dist_idx = [i for i, c in enumerate(circuits) if c.observable is None]
        children: list[ChildResult | None] = [None] * len(circuits)
        if exp_idx:
            vals = self._expectations([circuits[i] for i in exp_idx], n)
            for i, v in zip(exp_idx, vals):
                children[i] = ChildResult(name=circuits[i].name, expectation=float(v))
        if dist_idx:
            dists = self._distributions([circuits[i] for i in dist_idx], n)
            for i, d in zip(dist_idx, dists):
                children[i] = ChildResult(name=circuits[i].name, distribution=d)
        return children
