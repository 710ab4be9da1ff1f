"""TEST INFRASTRUCTURE ONLY -- never imported by the product package.

CPU restatement (numpy, complex128) of the reference's hot path, used as the
parity checker for the B200 kernels and as the CPU "port" baseline in
bench.py.  Every function cites the reference lines it restates
(/root/reference/pkg/src/qvirt/...).  Pinned against golden vectors produced
by the reference itself (tests/golden/make_golden.py, fixtures in
tests/golden/*.json; checked by tests/test_oracle.py).

Index convention (kernels.py:3-7): qubit 0 is the most significant bit;
qubit q flips index bit n-1-q, i.e. stride 1 << (n-1-q).
"""

from __future__ import annotations

import math
from typing import Iterable, Mapping, Sequence

import numpy as np

INV_SQRT2 = 1.0 / np.sqrt(2.0)   # kernels.py:21


def _pair_view(amps: np.ndarray, n: int, q: int) -> np.ndarray:
    """View with axis 1 = the bit of qubit q (stride 1 << (n-1-q))."""
    stride = 1 << (n - 1 - q)
    return amps.reshape(-1, 2, stride)


def zero_state(n: int) -> np.ndarray:
    """|0..0> (backend.py:57-63; the reference caps n at 30)."""
    a = np.zeros(1 << n, dtype=np.complex128)
    a[0] = 1.0
    return a


def apply_h(amps: np.ndarray, n: int, q: int) -> None:
    """kernels.py:18-27: (a0 + a1) * inv, (a0 - a1) * inv."""
    v = _pair_view(amps, n, q)
    a0 = v[:, 0, :].copy()
    a1 = v[:, 1, :].copy()
    v[:, 0, :] = (a0 + a1) * INV_SQRT2
    v[:, 1, :] = (a0 - a1) * INV_SQRT2


def apply_x(amps: np.ndarray, n: int, q: int) -> None:
    """kernels.py:30-37: swap the pair."""
    v = _pair_view(amps, n, q)
    v[:, [0, 1], :] = v[:, [1, 0], :]


def apply_ry(amps: np.ndarray, n: int, q: int, theta: float) -> None:
    """kernels.py:40-50: c = cos(theta/2), s = sin(theta/2); c a0 - s a1, s a0 + c a1."""
    c = np.cos(theta / 2.0)
    s = np.sin(theta / 2.0)
    v = _pair_view(amps, n, q)
    a0 = v[:, 0, :].copy()
    a1 = v[:, 1, :].copy()
    v[:, 0, :] = c * a0 - s * a1
    v[:, 1, :] = s * a0 + c * a1


def apply_rz(amps: np.ndarray, n: int, q: int, theta: float) -> None:
    """kernels.py:53-59: bit 0 -> exp(-i theta/2), bit 1 -> exp(+i theta/2)."""
    v = _pair_view(amps, n, q)
    v[:, 0, :] *= np.exp(-0.5j * theta)
    v[:, 1, :] *= np.exp(0.5j * theta)


def apply_rx(amps: np.ndarray, n: int, q: int, theta: float) -> None:
    """Extension gate (not in the reference set): [[c, -is], [-is, c]]."""
    c = np.cos(theta / 2.0)
    s = np.sin(theta / 2.0)
    v = _pair_view(amps, n, q)
    a0 = v[:, 0, :].copy()
    a1 = v[:, 1, :].copy()
    v[:, 0, :] = c * a0 - 1j * s * a1
    v[:, 1, :] = -1j * s * a0 + c * a1


def apply_cnot(amps: np.ndarray, n: int, control: int, target: int) -> None:
    """kernels.py:62-70: swap a[i], a[i | t] where the control bit is set and
    the target bit is clear."""
    idx = np.arange(1 << n, dtype=np.int64)
    cm = 1 << (n - 1 - control)
    tm = 1 << (n - 1 - target)
    sel = idx[((idx & cm) != 0) & ((idx & tm) == 0)]
    lo = amps[sel].copy()
    amps[sel] = amps[sel | tm]
    amps[sel | tm] = lo


def apply_cz(amps: np.ndarray, n: int, a: int, b: int) -> None:
    """Extension gate: phase -1 where both bits are set."""
    idx = np.arange(1 << n, dtype=np.int64)
    both = ((idx >> (n - 1 - a)) & 1) & ((idx >> (n - 1 - b)) & 1)
    amps[both == 1] *= -1.0


def apply_gate(amps: np.ndarray, n: int, kind: str, targets: Sequence[int], angle: float | None) -> None:
    """Dispatch of backend.py:66-85 (measure_all is a no-op in exact mode)."""
    if kind == "h":
        apply_h(amps, n, targets[0])
    elif kind == "x":
        apply_x(amps, n, targets[0])
    elif kind == "ry":
        apply_ry(amps, n, targets[0], angle)
    elif kind == "rz":
        apply_rz(amps, n, targets[0], angle)
    elif kind == "rx":
        apply_rx(amps, n, targets[0], angle)
    elif kind == "cnot":
        apply_cnot(amps, n, targets[0], targets[1])
    elif kind == "cz":
        apply_cz(amps, n, targets[0], targets[1])
    elif kind != "measure_all":
        raise ValueError(f"unsupported gate {kind}")


def run_gates(n: int, gates: Iterable[tuple[str, Sequence[int], float | None]]) -> np.ndarray:
    """allocate + run_gates (backend.py:57-91) from (kind, targets, angle) tuples."""
    amps = zero_state(n)
    for kind, targets, angle in gates:
        apply_gate(amps, n, kind, targets, angle)
    return amps


def gate_tuples(circuit) -> list[tuple[str, tuple[int, ...], float | None]]:
    """(kind, targets, angle) of any reference-shaped circuit object."""
    return [(g.kind.value, tuple(g.targets), g.angle) for g in circuit.gates]


def pauli_expectation(amps: np.ndarray, n: int, xmask: int, ymask: int, zmask: int, ny: int) -> float:
    """kernels.py:73-87: Re(i^ny * sum_i conj(a[i ^ flip]) a[i] (-1)^popcount(i & (y|z)))."""
    idx = np.arange(1 << n, dtype=np.uint64)
    flip = np.uint64(xmask | ymask)
    phase = np.uint64(ymask | zmask)
    sign = 1.0 - 2.0 * (np.bitwise_count(idx & phase) & 1)
    acc = np.sum(np.conj(amps[(idx ^ flip).astype(np.int64)]) * amps * sign)
    return float(((1j ** ny) * acc).real)


def term_masks(factors: Sequence[tuple[int, str]], n: int) -> tuple[int, int, int, int]:
    """backend.py:104-119: bit 1 << (n-1-q) per factor; returns (x, y, z, ny)."""
    m = {"X": 0, "Y": 0, "Z": 0}
    for q, letter in factors:
        m[letter] |= 1 << (n - 1 - q)
    return m["X"], m["Y"], m["Z"], bin(m["Y"]).count("1")


def expectation(amps: np.ndarray, n: int, terms: Sequence[tuple[Sequence[tuple[int, str]], float]],
                constant: float | None) -> float:
    """backend.py:94-101: coeff * <P> for one term (constant None), else
    constant + sum_i c_i <P_i> in term order."""
    if constant is None:
        (factors, coeff), = terms
        return coeff * pauli_expectation(amps, n, *term_masks(factors, n))
    total = constant
    for factors, coeff in terms:
        total += coeff * pauli_expectation(amps, n, *term_masks(factors, n))
    return total


def born_probabilities(amps: np.ndarray) -> np.ndarray:
    """kernels.py:90-94: re^2 + im^2."""
    return amps.real * amps.real + amps.imag * amps.imag


def normalized_probabilities(amps: np.ndarray) -> np.ndarray:
    """backend.py:122-129: probs / probs.sum()."""
    p = born_probabilities(amps)
    total = p.sum()
    if not total > 0.0:
        raise ValueError("state has zero norm")
    return p / total


def born_distribution(amps: np.ndarray, n: int) -> dict[str, float]:
    """backend.py:132-137: {bitstring: p} for p > 0."""
    p = normalized_probabilities(amps)
    return {format(i, f"0{n}b"): float(v) for i, v in enumerate(p) if v > 0.0}


def js_divergence(p: Mapping[str, float], q: Mapping[str, float]) -> float:
    """ddcl.py:37-61 (natural log, sorted key union, zero terms skipped)."""
    acc = 0.0
    for b in sorted(set(p) | set(q)):
        pb = p.get(b, 0.0)
        qb = q.get(b, 0.0)
        m = 0.5 * (pb + qb)
        if pb > 0.0:
            acc += 0.5 * pb * math.log(pb / m)
        if qb > 0.0:
            acc += 0.5 * qb * math.log(qb / m)
    return acc


def js_support_remainder(target: Mapping[str, float], probs: np.ndarray) -> float:
    """The identity the device epilogue uses:
    JS(P,Q) = sum_{b in supp P}[.5 p ln(p/m) + .5 q ln(q/m)] + (ln 2 / 2)(1 - sum_{b in supp P} q)."""
    acc = 0.0
    qs = 0.0
    for b in sorted(target):
        pb = float(target[b])
        qb = float(probs[int(b, 2)])
        m = 0.5 * (pb + qb)
        if pb > 0.0:
            acc += 0.5 * pb * math.log(pb / m)
        if qb > 0.0:
            acc += 0.5 * qb * math.log(qb / m)
        qs += qb
    return acc + 0.5 * math.log(2.0) * (1.0 - qs)


# ---- workload drivers (restated) -------------------------------------------

def ddcl_template_gates(n: int, layers: int) -> list[tuple[str, tuple[int, ...], int | None]]:
    """ddcl.py:109-132 with parameter indices in place of angles."""
    gates: list[tuple[str, tuple[int, ...], int | None]] = []
    for i in range(n // 2):
        gates.append(("h", (2 * i,), None))
        gates.append(("cnot", (2 * i, 2 * i + 1), None))
    k = 0
    for _ in range(layers):
        for q in range(n):
            gates += [("rz", (q,), k), ("ry", (q,), k + 1), ("rz", (q,), k + 2)]
            k += 3
        for q in range(n - 1):
            gates.append(("cnot", (q, q + 1), None))
        for q in range(n):
            gates += [("rz", (q,), k), ("ry", (q,), k + 1), ("rz", (q,), k + 2)]
            k += 3
    return gates


def bind_template(template, theta: Sequence[float]):
    return [(kind, t, None if p is None else float(theta[p])) for kind, t, p in template]


def shifted_thetas(theta: Sequence[float]) -> list[list[float]]:
    """gradients.py:33-46: k-major, '+' then '-', theta[k] += sign * pi/2."""
    out = []
    base = [float(v) for v in theta]
    for k in range(len(base)):
        for sign in (1.0, -1.0):
            row = list(base)
            row[k] += sign * (math.pi / 2)
            out.append(row)
    return out


def random_angles(count: int, seed: int) -> list[float]:
    """mcvqe.py:181-184."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return [float(t) for t in rng.uniform(-math.pi, math.pi, size=count)]


def random_target_distribution(n: int, seed: int) -> dict[str, float]:
    """ddcl.py:147-157."""
    size = 1 << min(n, 10)
    w = np.random.Generator(np.random.PCG64(seed)).uniform(0.0, 1.0, size=size)
    w /= w.sum()
    return {format(i, f"0{n}b"): float(v) for i, v in enumerate(w)}


def ddcl_losses(n: int, layers: int, theta: Sequence[float], target: Mapping[str, float]) -> list[float]:
    """Per-circuit JS losses of the shifted batch (ddcl.py:197-221)."""
    tpl = ddcl_template_gates(n, layers)
    out = []
    for row in shifted_thetas(theta):
        amps = run_gates(n, bind_template(tpl, row))
        out.append(js_divergence(target, born_distribution(amps, n)))
    return out


def ddcl_gradient(n: int, layers: int, theta: Sequence[float], target: Mapping[str, float]) -> list[float]:
    """ddcl.py:222-225: 0.5 (L[2k] - L[2k+1])."""
    losses = ddcl_losses(n, layers, theta, target)
    return [0.5 * (losses[2 * k] - losses[2 * k + 1]) for k in range(len(theta))]


def w_state_gates(a: Sequence[float]) -> list[tuple[str, tuple[int, ...], float | None]]:
    """mcvqe.py:72-107."""
    n = len(a)
    gates = [("x", (0,), None)]
    res = [0.0] * (n + 1)
    for k in range(n - 1, -1, -1):
        res[k] = math.hypot(a[k], res[k + 1])
    for k in range(1, n):
        half = math.atan2(res[k], a[k - 1]) if k < n - 1 else math.atan2(a[n - 1], a[n - 2])
        gates += [("ry", (k,), half), ("cnot", (k - 1, k), None), ("ry", (k,), -half),
                  ("cnot", (k - 1, k), None), ("cnot", (k, k - 1), None)]
    return gates


def mcvqe_template_gates(a: Sequence[float]) -> list[tuple[str, tuple[int, ...], object]]:
    """mcvqe.py:124-149 (merged angles); entries are literal floats for the
    W-prep and ('p', index) for parameters."""
    n = len(a)
    gates: list = [(k, t, ang) for k, t, ang in w_state_gates(a)]
    P = lambda i: ("p", i)
    gates += [("ry", (0,), P(0)), ("ry", (1,), P(1)), ("cnot", (0, 1), None), ("ry", (0,), P(2)),
              ("ry", (1,), P(3)), ("cnot", (0, 1), None), ("ry", (0,), P(4)), ("ry", (1,), P(5))]
    for j in range(1, n - 1):
        b = 6 + 5 * (j - 1)
        gates += [("ry", (j + 1,), P(b)), ("cnot", (j, j + 1), None), ("ry", (j,), P(b + 1)),
                  ("ry", (j + 1,), P(b + 2)), ("cnot", (j, j + 1), None), ("ry", (j,), P(b + 3)),
                  ("ry", (j + 1,), P(b + 4))]
    return gates


def bind_mcvqe(template, theta):
    return [(k, t, float(theta[a[1]]) if isinstance(a, tuple) else a) for k, t, a in template]


def aiem_terms(coeff_seed: int, n: int) -> tuple[list[tuple[list[tuple[int, str]], float]], float]:
    """pauli.py:221-244: coefficient draws and term order."""
    rng = np.random.Generator(np.random.PCG64(coeff_seed))
    one = rng.uniform(-1.0, 1.0, size=(2, n))
    two = rng.uniform(-1.0, 1.0, size=(4, n - 1))
    offset = float(rng.uniform(-1.0, 1.0))
    terms = []
    for a in range(n):
        terms.append(([(a, "X")], float(one[0][a])))
        terms.append(([(a, "Z")], float(one[1][a])))
    for a in range(n - 1):
        b = a + 1
        terms += [([(a, "X"), (b, "X")], float(two[0][a])), ([(a, "X"), (b, "Z")], float(two[1][a])),
                  ([(a, "Z"), (b, "X")], float(two[2][a])), ([(a, "Z"), (b, "Z")], float(two[3][a]))]
    return terms, offset


def random_cis_amplitudes(n: int, seed: int) -> list[float]:
    """mcvqe.py:173-178."""
    v = np.random.Generator(np.random.PCG64(seed)).normal(size=n)
    v /= np.linalg.norm(v)
    return [float(x) for x in v]


def mcvqe_values(n: int, coeff_seed: int, cis_seed: int, theta_seed: int) -> tuple[np.ndarray, list, float]:
    """Per-circuit <P_t> of the gradient batch (mcvqe.py:194-210 order:
    parameter, then +/-, then term) -- one simulation per shifted state."""
    terms, offset = aiem_terms(coeff_seed, n)
    a = random_cis_amplitudes(n, cis_seed)
    theta = random_angles(5 * n - 4, theta_seed)
    tpl = mcvqe_template_gates(a)
    vals = []
    for row in shifted_thetas(theta):
        amps = run_gates(n, bind_mcvqe(tpl, row))
        for factors, _ in terms:
            vals.append(pauli_expectation(amps, n, *term_masks(factors, n)))
    return np.asarray(vals), terms, offset


def mcvqe_gradient(n: int, coeff_seed: int, cis_seed: int, theta_seed: int) -> list[float]:
    """mcvqe.py:244-247: E = const + V @ c; grad = 0.5 (E+ - E-)."""
    vals, terms, offset = mcvqe_values(n, coeff_seed, cis_seed, theta_seed)
    c = np.array([t[1] for t in terms])
    e = offset + vals.reshape(-1, 2, len(terms)) @ c
    return [float(g) for g in 0.5 * (e[:, 0] - e[:, 1])]


# ---- dense-matrix oracle (restates pkg/tests/oracles.py:28-93) --------------

_I2 = np.eye(2, dtype=complex)
_P = {"X": np.array([[0, 1], [1, 0]], complex), "Y": np.array([[0, -1j], [1j, 0]]),
      "Z": np.array([[1, 0], [0, -1]], complex)}


def _kron(fs):
    out = fs[0]
    for f in fs[1:]:
        out = np.kron(out, f)
    return out


def dense_gate(n: int, kind: str, targets, angle) -> np.ndarray:
    if kind == "measure_all":
        return np.eye(1 << n, dtype=complex)
    if kind in ("cnot", "cz"):
        c, t = targets
        keep = [_I2] * n
        keep[c] = np.diag([1.0, 0.0]).astype(complex)
        flip = [_I2] * n
        flip[c] = np.diag([0.0, 1.0]).astype(complex)
        flip[t] = _P["X"] if kind == "cnot" else _P["Z"]
        return _kron(keep) + _kron(flip)
    if kind == "h":
        m = np.array([[1, 1], [1, -1]], complex) / np.sqrt(2)
    elif kind == "x":
        m = _P["X"]
    elif kind == "ry":
        c, s = np.cos(angle / 2), np.sin(angle / 2)
        m = np.array([[c, -s], [s, c]], complex)
    elif kind == "rz":
        m = np.diag([np.exp(-0.5j * angle), np.exp(0.5j * angle)])
    elif kind == "rx":
        c, s = np.cos(angle / 2), np.sin(angle / 2)
        m = np.array([[c, -1j * s], [-1j * s, c]])
    else:
        raise ValueError(kind)
    fs = [_I2] * n
    fs[targets[0]] = m
    return _kron(fs)


def dense_state(n: int, gates) -> np.ndarray:
    u = np.eye(1 << n, dtype=complex)
    for kind, t, ang in gates:
        u = dense_gate(n, kind, t, ang) @ u
    e0 = np.zeros(1 << n, complex)
    e0[0] = 1.0
    return u @ e0


def dense_expectation(state: np.ndarray, n: int, factors, coeff: float = 1.0) -> float:
    fs = [_I2] * n
    for q, letter in factors:
        fs[q] = _P[letter]
    m = coeff * _kron(fs)
    return float(np.real(np.conj(state) @ (m @ state)))


def random_circuit_gates(rng: np.random.Generator, n: int, n_gates: int, extended: bool = False):
    """pkg/tests/oracles.py:96-114 draw order (uniform over H/X/CNOT/Ry/Rz);
    `extended` adds RX and CZ draws for the extension gates."""
    gates = []
    kinds = 7 if extended else 5
    for _ in range(n_gates):
        kind = rng.integers(0, kinds)
        q = int(rng.integers(0, n))
        if kind == 0:
            gates.append(("h", (q,), None))
        elif kind == 1:
            gates.append(("x", (q,), None))
        elif kind == 2 and n > 1:
            t = int(rng.integers(0, n - 1))
            t += t >= q
            gates.append(("cnot", (q, t), None))
        elif kind == 3:
            gates.append(("ry", (q,), float(rng.uniform(-np.pi, np.pi))))
        elif kind == 5:
            gates.append(("rx", (q,), float(rng.uniform(-np.pi, np.pi))))
        elif kind == 6 and n > 1:
            t = int(rng.integers(0, n - 1))
            t += t >= q
            gates.append(("cz", (q, t), None))
        else:
            gates.append(("rz", (q,), float(rng.uniform(-np.pi, np.pi))))
    return gates
