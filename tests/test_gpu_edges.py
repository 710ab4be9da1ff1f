"""Edge cases against the dense oracle: 1-3 qubit registers, the tile
boundary (11-13 qubits), empty circuits, support indices at both ends of the
register, every result kind, and a batch mixing topologies, duplicates and an
empty circuit (reference backend.py:57-137 semantics)."""

import numpy as np
import pytest

import paper_2406_03466_b200 as qv
from oracle import statevector as sv

TOL = 1e-12


def _circuit(n, ng, seed):
    r = np.random.Generator(np.random.PCG64(seed))
    gates = []
    for _ in range(ng):
        k, q = int(r.integers(0, 5)), int(r.integers(0, n))
        if k == 0:
            gates.append(qv.h(q))
        elif k == 1:
            gates.append(qv.ry(q, float(r.uniform(-3, 3))))
        elif k == 2:
            gates.append(qv.rz(q, float(r.uniform(-3, 3))))
        elif n > 1:
            t = int(r.integers(0, n - 1))
            gates.append(qv.cnot(q, t if t < q else t + 1))
    return qv.Circuit(n, tuple(gates), name=f"edge{seed}")


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3, 11, 12, 13, 16])
@pytest.mark.parametrize("ng", [0, 1, 40])
def test_edge_registers_every_output(gpu, n, ng):
    b = qv.B200Backend(device=0)
    c = _circuit(n, ng, 100 * n + ng)
    amps = sv.run_gates(n, sv.gate_tuples(c))
    probs = np.abs(amps) ** 2
    dim = 1 << n
    sup = sorted({0, dim - 1, dim // 2, (dim - 1) // 3})
    assert np.max(np.abs(b.support_probabilities([c], n, sup)[0] - probs[sup])) < TOL
    keys = [format(i, f"0{n}b") for i in sorted({0, dim - 1})]
    target = {k: 1.0 / len(keys) for k in keys}
    ref = sv.js_divergence(target, {format(i, f"0{n}b"): float(p) for i, p in enumerate(probs) if p > 0})
    assert abs(b.js_losses([c], n, target)[0] - ref) < TOL
    factors = {0: "Z"} if n == 1 else {0: "X", n - 1: "Y"}
    obs = qv.Observable((qv.pauli(factors, 0.5),), 0.25)
    ref = sv.expectation(amps, n, [(sorted(factors.items()), 0.5)], 0.25)
    assert abs(b.expectation_values([c.with_observable(obs)], n)[0] - ref) < TOL


@pytest.mark.gpu
def test_mixed_topologies_duplicates_and_empty_circuit(gpu):
    b = qv.B200Backend(device=0)
    n = 14
    cs = [_circuit(n, 30, 7), _circuit(n, 0, 8), _circuit(n, 30, 7), _circuit(n, 55, 9)]
    sup = [0, 5, (1 << n) - 1]
    got = b.support_probabilities(cs, n, sup)
    for i, c in enumerate(cs):
        p = np.abs(sv.run_gates(n, sv.gate_tuples(c))) ** 2
        assert np.max(np.abs(got[i] - p[sup])) < TOL, i
    assert np.array_equal(got[0], got[2])
