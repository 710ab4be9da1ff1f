"""Host-side logic of the reference-interface mirror (no GPU): IR validation,
lazy binding, the shift table, lowering, observables, partition, merge.
Modelled on the reference's own unit tests (pkg/tests/test_circuits.py,
test_pauli.py, test_pool.py, test_buffers.py, test_ddcl.py, test_mcvqe.py)."""

import math

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2406_03466_b200 as qv
from oracle import statevector as sv


# ---- IR -------------------------------------------------------------------

def test_gate_validation():
    with pytest.raises(ValueError):
        qv.Gate(qv.GateKind.H, (0, 1))
    with pytest.raises(ValueError):
        qv.cnot(1, 1)
    with pytest.raises(ValueError):
        qv.h(-1)
    with pytest.raises(ValueError):
        qv.Gate(qv.GateKind.RY, (0,))
    with pytest.raises(ValueError):
        qv.ry(0, float("nan"))
    with pytest.raises(ValueError):
        qv.Gate(qv.GateKind.H, (0,), 0.5)
    assert qv.ry(0, "t").is_parameterized and not qv.ry(0, 1).is_parameterized
    assert qv.measure_all().touches(5)


def test_circuit_validation_and_bind():
    with pytest.raises(ValueError):
        qv.Circuit(0)
    with pytest.raises(ValueError):
        qv.Circuit(2, (qv.x(2),))
    with pytest.raises(ValueError):
        qv.Circuit(1, (qv.ry(0, "a"),))
    with pytest.raises(ValueError):
        qv.Circuit(1, name="")
    tpl = qv.Circuit(2, (qv.ry(0, "a"), qv.cnot(0, 1), qv.rz(1, "b")), params=("a", "b"))
    assert tpl.is_parameterized
    with pytest.raises(ValueError):
        qv.bind(tpl, [1.0])
    bound = qv.bind(tpl, [0.25, -1.5])
    assert not bound.is_parameterized and bound.params == ()
    assert [g.angle for g in bound.gates] == [0.25, None, -1.5]
    assert [g.kind for g in bound.gates] == [qv.GateKind.RY, qv.GateKind.CNOT, qv.GateKind.RZ]
    renamed = bound.with_name("z").with_observable(qv.pauli({0: "Z"}))
    assert renamed.name == "z" and renamed.gates == bound.gates


def test_shift_table_matches_reference_arithmetic():
    """gradients.py:33-46: values.copy(); shifted[k] += sign * SHIFT."""
    theta = qv.random_angles(30, 4)
    table = qv.shift_table(theta)
    for k in range(30):
        for s, (sign, _) in enumerate(qv.SHIFT_TAGS):
            row = [float(v) for v in theta]
            row[k] += sign * qv.SHIFT
            assert table[2 * k + s].tolist() == row   # bitwise


def test_shifted_circuits_order_and_lazy_gates():
    n, layers = 4, 1
    tpl = qv.ddcl_circuit_template(n, layers)
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), 9)
    items = list(qv.shifted_circuits(tpl, theta))
    assert [(k, t) for k, t, _ in items[:4]] == [(0, "+"), (0, "-"), (1, "+"), (1, "-")]
    k, tag, c = items[7]
    want = sv.bind_template(sv.ddcl_template_gates(n, layers), sv.shifted_thetas(theta)[7])
    assert [(g.kind.value, g.targets, g.angle) for g in c.gates] == [(a, tuple(b), d) for a, b, d in want]


def test_lowering_uniform_batch():
    spec = qv.DdclSpec(4, 2, qv.random_angles(48, 1), qv.random_target_distribution(4, 2))
    batch = qv.ddcl_batch(spec)
    lw = qv.lower_batch(batch)
    assert lw.uniform and lw.angles.shape == (96, 58) and lw.n_gates == 58
    rows = sv.shifted_thetas(spec.theta)
    tpl = sv.ddcl_template_gates(4, 2)
    for i in (0, 5, 95):
        want = [a if a is not None else 0.0 for _, _, a in sv.bind_template(tpl, rows[i])]
        assert lw.angles[i].tolist() == want
    mixed = qv.lower_batch([batch[0], qv.Circuit(4, (qv.h(0), qv.cz(0, 3)), name="m")])
    assert not mixed.uniform and mixed.gate_offsets.tolist() == [0, 58, 60]
    assert mixed.kinds[-1] == 7


# ---- observables ----------------------------------------------------------

def test_aiem_counts_and_masks():
    for n in range(2, 40):
        ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(n, 0))
        assert len(ham.terms) == qv.measurable_term_count(n) == 6 * n - 4
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(2, 0))
    assert [t.factors_text() for t in ham.terms] == ["X0", "Z0", "X1", "Z1", "X0 X1", "X0 Z1", "Z0 X1", "Z0 Z1"]
    terms, offset = sv.aiem_terms(0, 2)
    assert [t.coefficient for t in ham.terms] == [c for _, c in terms] and ham.constant == offset
    assert qv.term_masks(qv.pauli({0: "X", 2: "Y", 3: "Z"}), 4) == (0b1000, 0b0010, 0b0001)
    with pytest.raises(ValueError):
        qv.term_masks(qv.pauli({4: "Z"}), 4)


def test_combine_and_observable_validation():
    obs = qv.combine([qv.pauli({0: "Z"}, 1.0), qv.pauli({}, 2.0), qv.pauli({0: "Z"}, 0.5)], constant=1.0)
    assert obs.constant == 3.0 and len(obs.terms) == 1 and obs.terms[0].coefficient == 1.5
    with pytest.raises(ValueError):
        qv.Observable((qv.pauli({0: "Z"}), qv.pauli({0: "Z"})))
    with pytest.raises(ValueError):
        qv.PauliTerm(((0, "Q"),))


def test_expectation_from_counts():
    assert qv.expectation_from_counts({"00": 3, "11": 1}, qv.pauli({0: "Z", 1: "Z"})) == 1.0
    assert qv.expectation_from_counts({"01": 1, "00": 1}, qv.pauli({1: "Z"})) == 0.0


# ---- pool / buffers -------------------------------------------------------

def test_partition_examples():
    assert [b.size for b in qv.partition(10, 4)] == [3, 3, 2, 2]
    sizes = [b.size for b in qv.partition(13984, 256)]
    assert sizes.count(55) == 160 and sizes.count(54) == 96
    assert [b.size for b in qv.partition(3, 8)] == [1, 1, 1, 0, 0, 0, 0, 0]


@given(st.integers(0, 5000), st.integers(1, 300))
@settings(max_examples=80, deadline=None)
def test_partition_properties(n_circuits, n_vqpus):
    blocks = qv.partition(n_circuits, n_vqpus)
    sizes = [b.size for b in blocks]
    assert len(blocks) == n_vqpus and blocks[0].start == 0 and blocks[-1].end == n_circuits
    assert all(a.end == b.start for a, b in zip(blocks, blocks[1:]))
    assert max(sizes) - min(sizes) <= 1 and sorted(sizes, reverse=True) == sizes


def test_merge_orders_and_rejects_gaps():
    def local(names):
        buf = qv.ResultBuffer(n_qubits=1)
        for nm in names:
            buf.append_child(qv.ChildResult(name=nm))
        return buf
    assert [c.name for c in qv.consolidate([((2, 4), local(["c", "d"])), ((0, 2), local(["a", "b"]))])] == list("abcd")
    with pytest.raises(ValueError):
        qv.merge(qv.ResultBuffer(1), [((1, 2), local(["x"]))])


def test_child_validation():
    with pytest.raises(ValueError):
        qv.ChildResult("c", distribution={"0": 0.5}).validate(1)
    with pytest.raises(ValueError):
        qv.ChildResult("c", distribution={"01": 1.0}).validate(1)
    with pytest.raises(ValueError):
        qv.ChildResult("c", counts={"0": 2}, shots=3).validate(1)
    qv.ChildResult("c", distribution={"0": 0.25, "1": 0.75}).validate(1)


def test_pool_config_validation():
    for bad in ({"n_virtual_qpus": 0}, {"mode": "exact"}, {"shots": 0}):
        with pytest.raises(ValueError):
            qv.VqpuPoolConfig(**bad)
    with pytest.raises(ValueError):
        qv.ExecutionConfig(first_global_index=-1)


def test_empty_and_duplicate_batches_rejected():
    buf = qv.ResultBuffer(n_qubits=1)
    with pytest.raises(ValueError):
        qv.execute_parallel(buf, [], qv.VqpuPoolConfig())
    dup = [qv.Circuit(1, (qv.x(0),), name="s"), qv.Circuit(1, (qv.h(0),), name="s")]
    with pytest.raises(ValueError):
        qv.execute_parallel(buf, dup, qv.VqpuPoolConfig())
    with pytest.raises(ValueError, match="wide"):
        qv.execute_parallel(qv.ResultBuffer(3), [qv.Circuit(4, (qv.x(3),), name="wide")], qv.VqpuPoolConfig())


# ---- workloads ------------------------------------------------------------

def test_ddcl_counts_and_template():
    for n, p, c in ((20, 1200, 2400), (22, 1320, 2640), (24, 1440, 2880), (26, 1560, 3120)):
        assert qv.ddcl_parameter_count(n, 10) == p and qv.ddcl_execution_count(n, 10) == c
    with pytest.raises(ValueError):
        qv.ddcl_parameter_count(3, 1)
    tpl = qv.ddcl_circuit_template(4, 2)
    kinds = [g.kind for g in tpl.gates]
    assert kinds[:4] == [qv.GateKind.H, qv.GateKind.CNOT] * 2
    layer = kinds[4: 4 + 6 * 4 + 3]
    assert layer.count(qv.GateKind.CNOT) == 3 and layer.count(qv.GateKind.RZ) == 16
    want = sv.ddcl_template_gates(4, 2)
    assert [(g.kind.value, g.targets) for g in tpl.gates] == [(k, tuple(t)) for k, t, _ in want]


def test_ddcl_spec_validation_and_targets():
    with pytest.raises(ValueError):
        qv.DdclSpec(3, 1, (0.0,) * 18, {"000": 1.0})
    with pytest.raises(ValueError):
        qv.DdclSpec(2, 1, (0.0,) * 12, {"00": 0.7})
    t = qv.random_target_distribution(12, 3)
    assert len(t) == 1024 and set(t) == {format(i, "012b") for i in range(1024)}
    assert t == sv.random_target_distribution(12, 3)


def test_js_divergence_mirror():
    p = qv.random_target_distribution(5, 1)
    q = qv.random_target_distribution(5, 2)
    assert qv.js_divergence(p, q) == sv.js_divergence(p, q)
    with pytest.raises(ValueError):
        qv.js_divergence({"0": 0.9}, {"0": 1.0})


def test_mcvqe_counts_batch_and_wstate():
    for n, c in ((16, 13984), (18, 17888), (20, 22272), (22, 27136)):
        assert qv.mcvqe_execution_count(n) == c
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(3, 0))
    spec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(3, 1), qv.random_angles(11, 2))
    batch = qv.mcvqe_gradient_batch(ham, spec)
    assert len(batch) == qv.mcvqe_execution_count(3)
    assert batch[0].name == "k0+ X0" and batch[len(ham.terms)].name == "k0- X0"
    assert all(c.observable.coefficient == 1.0 for c in batch)
    a = qv.random_cis_amplitudes(5, 3)
    amps = sv.run_gates(5, [(g.kind.value, g.targets, g.angle) for g in qv.w_state_prep(a).gates])
    for k in range(5):
        assert amps[1 << (4 - k)].real == pytest.approx(a[k], abs=1e-12)
    assert [(g.kind.value, g.targets, g.angle) for g in qv.w_state_prep(a).gates] == \
        [(k, tuple(t), ang) for k, t, ang in sv.w_state_gates(a)]


class _OracleRowsBackend:
    """CPU stand-in exposing `pauli_values` (the B200 fast-path entry point)
    computed with the numpy oracle: exercises mcvqe_gradient's row
    bookkeeping (state / term grouping per vQPU block) without a GPU."""

    def __init__(self):
        self.calls = 0

    def pauli_values(self, circuits, n, offsets, xm, ym, zm):
        self.calls += 1
        out = []
        for i, c in enumerate(circuits):
            amps = sv.run_gates(n, [(g.kind.value, g.targets, g.angle) for g in c.gates])
            for j in range(int(offsets[i]), int(offsets[i + 1])):
                ny = bin(int(ym[j])).count("1")
                out.append(sv.pauli_expectation(amps, n, int(xm[j]), int(ym[j]), int(zm[j]), ny))
        return np.asarray(out)


@pytest.mark.parametrize("n_vqpus", [1, 5, 17])
def test_mcvqe_row_fast_path_matches_reference(golden_small, n_vqpus):
    case = golden_small["mcvqe"][2]   # 3 monomers
    n = case["n"]
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(n, case["coeff_seed"]))
    spec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(n, case["cis_seed"]),
                              qv.random_angles(qv.mcvqe_parameter_count(n), case["theta_seed"]))
    backend = _OracleRowsBackend()
    rep = qv.mcvqe_gradient(ham, spec, qv.VqpuPoolConfig(n_virtual_qpus=n_vqpus), backend_factory=lambda: backend)
    assert rep.n_circuit_executions == case["n_circuits"]
    assert np.max(np.abs(np.asarray(rep.gradient) - case["gradient"])) < 1e-10


def test_foreign_circuits_lowered_like_a_per_gate_loop():
    """Reference-shaped circuits (duck-typed .gates with .kind.value /
    .targets / .angle, e.g. qvirt.Circuit) lower through the topology-reusing
    fast path to exactly the arrays a per-gate loop gives; a changed topology
    in the middle of a batch is detected; unbound parameters are rejected."""
    import enum
    from types import SimpleNamespace as NS

    from paper_2406_03466_b200.backend import lower_batch
    from paper_2406_03466_b200.ir import CODE_BY_VALUE

    class Kind(enum.Enum):
        H = "h"
        CNOT = "cnot"
        RY = "ry"
        RZ = "rz"

    def circ(angles, extra=False):
        gates = [NS(kind=Kind.H, targets=(0,), angle=None), NS(kind=Kind.CNOT, targets=(0, 1), angle=None)]
        gates += [NS(kind=Kind.RZ if i % 2 else Kind.RY, targets=(i % 3,), angle=a) for i, a in enumerate(angles)]
        if extra:
            gates.append(NS(kind=Kind.CNOT, targets=(2, 1), angle=None))
        return NS(gates=tuple(gates), n_qubits=3, name="f")

    batch = [circ([0.1 * k + j for j in range(5)]) for k in range(4)] + [circ([1.0, 2.0, 3.0, 4.0, 5.0], extra=True)]
    lb = lower_batch(batch)
    for ci, c in enumerate(batch):
        o0, o1 = lb.gate_offsets[ci], lb.gate_offsets[ci + 1]
        want_k = [CODE_BY_VALUE[g.kind.value] for g in c.gates]
        want_a = [g.angle if g.angle is not None else 0.0 for g in c.gates]
        want_q0 = [g.targets[0] for g in c.gates]
        want_q1 = [g.targets[1] if len(g.targets) > 1 else -1 for g in c.gates]
        assert lb.kinds[o0:o1].tolist() == want_k
        assert lb.angles[o0:o1].tolist() == want_a
        assert lb.q0[o0:o1].tolist() == want_q0
        assert lb.q1[o0:o1].tolist() == want_q1
    with pytest.raises(ValueError, match="unbound"):
        lower_batch([circ([0.1, "t1", 0.3, 0.4, 0.5])])


def test_support_keys_of_mixed_width_rejected():
    """'0' + '111' joins to n * len bits for n = 2 but is not a 2-qubit support."""
    from paper_2406_03466_b200.backend import support_indices
    with pytest.raises(ValueError):
        support_indices(["0", "111"], 2)
    assert support_indices(["01", "11", "00"], 2).tolist() == [0, 1, 3]
