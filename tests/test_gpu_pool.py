"""Pool semantics on the GPU: serial equivalence (bitwise across virtual-QPU
counts and batch composition), failure isolation, size-independent
properties at large registers, and the drop-in into the reference's own
drivers.  Modelled on reference pkg/tests/test_pool.py and test_acceptance.py."""

import math
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

import paper_2406_03466_b200 as qv
from oracle import statevector as sv

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def random_batch(count, n=3, seed=17):
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for i in range(count):
        gates = sv.random_circuit_gates(rng, n, 10)
        size = int(rng.integers(1, n + 1))
        qubits = rng.choice(n, size=size, replace=False)
        term = qv.pauli({int(q): "XZ"[rng.integers(0, 2)] for q in qubits}, float(rng.uniform(-2, 2)))
        c = qv.Circuit(n, tuple(qv.Gate(qv.GateKind(k), t, a) for k, t, a in gates), name=f"c{i}")
        out.append(c.with_observable(term))
    return out


@pytest.mark.parametrize("n_vqpus", [1, 2, 3, 8, 256])
def test_serial_equivalence_bitwise(gpu, n_vqpus):
    batch = random_batch(12)
    serial = qv.ResultBuffer(n_qubits=3)
    qv.B200Backend(device=0).execute(serial, batch, qv.ExecutionConfig())
    buf = qv.ResultBuffer(n_qubits=3)
    qv.execute_parallel(buf, batch, qv.VqpuPoolConfig(n_virtual_qpus=n_vqpus))
    assert buf.metadata["vqpu_count"] == n_vqpus
    assert buf.child_names() == serial.child_names()
    assert [c.expectation for c in buf.children] == [c.expectation for c in serial.children]


def test_gradient_bitwise_across_vqpus_and_prefix_sharing(gpu):
    """14 qubits (multi-pass, HBM-resident): the same circuit's loss is
    bit-identical alone, inside the full shifted batch (trunk sharing), and
    under any pool split."""
    n, layers = 14, 1
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), 21)
    target = qv.random_target_distribution(n, 22)
    spec = qv.DdclSpec(n, layers, theta, target)
    grads = [qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=v)).gradient for v in (1, 2, 7)]
    assert grads[0] == grads[1] == grads[2]
    batch = qv.ddcl_batch(spec)
    backend = qv.B200Backend(device=0)
    full = backend.js_losses(batch, n, target)
    stats = backend.last_stats
    assert stats["sweeps"] < stats["sweeps_unshared"]
    for i in (0, 77, len(batch) - 1):
        alone = backend.js_losses([batch[i]], n, target)
        assert alone[0] == full[i]


def test_mcvqe_bitwise_across_vqpus(gpu):
    n = 6
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(n, 3))
    spec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(n, 4), qv.random_angles(qv.mcvqe_parameter_count(n), 5))
    g = [qv.mcvqe_gradient(ham, spec, qv.VqpuPoolConfig(n_virtual_qpus=v)).gradient for v in (1, 8)]
    assert g[0] == g[1]


class PoisonBackend(qv.B200Backend):
    def execute(self, buffer, circuits, config):
        for c in circuits:
            if c.name == "poison":
                raise qv.ExecutionError(c.name, "injected failure")
        super().execute(buffer, circuits, config)


def test_failure_aborts_batch_and_leaves_buffer_untouched(gpu):
    batch = random_batch(8)
    batch[5] = batch[5].with_name("poison")
    buf = qv.ResultBuffer(n_qubits=3)
    with pytest.raises(qv.ExecutionError, match="poison"):
        qv.execute_parallel(buf, batch, qv.VqpuPoolConfig(n_virtual_qpus=3), backend_factory=PoisonBackend)
    assert buf.children == [] and "vqpu_count" not in buf.metadata


def test_execute_failure_names_circuit(gpu):
    buf = qv.ResultBuffer(n_qubits=2)
    with pytest.raises(qv.ExecutionError, match="too-wide"):
        qv.B200Backend(device=0).execute(buf, [qv.Circuit(3, (qv.x(2),), name="too-wide")], qv.ExecutionConfig())
    assert buf.children == []
    ok = qv.Circuit(2, (qv.h(0),), name="ok", observable=qv.pauli({0: "X"}))
    bad = qv.Circuit(2, (qv.h(0),), name="bad", observable=qv.pauli({2: "Z"}))
    with pytest.raises(qv.ExecutionError, match="bad"):
        qv.B200Backend(device=0).execute(buf, [ok, bad], qv.ExecutionConfig())
    assert buf.child_names() == ["ok"] and buf.children[0].expectation == pytest.approx(1.0)


class RecordingBackend(qv.B200Backend):
    instances = []

    def __init__(self):
        super().__init__()
        self.threads = set()
        RecordingBackend.instances.append(self)

    def execute(self, buffer, circuits, config):
        self.threads.add(threading.get_ident())
        super().execute(buffer, circuits, config)


def test_private_backends_per_worker(gpu):
    RecordingBackend.instances = []
    buf = qv.ResultBuffer(n_qubits=3)
    qv.execute_parallel(buf, random_batch(3), qv.VqpuPoolConfig(n_virtual_qpus=256), backend_factory=RecordingBackend)
    assert len(RecordingBackend.instances) == 3
    assert all(len(b.threads) == 1 for b in RecordingBackend.instances)


def test_known_answers(gpu):
    b = qv.B200Backend(device=0)
    buf = qv.ResultBuffer(n_qubits=2)
    batch = [qv.Circuit(2, (qv.h(0),), name="a", observable=qv.pauli({0: "Z"})),
             qv.Circuit(2, (qv.x(0),), name="b", observable=qv.pauli({0: "Z"})),
             qv.Circuit(2, (), name="c", observable=qv.pauli({0: "Z"})),
             qv.Circuit(2, (qv.h(0), qv.cnot(0, 1)), name="bell", observable=qv.pauli({0: "X", 1: "X"})),
             qv.Circuit(2, (qv.h(0), qv.cnot(0, 1)), name="dist")]
    b.execute(buf, batch, qv.ExecutionConfig())
    assert [c.expectation for c in buf.children[:4]] == pytest.approx([0.0, -1.0, 1.0, 1.0], abs=1e-12)
    assert set(buf.children[4].distribution) == {"00", "11"}
    spec = qv.DdclSpec(2, 1, (0.0,) * 12, {"00": 0.5, "11": 0.5})
    assert qv.ddcl_distribution(spec) == pytest.approx({"00": 0.5, "10": 0.5}, abs=1e-12)


def test_stationary_gradient_at_zero_angles(gpu):
    """reference test_ddcl.py:162-168: target = the circuit's own distribution."""
    n, layers = 4, 2
    theta = (0.0,) * qv.ddcl_parameter_count(n, layers)
    own = qv.ddcl_distribution(qv.DdclSpec(n, layers, theta, {"0" * n: 1.0}))
    rep = qv.ddcl_gradient(qv.DdclSpec(n, layers, theta, own), qv.VqpuPoolConfig())
    assert max(abs(g) for g in rep.gradient) < 1e-9


@pytest.mark.parametrize("n,layers", [(22, 2), (26, 1)])
def test_large_register_properties(gpu, n, layers):
    """Size-independent checks where the oracle is too slow: the state norm
    stays 1, shifted pairs differ, support probabilities are in [0, 1]."""
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), 31)
    target = qv.random_target_distribution(n, 32)
    spec = qv.DdclSpec(n, layers, theta, target)
    batch = qv.ddcl_batch(spec)
    pick = [0, 1, len(batch) // 2, len(batch) - 1]
    backend = qv.B200Backend(device=0, support=target)
    buf = qv.ResultBuffer(n_qubits=n)
    backend.execute(buf, [batch[i] for i in pick], qv.ExecutionConfig())
    losses = backend.js_losses([batch[i] for i in pick], n, target)
    for child, loss in zip(buf.children, losses):
        d = child.distribution
        assert abs(math.fsum(d.values()) - 1.0) < 1e-12
        assert 0.0 <= loss <= math.log(2)
        assert qv.js_divergence(target, d) == pytest.approx(loss, abs=1e-12)
    assert losses[0] != losses[1]


def test_drop_in_reference_drivers(gpu, golden_small):
    """The reference's own ddcl_gradient / mcvqe_gradient / execute_parallel
    (unmodified, from baseline/_ref) driving B200Backend."""
    ref_path = ROOT / "baseline" / "_ref"
    if not (ref_path / "qvirt").exists():
        pytest.skip("baseline/_ref not installed")
    import os
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba-qvirt")
    sys.path.insert(0, str(ref_path))
    try:
        import qvirt
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"reference not importable: {exc}")
    finally:
        sys.path.remove(str(ref_path))
    cfg = golden_small["qcl_config1"]
    pt = cfg["points"][5]
    theta = qvirt.random_angles(qvirt.ddcl_parameter_count(4, 2), pt["theta_seed"])
    target = qvirt.random_target_distribution(4, pt["target_seed"])
    spec = qvirt.DdclSpec(4, 2, theta, target)
    rep = qvirt.ddcl_gradient(spec, qvirt.VqpuPoolConfig(n_virtual_qpus=4, mode="expectation"),
                              backend_factory=lambda: qv.B200Backend(support=target))
    assert np.max(np.abs(np.array(rep.gradient) - pt["gradient"])) < 1e-10
    mc = golden_small["mcvqe"][1]
    ham = qvirt.aiem_hamiltonian(qvirt.random_aiem_coefficients(4, mc["coeff_seed"]))
    mspec = qvirt.McvqeAnsatzSpec(qvirt.random_cis_amplitudes(4, mc["cis_seed"]),
                                  qvirt.random_angles(qvirt.mcvqe_parameter_count(4), mc["theta_seed"]))
    mrep = qvirt.mcvqe_gradient(ham, mspec, qvirt.VqpuPoolConfig(n_virtual_qpus=2), backend_factory=qv.B200Backend)
    assert np.max(np.abs(np.array(mrep.gradient) - mc["gradient"])) < 1e-10


def test_28_qubit_shift_pairs_against_direct_circuits(gpu):
    """The benchmark's register size: shift-pair losses (Psi0 -+ i Xi_k on the
    support's light cone) against direct simulation of the shifted circuits
    (prefix-shared, every pass full-width for the children path), for the
    first, a middle and the last parameter."""
    n, layers = 28, 2
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), 41)
    target = qv.random_target_distribution(n, 42)
    spec = qv.DdclSpec(n, layers, theta, target)
    backend = qv.B200Backend(device=0, support=target)
    ks = [0, len(theta) // 2, len(theta) - 1]
    pair = backend.shift_js_losses(qv.ddcl_circuit_template(n, layers), theta, target, ks)
    batch = qv.ddcl_batch(spec)
    direct = backend.js_losses([batch[2 * k + s] for k in ks for s in (0, 1)], n, target)
    assert np.max(np.abs(pair - direct)) < 1e-12
    buf = qv.ResultBuffer(n_qubits=n)
    backend.execute(buf, [batch[2 * ks[1]]], qv.ExecutionConfig())
    assert qv.js_divergence(target, buf.children[0].distribution) == pytest.approx(pair[2], abs=1e-12)


def test_28_qubit_light_cone_against_full_width_passes(gpu):
    """Support probabilities on the 2^10 low indices (light cone: the last
    passes sweep 1, 4, 1024 tiles; norm taken as 1) against the same support
    plus index 2^28 - 1, which makes every pass full-width and sweeps the
    norm: equal to FP64 rounding."""
    n, layers = 28, 2
    spec = qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 43),
                       qv.random_target_distribution(n, 44))
    backend = qv.B200Backend(device=0)
    circ = [qv.ddcl_circuit(spec)]
    low = np.arange(1 << 10, dtype=np.uint64)
    narrow = backend.support_probabilities(circ, n, low)
    wide = backend.support_probabilities(circ, n, np.append(low, np.uint64((1 << n) - 1)))
    assert np.max(np.abs(narrow[0] - wide[0, : low.size])) < 1e-14
    assert 0.0 < narrow.sum() < 1.0
