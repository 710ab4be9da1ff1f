"""Parity of the B200 executor with the reference, on the GPU.

Golden vectors come from the reference implementation (tests/golden/);
tolerances are the north star's: 1e-10 absolute for complex128 states,
1e-5 for complex64.  Everything goes through the public API and the C ABI.
"""

import math

import numpy as np
import pytest

import paper_2406_03466_b200 as qv
from oracle import statevector as sv

pytestmark = pytest.mark.gpu

TOL128 = 1e-10
TOL64 = 1e-5


def circuit_from_case(case, name="c"):
    gates = tuple(qv.Gate(qv.GateKind(k), tuple(t), a) for k, t, a in case["gates"])
    return qv.Circuit(case["n"], gates, name=name)


def observable_from_case(case):
    obs = case["observable"]
    terms = [qv.PauliTerm(tuple(tuple(f) for f in factors), c) for factors, c in obs["terms"]]
    if obs["constant"] is None:
        return terms[0]
    return qv.Observable(tuple(terms), obs["constant"])


def test_random_circuit_expectations(gpu, golden_small):
    backend = qv.B200Backend(device=0)
    for case in golden_small["random_circuits"]:
        c = circuit_from_case(case).with_observable(observable_from_case(case))
        buf = qv.ResultBuffer(n_qubits=case["n"])
        backend.execute(buf, [c], qv.ExecutionConfig())
        assert buf.children[0].expectation == pytest.approx(case["expectation"], abs=TOL128), case["n"]


def test_random_circuit_distributions(gpu, golden_small):
    backend = qv.B200Backend(device=0)
    for case in golden_small["random_circuits"]:
        if "distribution" not in case:
            continue
        buf = qv.ResultBuffer(n_qubits=case["n"])
        backend.execute(buf, [circuit_from_case(case)], qv.ExecutionConfig())
        got, want = buf.children[0].distribution, case["distribution"]
        keys = set(got) | set(want)
        assert max(abs(got.get(k, 0.0) - want.get(k, 0.0)) for k in keys) < TOL128


def test_qcl_config1_gradients(gpu, golden_small):
    """Config 1: QCL 4 qubits x 2 layers, 64 synthetic points."""
    cfg = golden_small["qcl_config1"]
    n, layers = cfg["n"], cfg["layers"]
    worst = 0.0
    for pt in cfg["points"]:
        theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), pt["theta_seed"])
        target = qv.random_target_distribution(n, pt["target_seed"])
        rep = qv.ddcl_gradient(qv.DdclSpec(n, layers, theta, target), qv.VqpuPoolConfig())
        worst = max(worst, float(np.max(np.abs(np.array(rep.gradient) - pt["gradient"]))))
        assert rep.n_circuit_executions == 2 * len(theta)
    assert worst < TOL128


def test_qcl_children_path_matches_losses(gpu, golden_small):
    """Through execute_parallel + ChildResult distributions (support +
    remainder), the reference's own JS on the children reproduces the losses."""
    cfg = golden_small["qcl_config1"]
    n, layers = cfg["n"], cfg["layers"]
    pt = cfg["points"][3]
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), pt["theta_seed"])
    target = qv.random_target_distribution(n, pt["target_seed"])
    buf = qv.ResultBuffer(n_qubits=n)
    rep = qv.ddcl_gradient(qv.DdclSpec(n, layers, theta, target), qv.VqpuPoolConfig(n_virtual_qpus=3), buffer=buf)
    losses = [qv.js_divergence(target, c.distribution) for c in buf.children]
    assert np.max(np.abs(np.array(losses) - pt["losses"])) < TOL128
    assert np.max(np.abs(np.array(rep.gradient) - pt["gradient"])) < TOL128
    assert buf.child_names()[:2] == ["k0+", "k0-"]


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_mcvqe_gradients(gpu, golden_small, idx):
    case = golden_small["mcvqe"][idx]
    n = case["n"]
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(n, case["coeff_seed"]))
    spec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(n, case["cis_seed"]),
                              qv.random_angles(qv.mcvqe_parameter_count(n), case["theta_seed"]))
    rep = qv.mcvqe_gradient(ham, spec, qv.VqpuPoolConfig())
    assert rep.n_circuit_executions == case["n_circuits"]
    assert np.max(np.abs(np.array(rep.gradient) - case["gradient"])) < TOL128
    buf = qv.ResultBuffer(n_qubits=n)
    rep2 = qv.mcvqe_gradient(ham, spec, qv.VqpuPoolConfig(n_virtual_qpus=4), buffer=buf)
    vals = np.array([c.expectation for c in buf.children])
    assert np.max(np.abs(vals - case["values"])) < TOL128
    assert buf.child_names()[: len(case["names"])] == case["names"]
    assert np.max(np.abs(np.array(rep2.gradient) - case["gradient"])) < TOL128
    assert qv.mcvqe_energy(ham, spec) == pytest.approx(case["energy"], abs=TOL128)


def test_qcl_forward_and_shifted_losses(gpu, golden_large):
    backend = qv.B200Backend(device=0)
    for case in golden_large["qcl_forward"]:
        n, layers = case["n"], case["layers"]
        theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), case["theta_seed"])
        target = qv.random_target_distribution(n, case["target_seed"])
        spec = qv.DdclSpec(n, layers, theta, target)
        js = backend.js_losses([qv.ddcl_circuit(spec)], n, target)[0]
        assert js == pytest.approx(case["js"], abs=TOL128), n
        if case["shifted"]:
            batch = qv.ddcl_batch(spec)
            pick = [2 * s["k"] + (0 if s["tag"] == "+" else 1) for s in case["shifted"]]
            got = backend.js_losses([batch[i] for i in pick], n, target)
            assert np.max(np.abs(got - [s["js"] for s in case["shifted"]])) < TOL128, n


@pytest.mark.parametrize("idx", [0, 1])
def test_qcl_full_gradient_multi_tile(gpu, golden_large, idx):
    """Whole shifted batch through the prefix-sharing scheduler (14q: state
    in HBM, several passes per circuit)."""
    case = golden_large["qcl_gradient"][idx]
    n, layers = case["n"], case["layers"]
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), case["theta_seed"])
    target = qv.random_target_distribution(n, case["target_seed"])
    spec = qv.DdclSpec(n, layers, theta, target)
    backend = qv.B200Backend(device=0)
    losses = backend.js_losses(qv.ddcl_batch(spec), n, target)
    assert np.max(np.abs(losses - case["losses"])) < TOL128
    rep = qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=5))
    assert np.max(np.abs(np.array(rep.gradient) - case["gradient"])) < TOL128


def test_shift_pairs_match_reference_and_direct(gpu, golden_large):
    """qv_shift_js (Psi0 -+ i Xi forms) against the reference's losses of the
    directly shifted circuits, and against direct simulation on the GPU."""
    backend = qv.B200Backend(device=0)
    for case in golden_large["qcl_forward"]:
        n, layers = case["n"], case["layers"]
        if n <= 12 or not case["shifted"]:
            continue
        theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), case["theta_seed"])
        target = qv.random_target_distribution(n, case["target_seed"])
        tpl = qv.ddcl_circuit_template(n, layers)
        ks = sorted({s["k"] for s in case["shifted"]})
        losses = backend.shift_js_losses(tpl, theta, target, ks)
        for s in case["shifted"]:
            got = losses[2 * ks.index(s["k"]) + (0 if s["tag"] == "+" else 1)]
            assert got == pytest.approx(s["js"], abs=TOL128), (n, s)
    case = golden_large["qcl_gradient"][0]   # 14 qubits x 1 layer, every parameter
    n, layers = case["n"], case["layers"]
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), case["theta_seed"])
    target = qv.random_target_distribution(n, case["target_seed"])
    pair = backend.shift_js_losses(qv.ddcl_circuit_template(n, layers), theta, target, list(range(len(theta))))
    assert np.max(np.abs(pair - case["losses"])) < TOL128
    direct = backend.js_losses(qv.ddcl_batch(qv.DdclSpec(n, layers, theta, target)), n, target)
    assert np.max(np.abs(pair - direct)) < 1e-13
    rep_pair = qv.ddcl_gradient(qv.DdclSpec(n, layers, theta, target), qv.VqpuPoolConfig(n_virtual_qpus=3))
    rep_direct = qv.ddcl_gradient(qv.DdclSpec(n, layers, theta, target), qv.VqpuPoolConfig(), shift_mode="direct")
    assert np.max(np.abs(np.array(rep_pair.gradient) - case["gradient"])) < TOL128
    assert np.max(np.abs(np.array(rep_direct.gradient) - case["gradient"])) < TOL128
    with pytest.raises(qv.ExecutionError):   # one tile: use js_losses
        backend.shift_js_losses(qv.ddcl_circuit_template(4, 1), [0.1] * 24, qv.random_target_distribution(4, 1), [0])


def test_complex64_within_1e5(gpu, golden_small, golden_large):
    cfg = golden_small["qcl_config1"]
    n, layers = cfg["n"], cfg["layers"]
    pt = cfg["points"][0]
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), pt["theta_seed"])
    target = qv.random_target_distribution(n, pt["target_seed"])
    rep = qv.ddcl_gradient(qv.DdclSpec(n, layers, theta, target), qv.VqpuPoolConfig(),
                           backend_factory=lambda: qv.B200Backend(precision="complex64", support=target))
    # children path (custom factory) in complex64
    assert np.max(np.abs(np.array(rep.gradient) - pt["gradient"])) < TOL64
    backend = qv.B200Backend(device=0, precision="complex64")
    for case in golden_large["qcl_forward"]:
        n, layers = case["n"], case["layers"]
        theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), case["theta_seed"])
        target = qv.random_target_distribution(n, case["target_seed"])
        js = backend.js_losses([qv.ddcl_circuit(qv.DdclSpec(n, layers, theta, target))], n, target)[0]
        assert js == pytest.approx(case["js"], abs=TOL64), n
    mc = golden_small["mcvqe"][0]
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(8, mc["coeff_seed"]))
    spec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(8, mc["cis_seed"]), qv.random_angles(36, mc["theta_seed"]))
    vals = backend.expectation_values(qv.mcvqe_gradient_batch(ham, spec), 8)
    assert np.max(np.abs(vals - mc["values"])) < TOL64


def test_extension_gates_rx_cz_against_oracle(gpu):
    backend = qv.B200Backend(device=0)
    for seed, n in ((1, 3), (2, 7), (3, 13), (4, 15)):
        rng = np.random.Generator(np.random.PCG64(seed))
        gates = sv.random_circuit_gates(rng, n, 150, extended=True)
        circ = qv.Circuit(n, tuple(qv.Gate(qv.GateKind(k), t, a) for k, t, a in gates), name="e")
        term = qv.pauli({0: "Y", n - 1: "X"}, 0.7)
        got = backend.expectation_values([circ.with_observable(term)], n)[0]
        amps = sv.run_gates(n, gates)
        want = 0.7 * sv.pauli_expectation(amps, n, *sv.term_masks(term.factors, n))
        assert got == pytest.approx(want, abs=TOL128), n


def test_light_cone_untouched_qubits_and_scattered_support(gpu):
    """Support-restricted runs sweep only the light cone (forward from |0>,
    backward from the support).  Qubits 0 and 1 carry no gate (their bits are
    never in a tile), the support mixes indices inside and outside that
    reach, and the shifted losses come from the pair path: all against the
    dense oracle."""
    n = 15
    rng = np.random.Generator(np.random.PCG64(77))
    names = [f"p{i}" for i in range(3 * (n - 2))]
    it = iter(names)
    gates = []
    for q in range(2, n):
        gates += [qv.h(q), qv.ry(q, next(it))]
    gates += [qv.cnot(q, q + 1) for q in range(2, n - 1)]
    for q in range(2, n):
        gates += [qv.rz(q, next(it)), qv.ry(q, next(it))]
    tpl = qv.Circuit(n, tuple(gates), name="cone", params=tuple(names))
    theta = rng.uniform(0, 2 * math.pi, len(names))
    idx = np.unique(np.concatenate([rng.integers(0, 1 << n, 200), rng.integers(0, 1 << (n - 2), 200)]))
    w = rng.uniform(0.0, 1.0, idx.size)
    target = {format(int(i), f"0{n}b"): float(v / w.sum()) for i, v in zip(idx, w)}
    backend = qv.B200Backend(device=0)

    def oracle_js(values):
        circ = qv.bind(tpl, values)
        amps = sv.run_gates(n, [(g.kind.value, g.targets, g.angle) for g in circ.gates])
        return sv.js_divergence(target, sv.born_distribution(amps, n))

    got = backend.js_losses([qv.bind(tpl, theta)], n, target)[0]
    assert got == pytest.approx(oracle_js(theta), abs=TOL128)
    ks = [0, 5, len(names) - 1]
    pair = backend.shift_js_losses(tpl, theta, target, ks)
    for j, k in enumerate(ks):
        for s, sign in enumerate((1.0, -1.0)):
            shifted = theta.copy()
            shifted[k] += sign * math.pi / 2
            assert pair[2 * j + s] == pytest.approx(oracle_js(shifted), abs=TOL128), (k, sign)


def test_forward_losses_batch_of_points(gpu, golden_large):
    """Config 3's forward pass: one circuit per data point, each against its
    own target, in one device batch -- against the reference's JS values and
    against per-point device losses."""
    backend = qv.B200Backend(device=0)
    for case in golden_large["qcl_forward"]:
        n, layers = case["n"], case["layers"]
        spec = qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), case["theta_seed"]),
                           qv.random_target_distribution(n, case["target_seed"]))
        assert qv.ddcl_forward_losses([spec], backend)[0] == pytest.approx(case["js"], abs=TOL128), n
    n, layers = 14, 2
    specs = [qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 1 + i),
                         qv.random_target_distribution(n, 2 + i)) for i in range(5)]
    batch = qv.ddcl_forward_losses(specs, backend)
    single = [backend.js_losses([qv.ddcl_circuit(s)], n, s.target)[0] for s in specs]
    assert np.max(np.abs(batch - np.asarray(single))) < 1e-13


@pytest.mark.parametrize("n", [8, 14])
def test_js_losses_against_own_targets(gpu, n):
    """QV_RES_TARGET_ROWS: each circuit against its own target row equals
    `js_losses` of that circuit alone with that target -- incl. duplicate
    circuits (one unique state, two targets) and a batch of two topologies
    (non-contiguous rows per topology group)."""
    backend = qv.B200Backend(device=0)
    layers = 2
    specs = [qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 30 + i),
                         qv.random_target_distribution(n, 40 + i)) for i in range(4)]
    circuits = [qv.ddcl_circuit(s) for s in specs]
    circuits.append(qv.ddcl_circuit(specs[0]))   # duplicate state, other target below
    other = qv.Circuit(n, tuple([qv.h(0)] + [qv.cnot(q, q + 1) for q in range(n - 1)]), name="ghz")
    circuits.insert(2, other)
    targets = [s.target for s in specs[:2]] + [specs[3].target] + [s.target for s in specs[2:]] + [specs[1].target]
    keys = sorted(targets[0])
    rows = np.asarray([[t[k] for k in keys] for t in targets])
    got = backend.js_losses_targets(circuits, n, keys, rows)
    want = [backend.js_losses([c], n, t)[0] for c, t in zip(circuits, targets)]
    assert np.max(np.abs(got - np.asarray(want))) < 1e-13
    assert got[0] != got[-1]   # same state, different targets
    with pytest.raises(ValueError):
        backend.js_losses_targets(circuits, n, keys, rows[:-1])
    # target rows are a JS-only option; unknown flags are rejected
    from paper_2406_03466_b200 import native
    from paper_2406_03466_b200.backend import lower_batch
    sup = np.asarray([0, 1], np.uint64)
    for kind, flags in ((native.QV_OUT_SUPPORT, native.QV_RES_TARGET_ROWS), (native.QV_OUT_JS, 6)):
        with pytest.raises(native.NativeError):
            backend._engine.execute(n, lower_batch(circuits[:1]), kind, support=sup, target=np.zeros(2), flags=flags)
    # empty support: only the remainder term (1 - 0)/2 ln 2, as without rows
    empty = backend.js_losses_targets(circuits[:2], n, [], np.zeros((2, 0)))
    assert np.array_equal(empty, np.full(2, 0.5 * math.log(2.0)))
    assert np.array_equal(backend.js_losses(circuits[:2], n, {}), empty)
    norms = backend.support_probabilities(circuits[:2], n, [])
    assert norms.shape == (2, 0)
    if n > backend.tile_qubits():
        pair = backend.shift_js_losses(qv.ddcl_circuit_template(n, layers), specs[0].theta, {}, [0, 5])
        assert np.max(np.abs(pair - 0.5 * math.log(2.0))) < 1e-15


@pytest.mark.parametrize("seed", range(8))
def test_random_multi_tile_circuits_fuzz(gpu, seed):
    """Random circuits on 13-18 qubits (several tiles, all gate kinds incl.
    the RX / CZ extensions): support probabilities on a scattered support
    (light-cone passes) and a random Pauli term (full-width passes) against
    the dense oracle."""
    rng = np.random.Generator(np.random.PCG64(900 + seed))
    n = 13 + seed % 6
    gates = sv.random_circuit_gates(rng, n, 240, extended=True)
    circ = qv.Circuit(n, tuple(qv.Gate(qv.GateKind(k), t, a) for k, t, a in gates), name="f")
    amps = sv.run_gates(n, gates)
    backend = qv.B200Backend(device=0)
    sup = np.unique(rng.integers(0, 1 << n, 64).astype(np.uint64))
    got = backend.support_probabilities([circ], n, sup)[0]
    assert np.max(np.abs(got - np.abs(amps[sup.astype(np.int64)]) ** 2)) < 1e-12
    letters = rng.choice(list("XYZ"), size=3)
    qubits = rng.choice(n, size=3, replace=False)
    term = qv.pauli({int(q): str(p) for q, p in zip(qubits, letters)}, 0.5)
    want = 0.5 * sv.pauli_expectation(amps, n, *sv.term_masks(term.factors, n))
    assert backend.expectation_values([circ.with_observable(term)], n)[0] == pytest.approx(want, abs=TOL128)
