"""Parity at the BASELINE's benchmark sizes (configs 3, 4, 5) against goldens
the REFERENCE produced with its own numba kernels (tests/golden/
make_golden_big.py: reference allocate / run_gates / born_probabilities,
backend.py:57-91, 122-129, kernels.py:18-94; JS by the support + remainder
form of ddcl.py:37-61; shifted circuits bound by gradients.py:33-46).

Tolerances are the north star's: 1e-10 absolute in complex128, 1e-5 in
complex64 (against the reference's complex128 answer).
"""

import numpy as np
import pytest

import paper_2406_03466_b200 as qv
from paper_2406_03466_b200 import native

pytestmark = pytest.mark.gpu

TOL128 = 1e-10
TOL64 = 1e-5


@pytest.fixture(autouse=True)
def _free_states():
    """Registers here take 4-64 GiB per state: give the device memory back
    after each test so the next one (other precision, larger state) fits."""
    yield
    for precision in ("complex128", "complex64"):
        native.release_engine(0, precision)


def _spec(case):
    n, layers = case["n"], case["layers"]
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), case["theta_seed"])
    target = qv.random_target_distribution(n, case["target_seed"])
    return qv.DdclSpec(n, layers, theta, target)


def _want_losses(case, ks):
    return np.array([case["losses"][f"k{k}{t}"] for k in ks for t in "+-"])


def _case(golden_big, name):
    if name not in golden_big:
        pytest.fail(f"tests/golden/golden_big_{name}.json is missing (tests/golden/make_golden_big.py {name})")
    return golden_big[name]["qcl"]


# ---------------------------------------------------------------- config 4
def test_config4_28q_shift_pairs_and_direct(gpu, golden_big):
    """28 qubits x 8 layers, complex128: the shift-pair path and directly
    simulated shifted circuits, k = first / middle / last parameter."""
    case = _case(golden_big, "qcl28")
    spec = _spec(case)
    ks = case["ks"]
    backend = qv.B200Backend(device=0)
    tpl = qv.ddcl_circuit_template(spec.n_qubits, spec.n_layers)
    pair = backend.shift_js_losses(tpl, spec.theta, spec.target, ks)
    want = _want_losses(case, ks)
    assert np.max(np.abs(pair - want)) < TOL128
    batch = qv.ddcl_batch(spec)
    direct = backend.js_losses([qv.ddcl_circuit(spec)] + [batch[2 * k + s] for k in ks for s in (0, 1)],
                               spec.n_qubits, spec.target)
    assert abs(direct[0] - case["js"]) < TOL128
    assert np.max(np.abs(direct[1:] - want)) < TOL128
    # support probabilities of the unshifted circuit (each ~1e-9: relative check)
    probs = backend.support_probabilities([qv.ddcl_circuit(spec)], spec.n_qubits, spec.target)[0]
    ref = np.asarray(case["support_probs"])
    assert np.max(np.abs(probs - ref)) < 1e-9 * np.max(ref)


def test_config4_28q_full_gradient(gpu, golden_big):
    """The production path of the bench: ddcl_gradient over the whole
    2,688-circuit shift table (shift pairs, prefix sharing, light cone, TMA
    pass kernel) matches the reference's gradient entries."""
    case = _case(golden_big, "qcl28")
    spec = _spec(case)
    rep = qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=1))
    assert rep.n_circuit_executions == 2 * len(spec.theta)
    grad = np.asarray(rep.gradient)
    assert np.all(np.isfinite(grad))
    for k in case["ks"]:
        assert abs(grad[k] - case["gradient"][str(k)]) < TOL128, k


def test_config4_28q_complex64(gpu, golden_big):
    """complex64 at 28 qubits x 8 layers against the reference's complex128:
    the complex64 shift-pair path (qv_shift_js in float, incl. the
    per-parameter phase rotation of finalize_pair_kernel), direct losses, and
    the children path through Accelerator.execute()."""
    case = _case(golden_big, "qcl28")
    spec = _spec(case)
    ks = case["ks"]
    backend = qv.B200Backend(device=0, precision="complex64")
    tpl = qv.ddcl_circuit_template(spec.n_qubits, spec.n_layers)
    pair = backend.shift_js_losses(tpl, spec.theta, spec.target, ks)
    want = _want_losses(case, ks)
    assert np.max(np.abs(pair - want)) < TOL64
    batch = qv.ddcl_batch(spec)
    circuits = [batch[2 * ks[0]], batch[2 * ks[0] + 1]]
    direct = backend.js_losses(circuits, spec.n_qubits, spec.target)
    assert np.max(np.abs(direct - want[:2])) < TOL64
    # children: support + one remainder key per child, reference js_divergence
    child_backend = qv.B200Backend(device=0, precision="complex64", support=spec.target)
    buf = qv.ResultBuffer(n_qubits=spec.n_qubits)
    child_backend.execute(buf, circuits, qv.ExecutionConfig())
    got = [qv.js_divergence(spec.target, c.distribution) for c in buf.children]
    assert np.max(np.abs(np.asarray(got) - want[:2])) < TOL64


# ---------------------------------------------------------------- config 3
def test_config3_20q_gradient_entries(gpu, golden_big):
    """20 qubits x 6 layers: gradient entries at 10 parameters (shift pairs
    and direct shifted circuits) and the forward JS of batch points 0 / 511 /
    1023 (theta seed 1+i, target seed 2+i)."""
    g = golden_big.get("qcl20") or pytest.fail("golden_big_qcl20.json missing")
    case = g["qcl"]
    spec = _spec(case)
    for mode in ("pair", "direct"):
        rep = qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=4), shift_mode=mode)
        grad = np.asarray(rep.gradient)
        for k in case["ks"]:
            assert abs(grad[k] - case["gradient"][str(k)]) < TOL128, (mode, k)
    n, layers = spec.n_qubits, spec.n_layers
    specs = [qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), p["theta_seed"]),
                         qv.random_target_distribution(n, p["target_seed"])) for p in g["points"]]
    fwd = qv.ddcl_forward_losses(specs, qv.B200Backend(device=0))
    assert np.max(np.abs(fwd - [p["js"] for p in g["points"]])) < TOL128


# ---------------------------------------------------------------- config 5
def test_config5_geometry_30q(gpu, golden_big):
    """Config 5's circuit (4 layers) at the reference's 30-qubit cap
    (backend.py:31): complex128 within 1e-10 and complex64 within 1e-5 of
    the reference, forward loss and the shift pair of parameter 0."""
    case = _case(golden_big, "qcl30c5")
    spec = _spec(case)
    tpl = qv.ddcl_circuit_template(spec.n_qubits, spec.n_layers)
    want = _want_losses(case, case["ks"])
    for precision, tol in (("complex128", TOL128), ("complex64", TOL64)):
        backend = qv.B200Backend(device=0, precision=precision)
        fwd = backend.js_losses([qv.ddcl_circuit(spec)], spec.n_qubits, spec.target)[0]
        assert abs(fwd - case["js"]) < tol, precision
        pair = backend.shift_js_losses(tpl, spec.theta, spec.target, case["ks"])
        assert np.max(np.abs(pair - want)) < tol, precision
        native.release_engine(0, precision)


def test_config5_32q_complex64_against_complex128(gpu):
    """Config 5 itself (32 qubits x 4 layers) is beyond the reference
    (n > 30): complex64 shift pairs against this executor's complex128
    direct simulation (one 64 GiB state at a time) within 1e-5."""
    n, layers = 32, 4
    spec = qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 1),
                       qv.random_target_distribution(n, 2))
    ks = [0, 383, 767]
    batch = qv.ddcl_batch(spec)
    b128 = qv.B200Backend(device=0, precision="complex128")
    ref = np.concatenate([b128.js_losses([batch[2 * k], batch[2 * k + 1]], n, spec.target) for k in ks])
    fwd128 = b128.js_losses([qv.ddcl_circuit(spec)], n, spec.target)[0]
    native.release_engine(0, "complex128")
    b64 = qv.B200Backend(device=0, precision="complex64")
    pair = b64.shift_js_losses(qv.ddcl_circuit_template(n, layers), spec.theta, spec.target, ks)
    assert np.max(np.abs(pair - ref)) < TOL64
    fwd64 = b64.js_losses([qv.ddcl_circuit(spec)], n, spec.target)[0]
    assert abs(fwd64 - fwd128) < TOL64
    native.release_engine(0, "complex64")


# ------------------------------------------------------- MC-VQE, n = 16
def test_mcvqe16_fused_pauli_terms(gpu, golden_big):
    """MC-VQE at 16 chromophores (multi-tile registers): every one of the
    13,984 shifted-circuit expectations and the gradient against the
    reference (mcvqe.py:194-247, kernels.py:73-87), with each term evaluated
    inside a pass (the state's last pass or a read-only window sweep) -- at
    most two whole-state reads per distinct state instead of one per term
    (N_H = 6n - 4 = 92)."""
    if "mcvqe16" not in golden_big:
        pytest.fail("tests/golden/golden_big_mcvqe16.json is missing (make_golden_big.py mcvqe16)")
    case = golden_big["mcvqe16"]["mcvqe"]
    n = case["n"]
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(n, case["coeff_seed"]))
    spec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(n, case["cis_seed"]),
                              qv.random_angles(qv.mcvqe_parameter_count(n), case["theta_seed"]))
    backend = qv.B200Backend(device=0)
    vals = backend.expectation_values(qv.mcvqe_gradient_batch(ham, spec), n)
    assert len(vals) == case["n_circuits"]
    assert np.max(np.abs(vals - case["values"])) < TOL128
    st = native.engine(0).last_stats
    assert st["pauli_state_reads"] <= 2 * st["unique_states"], st
    rep = qv.mcvqe_gradient(ham, spec, qv.VqpuPoolConfig(n_virtual_qpus=3))
    assert np.max(np.abs(np.asarray(rep.gradient) - case["gradient"])) < TOL128
    assert qv.mcvqe_energy(ham, spec) == pytest.approx(case["energy"], abs=TOL128)


# ------------------------------------- the literal drop-in at config 3 size
def _reference_qvirt():
    """The unmodified reference package installed in baseline/_ref."""
    import os
    import sys
    from pathlib import Path
    ref = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
    if not (ref / "qvirt").exists():
        pytest.skip("baseline/_ref not installed")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba-qvirt")
    sys.path.insert(0, str(ref))
    try:
        import qvirt
    finally:
        sys.path.remove(str(ref))
    return qvirt


def test_config3_reference_driver_on_b200(gpu, golden_big):
    """The reference's own ddcl_gradient -> shifted_circuits ->
    execute_parallel -> Accelerator.execute path (ddcl.py:197-226,
    gradients.py:33-46, pool.py:88-138, backend.py:189-227), unmodified, with
    B200Backend as the backend factory, at 20 qubits x 6 layers: its
    gradient matches the reference's golden entries."""
    qvirt = _reference_qvirt()
    g = golden_big.get("qcl20") or pytest.fail("golden_big_qcl20.json missing")
    case = g["qcl"]
    n, layers = case["n"], case["layers"]
    theta = qvirt.random_angles(qvirt.ddcl_parameter_count(n, layers), case["theta_seed"])
    target = qvirt.random_target_distribution(n, case["target_seed"])
    spec = qvirt.DdclSpec(n, layers, theta, target)
    rep = qvirt.ddcl_gradient(spec, qvirt.VqpuPoolConfig(n_virtual_qpus=4, mode="expectation"),
                              backend_factory=lambda: qv.B200Backend(support=target))
    assert rep.n_circuit_executions == 2 * len(theta)
    for k in case["ks"]:
        assert abs(rep.gradient[k] - case["gradient"][str(k)]) < TOL128, k
