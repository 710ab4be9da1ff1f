"""Pin the CPU oracle (oracle/statevector.py) against golden vectors produced
by the reference implementation itself (tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

from oracle import statevector as sv


def gates_of(case):
    return [(k, tuple(t), a) for k, t, a in case["gates"]]


def test_random_circuit_states_and_expectations(golden_small):
    for case in golden_small["random_circuits"]:
        n = case["n"]
        if n > 14:
            continue
        amps = sv.run_gates(n, gates_of(case))
        obs = case["observable"]
        terms = [([tuple(f) for f in factors], c) for factors, c in obs["terms"]]
        assert sv.expectation(amps, n, terms, obs["constant"]) == pytest.approx(case["expectation"], abs=1e-12)
        if "state" in case:
            want = np.array([complex(r, i) for r, i in case["state"]])
            assert np.max(np.abs(amps - want)) < 1e-13
        if "distribution" in case:
            got = sv.born_distribution(amps, n)
            assert set(got) == set(case["distribution"])
            assert max(abs(got[k] - v) for k, v in case["distribution"].items()) < 1e-13


def test_dense_oracle_agrees(golden_small):
    for case in golden_small["random_circuits"][:6]:
        n = case["n"]
        dense = sv.dense_state(n, gates_of(case))
        assert np.max(np.abs(dense - sv.run_gates(n, gates_of(case)))) < 1e-12


def test_qcl_config1_gradients(golden_small):
    cfg = golden_small["qcl_config1"]
    for pt in cfg["points"][:8]:
        theta = sv.random_angles(6 * cfg["n"] * cfg["layers"], pt["theta_seed"])
        target = sv.random_target_distribution(cfg["n"], pt["target_seed"])
        losses = sv.ddcl_losses(cfg["n"], cfg["layers"], theta, target)
        assert np.max(np.abs(np.array(losses) - pt["losses"])) < 1e-13
        grad = [0.5 * (losses[2 * k] - losses[2 * k + 1]) for k in range(len(theta))]
        assert np.max(np.abs(np.array(grad) - pt["gradient"])) < 1e-13


def test_mcvqe_gradients(golden_small):
    for case in golden_small["mcvqe"]:
        vals, terms, offset = sv.mcvqe_values(case["n"], case["coeff_seed"], case["cis_seed"], case["theta_seed"])
        assert len(vals) == case["n_circuits"]
        assert np.max(np.abs(vals - case["values"])) < 1e-12
        grad = sv.mcvqe_gradient(case["n"], case["coeff_seed"], case["cis_seed"], case["theta_seed"])
        assert np.max(np.abs(np.array(grad) - case["gradient"])) < 1e-12


def test_survey_recorded_values(golden_small, golden_large):
    """Numbers recorded in SURVEY.md section 8c from the reference."""
    mc = golden_small["mcvqe"][0]
    assert mc["gradient"][:3] == pytest.approx([0.17960268727710282, 0.4516317340310676, 0.18203194382944154], abs=1e-12)
    js = {(c["n"], c["layers"]): c["js"] for c in golden_large["qcl_forward"]}
    assert js[(4, 2)] == pytest.approx(0.07447458464324513, abs=1e-12)
    assert js[(12, 2)] == pytest.approx(0.44845454299707344, abs=1e-12)
    assert js[(14, 3)] == pytest.approx(0.5839742751341225, abs=1e-12)
    assert js[(20, 6)] == pytest.approx(0.6918049656935581, abs=1e-12)


def test_support_remainder_identity(golden_large):
    """JS with the off-support mass lumped equals the full JS (the identity
    the device epilogue relies on)."""
    for case in golden_large["qcl_forward"]:
        n, layers = case["n"], case["layers"]
        if n > 14:
            continue
        theta = sv.random_angles(6 * n * layers, case["theta_seed"])
        target = sv.random_target_distribution(n, case["target_seed"])
        amps = sv.run_gates(n, sv.bind_template(sv.ddcl_template_gates(n, layers), theta))
        probs = sv.normalized_probabilities(amps)
        full = sv.js_divergence(target, sv.born_distribution(amps, n))
        assert full == pytest.approx(case["js"], abs=1e-13)
        assert sv.js_support_remainder(target, probs) == pytest.approx(full, abs=1e-14)


def test_zero_angle_known_answer(golden_small):
    """reference test_ddcl.py:105-108: {'00': .5, '10': .5}."""
    amps = sv.run_gates(2, sv.bind_template(sv.ddcl_template_gates(2, 1), [0.0] * 12))
    got = sv.born_distribution(amps, 2)
    want = golden_small["zero_angle_distribution"]["distribution"]
    assert set(got) == set(want) == {"00", "10"}
    assert all(abs(got[k] - want[k]) < 1e-15 for k in want)


def test_js_closed_forms():
    """reference test_ddcl.py:30-43."""
    p = {"00": 0.25, "01": 0.75}
    assert sv.js_divergence(p, dict(p)) == 0.0
    assert sv.js_divergence({"0": 1.0}, {"1": 1.0}) == pytest.approx(math.log(2), abs=1e-12)
    want = 0.5 * (math.log(4 / 3) + 0.5 * math.log(2 / 3) + 0.5 * math.log(2))
    assert sv.js_divergence({"0": 1.0}, {"0": 0.5, "1": 0.5}) == pytest.approx(want, abs=1e-12)


def test_oracle_against_reference_at_config3_size():
    """The oracle restatement against the reference's own 20-qubit x 6-layer
    goldens (tests/golden/make_golden_big.py qcl20): forward JS and the
    parameter-0 shifted losses (support + remainder form, normalised by the
    swept sum as backend.py:122-129 does)."""
    import json
    from pathlib import Path
    g = json.loads((Path(__file__).resolve().parent / "golden" / "golden_big_qcl20.json").read_text())
    case = g["qcl"]
    n, layers = case["n"], case["layers"]
    theta = sv.random_angles(6 * n * layers, case["theta_seed"])
    target = sv.random_target_distribution(n, case["target_seed"])
    tpl = sv.ddcl_template_gates(n, layers)

    def loss(row):
        probs = sv.normalized_probabilities(sv.run_gates(n, sv.bind_template(tpl, row)))
        return sv.js_support_remainder(target, probs)

    assert abs(loss(theta) - case["js"]) < 1e-12
    rows = sv.shifted_thetas(theta)
    assert abs(loss(rows[0]) - case["losses"]["k0+"]) < 1e-12
    assert abs(loss(rows[1]) - case["losses"]["k0-"]) < 1e-12
