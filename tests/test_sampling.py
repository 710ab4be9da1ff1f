"""Counts mode.

CPU: the PCG64 restatement the device sampler uses (128-bit LCG step,
XSL-RR output, Brown jump-ahead, (x >> 11) * 2^-53 doubles) against numpy,
and the restated sampler against the reference's counts (golden vectors).
GPU: B200Backend counts mode and the counts-mode gradients against the
reference's own samples.
"""

import numpy as np
import pytest

import paper_2406_03466_b200 as qv
from oracle import statevector as sv

MULT = (2549297995355413924 << 64) + 4865540595714422341
M128 = (1 << 128) - 1
M64 = (1 << 64) - 1


def pcg_next(state, inc):
    state = (state * MULT + inc) & M128
    hi, lo = state >> 64, state & M64
    x, rot = hi ^ lo, hi >> 58
    return state, ((x >> rot) | (x << ((64 - rot) & 63))) & M64


def pcg_advance(state, inc, delta):
    """Brown's LCG skip, the same loop as sampling.cuh Pcg64::advance."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, MULT, inc
    while delta:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = ((cur_mult + 1) * cur_plus) & M128
        cur_mult = (cur_mult * cur_mult) & M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & M128


def uniforms(seed, start, count):
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    s = pcg_advance(s, inc, start)
    out = []
    for _ in range(count):
        s, v = pcg_next(s, inc)
        out.append((v >> 11) * (1.0 / 9007199254740992.0))
    return out


@pytest.mark.parametrize("seed", [0, 5, 123456789, 2 ** 40 + 7])
def test_pcg64_restatement_and_jump_ahead(seed):
    want = np.random.Generator(np.random.PCG64(seed)).random(300)
    assert uniforms(seed, 0, 300) == want.tolist()
    assert uniforms(seed, 137, 50) == want[137:187].tolist()


def restated_counts(amps, n, shots, seed):
    """Reference sampler (backend.py:140-157) on the oracle's probabilities."""
    probs = sv.normalized_probabilities(amps)
    edges = np.cumsum(probs)
    u = np.asarray(uniforms(seed, 0, shots))
    draws = np.minimum(np.searchsorted(edges, u, side="right"), probs.shape[0] - 1)
    hits = np.bincount(draws, minlength=probs.shape[0])
    return {format(i, f"0{n}b"): int(c) for i, c in enumerate(hits) if c}


def test_restated_sampler_matches_reference_counts(golden_counts):
    for case in golden_counts["circuits"]:
        n = case["n"]
        for off, (c, want) in enumerate(zip(case["batch"], case["counts"])):
            gates = [(k, tuple(t), a) for k, t, a in c["gates"]]
            if c["observable"]:
                (factors, _), = c["observable"]["terms"]
                gates += [("h", (q,), None) for q, letter in factors if letter == "X"]
            amps = sv.run_gates(n, gates)
            got = restated_counts(amps, n, case["shots"], case["seed"] + case["first_global_index"] + off)
            assert got == want


@pytest.fixture(scope="session")
def golden_counts():
    import json
    from pathlib import Path
    path = Path(__file__).resolve().parent / "golden" / "golden_counts.json"
    return json.loads(path.read_text())


def _circuit(c, n):
    gates = tuple(qv.Gate(qv.GateKind(k), tuple(t), a) for k, t, a in c["gates"])
    obs = None
    if c["observable"]:
        (factors, coeff), = c["observable"]["terms"]
        obs = qv.PauliTerm(tuple(tuple(f) for f in factors), coeff)
    return qv.Circuit(n, gates, name=c["name"], observable=obs)


@pytest.mark.gpu
def test_device_counts_match_reference(gpu, golden_counts):
    backend = qv.B200Backend(device=0)
    for case in golden_counts["circuits"]:
        n = case["n"]
        batch = [_circuit(c, n) for c in case["batch"]]
        buf = qv.ResultBuffer(n_qubits=n)
        backend.execute(buf, batch, qv.ExecutionConfig(mode="counts", shots=case["shots"], seed=case["seed"],
                                                       first_global_index=case["first_global_index"]))
        for child, want in zip(buf.children, case["counts"]):
            assert child.shots == case["shots"]
            assert child.counts == want, (n, child.name)


@pytest.mark.gpu
def test_counts_gradients_match_reference(gpu, golden_counts):
    d = golden_counts["ddcl"]
    spec = qv.DdclSpec(d["n"], d["layers"], qv.random_angles(qv.ddcl_parameter_count(d["n"], d["layers"]), d["theta_seed"]),
                       qv.random_target_distribution(d["n"], d["target_seed"]), shots=d["shots"])
    rep = qv.ddcl_gradient(spec, qv.VqpuPoolConfig(mode="counts", shots=d["shots"], base_seed=d["base_seed"]))
    assert np.max(np.abs(np.array(rep.gradient) - d["gradient"])) < 1e-12
    rep4 = qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=4, mode="counts", shots=d["shots"],
                                                    base_seed=d["base_seed"]))
    assert rep4.gradient == rep.gradient   # bitwise across vQPU counts (global seeding)
    m = golden_counts["mcvqe"]
    ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(m["n"], m["coeff_seed"]))
    mspec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(m["n"], m["cis_seed"]),
                               qv.random_angles(qv.mcvqe_parameter_count(m["n"]), m["theta_seed"]))
    mrep = qv.mcvqe_gradient(ham, mspec, qv.VqpuPoolConfig(mode="counts", shots=m["shots"], base_seed=m["base_seed"]))
    assert np.max(np.abs(np.array(mrep.gradient) - m["gradient"])) < 1e-12


@pytest.mark.gpu
def test_counts_mode_rules(gpu):
    b = qv.B200Backend(device=0)
    bell = qv.Circuit(2, (qv.h(0), qv.cnot(0, 1)), name="xx", observable=qv.pauli({0: "X", 1: "X"}))
    buf = qv.ResultBuffer(n_qubits=2)
    b.execute(buf, [bell], qv.ExecutionConfig(mode="counts", shots=500, seed=3))
    assert set(buf.children[0].counts) <= {"00", "11"} and buf.children[0].shots == 500
    shifted, direct = qv.ResultBuffer(2), qv.ResultBuffer(2)
    b.execute(shifted, [bell], qv.ExecutionConfig(mode="counts", shots=500, seed=3, first_global_index=4))
    b.execute(direct, [bell], qv.ExecutionConfig(mode="counts", shots=500, seed=7))
    assert shifted.children[0].counts == direct.children[0].counts
    with pytest.raises(qv.ExecutionError, match="Y"):
        b.execute(qv.ResultBuffer(1), [qv.Circuit(1, (), name="y", observable=qv.pauli({0: "Y"}))],
                  qv.ExecutionConfig(mode="counts"))
    assert b.execute(qv.ResultBuffer(1), [qv.Circuit(1, (), name="z")], qv.ExecutionConfig(mode="counts", shots=100)) is None
