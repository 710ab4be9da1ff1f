"""Generate golden vectors by running the REFERENCE implementation (`qvirt`).

Run in the build container, where the read-only reference is mounted:

    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests \
        python tests/golden/make_golden.py

Writes tests/golden/*.json (committed).  Every case stores its seeds so it can
be regenerated; floats are written with repr precision (exact round trip).
Nothing on the GPU box reads /root/reference: tests use these fixtures.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("QVIRT_REFERENCE", "/root/reference/pkg"))
sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba-golden")

import oracles  # noqa: E402  (reference pkg/tests/oracles.py)
import qvirt  # noqa: E402
from qvirt import (  # noqa: E402
    DdclSpec, ExecutionConfig, McvqeAnsatzSpec, ResultBuffer, StatevectorBackend, VqpuPoolConfig,
    aiem_hamiltonian, ddcl_circuit, ddcl_circuit_template, ddcl_gradient, ddcl_parameter_count,
    js_divergence, mcvqe_energy, mcvqe_gradient, mcvqe_gradient_batch, mcvqe_parameter_count,
    random_aiem_coefficients, random_angles, random_cis_amplitudes, random_target_distribution,
)
from qvirt.backend import allocate, born_distribution, expectation, run_gates  # noqa: E402
from qvirt.gradients import shifted_circuits  # noqa: E402

OUT = Path(__file__).resolve().parent


def gates_json(circuit):
    return [[g.kind.value, list(g.targets), g.angle] for g in circuit.gates]


def obs_json(obs):
    if obs is None:
        return None
    if isinstance(obs, qvirt.PauliTerm):
        return {"terms": [[[list(f) for f in obs.factors], obs.coefficient]], "constant": None}
    return {"terms": [[[list(f) for f in t.factors], t.coefficient] for t in obs.terms], "constant": obs.constant}


def random_circuits():
    """Random circuits over the full gate set (pkg/tests/oracles.py:96-129)
    with random observables: final states for n <= 6, expectations for all."""
    cases = []
    specs = [(s, n, g) for s, (n, g) in enumerate([(1, 5), (2, 9), (3, 12), (4, 16), (5, 25), (6, 40),
                                                     (8, 60), (10, 120), (12, 160), (13, 200), (14, 220),
                                                     (16, 260), (18, 300)])]
    for seed, n, n_gates in specs:
        rng = np.random.Generator(np.random.PCG64(1000 + seed))
        circuit = oracles.random_circuit(rng, n, n_gates, name=f"rc{seed}")
        obs = oracles.random_observable(np.random.Generator(np.random.PCG64(2000 + seed)), n, 4)
        state = run_gates(allocate(n), circuit.gates)
        case = {"seed": seed, "n": n, "gates": gates_json(circuit), "observable": obs_json(obs),
                "expectation": expectation(state, obs)}
        if n <= 6:
            case["state"] = [[float(a.real), float(a.imag)] for a in state.amplitudes]
        if n <= 12:
            dist = born_distribution(state)
            case["distribution"] = {k: v for k, v in dist.items()}
        cases.append(case)
    return cases


def qcl_config1(points=64, base_seed=0):
    """Config 1: QCL 4 qubits x 2 layers, parameter-shift gradient over 64
    synthetic points; point i = (theta seed base+1+i, target seed base+2+i)."""
    n, layers = 4, 2
    count = ddcl_parameter_count(n, layers)
    out = []
    for i in range(points):
        theta = random_angles(count, base_seed + 1 + i)
        target = random_target_distribution(n, base_seed + 2 + i)
        spec = DdclSpec(n, layers, theta, target)
        buf = ResultBuffer(n_qubits=n)
        rep = ddcl_gradient(spec, VqpuPoolConfig(mode="expectation"), buffer=buf)
        losses = [js_divergence(target, c.distribution) for c in buf.children]
        out.append({"point": i, "theta_seed": base_seed + 1 + i, "target_seed": base_seed + 2 + i,
                    "gradient": list(rep.gradient), "losses": losses})
    return {"n": n, "layers": layers, "points": out}


def mcvqe_case(n, coeff_seed, cis_seed, theta_seed, keep_values=True):
    ham = aiem_hamiltonian(random_aiem_coefficients(n, coeff_seed))
    spec = McvqeAnsatzSpec(random_cis_amplitudes(n, cis_seed), random_angles(mcvqe_parameter_count(n), theta_seed))
    buf = ResultBuffer(n_qubits=n)
    rep = mcvqe_gradient(ham, spec, VqpuPoolConfig(mode="expectation"), buffer=buf)
    case = {"n": n, "coeff_seed": coeff_seed, "cis_seed": cis_seed, "theta_seed": theta_seed,
            "gradient": list(rep.gradient), "energy": mcvqe_energy(ham, spec),
            "n_circuits": rep.n_circuit_executions}
    if keep_values:
        case["values"] = [c.expectation for c in buf.children]
        case["names"] = [c.name for c in buf.children[:50]]
    return case


def qcl_forward(n, layers, theta_seed=1, target_seed=2, shifted=()):
    """JS loss of the unshifted circuit and of selected shifted circuits."""
    count = ddcl_parameter_count(n, layers)
    theta = random_angles(count, theta_seed)
    target = random_target_distribution(n, target_seed)
    spec = DdclSpec(n, layers, theta, target)
    state = run_gates(allocate(n), ddcl_circuit(spec).gates)
    case = {"n": n, "layers": layers, "theta_seed": theta_seed, "target_seed": target_seed,
            "js": js_divergence(target, born_distribution(state)), "shifted": []}
    if shifted:
        template = ddcl_circuit_template(n, layers)
        wanted = set(shifted)
        for k, tag, bound in shifted_circuits(template, theta):
            if (k, tag) in wanted:
                st = run_gates(allocate(n), bound.gates)
                case["shifted"].append({"k": k, "tag": tag, "js": js_divergence(target, born_distribution(st))})
    return case


def qcl_gradient_case(n, layers, theta_seed, target_seed):
    count = ddcl_parameter_count(n, layers)
    theta = random_angles(count, theta_seed)
    target = random_target_distribution(n, target_seed)
    buf = ResultBuffer(n_qubits=n)
    rep = ddcl_gradient(DdclSpec(n, layers, theta, target), VqpuPoolConfig(n_virtual_qpus=8), buffer=buf)
    losses = [js_divergence(target, c.distribution) for c in buf.children]
    return {"n": n, "layers": layers, "theta_seed": theta_seed, "target_seed": target_seed,
            "gradient": list(rep.gradient), "losses": losses}


def counts_cases():
    """Counts mode (backend.py:140-157, 220-227): sampled tallies from the
    reference for random circuits (with and without X/Z terms), and the
    counts-mode DDCL / MC-VQE gradients."""
    out = {"circuits": []}
    for seed, n, n_gates, shots in ((1, 2, 6, 500), (2, 5, 30, 1000), (3, 8, 60, 4096), (4, 11, 90, 8192),
                                     (5, 14, 120, 2000)):
        rng = np.random.Generator(np.random.PCG64(3000 + seed))
        batch = []
        for i in range(4):
            c = oracles.random_circuit(rng, n, n_gates, name=f"s{seed}c{i}")
            if i % 2:
                c = c.with_observable(oracles.random_pauli_term(rng, n, letters="XZ"))
            batch.append(c)
        buf = ResultBuffer(n_qubits=n)
        StatevectorBackend().execute(buf, batch, ExecutionConfig(mode="counts", shots=shots, seed=11 * seed,
                                                                  first_global_index=seed))
        out["circuits"].append({
            "n": n, "shots": shots, "seed": 11 * seed, "first_global_index": seed,
            "batch": [{"gates": gates_json(c), "observable": obs_json(c.observable), "name": c.name} for c in batch],
            "counts": [ch.counts for ch in buf.children]})
    theta = random_angles(ddcl_parameter_count(4, 1), 7)
    spec = DdclSpec(4, 1, theta, random_target_distribution(4, 8), shots=2048)
    rep = ddcl_gradient(spec, VqpuPoolConfig(mode="counts", shots=2048, base_seed=6))
    out["ddcl"] = {"n": 4, "layers": 1, "theta_seed": 7, "target_seed": 8, "shots": 2048, "base_seed": 6,
                   "gradient": list(rep.gradient)}
    ham = aiem_hamiltonian(random_aiem_coefficients(3, 8))
    mspec = McvqeAnsatzSpec(random_cis_amplitudes(3, 9), random_angles(mcvqe_parameter_count(3), 10))
    mrep = mcvqe_gradient(ham, mspec, VqpuPoolConfig(mode="counts", shots=512, base_seed=1))
    out["mcvqe"] = {"n": 3, "coeff_seed": 8, "cis_seed": 9, "theta_seed": 10, "shots": 512, "base_seed": 1,
                    "gradient": list(mrep.gradient)}
    return out


def buffer_cases():
    """The reference's text form of result buffers (buffers.py:129-152):
    exact-mode distributions and expectations, counts, metadata, awkward
    names and floats, plus the reference's pool output of a small batch."""
    from qvirt.buffers import ChildResult, serialize
    cases = []
    buf = ResultBuffer(n_qubits=3)
    buf.metadata.update({"vqpu_count": 4, "label": "run 1", "ok": True, "scale": 0.1 + 0.2, "a.b-c_d": -7})
    buf.append_child(ChildResult(name="k0+", expectation=1.0 / 3.0))
    buf.append_child(ChildResult(name="with space", expectation=-2.5e-17))
    buf.append_child(ChildResult(name="c", counts={"101": 5, "000": 2, "011": 1}, shots=8))
    buf.append_child(ChildResult(name="d", distribution={"111": 0.6, "001": 0.1 + 0.2, "000": 0.1}))
    cases.append({"text": serialize(buf)})
    rng = np.random.default_rng(5)
    batch = []
    for i in range(4):
        c = oracles.random_circuit(rng, 3, 12, name=f"p{i}")
        if i % 2:
            c = c.with_observable(oracles.random_pauli_term(rng, 3, letters="XZ"))
        batch.append(c)
    pool = ResultBuffer(n_qubits=3)
    qvirt.execute_parallel(pool, batch, VqpuPoolConfig(n_virtual_qpus=2))
    cases.append({"text": serialize(pool), "n": 3, "n_virtual_qpus": 2,
                  "batch": [{"gates": gates_json(c), "observable": obs_json(c.observable), "name": c.name}
                            for c in batch]})
    counted = ResultBuffer(n_qubits=3)
    StatevectorBackend().execute(counted, batch, ExecutionConfig(mode="counts", shots=100, seed=3))
    cases.append({"text": serialize(counted)})
    return cases


def main():
    if "--counts-only" in sys.argv:
        (OUT / "golden_counts.json").write_text(json.dumps(counts_cases()))
        return
    if "--buffers-only" in sys.argv:
        (OUT / "golden_buffers.json").write_text(json.dumps(buffer_cases()))
        return
    (OUT / "golden_buffers.json").write_text(json.dumps(buffer_cases()))
    t0 = time.time()
    (OUT / "golden_counts.json").write_text(json.dumps(counts_cases()))
    small = {"generator": "tests/golden/make_golden.py", "reference": str(REF),
             "random_circuits": random_circuits()}
    print(f"random circuits {time.time() - t0:.1f}s", flush=True)
    small["qcl_config1"] = qcl_config1()
    print(f"config1 {time.time() - t0:.1f}s", flush=True)
    small["mcvqe"] = [mcvqe_case(8, 0, 1, 2), mcvqe_case(4, 7, 8, 11), mcvqe_case(3, 3, 4, 5)]
    print(f"mcvqe {time.time() - t0:.1f}s", flush=True)
    small["zero_angle_distribution"] = {
        "n": 2, "layers": 1,
        "distribution": born_distribution(run_gates(allocate(2), ddcl_circuit(
            DdclSpec(2, 1, (0.0,) * 12, {"00": 0.5, "11": 0.5})).gates))}
    (OUT / "golden_small.json").write_text(json.dumps(small))
    large = {"generator": "tests/golden/make_golden.py", "reference": str(REF), "qcl_forward": []}
    for n, layers, sh in ((4, 2, ()), (12, 2, ((0, "+"), (0, "-"), (143, "-"))),
                          (14, 3, ((0, "+"), (100, "-"), (251, "+"))), (16, 2, ((5, "+"), (191, "-"))),
                          (20, 6, ((0, "+"), (719, "-")))):
        large["qcl_forward"].append(qcl_forward(n, layers, shifted=sh))
        print(f"forward n={n} {time.time() - t0:.1f}s", flush=True)
    large["qcl_gradient"] = [qcl_gradient_case(14, 1, 5, 6), qcl_gradient_case(10, 2, 3, 4)]
    print(f"gradients {time.time() - t0:.1f}s", flush=True)
    (OUT / "golden_large.json").write_text(json.dumps(large))


if __name__ == "__main__":
    main()
