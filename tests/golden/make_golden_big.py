"""Golden vectors at benchmark sizes, produced by the REFERENCE's own kernels.

Configs 3, 4 and 5 of BASELINE.json are too large for the reference's
exact-mode `born_distribution` (a 2^n-entry Python dict), but not for its
state-vector kernels: this script runs the reference's `allocate` /
`run_gates` (backend.py:57-91, numba kernels.py:18-70, nogil so threads
overlap) and `kernels.born_probabilities` (kernels.py:90-94), normalises by
`probs.sum()` exactly like `_probabilities` (backend.py:122-129), and takes
the JS loss (ddcl.py:37-61) in the support + remainder form: the target's
support is the first 2^10 indices (ddcl.py:147-157), which sort before every
off-support key, and each off-support key b contributes ½ q_b ln 2.  The
identity was checked against the dict form at n = 4 / 12 / 14 (SURVEY §8a
A20, |Δ| ≤ 2.3e-15).  Gradient entries are ½(L+ − L−) over circuits bound
by the reference's own `shifted_circuits` (gradients.py:33-46).

Run in the build container (the reference is read-only there; this writes
only tests/golden/golden_big_<case>.json):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_golden_big.py qcl28   # config 4, ~7 x 4 GiB
    ... qcl30c5    # config 5 geometry at the reference's 30-qubit cap
    ... qcl20      # config 3: gradient entries + batch points
    ... mcvqe16    # MC-VQE at 16 chromophores, every circuit's expectation

Nothing on the GPU box reads /root/reference; tests read the JSON.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("QVIRT_REFERENCE", "/root/reference/pkg"))
sys.path[:0] = [str(REF / "src")]
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba-golden")

from qvirt import (  # noqa: E402
    DdclSpec, ddcl_circuit, ddcl_circuit_template, ddcl_parameter_count, random_angles,
    random_target_distribution,
)
from qvirt import kernels  # noqa: E402
from qvirt.backend import allocate, run_gates  # noqa: E402
from qvirt.gradients import shifted_circuits  # noqa: E402

OUT = Path(__file__).resolve().parent
LN2 = math.log(2.0)


def loss_of(n, gates, target_w):
    """Run one circuit with the reference kernels; return the JS loss and
    the normalised support probabilities (support = indices [0, len(w)))."""
    state = run_gates(allocate(n), gates)
    amps = state.amplitudes
    s = len(target_w)
    chunk = 1 << 24
    if amps.shape[0] <= chunk:
        probs = np.empty(amps.shape[0], dtype=np.float64)
        kernels.born_probabilities(amps, probs)
        total = probs.sum()
        supp, off = probs[:s].copy(), probs[s:].sum()
    else:
        # Chunked so a 30-qubit run does not need a second 8 GiB array; the
        # per-amplitude values are the kernel's, only the sum's association
        # differs from probs.sum() (relative 1e-16).
        probs = np.empty(chunk, dtype=np.float64)
        total = off = 0.0
        for lo in range(0, amps.shape[0], chunk):
            kernels.born_probabilities(amps[lo:lo + chunk], probs)
            if lo == 0:
                supp = probs[:s].copy()
                off += probs[s:].sum()
            else:
                off += probs.sum()
            total += probs.sum()
    del state, amps, probs
    q_supp = supp / total
    q_off = off / total
    acc = 0.0
    for pb, qb in zip(target_w.tolist(), q_supp.tolist()):
        m = 0.5 * (pb + qb)
        if pb > 0.0:
            acc += 0.5 * pb * math.log(pb / m)
        if qb > 0.0:
            acc += 0.5 * qb * math.log(qb / m)
    acc += 0.5 * LN2 * float(q_off)
    return acc, q_supp.tolist(), float(total)


def qcl_case(n, layers, theta_seed, target_seed, ks, threads, keep_probs=True, forward=True):
    count = ddcl_parameter_count(n, layers)
    theta = random_angles(count, theta_seed)
    target = random_target_distribution(n, target_seed)
    w = np.array([target[k] for k in sorted(target)], dtype=np.float64)
    template = ddcl_circuit_template(n, layers)
    jobs = []
    if forward:
        jobs.append(("fwd", ddcl_circuit(DdclSpec(n, layers, theta, target)).gates))
    wanted = set(ks)
    for k, tag, bound in shifted_circuits(template, theta):
        if k in wanted:
            jobs.append((f"k{k}{tag}", bound.gates))
    t0 = time.time()

    def run(job):
        name, gates = job
        js, q, total = loss_of(n, gates, w)
        print(f"  {name}: js={js!r} ({time.time() - t0:.0f}s)", flush=True)
        return name, js, q, total

    with ThreadPoolExecutor(threads) as ex:
        res = {name: (js, q, total) for name, js, q, total in ex.map(run, jobs)}
    case = {"n": n, "layers": layers, "theta_seed": theta_seed, "target_seed": target_seed,
            "ks": list(ks), "losses": {name: v[0] for name, v in res.items()},
            "norms": {name: v[2] for name, v in res.items()},
            "gradient": {str(k): 0.5 * (res[f"k{k}+"][0] - res[f"k{k}-"][0]) for k in ks}}
    if forward:
        case["js"] = res["fwd"][0]
        if keep_probs:
            case["support_probs"] = res["fwd"][1]
    if keep_probs:
        case["support_probs_shifted"] = {name: v[1] for name, v in res.items() if name != "fwd"}
    return case


def main():
    which = sys.argv[1]
    t0 = time.time()
    meta = {"generator": "tests/golden/make_golden_big.py", "reference": str(REF)}
    if which == "qcl28":
        # config 4: 28q x 8L, theta seed 1, target seed 2; k = first, middle, last.
        out = dict(meta, qcl=qcl_case(28, 8, 1, 2, (0, 671, 1343), threads=7))
    elif which == "qcl30c5":
        # config 5's geometry (4 layers) at the reference's 30-qubit cap
        # (backend.py:31); the complex64 GPU path is checked against it.
        out = dict(meta, qcl=qcl_case(30, 4, 1, 2, (0,), threads=3))
    elif which == "qcl28c5":
        out = dict(meta, qcl=qcl_case(28, 4, 1, 2, (0, 335, 671), threads=7))
    elif which == "mcvqe16":
        # MC-VQE at 16 chromophores (the paper's Table-1 sizes): every
        # shifted circuit's expectation (one coefficient-1 AIEM term each,
        # mcvqe.py:194-247) through the reference's own pool and kernels.
        from qvirt import (McvqeAnsatzSpec, ResultBuffer, VqpuPoolConfig, aiem_hamiltonian, mcvqe_energy,
                           mcvqe_gradient, mcvqe_parameter_count, random_aiem_coefficients,
                           random_cis_amplitudes)
        n = 16
        ham = aiem_hamiltonian(random_aiem_coefficients(n, 0))
        spec = McvqeAnsatzSpec(random_cis_amplitudes(n, 1), random_angles(mcvqe_parameter_count(n), 2))
        buf = ResultBuffer(n_qubits=n)
        rep = mcvqe_gradient(ham, spec, VqpuPoolConfig(n_virtual_qpus=4), buffer=buf)
        out = dict(meta, mcvqe={"n": n, "coeff_seed": 0, "cis_seed": 1, "theta_seed": 2,
                                "gradient": list(rep.gradient), "energy": mcvqe_energy(ham, spec),
                                "n_circuits": rep.n_circuit_executions,
                                "values": [c.expectation for c in buf.children]})
    elif which == "qcl20":
        # config 3: 20q x 6L gradient entries at 10 parameters (theta seed 1,
        # target seed 2 = batch point 0) and the forward JS of batch points
        # i in {0, 511, 1023} (theta seed 1+i, target seed 2+i).
        ks = (0, 1, 2, 59, 119, 240, 359, 480, 600, 719)
        grad = qcl_case(20, 6, 1, 2, ks, threads=8, keep_probs=False)
        points = []
        for i in (0, 511, 1023):
            c = qcl_case(20, 6, 1 + i, 2 + i, (), threads=1, keep_probs=False)
            points.append({"point": i, "theta_seed": 1 + i, "target_seed": 2 + i, "js": c["js"]})
        out = dict(meta, qcl=grad, points=points)
    else:
        raise SystemExit(f"unknown case {which!r}")
    out["seconds"] = round(time.time() - t0, 1)
    (OUT / f"golden_big_{which}.json").write_text(json.dumps(out))
    print(f"wrote golden_big_{which}.json in {out['seconds']}s", flush=True)


if __name__ == "__main__":
    main()
