"""Where a small workload's end-to-end time goes (GPU box): per call of the
native executor, host wall ms of the whole call, host ms before its first
kernel, device ms, and the Python time around it.

    python tools/host_overhead.py qcl4|qcl20|mcvqe8|qcl20fwd [reps]
"""

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2406_03466_b200 as qv  # noqa: E402
from paper_2406_03466_b200 import native  # noqa: E402


def main():
    what = sys.argv[1]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    eng = native.engine(0, "complex128")
    if what == "qcl4":
        spec = qv.DdclSpec(4, 2, qv.random_angles(qv.ddcl_parameter_count(4, 2), 1), qv.random_target_distribution(4, 2))
        run = lambda: qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=1))  # noqa: E731
    elif what == "qcl20":
        spec = qv.DdclSpec(20, 6, qv.random_angles(qv.ddcl_parameter_count(20, 6), 1),
                           qv.random_target_distribution(20, 2))
        run = lambda: qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=1))  # noqa: E731
    elif what == "mcvqe8":
        ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(8, 0))
        ms = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(8, 1), qv.random_angles(qv.mcvqe_parameter_count(8), 2))
        run = lambda: qv.mcvqe_gradient(ham, ms, qv.VqpuPoolConfig(n_virtual_qpus=1))  # noqa: E731
    else:
        specs = [qv.DdclSpec(20, 6, qv.random_angles(qv.ddcl_parameter_count(20, 6), 1 + i),
                             qv.random_target_distribution(20, 2 + i)) for i in range(1024)]
        b = qv.B200Backend()
        run = lambda: qv.ddcl_forward_losses(specs, b)  # noqa: E731
    for _ in range(3):
        run()
    rows = []
    for _ in range(reps):
        before = dict(eng.total_stats)
        t0 = time.perf_counter()
        run()
        wall = (time.perf_counter() - t0) * 1e3
        d = {k: eng.total_stats[k] - before[k] for k in ("host_ms", "host_prep_ms", "device_ms")}
        d["wall_ms"] = wall
        rows.append(d)
    med = {k: float(np.median([r[k] for r in rows])) for k in rows[0]}
    print(json.dumps({"workload": what, **med}))


if __name__ == "__main__":
    main()
