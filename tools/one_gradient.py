"""One full parameter-shift gradient of a BASELINE QCL config through the
public API (for launch lists under ncu).

    python tools/one_gradient.py [n] [layers] [precision]
"""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2406_03466_b200 as qv  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    precision = sys.argv[3] if len(sys.argv) > 3 else "complex128"
    spec = qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 1),
                       qv.random_target_distribution(n, 2))
    factory = lambda: qv.B200Backend(device=0, precision=precision)  # noqa: E731
    t0 = time.perf_counter()
    report = qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=1), backend_factory=factory)
    print(f"gradient of {len(report.gradient)} parameters in {time.perf_counter() - t0:.2f} s")


if __name__ == "__main__":
    main()
