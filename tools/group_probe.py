"""Compute-only probe of the register-group math: batches of 12-qubit random
rotation circuits run entirely in shared memory (single tile, no HBM state
traffic), so the pass kernel's FP64 rate is the group math's rate.

    python tools/group_probe.py [circuits] [layers] [precision]
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2406_03466_b200 as qv  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    precision = sys.argv[3] if len(sys.argv) > 3 else "complex128"
    n = 12
    spec = qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 1),
                       qv.random_target_distribution(n, 2))
    batch = qv.ddcl_batch(spec)[:count]
    backend = qv.B200Backend(device=0, precision=precision)
    for _ in range(2):
        backend.js_losses(batch, n, spec.target)
    st = backend.last_stats
    print(f"{precision} n={n} L={layers} circuits={len(batch)}: {st['pass_flops'] / st['pass_ms'] / 1e9:.2f} TFLOP/s "
          f"in {st['pass_ms']:.2f} ms")


if __name__ == "__main__":
    main()
