"""Short driver for ncu: a few forward QCL circuits at n qubits through the
public API, so every pass kernel launch is a full-size sweep.

    python tools/profile_pass.py [n] [layers] [circuits] [precision]
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2406_03466_b200 as qv  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    count = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    precision = sys.argv[4] if len(sys.argv) > 4 else "complex128"
    theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), 1)
    target = qv.random_target_distribution(n, 2)
    spec = qv.DdclSpec(n, layers, theta, target)
    batch = qv.ddcl_batch(spec)
    pick = [batch[2 * i * (len(batch) // (2 * count))] for i in range(count)]
    backend = qv.B200Backend(device=0, precision=precision)
    for _ in range(2):
        losses = backend.js_losses(pick, n, target)
    st = backend.last_stats
    print("losses", losses.tolist())
    print({k: round(v, 3) for k, v in st.items()})
    print(f"pass kernel {st['pass_bytes'] / st['pass_ms'] / 1e6:.1f} GB/s, {st['pass_flops'] / st['pass_ms'] / 1e9:.2f} TFLOP/s, "
          f"{st['pass_ms'] / max(st['sweeps'], 1):.3f} ms per sweep")


if __name__ == "__main__":
    main()
