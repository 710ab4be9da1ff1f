"""A/B of the TMA pass kernel against pass_kernel on one QCL gradient.

    python tools/ab_tma.py n layers precision [tag]        (QVB200_TMA=0 disables TMA)

Prints one JSON line (gradient seconds, pass-kernel device ms, launch counts,
a checksum of the gradient) and writes the gradient to gpurun_out/ab_<tag>.npy
so two runs can be compared bit for bit: store-only passes do the same
arithmetic on either kernel, so the gradients must be identical.
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2406_03466_b200 as qv  # noqa: E402
from paper_2406_03466_b200 import native  # noqa: E402


def main():
    n, layers = int(sys.argv[1]), int(sys.argv[2])
    precision = sys.argv[3] if len(sys.argv) > 3 else "complex128"
    tag = sys.argv[4] if len(sys.argv) > 4 else f"{n}x{layers}_{precision}_tma{os.environ.get('QVB200_TMA', '1')}"
    reps = int(os.environ.get("AB_REPS", "2"))
    spec = qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 1),
                       qv.random_target_distribution(n, 2))
    factory = lambda: qv.B200Backend(device=0, precision=precision)  # noqa: E731
    eng = native.engine(0, precision)
    qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=1), backend_factory=factory)   # warm-up
    best = None
    for _ in range(reps):
        before = dict(eng.total_stats)
        t0 = time.perf_counter()
        rep = qv.ddcl_gradient(spec, qv.VqpuPoolConfig(n_virtual_qpus=1), backend_factory=factory)
        dt = time.perf_counter() - t0
        st = {k: eng.total_stats[k] - before[k] for k in native.STAT_NAMES}
        if best is None or dt < best[0]:
            best = (dt, st)
    g = np.array(rep.gradient)
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    np.save(out / f"ab_{tag}.npy", g)
    dt, st = best
    print(json.dumps({"tag": tag, "n": n, "layers": layers, "precision": precision, "seconds": round(dt, 4),
                      "pass_ms": round(st["pass_ms"], 2), "device_ms": round(st["device_ms"], 2),
                      "launches": st["launches"], "tma_launches": st["tma_launches"],
                      "hbm_frac": st["pass_bytes"] / (st["pass_ms"] * 1e-3) / 6539.9e9 if st["pass_ms"] else None,
                      "checksum": float(np.sum(g * np.arange(1, len(g) + 1)))}), flush=True)


if __name__ == "__main__":
    main()
