"""Phase timeline of the two CTAs sharing an SM (blockIdx 0 and gridDim/2)
on the global timer (ns), from the QV_TRACE build.

    QVB200_TRACE_MIN_M0=97 python tools/trace_pair.py 28 8 2
"""

import os
import struct
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def main():
    args = sys.argv[1:] or ["28", "8", "2"]
    out = "/tmp/qv_trace.bin"
    lib = os.environ.get("QVB200_TRACE_LIB") or str(ROOT / "paper_2406_03466_b200" / "libqvb200_trace.so")
    env = dict(os.environ, QVB200_LIB=lib, QVB200_TRACE_OUT=out)
    subprocess.run([sys.executable, str(ROOT / "tools" / "profile_pass.py"), *args], env=env, check=True,
                   stdout=subprocess.DEVNULL)
    raw = Path(out).read_bytes()
    k, ng, nm, threads = struct.unpack("4i", raw[:16])
    tr = np.frombuffer(raw[16:], dtype=np.int64).reshape(8, 64, 16)
    sm_a, sm_b = tr[0, 63, 0], tr[0, 63, 8]
    print(f"k={k} groups={ng} mats={nm}; CTA 0 on SM {sm_a}, partner on SM {sm_b}")
    t0 = min(v for v in tr[:, 0, :].ravel() if v > 0)
    events = [(0, "start"), (1, "resident")] + [(3 + 2 * g, f"g{g}") for g in range(ng)] + [(62, "stored")]
    for cta, lo in (("A", 0), ("B", 8)):
        for item in range(8):
            cells = []
            for ev, name in events:
                v = tr[item, ev, lo:lo + 8]
                v = v[v > 0]
                if v.size:
                    cells.append(f"{name}:{(np.median(v) - t0) / 1000:.2f}")
            print(f"{cta} item {item}: " + "  ".join(cells) + "  (us)")


if __name__ == "__main__":
    main()
