"""Per-phase timeline of one persistent CTA of the pass kernel (debug build).

    python tools/trace_pass.py [n] [layers] [circuits]        # on a GPU box
Runs tools/profile_pass.py against libqvb200_trace.so and prints, for the
first 8 work items of CTA 0, the cycles each warp spends per phase.
"""

import os
import struct
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def main():
    args = sys.argv[1:] or ["26", "2", "2"]
    out = "/tmp/qv_trace.bin"
    lib = os.environ.get("QVB200_TRACE_LIB") or str(ROOT / "paper_2406_03466_b200" / "libqvb200_trace.so")
    env = dict(os.environ, QVB200_LIB=lib,
               QVB200_TRACE_OUT=out)
    subprocess.run([sys.executable, str(ROOT / "tools" / "profile_pass.py"), *args], env=env, check=True)
    raw = Path(out).read_bytes()
    k, ng, nm, threads = struct.unpack("4i", raw[:16])
    tr = np.frombuffer(raw[16:], dtype=np.int64).reshape(8, 64, 16)
    warps = min(16, threads // 32)
    print(f"k={k} groups={ng} mats={nm} threads={threads} nonzero={np.count_nonzero(tr)}")
    for item in range(8):
        starts = tr[item, 0, :warps]
        starts = starts[starts > 0]
        if not starts.size:
            continue
        t0 = starts[starts > 0].min()
        rows = [("start", 0), ("resident", 1)]
        for g in range(min(ng, 29)):
            rows += [(f"g{g} math", 2 + 2 * g), (f"g{g} sync", 3 + 2 * g)]
        rows.append(("stored", 62))
        line = []
        prev = t0
        for name, ev in rows:
            v = tr[item, ev, :warps]
            v = v[v > 0]   # the ring kernel's items run on half the warps
            if not v.size:
                continue
            line.append(f"{name}:{int(np.median(v) - t0)}[{int(v.min() - t0)},{int(v.max() - t0)}]")
        nxt = tr[item + 1, 0, :warps] if item + 1 < 8 else None
        gap = f"  next item +{int(nxt[nxt > 0].min() - t0)}" if nxt is not None and nxt.any() else ""
        print(f"item {item}: " + "  ".join(line) + gap)


if __name__ == "__main__":
    main()
