"""Shared-memory bank behaviour of a plan's register groups (CPU).

For every group and register index j, the 32 lanes of warp 0 access slots
base(lane) ^ combo[j] (16-byte complex128 / 8-byte complex64 amplitudes).
A 128-bit access needs at least 4 wavefronts (8 lanes x 16 B per 128-byte
bank row); lanes that hit the same 16-byte bank quad at different addresses
serialise.  Prints the wavefront count against the ideal per pass.

    python tools/bank_check.py [n] [layers] [precision 0|1]
"""

import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import statevector as sv  # noqa: E402
from paper_2406_03466_b200 import build  # noqa: E402
from paper_2406_03466_b200.ir import CODE_BY_VALUE  # noqa: E402

GROUP = np.dtype([("combo", "<u4", 16), ("tcol", "<u4", 11), ("cta_sync", "<i4"), ("mat", "<i4", 4)])
PASS = np.dtype({"names": ["k", "n_outer", "g0", "ng", "m0", "nm"], "formats": ["<i4"] * 6,
                 "offsets": [0, 4, 8, 12, 16, 20], "itemsize": 352})


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    prec = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    lib = ctypes.CDLL(str(build.build_plancheck()))
    f = lib.qvp_plan_descriptors
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                                                            ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32,
                                                                            ctypes.c_void_p]
    gates = sv.bind_template(sv.ddcl_template_gates(n, layers), [0.1] * (6 * n * layers))
    kinds = np.array([CODE_BY_VALUE[k] for k, _, _ in gates], np.uint8)
    q0 = np.array([t[0] for _, t, _ in gates], np.int32)
    q1 = np.array([t[1] if len(t) > 1 else -1 for _, t, _ in gates], np.int32)
    groups = np.zeros(4096, GROUP)
    passes = np.zeros(256, PASS)
    npass = ctypes.c_int32(0)
    ng = f(n, len(gates), kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data, prec, 0, groups.ctypes.data, 4096,
           passes.ctypes.data, 256, ctypes.byref(npass))
    amp = 16 if prec == 0 else 8
    lanes = np.arange(32)
    total = ideal = 0
    for p in range(npass.value):
        pd = passes[p]
        wf = 0
        for g in range(pd["g0"], pd["g0"] + pd["ng"]):
            G = groups[g]
            base = np.zeros(32, np.uint32)
            for m in range(5):
                base ^= np.where((lanes >> m) & 1, G["tcol"][m], 0).astype(np.uint32)
            for j in range(16):
                slots = (base ^ G["combo"][j]) // amp
                quads = (slots * amp // 16) % 8 if amp == 16 else (slots * amp // 8) % 32
                per = np.bincount(quads, minlength=8 if amp == 16 else 32)
                wf += 2 * int(per.max() if amp == 16 else max(1, per.max()))   # load + store
        ideal_p = pd["ng"] * 16 * 2 * (4 if amp == 16 else 2)
        total += wf
        ideal += ideal_p
        print(f"pass {p:2d}: groups {pd['ng']:2d} mats {pd['nm']:2d}  wavefronts {wf:5d} ideal {ideal_p:5d}  x{wf / ideal_p:.2f}")
    print(f"total x{total / ideal:.3f}")


if __name__ == "__main__":
    main()
