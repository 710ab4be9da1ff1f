"""Print the planner's pass/group structure for the BASELINE QCL configs (CPU)."""

import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import statevector as sv  # noqa: E402
from paper_2406_03466_b200 import build  # noqa: E402
from paper_2406_03466_b200.ir import CODE_BY_VALUE  # noqa: E402


def main():
    lib = ctypes.CDLL(str(build.build_plancheck()))
    lib.qvp_plan_stats.restype = ctypes.c_int
    lib.qvp_plan_stats.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 3 + [
        ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
    configs = [(28, 8, 0), (26, 2, 0), (20, 6, 0), (32, 4, 1)]
    for n, layers, prec in configs:
        gates = sv.bind_template(sv.ddcl_template_gates(n, layers), [0.1] * (6 * n * layers))
        kinds = np.array([CODE_BY_VALUE[k] for k, _, _ in gates], np.uint8)
        q0 = np.array([t[0] for _, t, _ in gates], np.int32)
        q1 = np.array([t[1] if len(t) > 1 else -1 for _, t, _ in gates], np.int32)
        st = np.zeros(7, np.int64)
        pm = np.zeros(128, np.int32)
        rc = lib.qvp_plan_stats(n, len(gates), kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data, prec, 0,
                                st.ctypes.data, pm.ctypes.data, 128)
        assert rc == 0
        print(f"n={n} L={layers} prec={prec}: passes={st[0]} groups={st[1]} cta_barriers={st[6]} mats={st[2]} "
              f"fill={st[2] / (4 * st[1]):.2f} per-pass mats={pm[:st[0]].tolist()}")


if __name__ == "__main__":
    main()
