"""Do two independent launches sharing each SM (one CTA each, separate
engines and streams) overlap better than one launch with two CTAs per SM?

    python tools/concurrent_probe.py [n] [layers] [circuits per engine]
Runs the same total work (2 x circuits forward JS losses at n qubits) as
(a) one engine, both batches back to back, and (b) two engines in two
threads with QVB200_CTAS_PER_SM=1 set by the caller for (b).
"""

import sys
import threading
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_2406_03466_b200 as qv  # noqa: E402
from paper_2406_03466_b200 import backend as bk, native  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    layers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    count = int(sys.argv[3]) if len(sys.argv) > 3 else 8
    mode = sys.argv[4] if len(sys.argv) > 4 else "one"
    target = qv.random_target_distribution(n, 2)
    tpl = qv.ddcl_circuit_template(n, layers)
    rng = np.random.default_rng(0)
    batches = [qv.bind_rows(tpl, rng.uniform(-3, 3, (count, len(tpl.params))), [f"b{j}c{i}" for i in range(count)])
               for j in range(2)]
    keys = sorted(target)
    sup = bk.support_indices(keys, n)
    p = np.asarray([target[k] for k in keys])
    budget = 60 << 30
    engines = [native.Engine(0, "complex128", budget) for _ in range(2 if mode == "two" else 1)]
    lowered = [bk.lower_batch(b) for b in batches]

    def run(e, lw):
        e.execute(n, lw, native.QV_OUT_JS, support=sup, target=p)

    for _ in range(2):   # warm-up + timed
        t0 = time.perf_counter()
        if mode == "one":
            for lw in lowered:
                run(engines[0], lw)
        else:
            ths = [threading.Thread(target=run, args=(engines[i], lowered[i])) for i in range(2)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
        dt = time.perf_counter() - t0
    print(f"{mode}: {2 * count} circuits of {n}q x {layers}L in {dt:.3f} s")


if __name__ == "__main__":
    main()
