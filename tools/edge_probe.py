"""Edge-case sweep of the executor against the dense oracle (GPU box):
tiny and tile-boundary registers, empty circuits, extreme support indices,
every output kind.  Prints one line per case: ok / MISMATCH / ERROR."""

import sys
import traceback
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2406_03466_b200 as qv  # noqa: E402
from oracle import statevector as sv  # noqa: E402


def oracle_amps(c):
    return sv.run_gates(c.n_qubits, sv.gate_tuples(c))


def case(name, fn):
    try:
        msg = fn()
        print(f"{name}: {msg or 'ok'}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name}: ERROR {e!r}", flush=True)
        traceback.print_exc(limit=2)


def main():
    b = qv.B200Backend(device=0)
    rng = np.random.Generator(np.random.PCG64(5))

    def rand_circuit(n, ng, seed):
        r = np.random.Generator(np.random.PCG64(seed))
        gates = []
        for _ in range(ng):
            k = r.integers(0, 5)
            q = int(r.integers(0, n))
            if k == 0:
                gates.append(qv.h(q))
            elif k == 1:
                gates.append(qv.ry(q, float(r.uniform(-3, 3))))
            elif k == 2:
                gates.append(qv.rz(q, float(r.uniform(-3, 3))))
            elif n > 1:
                t = int(r.integers(0, n - 1))
                t = t if t < q else t + 1
                gates.append(qv.cnot(q, t))
        return qv.Circuit(n, tuple(gates), name=f"r{seed}")

    for n in (1, 2, 3, 11, 12, 13, 16):
        for ng in (0, 1, 40):
            c = rand_circuit(n, ng, 100 * n + ng)
            amps = oracle_amps(c)
            probs = np.abs(amps) ** 2

            def sup_case(c=c, n=n, probs=probs):
                dim = 1 << n
                sup = sorted({0, dim - 1, dim // 2, (dim - 1) // 3})
                got = b.support_probabilities([c], n, sup)[0]
                err = np.max(np.abs(got - probs[sup]))
                return None if err < 1e-12 else f"MISMATCH {err:.2e}"
            case(f"support n={n} gates={ng}", sup_case)

            def js_case(c=c, n=n, probs=probs):
                dim = 1 << n
                keys = [format(i, f"0{n}b") for i in sorted({0, dim - 1})]
                tgt = {k: 1.0 / len(keys) for k in keys}
                got = b.js_losses([c], n, tgt)[0]
                ref = sv.js_divergence(tgt, {format(i, f"0{n}b"): float(p) for i, p in enumerate(probs) if p > 0})
                return None if abs(got - ref) < 1e-12 else f"MISMATCH {got} {ref}"
            case(f"js n={n} gates={ng}", js_case)

            def pauli_case(c=c, n=n, amps=amps):
                fac = {0: "Z"} if n == 1 else {0: "X", n - 1: "Y"}
                obs = qv.Observable((qv.pauli(fac, 0.5),), 0.25)
                got = b.expectation_values([c.with_observable(obs)], n)[0]
                ref = sv.expectation(amps, n, [(sorted(fac.items()), 0.5)], 0.25)
                return None if abs(got - ref) < 1e-12 else f"MISMATCH {got} {ref}"
            case(f"pauli n={n} gates={ng}", pauli_case)

    # batches mixing topologies, duplicates and an empty circuit
    def mixed():
        n = 14
        cs = [rand_circuit(n, 30, 7), rand_circuit(n, 0, 8), rand_circuit(n, 30, 7), rand_circuit(n, 55, 9)]
        sup = [0, 5, (1 << n) - 1]
        got = b.support_probabilities(cs, n, sup)
        for i, c in enumerate(cs):
            p = np.abs(oracle_amps(c)) ** 2
            if np.max(np.abs(got[i] - p[sup])) > 1e-12:
                return f"MISMATCH circuit {i}"
    case("mixed batch n=14", mixed)


if __name__ == "__main__":
    main()
