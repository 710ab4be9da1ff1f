"""Benchmark: parameter-shift gradient of a QCL (DDCL) circuit on B200.

Metric (BASELINE.json): circuit evals/sec & full-gradient time at 1/2/4/8
B200, by qubits x layers.  Default workload = config 4, the north star's:
QCL 28 qubits x 8 layers, complex128, one step = one full parameter-shift
gradient (2 * 6nL = 2688 circuits), strong scaling over GPUs.

    python bench.py [--gpus N --steps K --warmup W] [--workload qcl28|qcl20|qcl20fwd|qcl20b|qcl32|qcl4|mcvqe8]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the reference CPU implementation

Timing: W untimed steps, then K steps between barrier + device synchronise,
CUDA events on the launching streams, max over ranks.  `value` is the device
busy span of the executor (first to last kernel of each step: inputs already
resident); `e2e` times the public call `ddcl_gradient(...)` end to end (host
lowering, H2D of the fused matrices, D2H of the losses) with CUDA events.
States (4 GiB at 28 qubits) are far larger than L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "circuit evals/sec & full-gradient time at 1/2/4/8 B200, by qubits x layers"
UNIT = "circuit evals/s"

WORKLOADS = {
    # name: (kind, n, layers, precision, description)
    "qcl28": ("qcl", 28, 8, "complex128", "config 4: QCL 28 qubits x 8 layers full parameter-shift gradient, complex128"),
    "qcl20": ("qcl", 20, 6, "complex128", "config 3: QCL 20 qubits x 6 layers full gradient for one data point, complex128"),
    "qcl20fwd": ("qcl_fwd", 20, 6, "complex128",
                 "config 3: QCL 20 qubits x 6 layers forward losses of a batch of 1024 data points (one circuit each)"),
    "qcl20b": ("qcl_batch", 20, 6, "complex128",
               "config 3: QCL 20 qubits x 6 layers full gradients of all 1024 data points (1,474,560 circuits)"),
    "qcl32": ("qcl", 32, 4, "complex64", "config 5: QCL 32 qubits x 4 layers full gradient, complex64"),
    "qcl4": ("qcl", 4, 2, "complex128", "config 1: QCL 4 qubits x 2 layers gradient (one data point)"),
    # the paper's own DDCL strong-scaling workloads (Table 2/3: L = 10)
    "ddcl20l10": ("qcl", 20, 10, "complex128", "paper Table 3: DDCL 20 qubits x 10 layers full gradient (2400 circuits)"),
    "ddcl26l10": ("qcl", 26, 10, "complex128", "paper Table 3: DDCL 26 qubits x 10 layers full gradient (3120 circuits)"),
    "mcvqe8": ("mcvqe", 8, 0, "complex128", "config 2: MC-VQE 8-chromophore parameter-shift gradient"),
    "mcvqe16": ("mcvqe", 16, 0, "complex128", "MC-VQE 16-chromophore parameter-shift gradient (paper Table 1 size)"),
    # the literal drop-in: the UNMODIFIED reference driver (baseline/_ref
    # qvirt.ddcl_gradient -> shifted_circuits -> execute_parallel) calling
    # B200Backend.execute on every shifted circuit -- its own circuit objects,
    # no shift pairs; host time of the reference driver is inside the step
    "qcl28dropin": ("qcl_dropin", 28, 8, "complex128",
                    "config 4 through the unmodified reference ddcl_gradient with B200Backend as backend_factory"),
    "qcl20dropin": ("qcl_dropin", 20, 6, "complex128",
                    "config 3 (one point) through the unmodified reference ddcl_gradient with B200Backend"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="qcl28")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-f", self.path], stdout=subprocess.DEVNULL,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        try:
            lines = Path(self.path).read_text().splitlines()
        except Exception:
            lines = []
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9 or not parts[0].isdigit() or int(parts[0]) not in self.gpus:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baselines

def _reference_module():
    """The unmodified reference (`qvirt`) installed under baseline/_ref."""
    ref = ROOT / "baseline" / "_ref"
    os.environ.setdefault("NUMBA_CACHE_DIR", str(Path(tempfile.gettempdir()) / "numba-qvirt"))
    if (ref / "qvirt").exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import qvirt  # noqa: F401
    from qvirt import backend as qb
    return qvirt, qb


REFERENCE_MAX_QUBITS = 30   # qvirt.backend.MAX_QUBITS (backend.py:31)


class NotRunnable(RuntimeError):
    """The reference cannot run this configuration at all."""


def cpu_sample_rate(kind, n, layers, threads, budget_s=12.0, seed=0):
    """Time the reference CPU implementation on a bounded sample of the
    workload, all `threads` host threads busy; returns (evals/s, sample text,
    implementation kind).  QCL at n >= 20: each thread applies the first gates
    of its own shifted circuit with the reference's numba kernels
    (`run_gates`, backend.py:88-91) until the budget is spent, and the
    measured gate-sweep rate is converted to circuits (gates per circuit
    G = n + L(7n-1)).  The exact-mode distribution dict the reference builds
    afterwards (infeasible at 28 qubits) is not charged -- generous to the CPU."""
    try:
        qvirt, qb = _reference_module()
        impl = "reference"
    except Exception:
        qvirt = qb = None
        impl = "port"
    from concurrent.futures import ThreadPoolExecutor
    import numpy as np

    if kind == "mcvqe" or (kind == "qcl" and n <= 12):
        # small registers: the reference's own pool over the full gradient
        if impl == "reference":
            def one():
                if kind == "mcvqe":
                    ham = qvirt.aiem_hamiltonian(qvirt.random_aiem_coefficients(n, seed))
                    spec = qvirt.McvqeAnsatzSpec(qvirt.random_cis_amplitudes(n, seed + 1),
                                                 qvirt.random_angles(qvirt.mcvqe_parameter_count(n), seed + 2))
                    rep = qvirt.mcvqe_gradient(ham, spec, qvirt.VqpuPoolConfig(n_virtual_qpus=1))
                else:
                    spec = qvirt.DdclSpec(n, layers, qvirt.random_angles(qvirt.ddcl_parameter_count(n, layers), seed + 1),
                                          qvirt.random_target_distribution(n, seed + 2))
                    rep = qvirt.ddcl_gradient(spec, qvirt.VqpuPoolConfig(n_virtual_qpus=1))
                return rep.n_circuit_executions
            one()   # JIT warm-up
            t0 = time.perf_counter()
            done = 0
            while time.perf_counter() - t0 < budget_s / 2:
                done += one()
            dt = time.perf_counter() - t0
            return done / dt, f"reference {kind} gradients through its pool (1 vQPU; more vQPUs anti-scale on the GIL)", impl, 1
        from oracle import statevector as sv
        t0 = time.perf_counter()
        done = 0
        while time.perf_counter() - t0 < budget_s / 2:
            if kind == "mcvqe":
                done += len(sv.mcvqe_values(n, seed, seed + 1, seed + 2)[0])
            else:
                theta = sv.random_angles(6 * n * layers, seed + 1)
                done += len(sv.ddcl_losses(n, layers, theta, sv.random_target_distribution(n, seed + 2)))
        return done / (time.perf_counter() - t0), f"numpy oracle port, {kind} gradients", impl, 1

    gates_per_circuit = n + layers * (7 * n - 1)
    if impl == "reference" and n > REFERENCE_MAX_QUBITS:
        raise NotRunnable(f"not runnable by the reference: n = {n} > {REFERENCE_MAX_QUBITS} "
                          "(allocate() guard, backend.py:31)")
    if impl == "reference":
        template = qvirt.ddcl_circuit_template(n, layers)
        theta = qvirt.random_angles(qvirt.ddcl_parameter_count(n, layers), seed + 1)
        circuit = qvirt.bind(template, theta)
        gates = circuit.gates
        qb.run_gates(qb.allocate(4), qvirt.ddcl_circuit_template(4, 1).gates[:4])   # JIT warm-up

        def worker(_):
            st = qb.allocate(n)
            t0 = time.perf_counter()
            count = 0
            while time.perf_counter() - t0 < budget_s:   # repeat the circuit until the budget is spent
                for g in gates:
                    qb.apply(st, g)
                    count += 1
                    if time.perf_counter() - t0 > budget_s:
                        break
            return count, time.perf_counter() - t0
    else:
        from oracle import statevector as sv
        tpl = sv.bind_template(sv.ddcl_template_gates(n, layers), sv.random_angles(6 * n * layers, seed + 1))

        def worker(_):
            amps = sv.zero_state(n)
            t0 = time.perf_counter()
            count = 0
            while time.perf_counter() - t0 < budget_s:
                for kind_, t, a in tpl:
                    sv.apply_gate(amps, n, kind_, t, a)
                    count += 1
                    if time.perf_counter() - t0 > budget_s:
                        break
            return count, time.perf_counter() - t0

    with ThreadPoolExecutor(max_workers=threads) as pool:
        res = list(pool.map(worker, range(threads)))
    sweeps = sum(c for c, _ in res)
    wall = max(t for _, t in res)
    rate = sweeps / wall / gates_per_circuit
    sample = (f"{threads} threads x one {n}-qubit state each, {sweeps} gate sweeps of a shifted "
              f"{n}q x {layers}L circuit in {wall:.1f} s, / {gates_per_circuit} gates per circuit")
    return rate, sample, impl, threads


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_threads_for(n):
    """Threads for the 28q+ CPU sample: one 2^n state per thread must fit in RAM."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 32 << 30
    per = 16 << n
    return max(1, min(host_threads(), int(avail * 0.5 // per)))


def run_reference(args):
    """--impl reference: the reference CPU implementation on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    kind, n, layers, precision, desc = WORKLOADS[args.workload]
    kind = "qcl" if kind.startswith("qcl") else kind   # same circuits, same per-circuit CPU cost
    threads = cpu_threads_for(n) if n > 12 else 1
    if n > REFERENCE_MAX_QUBITS:
        print(json.dumps({"impl": "reference", "unavailable": f"the reference rejects n = {n} > "
                          f"{REFERENCE_MAX_QUBITS} qubits (backend.py:31); config 5 is not runnable by it"}),
              flush=True)
        return
    for _ in range(args.warmup):
        cpu_sample_rate(kind, n, layers, threads, budget_s=4.0, seed=args.seed)
    rates, samples = [], []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rate, sample, impl, used = cpu_sample_rate(kind, n, layers, threads, budget_s=10.0, seed=args.seed)
        rates.append(rate)
        samples.append(sample)
    wall = time.perf_counter() - t0
    value = statistics.median(rates)
    circuits = circuits_per_step(kind, n, layers)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1000 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic (seeded PCG64 angles/targets, reference generators)",
        "config": {"workload": desc, "qubits": n, "layers": layers, "circuits_per_gradient": circuits,
                   "full_gradient_s_extrapolated": circuits / value},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": impl, "sample": samples[-1]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


POINTS = 1024   # config 3's batch of data points
BLOCKS_PER_RANK = 24   # vQPU blocks per GPU under torchrun, non-QCL workloads (see main)

# the paper's published strong-scaling fits (Table 3,
# PAPER.md:303-325), log10(seconds) = a * log2(GPUs) + b, V100 + cuStateVec,
# sampled counts mode -- the only published numbers for this path.
PAPER_FITS = {(20, 10): (-0.132, 2.622), (22, 10): (-0.137, 2.726), (24, 10): (-0.159, 2.958),
              (26, 10): (-0.204, 3.398)}


def paper_rate(n, layers, gpus):
    """Circuit evals/s of the paper's fit at this GPU count, or None."""
    fit = PAPER_FITS.get((n, layers))
    if fit is None:
        return None
    seconds = 10 ** (fit[0] * math.log2(gpus) + fit[1])
    return 12 * n * layers / seconds


def circuits_per_step(kind, n, layers):
    if kind == "mcvqe":
        return 2 * (6 * n - 4) * (5 * n - 4)
    if kind == "qcl_fwd":
        return POINTS
    if kind == "qcl_batch":
        return POINTS * 12 * n * layers
    return 12 * n * layers


class _Step:
    """Result of one multi-point step: circuits evaluated and a checksum vector."""

    def __init__(self, circuits, values):
        self.n_circuit_executions = circuits
        self.gradient = values


# ---------------------------------------------------------------------------

def fp64_peak_tflops(torch):
    """Measured FP64 ceiling on this GPU: cuBLAS DGEMM 8192^3 (2 N^3 flops),
    best of 5 -- the FP64 analogue of MEASURED_PEAKS.json's bf16 GEMM."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    best = math.inf
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * 8192 ** 3 / (best / 1e3) / 1e12


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    device = torch.cuda.current_device()

    import paper_2406_03466_b200 as qv
    from paper_2406_03466_b200 import native
    from paper_2406_03466_b200.vqpu import rank_local

    kind, n, layers, precision, desc = WORKLOADS[args.workload]
    s = args.seed
    if kind == "qcl_dropin":
        if world > 1:
            raise SystemExit("the reference driver's pool is single-process; run the drop-in leg with --gpus 1")
        qvirt = _reference_package()
        theta = qvirt.random_angles(qvirt.ddcl_parameter_count(n, layers), s + 1)
        target = qvirt.random_target_distribution(n, s + 2)
        ref_spec = qvirt.DdclSpec(n, layers, theta, target)
        ref_pool = qvirt.VqpuPoolConfig(n_virtual_qpus=1, mode="expectation")

        def step():
            return qvirt.ddcl_gradient(ref_spec, ref_pool,
                                       backend_factory=lambda: qv.B200Backend(device=device, precision=precision,
                                                                              support=target))
    elif kind == "qcl":
        theta = qv.random_angles(qv.ddcl_parameter_count(n, layers), s + 1)
        target = qv.random_target_distribution(n, s + 2)
        spec = qv.DdclSpec(n, layers, theta, target)
        def step():
            return qv.ddcl_gradient(spec, pool, backend_factory=_Factory(device, precision))
    elif kind in ("qcl_fwd", "qcl_batch"):
        # data point i: theta seed s+1+i, target seed s+2+i; points
        # are dealt to ranks round-robin, each rank runs its share on its GPU
        mine = range(rank, POINTS, world)
        specs = [qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), s + 1 + i),
                             qv.random_target_distribution(n, s + 2 + i)) for i in mine]
        fwd_backend = qv.B200Backend(device=device, precision=precision)
        one_pool = qv.VqpuPoolConfig(n_virtual_qpus=1)

        def step():
            if kind == "qcl_fwd":
                return _Step(POINTS, qv.ddcl_forward_losses(specs, fwd_backend))
            # the points are already dealt to ranks: each rank's gradients run
            # on its own GPU with no collective (vqpu.rank_local)
            with rank_local():
                grads = [qv.ddcl_gradient(sp, one_pool, backend_factory=_Factory(device, precision)).gradient
                         for sp in specs]
            return _Step(circuits_per_step(kind, n, layers), np.concatenate(grads))
    else:
        ham = qv.aiem_hamiltonian(qv.random_aiem_coefficients(n, s))
        mspec = qv.McvqeAnsatzSpec(qv.random_cis_amplitudes(n, s + 1), qv.random_angles(qv.mcvqe_parameter_count(n), s + 2))

        def step():
            return qv.mcvqe_gradient(ham, mspec, pool, backend_factory=_Factory(device, precision))

    # vQPU blocks dealt to ranks in zigzag order (vqpu.rank_of_block) so every
    # rank gets parameters from every depth; each rank runs its blocks as one
    # batch sharing one trunk.  QCL gradients: one vQPU per parameter (its ±
    # shift pair), the finest split that never cuts a pair -- tools/shard_probe.py,
    # 28q x 8L split 8 ways: max shard 4.62 s, vs 4.72 s with 24 blocks per rank
    # and 4.99 s with 8.  Other workloads: BLOCKS_PER_RANK blocks per rank.
    if world == 1:
        n_vqpus = 1
    elif kind == "qcl":
        n_vqpus = qv.ddcl_parameter_count(n, layers)
    else:
        n_vqpus = BLOCKS_PER_RANK * world
    pool = qv.VqpuPoolConfig(n_virtual_qpus=n_vqpus)
    engine = native.engine(device, precision)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[device])
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 0)):
        step()
    barrier()
    keys = ("device_ms", "pass_ms", "pass_bytes", "pass_flops", "launches", "sweeps", "sweeps_unshared",
            "h2d_bytes", "d2h_bytes", "tma_ms", "tma_bytes", "tma_launches")

    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    dev_ms = pass_ms = pass_bytes = pass_flops = launches = sweeps = unshared = h2d = d2h = 0.0
    tma_ms = tma_bytes = tma_launches = 0.0
    passes = tile = 0
    reports = []
    with ClockSampler(list(range(max(world, 1)))) as clocks:
        barrier()
        ev0.record()
        for _ in range(args.steps):
            before = dict(engine.total_stats)
            rep = step()
            st = {k: engine.total_stats[k] - before[k] for k in keys}   # every engine call of the step
            dev_ms += st["device_ms"]
            pass_ms += st["pass_ms"]
            pass_bytes += st["pass_bytes"]
            pass_flops += st["pass_flops"]
            launches += st["launches"]
            sweeps += st["sweeps"]
            unshared += st["sweeps_unshared"]
            h2d += st["h2d_bytes"]
            d2h += st["d2h_bytes"]
            tma_ms += st["tma_ms"]
            tma_bytes += st["tma_bytes"]
            tma_launches += st["tma_launches"]
            passes, tile = engine.total_stats["passes_per_circuit"], engine.total_stats["tile_bits"]
            reports.append(rep)
        ev1.record()
        barrier()
    e2e_ms = ev0.elapsed_time(ev1)

    agg = torch.tensor([e2e_ms, dev_ms, pass_ms, launches, pass_bytes, pass_flops, sweeps, unshared], dtype=torch.float64,
                       device="cuda")
    if world > 1:
        mx = agg.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = agg.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
    else:
        mx = sm = agg
    e2e_ms_max, dev_ms_max = float(mx[0]), float(mx[1])
    circuits = reports[-1].n_circuit_executions   # whole job (every rank's points)
    steps = args.steps
    value = circuits * steps / (dev_ms_max / 1e3)
    e2e_value = circuits * steps / (e2e_ms_max / 1e3)

    # roofline of the dominant kernel on this rank, from live CUDA events on
    # the engine stream: tma_pass_kernel when it ran (the store passes of
    # multi-tile states), else pass_kernel; all pass launches beside it
    hbm_peak = _measured_peaks().get("hbm_gbs", 6650.0)
    all_achieved = pass_bytes / (pass_ms / 1e3) / 1e9 if pass_ms else 0.0
    dominant = "tma_pass_kernel" if tma_ms > 0.5 * pass_ms else "pass_kernel"
    achieved = tma_bytes / (tma_ms / 1e3) / 1e9 if dominant == "tma_pass_kernel" else all_achieved
    fp_rate = pass_flops / (pass_ms / 1e3) / 1e12 if pass_ms else 0.0   # counted: 28 flop per amplitude pair
    fp64_peak = fp64_peak_tflops(torch) if (rank == 0 and precision == "complex128") else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads_for(n) if n > 12 else 1
        try:
            rate, sample, impl, used = cpu_sample_rate("qcl" if kind.startswith("qcl") else kind, n, layers,
                                                       threads, budget_s=12.0, seed=s)
            cpu = {"value": rate, "unit": UNIT, "cores": used, "kind": impl, "sample": sample}
        except NotRunnable as why:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": str(why)}

    if rank == 0:
        grad = np.asarray(reports[-1].gradient)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": dev_ms_max / steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": (value / paper_rate(n, layers, world)) if (kind == "qcl" and paper_rate(n, layers, world))
            else None,
            "dtype": "c128 (f64)" if precision == "complex128" else "c64 (f32, f64 reductions)",
            "data": "synthetic (seeded PCG64: theta seed s+1, target seed s+2, reference generators)",
            "config": {
                "workload": desc, "qubits": n, "layers": layers, "precision": precision,
                "circuits_per_step": circuits,
                "step": {"qcl_fwd": f"forward JS losses of {POINTS} data points",
                         "qcl_batch": f"full parameter-shift gradients of {POINTS} data points"}.get(
                             kind, "one full parameter-shift gradient"),
                "full_gradient_s": e2e_ms_max / steps / 1e3,
                "full_gradient_device_s": dev_ms_max / steps / 1e3,
                "parallelism": f"vqpu{pool.n_virtual_qpus}->gpu{world} (zigzag blocks), NCCL all-gather of losses",
                "shift_mode": "none (forward pass)" if kind == "qcl_fwd" else
                "direct (the reference driver's 2N shifted Circuit objects through B200Backend.execute; "
                "children carry support + remainder distributions)" if kind == "qcl_dropin" else
                "pair (psi+- = (Psi0 -+ i Xi_k)/sqrt2: one extra state per parameter)"
                if kind.startswith("qcl") and n > 12 else "direct",
                "passes_per_circuit": passes, "tile_bits": tile,
                "hbm_sweeps_per_step": float(sm[6]) / steps, "hbm_sweeps_without_prefix_sharing": float(sm[7]) / steps,
                "l2": "states (2^n x 16 B) far exceed the 126 MB L2; no flush needed",
                "gradient_checksum": float(np.sum(grad)), "seed": s,
                **({"vs_baseline_source": "paper Table 3 fit at this GPU count (V100 + cuStateVec, sampled "
                                          "counts mode; BASELINE.md section 1); this run is exact mode"}
                   if kind == "qcl" and paper_rate(n, layers, world) else {}),
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak if hbm_peak else None, **_ncu_traffic(dominant),
                         "kernel": dominant, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)",
                         "kernel_share_of_pass_time": (tma_ms / pass_ms) if (pass_ms and dominant == "tma_pass_kernel")
                         else 1.0,
                         "kernel_launches": int(tma_launches) if dominant == "tma_pass_kernel" else None,
                         "all_passes_achieved": all_achieved,
                         "all_passes_frac": all_achieved / hbm_peak if hbm_peak else None,
                         "bytes_rule": "per state-pass: read + write of the swept tiles; a chain's first pass reads "
                                       "the shared trunk once for the whole launch; a pair pass reads Xi and Psi0",
                         "fp64_achieved_tflops": fp_rate, "fp64_executed_tflops": fp_rate * 24.0 / 28.0,
                         "fp64_flop_rule": "counted 28 flop per amplitude pair per fused 2x2 matrix (complex 2x2 "
                                           "matvec); executed 24 (4 DMUL + 10 DFMA: m00 made real by the host)",
                         "fp64_peak_tflops": fp64_peak,
                         "fp64_peak_source": "cuBLAS DGEMM 8192^3 measured in this run" if fp64_peak else None},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d / steps,
                    "d2h_bytes_per_step": d2h / steps,
                    "api": {"qcl": "paper_2406_03466_b200.ddcl_gradient(spec, VqpuPoolConfig, B200Backend)",
                            "qcl_fwd": "paper_2406_03466_b200.ddcl_forward_losses(specs, B200Backend)",
                            "qcl_batch": "paper_2406_03466_b200.ddcl_gradient per data point",
                            "qcl_dropin": "unmodified reference qvirt.ddcl_gradient(spec, VqpuPoolConfig, "
                                          "backend_factory=lambda: B200Backend(support=target))"}.get(
                                kind, "paper_2406_03466_b200.mcvqe_gradient(...)")},
            "gpu_launches": int(float(sm[3])),
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class _Factory:
    """Zero-argument backend factory pinned to this rank's device.  A class
    (not a lambda) so the gradient drivers recognise a B200 factory and take
    the device-side loss path."""

    def __init__(self, device, precision):
        self.device = device
        self.precision = precision

    def __call__(self):
        import paper_2406_03466_b200 as qv
        return qv.B200Backend(device=self.device, precision=self.precision)


def _ncu_traffic(kernel="tma_pass_kernel"):
    """DRAM bytes of one launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_<kernel>.json: production launches of
    the bench's own gradient), beside that launch's algorithmic bytes; null
    if the capture is absent."""
    name = {"tma_pass_kernel": "ncu_tma_pass_kernel.json"}.get(kernel, "ncu_pass_kernel.json")
    try:
        prof = json.loads((ROOT / "profiles" / name).read_text())
        launch = prof["launches"][0]
        return {"traffic": launch["traffic_bytes"], "traffic_algorithmic_bytes": launch["algorithmic_bytes"],
                "traffic_launch": launch["what"], "traffic_source": f"profiles/{name}"}
    except Exception:
        return {"traffic": None}


def _reference_package():
    """The unmodified reference (`qvirt`) installed in baseline/_ref."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "qvirt").exists():
        raise SystemExit("baseline/_ref is not installed (see DESIGN.md section 7)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba-qvirt")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import qvirt
    return qvirt


def _measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


if __name__ == "__main__":
    main()
