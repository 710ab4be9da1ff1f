"""Per-rank shard times of the W-rank split of one full gradient, measured
on ONE GPU (for the strong-scaling target at a rank count the box does not
offer).

    python tools/shard_probe.py [world=8] [ranks=0..W-1] [n=28] [layers=8] [blocks_per_rank=8]

Each listed rank's share (the same blocks `vqpu.execute_row_values` hands
that rank under torch.distributed: `blocks_per_rank` vQPU blocks per rank,
zigzag order) is
evaluated on cuda:0 through the public `ddcl_gradient`, with a stand-in
process group whose all-gather only fills the rank's own row (the gathered
gradient is therefore partial -- only the time is used).  The W-GPU step time
is the max over ranks of the shard times plus the all-gather of W x width
doubles (microseconds over NVLink).  Prints one JSON line per rank and a
summary line.
"""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2406_03466_b200 as qv  # noqa: E402
from paper_2406_03466_b200 import native, vqpu  # noqa: E402


class _ShardGroup:
    """torch.distributed stand-in: rank r of W, all-gather fills row r only."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world

    def get_rank(self):
        return self.rank

    def get_world_size(self):
        return self.world

    def get_backend(self):
        return "nccl"

    def all_gather_into_tensor(self, recv, send):
        recv.zero_()
        recv[self.rank * send.numel():(self.rank + 1) * send.numel()] = send


def main():
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    ranks = [int(r) for r in sys.argv[2].split(",")] if len(sys.argv) > 2 and sys.argv[2] else list(range(world))
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 28
    layers = int(sys.argv[4]) if len(sys.argv) > 4 else 8
    per = int(sys.argv[5]) if len(sys.argv) > 5 else 8
    torch.cuda.set_device(0)
    spec = qv.DdclSpec(n, layers, qv.random_angles(qv.ddcl_parameter_count(n, layers), 1),
                       qv.random_target_distribution(n, 2))
    factory = lambda: qv.B200Backend(device=0)  # noqa: E731
    engine = native.engine(0, "complex128")
    pool = qv.VqpuPoolConfig(n_virtual_qpus=per * world)
    real = vqpu._dist_context
    times = {}
    try:
        for r in ranks:
            vqpu._dist_context = lambda r=r: _ShardGroup(r, world)
            qv.ddcl_gradient(spec, pool, backend_factory=factory)   # warm-up (planner, buffers)
            torch.cuda.synchronize()
            before = engine.total_stats["device_ms"]
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            qv.ddcl_gradient(spec, pool, backend_factory=factory)
            ev1.record()
            torch.cuda.synchronize()
            times[r] = ev0.elapsed_time(ev1) / 1e3
            print(json.dumps({"rank": r, "world": world, "blocks_per_rank": per, "shard_s": times[r],
                              "device_s": (engine.total_stats["device_ms"] - before) / 1e3}), flush=True)
    finally:
        vqpu._dist_context = real
    print(json.dumps({"world": world, "blocks_per_rank": per, "qubits": n, "layers": layers, "ranks": sorted(times),
                      "max_shard_s": max(times.values()), "min_shard_s": min(times.values()),
                      "sum_shard_s": sum(times.values())}), flush=True)


if __name__ == "__main__":
    main()
