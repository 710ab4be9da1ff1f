"""Multi-process path of the virtual-QPU pool on CPU (torch.distributed,
gloo, world size 2): block b runs on rank `rank_of_block(b, W)` (zigzag), per-circuit scalars are
exchanged with one padded all-gather, every rank ends with the full vector
in batch order.  A stub backend stands in for the GPU (the exchange logic is
what is under test; the B200 path runs the same code with NCCL)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2406_03466_b200 as qv


class StubBackend:
    """Deterministic per-circuit value: a function of the circuit alone."""

    executed: list = []

    def values(self, block):
        return np.array([float(c.name[1:]) * 1.5 + 0.25 for c in block])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_circuits, n_vqpus, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch = [qv.Circuit(2, (qv.h(0),), name=f"c{i}") for i in range(n_circuits)]
        seen = []

        def evaluate(backend, block):
            seen.extend(c.name for c in block)
            return backend.values(block)

        _, values = qv.execute_values(batch, 2, qv.VqpuPoolConfig(n_virtual_qpus=n_vqpus), StubBackend, evaluate)
        out[rank] = (values.tolist(), seen)
    finally:
        dist.destroy_process_group()


def test_zigzag_block_owner():
    assert [qv.vqpu.rank_of_block(b, 4) for b in range(10)] == [0, 1, 2, 3, 3, 2, 1, 0, 0, 1]
    assert [qv.vqpu.rank_of_block(b, 1) for b in range(3)] == [0, 0, 0]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_bench_blocks_keep_shift_pairs_whole(world):
    """bench.py's QCL pool (one vQPU per parameter) on the 28q x 8L shift
    table (2688 rows, rows 2k / 2k+1 = the +/- pair of parameter k): every
    block is one whole pair and every rank gets the same number of rows."""
    n_theta = qv.ddcl_parameter_count(28, 8)
    rows = 2 * n_theta
    blocks = [b for b in qv.partition(rows, n_theta) if b.size]
    assert all(b.start % 2 == 0 and b.size % 2 == 0 for b in blocks)
    per_rank = [sum(b.size for i, b in enumerate(blocks) if qv.vqpu.rank_of_block(i, world) == r)
                for r in range(world)]
    assert per_rank == [rows // world] * world


@pytest.mark.parametrize("n_circuits,n_vqpus", [(10, 4), (7, 16), (2688, 16), (5, 1)])
def test_execute_values_two_ranks(n_circuits, n_vqpus):
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(2, _free_port(), n_circuits, n_vqpus, out), nprocs=2, join=True)
    want = [i * 1.5 + 0.25 for i in range(n_circuits)]
    blocks = [b for b in qv.partition(n_circuits, n_vqpus) if b.size]
    for rank in range(2):
        values, seen = out[rank]
        assert values == want
        mine = [f"c{i}" for j, b in enumerate(blocks) if qv.vqpu.rank_of_block(j, 2) == rank
                for i in range(b.start, b.end)]
        assert seen == mine


def _row_worker(rank, world, port, n_rows, n_vqpus, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seen = []

        def evaluate_rows(backend, rows):
            seen.extend(int(r) for r in rows)
            return rows * 1.5 + 0.25

        _, values = qv.execute_row_values(n_rows, qv.VqpuPoolConfig(n_virtual_qpus=n_vqpus), StubBackend,
                                          evaluate_rows)
        out[rank] = (values.tolist(), seen)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_rows,n_vqpus", [(2688, 16), (9, 4)])
def test_execute_row_values_two_ranks(n_rows, n_vqpus):
    """The shift-table path of ddcl_gradient (rows, no Circuit objects): same
    blocks, zigzag ownership and all-gather as execute_values."""
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_row_worker, args=(2, _free_port(), n_rows, n_vqpus, out), nprocs=2, join=True)
    want = [i * 1.5 + 0.25 for i in range(n_rows)]
    blocks = [b for b in qv.partition(n_rows, n_vqpus) if b.size]
    for rank in range(2):
        values, seen = out[rank]
        assert values == want
        assert seen == [i for j, b in enumerate(blocks) if qv.vqpu.rank_of_block(j, 2) == rank
                        for i in range(b.start, b.end)]


def test_execute_row_values_single_process():
    _, values = qv.execute_row_values(10, qv.VqpuPoolConfig(n_virtual_qpus=3), StubBackend,
                                      lambda backend, rows: rows * 2.0)
    assert values.tolist() == [2.0 * i for i in range(10)]
    with pytest.raises(ValueError):
        qv.execute_row_values(0, qv.VqpuPoolConfig(), StubBackend, lambda b, r: r)


def _local_worker(rank, world, port, out):
    """Ranks with DIFFERENT batches inside vqpu.rank_local(): each runs its own
    rows on its own device, no collective (bench.py's per-rank data points)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_rows = 5 + 2 * rank
        with qv.vqpu.rank_local():
            _, values = qv.execute_row_values(n_rows, qv.VqpuPoolConfig(n_virtual_qpus=1), StubBackend,
                                              lambda backend, rows: rows * 1.5 + rank)
        # outside the block the collective path is back
        _, shared = qv.execute_row_values(4, qv.VqpuPoolConfig(n_virtual_qpus=2), StubBackend,
                                          lambda backend, rows: rows * 1.0)
        out[rank] = (values.tolist(), shared.tolist())
    finally:
        dist.destroy_process_group()


def test_rank_local_rows_per_rank():
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_local_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for rank in range(2):
        values, shared = out[rank]
        assert values == [i * 1.5 + rank for i in range(5 + 2 * rank)]
        assert shared == [0.0, 1.0, 2.0, 3.0]


def _failing_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def evaluate_rows(backend, rows):
            if rank == 1:
                raise ValueError("device fault on rank 1")
            return rows * 1.0

        try:
            qv.execute_row_values(8, qv.VqpuPoolConfig(n_virtual_qpus=2), StubBackend, evaluate_rows)
            out[rank] = "no error"
        except qv.ExecutionError as exc:
            out[rank] = f"ExecutionError: {exc}"
        except ValueError as exc:
            out[rank] = f"ValueError: {exc}"
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_failure_on_one_rank_aborts_every_rank():
    """A rank whose blocks raise still joins the all-gather (status slot), so
    its peers do not hang in the collective: every rank aborts the batch."""
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_failing_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[1] == "ValueError: device fault on rank 1"
    assert out[0].startswith("ExecutionError") and "rank 1" in out[0]
