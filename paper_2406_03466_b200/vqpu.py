"""Virtual-QPU pool: one batch split across parallel executors, mirroring the
reference's `qvirt.pool` (pkg/src/qvirt/pool.py:32-138) -- the paper's
HPCVirtDecorator.

`execute_parallel` keeps the reference contract exactly: contiguous blocks
(the first n mod v get one extra), a private backend per non-empty block from
a zero-argument factory, one thread per block, consolidation in global order,
abort-the-batch on any failure with the caller's buffer untouched.  With
`B200Backend` as the factory, blocks land round-robin on the visible GPUs
(vQPU b -> GPU b mod G) and the threads overlap because ctypes drops the GIL.

`execute_values` is the B200 fast path used by the gradient drivers: the same
partition and per-block backends, but each block returns one float64 per
circuit (an expectation value or a JS loss) instead of `ChildResult` objects.
Under torch.distributed (one process per GPU, NCCL over NVLink) block b runs
on rank b mod world_size, each rank executes its blocks as one batch on its
own GPU, and the per-circuit scalars are exchanged with a single padded
all-gather -- the MPI_Allgatherv of the paper's decorator.
"""

from __future__ import annotations

import contextlib
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from .backend import MODES, Accelerator, B200Backend, ExecutionConfig, ExecutionError
from .ir import Circuit
from .results import ChildResult, ResultBuffer, merge


@dataclass(frozen=True)
class VqpuPoolConfig:
    """Pool-level settings (reference pool.py:32-47)."""

    n_virtual_qpus: int = 1
    mode: str = "expectation"
    shots: int = 8192
    base_seed: int = 0

    def __post_init__(self) -> None:
        if self.n_virtual_qpus < 1:
            raise ValueError(f"n_virtual_qpus must be positive, got {self.n_virtual_qpus}")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.shots < 1:
            raise ValueError(f"shots must be positive, got {self.shots}")


@dataclass(frozen=True)
class Block:
    """Worker slice [start, end) of the batch."""

    vqpu_id: int
    start: int
    end: int

    @property
    def size(self) -> int:
        return self.end - self.start


def partition(n_circuits: int, n_vqpus: int) -> list[Block]:
    """Contiguous blocks whose sizes differ by at most one, larger first
    (reference pool.py:63-76)."""
    if n_circuits < 0:
        raise ValueError(f"n_circuits must be nonnegative, got {n_circuits}")
    if n_vqpus < 1:
        raise ValueError(f"n_vqpus must be positive, got {n_vqpus}")
    q, r = divmod(n_circuits, n_vqpus)
    bounds = [0]
    for v in range(n_vqpus):
        bounds.append(bounds[-1] + q + (v < r))
    return [Block(v, bounds[v], bounds[v + 1]) for v in range(n_vqpus)]


def consolidate(tagged_locals: Sequence[tuple[tuple[int, int], ResultBuffer]]) -> list[ChildResult]:
    """Children of per-worker buffers in global batch order (pool.py:79-85)."""
    if not tagged_locals:
        raise ValueError("nothing to consolidate")
    scratch = ResultBuffer(n_qubits=tagged_locals[0][1].n_qubits)
    merge(scratch, tagged_locals)
    return list(scratch.children)


def _validate_batch(circuits: Sequence[Circuit], n_qubits: int) -> None:
    """Up-front checks of pool.py:100-109."""
    if not circuits:
        raise ValueError("empty batch")
    names = [c.name for c in circuits]
    if len(set(names)) != len(names):
        raise ValueError("duplicate circuit names in batch")
    for c in circuits:
        if c.n_qubits != n_qubits:
            raise ValueError(f"circuit {c.name!r} has {c.n_qubits} qubits, buffer {n_qubits}")
        if c.is_parameterized:
            raise ValueError(f"circuit {c.name!r} has unbound parameters")


def _run_blocks(blocks, work):
    if len(blocks) == 1:
        return [work(blocks[0])]
    with ThreadPoolExecutor(max_workers=len(blocks)) as pool:
        futures = [pool.submit(work, b) for b in blocks]
        return [f.result() for f in futures]


def execute_parallel(buffer: ResultBuffer, circuits: Sequence[Circuit], config: VqpuPoolConfig,
                     backend_factory: Callable[[], Accelerator] = B200Backend) -> float:
    """Run a batch across the pool into `buffer`; returns the pool wall time
    (reference pool.py:88-138)."""
    _validate_batch(circuits, buffer.n_qubits)
    blocks = [b for b in partition(len(circuits), config.n_virtual_qpus) if b.size]

    def run_block(block: Block):
        backend = backend_factory()
        local = ResultBuffer(n_qubits=buffer.n_qubits)
        local.metadata["vqpu_id"] = block.vqpu_id
        cfg = ExecutionConfig(mode=config.mode, shots=config.shots, seed=config.base_seed,
                              first_global_index=block.start)
        backend.execute(local, circuits[block.start:block.end], cfg)
        return (block.start, block.end), local

    started = time.perf_counter()
    tagged = _run_blocks(blocks, run_block)
    elapsed = time.perf_counter() - started
    for child in consolidate(tagged):
        buffer.append_child(child)
    buffer.metadata["vqpu_count"] = config.n_virtual_qpus
    return elapsed


# ---------------------------------------------------------------------------
# B200 fast path: per-circuit scalars, optionally across torch.distributed ranks

_LOCAL = threading.local()


@contextlib.contextmanager
def rank_local():
    """Inside this block the scalar fast path ignores torch.distributed and
    runs every block on this process's GPU, with no collective.  For work a
    caller has already sharded across ranks (e.g. each rank owns its own data
    points): without it, every rank would hand the single block of its own
    batch to rank 0 and receive rank 0's values."""
    depth = getattr(_LOCAL, "depth", 0)
    _LOCAL.depth = depth + 1
    try:
        yield
    finally:
        _LOCAL.depth = depth


def _dist_context():
    if getattr(_LOCAL, "depth", 0):
        return None
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch is part of the image
        return None
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist
    return None


def rank_of_block(b: int, world: int) -> int:
    """Zigzag (boustrophedon) block -> rank map: 0,1,..,W-1,W-1,..,1,0,...
    Consecutive blocks of a shifted batch get steadily cheaper (later
    parameters branch off the shared trunk later), so plain round-robin would
    hand rank 0 the most expensive block of every round; zigzag cancels that
    gradient to first order."""
    r = b % (2 * world)
    return r if r < world else 2 * world - 1 - r


def execute_values(circuits: Sequence[Circuit], n_qubits: int, config: VqpuPoolConfig,
                   backend_factory: Callable[[], Accelerator], evaluate: Callable,
                   ) -> tuple[float, np.ndarray]:
    """Evaluate `evaluate(backend, block_circuits) -> float64[len(block)]` over
    the pool and return (pool wall seconds, values in batch order).

    Single process: one thread and backend per non-empty block (as
    `execute_parallel`).  Under torch.distributed with world size W > 1: block
    b belongs to rank `rank_of_block(b, W)`; each rank runs all of its blocks
    as one batch on its GPU, then one NCCL all-gather (gloo on CPU) shares the
    values.  Values are a function of each circuit alone, so every split gives
    bitwise-identical results.
    """
    _validate_batch(circuits, n_qubits)
    return execute_row_values(len(circuits), config, backend_factory,
                              lambda backend, rows: evaluate(backend, [circuits[i] for i in rows]))


def execute_row_values(n_rows: int, config: VqpuPoolConfig, backend_factory: Callable[[], Accelerator],
                       evaluate_rows: Callable) -> tuple[float, np.ndarray]:
    """`execute_values` over a batch known only by its row count: blocks,
    ranks and the all-gather are the same, `evaluate_rows(backend, rows)`
    gets the int64 row indices of its share (ascending).  Used when the batch
    is a parameter-shift table of one template, so no per-row `Circuit`
    objects are built (the template was validated when lowered)."""
    if n_rows < 1:
        raise ValueError("empty batch")
    if config.mode != "expectation":
        raise ValueError("the scalar fast path evaluates exact (expectation-mode) results")
    blocks = [b for b in partition(n_rows, config.n_virtual_qpus) if b.size]
    dist = _dist_context()
    started = time.perf_counter()
    if dist is None:
        def run_block(block: Block):
            backend = backend_factory()
            return evaluate_rows(backend, np.arange(block.start, block.end, dtype=np.int64))
        parts = _run_blocks(blocks, run_block)
        values = np.concatenate(parts) if parts else np.zeros(0)
        return time.perf_counter() - started, values

    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    owner = [rank_of_block(i, world) for i in range(len(blocks))]
    mine = [b for i, b in enumerate(blocks) if owner[i] == rank]
    index = np.concatenate([np.arange(b.start, b.end) for b in mine]) if mine else np.zeros(0, np.int64)
    local = np.zeros(0, np.float64)
    failure: BaseException | None = None
    if mine:
        try:
            backend = backend_factory()
            local = np.asarray(evaluate_rows(backend, index.astype(np.int64)), dtype=np.float64)
        except Exception as exc:   # reported to every rank through the gather below
            failure = exc
            local = np.zeros(0, np.float64)
    per_rank = [sum(b.size for i, b in enumerate(blocks) if owner[i] == r) for r in range(world)]
    width = max(per_rank)
    use_cuda = dist.get_backend() == "nccl"
    device = torch.device("cuda", torch.cuda.current_device()) if use_cuda else torch.device("cpu")
    # one extra slot per rank carries its status, so a rank whose blocks
    # failed still joins the collective and every rank aborts the batch
    # together (the reference aborts the whole batch, pool.py:96-98)
    send = torch.zeros(width + 1, dtype=torch.float64, device=device)
    if local.size:
        send[: local.size] = torch.from_numpy(local).to(device)
    send[width] = 1.0 if failure is not None else 0.0
    recv = torch.empty(world * (width + 1), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(recv, send)
    gathered = recv.cpu().numpy().reshape(world, width + 1)
    failed = [r for r in range(world) if gathered[r, width] != 0.0]
    if failure is not None:
        raise failure
    if failed:
        raise ExecutionError(f"rank {failed[0]}", f"a block on rank {failed[0]} failed; the batch is aborted")
    values = np.empty(n_rows, np.float64)
    for r in range(world):
        owned = [b for i, b in enumerate(blocks) if owner[i] == r]
        cursor = 0
        for b in owned:
            values[b.start:b.end] = gathered[r, cursor:cursor + b.size]
            cursor += b.size
    return time.perf_counter() - started, values
