"""CPU checks of the pass planner (no GPU).

libqvb200_plan.so interprets a plan exactly as the CUDA pass kernel does --
tile staging through the swizzled slot maps, 16-amplitude register groups,
CNOTs folded into GF(2) slot maps -- on the host.  Comparing it with the
oracle on random circuits, with tile sizes small enough to force many
passes, validates the planner's bookkeeping independently of the GPU.
"""

import ctypes

import numpy as np
import pytest

from oracle import statevector as sv
from paper_2406_03466_b200 import build as qbuild
from paper_2406_03466_b200.ir import CODE_BY_VALUE


@pytest.fixture(scope="module")
def plan_lib():
    path = qbuild.build_plancheck()
    lib = ctypes.CDLL(str(path))
    lib.qvp_simulate.restype = ctypes.c_int
    lib.qvp_simulate.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    lib.qvp_plan_stats.restype = ctypes.c_int
    lib.qvp_plan_stats.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
    return lib


def arrays(gates):
    kinds = np.array([CODE_BY_VALUE[k] for k, _, _ in gates] or [0], np.uint8)
    q0 = np.array([t[0] if t else 0 for _, t, _ in gates] or [0], np.int32)
    q1 = np.array([t[1] if len(t) > 1 else -1 for _, t, _ in gates] or [0], np.int32)
    ang = np.array([a if a is not None else 0.0 for _, _, a in gates] or [0.0], np.float64)
    return kinds, q0, q1, ang


def simulate(lib, n, gates, tile_bits, precision=0):
    kinds, q0, q1, ang = arrays(gates)
    out = np.zeros(2 << n, np.float64)
    passes = lib.qvp_simulate(n, len(gates), kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data,
                              ang.ctypes.data, precision, tile_bits, out.ctypes.data)
    assert passes > 0
    return out[0::2] + 1j * out[1::2], passes


def stats(lib, n, gates, tile_bits=0, precision=0):
    kinds, q0, q1, _ = arrays(gates)
    st = np.zeros(7, np.int64)
    pm = np.zeros(256, np.int32)
    assert lib.qvp_plan_stats(n, len(gates), kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data,
                              precision, tile_bits, st.ctypes.data, pm.ctypes.data, 256) == 0
    return st, pm[: st[0]]


@pytest.mark.parametrize("seed", range(24))
def test_random_circuits_match_oracle_across_tile_sizes(plan_lib, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    n = int(rng.integers(1, 11))
    gates = sv.random_circuit_gates(rng, n, int(rng.integers(0, 80)), extended=True)
    want = sv.run_gates(n, gates)
    for tile in (0, 5, 6, 8):
        for precision in (0, 1):
            if precision == 1 and tile == 5:
                continue   # complex64 needs >= 6 tile bits (4 coalescing + 2)
            got, _ = simulate(plan_lib, n, gates, tile, precision)
            assert np.max(np.abs(got - want)) < 1e-12, (tile, precision)


@pytest.mark.parametrize("n,layers,tile", [(8, 2, 5), (10, 2, 6), (12, 1, 7), (10, 3, 8)])
def test_ddcl_layers_multi_pass(plan_lib, n, layers, tile):
    tpl = sv.ddcl_template_gates(n, layers)
    theta = sv.random_angles(6 * n * layers, 7)
    gates = sv.bind_template(tpl, theta)
    got, passes = simulate(plan_lib, n, gates, tile)
    assert passes > 1
    assert np.max(np.abs(got - sv.run_gates(n, gates))) < 1e-12


@pytest.mark.parametrize("n,layers,precision", [(13, 2, 0), (14, 2, 1), (16, 1, 0), (15, 1, 1)])
def test_ddcl_production_tiles_and_warp_local_segments(plan_lib, n, layers, precision):
    """Production tile sizes (k = 12 for both precisions: 8 warps).  The interpreter
    returns -2 if a group without a CTA barrier makes any warp touch slots
    other than the ones it wrote in the previous group."""
    gates = sv.bind_template(sv.ddcl_template_gates(n, layers), sv.random_angles(6 * n * layers, n))
    got, passes = simulate(plan_lib, n, gates, 0, precision)
    assert passes > 1
    assert np.max(np.abs(got - sv.run_gates(n, gates))) < 1e-12
    st, _ = stats(plan_lib, n, gates, 0, precision)
    assert st[6] < st[1]   # some groups are warp-local


@pytest.mark.parametrize("seed", range(6))
def test_random_circuits_multi_warp_tiles(plan_lib, seed):
    rng = np.random.Generator(np.random.PCG64(100 + seed))
    n = 13 + seed % 2
    gates = sv.random_circuit_gates(rng, n, 120, extended=True)
    want = sv.run_gates(n, gates)
    for tile, precision in ((10, 0), (11, 1), (0, 0), (0, 1)):
        got, _ = simulate(plan_lib, n, gates, tile, precision)
        assert np.max(np.abs(got - want)) < 1e-12, (tile, precision)


def test_pass_counts_for_baseline_configs(plan_lib):
    """Regression guard on the planner: HBM sweeps per circuit."""
    expect_max = {(28, 8): 23, (20, 6): 11, (32, 4): 17}
    for (n, layers), cap in expect_max.items():
        gates = sv.bind_template(sv.ddcl_template_gates(n, layers), [0.1] * (6 * n * layers))
        precision = 1 if n == 32 else 0
        st, per_pass = stats(plan_lib, n, gates, 0, precision)
        assert st[5] == 0 and st[0] <= cap, (n, layers, st)
        assert per_pass.sum() == st[2]


def test_small_register_is_single_tile(plan_lib):
    gates = sv.bind_template(sv.ddcl_template_gates(4, 2), [0.3] * 48)
    st, _ = stats(plan_lib, 4, gates)
    assert st[5] == 1 and st[0] == 1 and st[4] == 4


def _simulate_cone(lib, n, gates, tile_bits, support, precision=0, tma=False):
    f = lib.qvp_simulate_cone_tma if tma else lib.qvp_simulate_cone
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 4 + [ctypes.c_int, ctypes.c_int,
                                                                            ctypes.c_void_p, ctypes.c_int64,
                                                                            ctypes.c_void_p, ctypes.c_void_p]
    kinds, q0, q1, ang = arrays(gates)
    sup = np.ascontiguousarray(support, dtype=np.uint64)
    out = np.zeros(sup.size, np.float64)
    visited = ctypes.c_int64(0)
    rc = f(n, len(gates), kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data, ang.ctypes.data, precision, tile_bits,
           sup.ctypes.data, sup.size, out.ctypes.data, ctypes.byref(visited))
    assert rc > 0
    return out, visited.value, rc


@pytest.mark.parametrize("seed", range(8))
def test_light_cone_restriction_reads_only_written_data(plan_lib, seed):
    """The product's light cone (csrc/plan.cpp light_cone / restrict_pass):
    each pass runs only on the tiles the support can see and zero-fills the
    slots of bits no earlier pass touched.  The interpreter starts from a
    NaN-filled state, so reading anything the restricted passes did not
    write would poison the support probabilities.  Random circuits (some
    qubits without gates), small tiles (many passes), scattered supports."""
    rng = np.random.Generator(np.random.PCG64(500 + seed))
    n = 12 + seed % 3
    idle = {int(q) for q in rng.choice(n, size=seed % 3, replace=False)}
    active = [q for q in range(n) if q not in idle]
    gates = [g for g in sv.random_circuit_gates(rng, n, 90, extended=True) if set(g[1]) <= set(active)]
    probs = np.abs(sv.run_gates(n, gates)) ** 2
    tile = (6, 7, 8)[seed % 3]
    supports = [np.arange(1 << 5, dtype=np.uint64),
                np.unique(rng.integers(0, 1 << n, 40).astype(np.uint64)),
                np.array([int(rng.integers(0, 1 << n))], np.uint64),
                np.array([0, (1 << n) - 1], np.uint64)]
    for sup in supports:
        for tma in (False, True):
            # tma: passes with a TMA layout load their whole box (fresh slots
            # included, NaN here) and zero the fresh registers on the first read
            got, visited, passes = _simulate_cone(plan_lib, n, gates, tile, sup, tma=tma)
            assert not np.any(np.isnan(got)), (sup, tma)
            assert np.max(np.abs(got - probs[sup.astype(np.int64)])) < 1e-12, (sup, tma)
    # the low-index support sweeps far fewer tiles than the full passes
    _, visited, passes = _simulate_cone(plan_lib, n, gates, tile, supports[0])
    assert visited < passes * (1 << (n - tile))


# ---------------------------------------------------------------------------
# TMA layouts (tma_pass.cuh): the interpreter loads and stores every pass with
# a TmaLayout through the TMA box layout computed from the layout's tensor
# dimensions (independently of the planner's slot columns; a mismatch returns
# -3), and the last register group writes in that layout.

@pytest.fixture(scope="module")
def tma_lib(plan_lib):
    for f in (plan_lib.qvp_simulate_tma, plan_lib.qvp_simulate_tma_direct):
        f.restype = ctypes.c_int
        f.argtypes = plan_lib.qvp_simulate.argtypes
    plan_lib.qvp_plan_tma.restype = ctypes.c_int
    plan_lib.qvp_plan_tma.argtypes = [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 3 + [
        ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int32]
    return plan_lib


def simulate_tma(lib, n, gates, tile_bits, precision=0, direct=False):
    """direct: the last register group stores straight to the state (the
    kernel's default); else through the TMA box layout and a TMA store."""
    kinds, q0, q1, ang = arrays(gates)
    out = np.zeros(2 << n, np.float64)
    fn = lib.qvp_simulate_tma_direct if direct else lib.qvp_simulate_tma
    passes = fn(n, len(gates), kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data,
                ang.ctypes.data, precision, tile_bits, out.ctypes.data)
    assert passes > 0, passes
    return out[0::2] + 1j * out[1::2]


def tma_layouts(lib, n, gates, tile_bits=0, precision=0):
    kinds, q0, q1, _ = arrays(gates)
    out = np.zeros(4 * 128, np.int64)
    passes = lib.qvp_plan_tma(n, len(gates), kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data, precision,
                              tile_bits, out.ctypes.data, 128)
    assert passes > 0
    return out[: 4 * passes].reshape(passes, 4)   # ok, ndim, wavefronts, groups


@pytest.mark.parametrize("seed", range(16))
def test_tma_layouts_match_oracle(tma_lib, seed):
    rng = np.random.Generator(np.random.PCG64(100 + seed))
    n = int(rng.integers(7, 12))
    gates = sv.random_circuit_gates(rng, n, int(rng.integers(1, 120)), extended=True)
    want = sv.run_gates(n, gates)
    for tile, precision in ((5, 0), (6, 0), (8, 0), (7, 1), (8, 1)):
        for direct in (False, True):
            got = simulate_tma(tma_lib, n, gates, tile, precision, direct)
            assert np.max(np.abs(got - want)) < 1e-12, (tile, precision, direct)


@pytest.mark.parametrize("n,layers,precision", [(28, 8, 0), (20, 6, 0), (32, 4, 1)])
def test_qcl_passes_have_tma_layouts(tma_lib, n, layers, precision):
    """Every pass of the benchmark circuits gets a <= 4-index-dimension TMA
    layout (plus the state dimension: rank <= 5)."""
    gates = sv.bind_template(sv.ddcl_template_gates(n, layers), [0.1] * (6 * n * layers))
    lay = tma_layouts(tma_lib, n, gates, 0, precision)
    assert (lay[:, 0] == 1).all()
    assert (lay[:, 1] >= 2).all() and (lay[:, 1] <= 4).all()


def test_tma_ddcl_multi_pass(tma_lib):
    tpl = sv.ddcl_template_gates(12, 3)
    gates = sv.bind_template(tpl, sv.random_angles(6 * 12 * 3, 9))
    for direct in (False, True):
        got = simulate_tma(tma_lib, 12, gates, 8, direct=direct)
        assert np.max(np.abs(got - sv.run_gates(12, gates))) < 1e-12
