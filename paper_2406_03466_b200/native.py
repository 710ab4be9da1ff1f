"""ctypes binding of libqvb200.so (include/qvb200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, `engine()` raises `NativeUnavailable` and the backend
fails loudly.  ctypes releases the GIL for the duration of every call, so
per-thread backends (one per virtual QPU) overlap on the host.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np

import os

# QVB200_LIB selects an alternative build (e.g. the clock64-traced debug
# library used by tools/tma_trace.py, or the diagnostic builds of
# build.build_variant); the default is the product library.
LIB_PATH = Path(os.environ.get("QVB200_LIB") or Path(__file__).resolve().parent / "libqvb200.so")

QV_OK, QV_ERR_ARGUMENT, QV_ERR_CIRCUIT, QV_ERR_CUDA, QV_ERR_INTERNAL = range(5)
QV_COMPLEX128, QV_COMPLEX64 = 0, 1
QV_OUT_PAULI, QV_OUT_SUPPORT, QV_OUT_FULL, QV_OUT_JS, QV_OUT_COUNTS = range(5)
QV_RES_TARGET_ROWS = 1

PRECISIONS = {"complex128": QV_COMPLEX128, "complex64": QV_COMPLEX64}

# Symbols include/qvb200.h declares (checked by the CPU test suite).
EXPORTS = ("qv_version", "qv_output_size", "qv_create", "qv_destroy", "qv_execute", "qv_shift_js",
           "qv_last_error", "qv_last_error_circuit", "qv_last_stats", "qv_device_count")

STAT_NAMES = ("launches", "sweeps", "sweeps_unshared", "unique_states", "pass_bytes",
              "pass_ms", "passes_per_circuit", "tile_bits", "device_ms", "h2d_bytes", "d2h_bytes",
              "pass_flops", "tma_launches", "pauli_state_reads", "tma_ms", "tma_bytes", "host_ms", "host_prep_ms")


class NativeUnavailable(RuntimeError):
    """libqvb200.so could not be loaded or no B200 is visible."""


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str, circuit: int):
        super().__init__(message)
        self.code = code
        self.circuit = circuit


class QvCircuits(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("n_circuits", ctypes.c_int32), ("uniform", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("n_gates", ctypes.c_int64),
                ("gate_offsets", ctypes.c_void_p), ("kinds", ctypes.c_void_p), ("q0", ctypes.c_void_p),
                ("q1", ctypes.c_void_p), ("angles", ctypes.c_void_p)]


class QvResults(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("flags", ctypes.c_int32), ("term_offsets", ctypes.c_void_p),
                ("xmask", ctypes.c_void_p), ("ymask", ctypes.c_void_p), ("zmask", ctypes.c_void_p),
                ("support_count", ctypes.c_int64), ("support", ctypes.c_void_p), ("target", ctypes.c_void_p),
                ("shots", ctypes.c_int64), ("rng_state", ctypes.c_void_p)]


_lib = None
_lib_lock = threading.Lock()


def load_library() -> ctypes.CDLL:
    global _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeUnavailable(f"{LIB_PATH} is missing; run __graft_entry__.build()")
            lib = ctypes.CDLL(str(LIB_PATH))
            lib.qv_version.restype = ctypes.c_char_p
            lib.qv_output_size.restype = ctypes.c_int64
            lib.qv_output_size.argtypes = [ctypes.POINTER(QvCircuits), ctypes.POINTER(QvResults)]
            lib.qv_create.restype = ctypes.c_int
            lib.qv_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
            lib.qv_destroy.restype = ctypes.c_int
            lib.qv_destroy.argtypes = [ctypes.c_void_p]
            lib.qv_execute.restype = ctypes.c_int
            lib.qv_execute.argtypes = [ctypes.c_void_p, ctypes.POINTER(QvCircuits), ctypes.POINTER(QvResults),
                                       ctypes.c_void_p, ctypes.c_int64]
            lib.qv_last_error.restype = ctypes.c_char_p
            lib.qv_last_error.argtypes = [ctypes.c_void_p]
            lib.qv_last_error_circuit.restype = ctypes.c_int64
            lib.qv_last_error_circuit.argtypes = [ctypes.c_void_p]
            lib.qv_last_stats.restype = ctypes.c_int
            lib.qv_last_stats.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
            lib.qv_device_count.restype = ctypes.c_int
            lib.qv_device_count.argtypes = []
            lib.qv_shift_js.restype = ctypes.c_int
            lib.qv_shift_js.argtypes = [ctypes.c_void_p, ctypes.POINTER(QvCircuits), ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.POINTER(QvResults), ctypes.c_void_p]
            _lib = lib
        return _lib


def _ptr(a: np.ndarray | None) -> int | None:
    return None if a is None else a.ctypes.data


class Engine:
    """One native executor (a qv_handle) on one device and precision."""

    def __init__(self, device: int, precision: str = "complex128", memory_budget: int = 0):
        lib = load_library()
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {tuple(PRECISIONS)}")
        handle = ctypes.c_void_p()
        code = lib.qv_create(int(device), PRECISIONS[precision], int(memory_budget), ctypes.byref(handle))
        if code != QV_OK:
            raise NativeUnavailable(f"qv_create(device={device}) failed with status {code} (no CUDA device?)")
        self._lib = lib
        self._handle = handle
        self.device = int(device)
        self.precision = precision
        self.last_stats: dict[str, float] = {}
        # running sums over every call (per-call values for the two shape stats)
        self.total_stats: dict[str, float] = dict.fromkeys(STAT_NAMES, 0.0)
        # Every backend on a device shares this engine (execute_parallel runs
        # up to V threads on it).  The handle serialises the calls themselves;
        # this lock also covers reading a call's error text, failing circuit
        # and stats, so no other thread's call can clear or replace them first.
        self._call_lock = threading.Lock()

    def close(self) -> None:
        if self._handle:
            self._lib.qv_destroy(self._handle)
            self._handle = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order varies
        try:
            self.close()
        except Exception:
            pass

    def execute(self, n_qubits: int, lowered: "LoweredBatch", result_kind: int, *,
                terms: tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray] | None = None,
                support: np.ndarray | None = None, target: np.ndarray | None = None,
                shots: int = 0, rng_state: np.ndarray | None = None, flags: int = 0) -> np.ndarray:
        """Run one batch; returns the flat float64 output (layout: qvb200.h)."""
        c = QvCircuits()
        c.n_qubits = n_qubits
        c.n_circuits = lowered.n_circuits
        c.uniform = 1 if lowered.uniform else 0
        c.n_gates = lowered.n_gates
        c.gate_offsets = _ptr(lowered.gate_offsets)
        c.kinds = _ptr(lowered.kinds)
        c.q0 = _ptr(lowered.q0)
        c.q1 = _ptr(lowered.q1)
        c.angles = _ptr(lowered.angles)
        r = QvResults()
        r.kind = result_kind
        r.flags = int(flags)
        keep = []
        if terms is not None:
            off, xm, ym, zm = (np.ascontiguousarray(a) for a in terms)
            keep += [off, xm, ym, zm]
            r.term_offsets, r.xmask, r.ymask, r.zmask = _ptr(off), _ptr(xm), _ptr(ym), _ptr(zm)
        if support is not None:
            support = np.ascontiguousarray(support, dtype=np.uint64)
            keep.append(support)
            r.support_count = support.shape[0]
            r.support = _ptr(support)
        if target is not None:
            target = np.ascontiguousarray(target, dtype=np.float64)
            keep.append(target)
            r.target = _ptr(target)
        if rng_state is not None:
            rng_state = np.ascontiguousarray(rng_state, dtype=np.uint64)
            keep.append(rng_state)
            r.rng_state = _ptr(rng_state)
            r.shots = int(shots)
        size = self._lib.qv_output_size(ctypes.byref(c), ctypes.byref(r))
        if size < 0:
            raise ValueError("malformed result request")
        out = np.empty(max(int(size), 1), dtype=np.float64)
        with self._call_lock:
            code = self._lib.qv_execute(self._handle, ctypes.byref(c), ctypes.byref(r), out.ctypes.data, out.shape[0])
            self._finish(code)
        return out[:size]

    def shift_js(self, n_qubits: int, base: "LoweredBatch", gate_index: np.ndarray, support: np.ndarray,
                 target: np.ndarray) -> np.ndarray:
        """qv_shift_js: JS losses at t_g +- pi/2 for each rotation gate g of one
        bound circuit; returns [2 * len(gate_index)] ('+' then '-' per gate)."""
        c = QvCircuits()
        c.n_qubits = n_qubits
        c.n_circuits = 1
        c.uniform = 1
        c.n_gates = base.n_gates
        c.kinds, c.q0, c.q1, c.angles = (_ptr(base.kinds), _ptr(base.q0), _ptr(base.q1), _ptr(base.angles))
        gates = np.ascontiguousarray(gate_index, dtype=np.int64)
        support = np.ascontiguousarray(support, dtype=np.uint64)
        target = np.ascontiguousarray(target, dtype=np.float64)
        r = QvResults()
        r.kind = QV_OUT_JS
        r.support_count = support.shape[0]
        r.support = _ptr(support)
        r.target = _ptr(target)
        out = np.empty(2 * gates.shape[0], dtype=np.float64)
        with self._call_lock:
            code = self._lib.qv_shift_js(self._handle, ctypes.byref(c), gates.shape[0], gates.ctypes.data,
                                         ctypes.byref(r), out.ctypes.data)
            self._finish(code)
        return out

    def _finish(self, code: int) -> None:
        """Stats and error of the call just made (caller holds _call_lock)."""
        stats = np.zeros(len(STAT_NAMES), dtype=np.float64)
        self._lib.qv_last_stats(self._handle, stats.ctypes.data, stats.shape[0])
        self.last_stats = dict(zip(STAT_NAMES, stats.tolist()))
        for k, v in self.last_stats.items():
            self.total_stats[k] = v if k in ("passes_per_circuit", "tile_bits") else self.total_stats[k] + v
        if code != QV_OK:
            msg = (self._lib.qv_last_error(self._handle) or b"").decode()
            raise NativeError(code, msg, int(self._lib.qv_last_error_circuit(self._handle)))


class LoweredBatch:
    """Gate arrays of a batch in the C-ABI layout (qv_circuits)."""

    __slots__ = ("n_circuits", "uniform", "n_gates", "gate_offsets", "kinds", "q0", "q1", "angles")

    def __init__(self, n_circuits, uniform, n_gates, gate_offsets, kinds, q0, q1, angles):
        self.n_circuits = int(n_circuits)
        self.uniform = bool(uniform)
        self.n_gates = int(n_gates)
        self.gate_offsets = None if gate_offsets is None else np.ascontiguousarray(gate_offsets, dtype=np.int64)
        self.kinds = np.ascontiguousarray(kinds, dtype=np.uint8)
        self.q0 = np.ascontiguousarray(q0, dtype=np.int32)
        self.q1 = np.ascontiguousarray(q1, dtype=np.int32)
        self.angles = np.ascontiguousarray(angles, dtype=np.float64)
        if self.kinds.shape[0] == 0:   # keep pointers valid for empty circuits
            self.kinds = np.zeros(1, np.uint8)
            self.q0 = np.zeros(1, np.int32)
            self.q1 = np.zeros(1, np.int32)
        if self.angles.size == 0:
            self.angles = np.zeros(1, np.float64)


_engines: dict[tuple[int, str], Engine] = {}
_engines_lock = threading.Lock()


def device_count() -> int:
    return int(load_library().qv_device_count())


def release_engine(device: int, precision: str = "complex128") -> None:
    """Destroy the process-wide engine of (device, precision) and free its
    device memory (e.g. a 64 GiB complex128 state before a complex64 run on
    the same GPU).  Backends created earlier must not be used afterwards."""
    with _engines_lock:
        eng = _engines.pop((int(device), precision), None)
    if eng is not None:
        with eng._call_lock:
            eng.close()


def engine(device: int, precision: str = "complex128") -> Engine:
    """Process-wide engine per (device, precision); calls on it serialise."""
    key = (int(device), precision)
    with _engines_lock:
        eng = _engines.get(key)
        if eng is None:
            eng = Engine(device, precision)
            _engines[key] = eng
        return eng
