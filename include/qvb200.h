/*
 * qvb200.h — C ABI of the B200 state-vector executor (libqvb200.so).
 *
 * This is the drop-in boundary for the reference's accelerator plugin
 * surface.  The reference binds no native code (its "kernels" are numba
 * functions), so each entry point below names the Python interface it
 * replaces; `INTEGRATION.md` shows the ctypes stub a maintainer of the
 * reference would add to `qvirt/backend.py`.
 *
 *   qv_create / qv_destroy   <- one `StatevectorBackend()` instance per
 *                               worker thread (reference pkg/src/qvirt/backend.py:189-201,
 *                               created by `backend_factory()` in pool.py:113-114).
 *   qv_execute               <- `StatevectorBackend.execute(buffer, circuits, config)`
 *                               in expectation mode (backend.py:199-219):
 *                               allocate (:57-63) -> run_gates (:88-91, kernels.py:18-70)
 *                               -> expectation (:94-119, kernels.py:73-87)
 *                               or born_distribution (:122-137, kernels.py:90-94).
 *   qv_last_error*           <- `ExecutionError(circuit_name, message)` (backend.py:36-41):
 *                               the failing circuit index lets the caller raise with the name.
 *
 * Conventions (same as the reference, kernels.py:3-7): qubit 0 is the MOST
 * significant bit of an amplitude index; qubit q flips index bit n-1-q.  All
 * pointers are host pointers owned by the caller for the duration of the call;
 * no CUDA or torch types cross this boundary.  Calls never throw; they return
 * a status code.  Calls on one handle are serialised by the handle; distinct
 * handles may be driven from distinct threads (ctypes releases the GIL).
 */
#ifndef QVB200_H
#define QVB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
#define QV_OK 0
#define QV_ERR_ARGUMENT 1   /* bad arguments / malformed batch (reference: ValueError)  */
#define QV_ERR_CIRCUIT 2    /* a circuit failed; see qv_last_error_circuit (ExecutionError) */
#define QV_ERR_CUDA 3       /* CUDA runtime failure (out of memory, launch error, no device) */
#define QV_ERR_INTERNAL 4

/* ---- gate kinds (reference circuits.py:27-33 GateKind; RX/CZ are extensions) */
#define QV_GATE_H 0
#define QV_GATE_X 1
#define QV_GATE_CNOT 2      /* q0 = control, q1 = target */
#define QV_GATE_RY 3
#define QV_GATE_RZ 4
#define QV_GATE_MEASURE_ALL 5 /* no-op in exact mode (backend.py:66-85) */
#define QV_GATE_RX 6        /* extension: [[c,-is],[-is,c]]                  */
#define QV_GATE_CZ 7        /* extension: diag(1,1,1,-1) on (q0,q1)           */

/* ---- amplitude precision -------------------------------------------------- */
#define QV_COMPLEX128 0     /* the reference's only precision (backend.py:61) */
#define QV_COMPLEX64 1      /* complex64 states, FP64 reductions                */

/* ---- result kinds --------------------------------------------------------- */
#define QV_OUT_PAULI 0      /* per circuit, per term: <P> (coefficient-free, kernels.py:73-87)  */
#define QV_OUT_SUPPORT 1    /* per circuit: normalised p on `support` + the norm (backend.py:122-129) */
#define QV_OUT_FULL 2       /* per circuit: all 2^n normalised probabilities (n <= 24)          */
#define QV_OUT_JS 3         /* per circuit: JS(target || p) via the support+remainder identity  */
                            /* (ddcl.py:37-61 over born_distribution)                            */
#define QV_RES_TARGET_ROWS 1 /* QV_OUT_JS: `target` holds one row of support_count probabilities   */
                            /* per circuit (circuit c at target + c * support_count), e.g. the   */
                            /* per-data-point targets of a QCL forward batch (ddcl.py:147-157)   */
#define QV_OUT_COUNTS 4     /* per circuit: `shots` samples of the outcome distribution with the  */
                            /* reference's sampler (backend.py:140-157): numpy PCG64 doubles,     */
                            /* inverse CDF on the sequential cumsum, side="right" (n <= 24)       */

typedef struct qv_engine* qv_handle;

/* A batch of bound circuits on one register width.
 * uniform = 1: every circuit has the same gate list (kinds/q0/q1 of length n_gates)
 *              and `angles` is an [n_circuits][n_gates] row-major table
 *              (the structure of a parameter-shift batch, gradients.py:33-46).
 * uniform = 0: circuit c owns gates [gate_offsets[c], gate_offsets[c+1]) of
 *              kinds/q0/q1/angles.
 * Angles of non-rotation gates are ignored.  q1 is ignored for 1-qubit gates. */
typedef struct qv_circuits {
    int32_t n_qubits;
    int32_t n_circuits;
    int32_t uniform;
    int32_t reserved;
    int64_t n_gates;               /* uniform = 1 */
    const int64_t* gate_offsets;   /* uniform = 0: n_circuits + 1 entries */
    const uint8_t* kinds;
    const int32_t* q0;
    const int32_t* q1;
    const double* angles;
} qv_circuits;

/* What to return for each circuit. */
typedef struct qv_results {
    int32_t kind;                  /* QV_OUT_* */
    int32_t flags;                 /* QV_RES_* (0 before this field was defined) */
    /* QV_OUT_PAULI: circuit c owns terms [term_offsets[c], term_offsets[c+1]);
     * a term is a Pauli product given by qubit-bit masks (bit n-1-q for qubit q),
     * exactly the (xmask, ymask, zmask) of backend.py:104-119.                 */
    const int64_t* term_offsets;
    const uint64_t* xmask;
    const uint64_t* ymask;
    const uint64_t* zmask;
    /* QV_OUT_SUPPORT / QV_OUT_JS: one support shared by the whole batch,
     * sorted ascending, unique amplitude indices; `target` (JS only) holds the
     * target probability of each support index.  These results are computed
     * on the support's light cone: a pass only sweeps the tiles the support
     * can see.  When the last pass is restricted that way the state norm is
     * not swept and is taken as 1 (the circuits are unitary; the reference's
     * normalising sum differs from 1 by ~1e-15), so the SUPPORT row's norm
     * entry then reads exactly 1.                                             */
    int64_t support_count;
    const uint64_t* support;
    const double* target;
    /* QV_OUT_COUNTS: shots per circuit, and each circuit's PCG64 generator
     * state as numpy's PCG64(seed).state holds it: rng_state[4c + 0..3] =
     * (state >> 64, state & (2^64-1), inc >> 64, inc & (2^64-1)).           */
    int64_t shots;
    const uint64_t* rng_state;
} qv_results;

/* Output sizes (doubles) written to `out`:
 *   PAULI   : term_offsets[n_circuits]                     (term t of circuit c at term_offsets[c]+t)
 *   SUPPORT : n_circuits * (support_count + 1)             (row: p_0..p_{S-1}, norm)
 *   FULL    : n_circuits * 2^n_qubits
 *   JS      : n_circuits
 *   COUNTS  : n_circuits * (2 * shots + 1); row: m, then m (outcome index, count)
 *             pairs in ascending index order                                          */
int64_t qv_output_size(const qv_circuits* circuits, const qv_results* results);

/* Create an executor bound to CUDA device `device`.  `memory_budget_bytes`
 * caps the device memory this handle keeps for state vectors (0 = whatever it
 * holds plus 90% of the device memory free at each call, less 1 GiB, so two
 * handles on one device -- e.g. one per precision -- share it). */
int qv_create(int device, int precision, uint64_t memory_budget_bytes, qv_handle* out);
int qv_destroy(qv_handle handle);

/* Execute a batch; blocks until `out` holds the results. */
int qv_execute(qv_handle handle, const qv_circuits* circuits, const qv_results* results,
               double* out, int64_t out_len);

/* Parameter-shift JS losses of ONE bound circuit without simulating two
 * shifted circuits per parameter.  For a rotation gate g (RX/RY/RZ, generator
 * P) at angle t, R(t +- pi/2) = R(t) (I -+ iP) / sqrt(2) exactly, so the two
 * shifted output states are (Psi0 -+ i Xi_g) / sqrt(2): Psi0 is the
 * unshifted output and Xi_g the output with P inserted at gate g.  One extra
 * state per shifted gate replaces two circuits; the two distributions are
 * formed in the final pass's epilogue.  Replaces the loss loop of reference
 * ddcl.py:210-225 over gradients.py:33-46 (theta[k] +- pi/2 for every k).
 *   base        : n_circuits = 1
 *   gate_index  : n_shift rotation-gate indices into base's gate list
 *   results     : kind = QV_OUT_JS (support + target)
 *   out         : 2 * n_shift doubles, out[2j] = JS at t_j + pi/2, out[2j+1] = JS at t_j - pi/2
 * Results agree with direct simulation of the shifted circuits to FP64
 * rounding (~1e-16), not bitwise; requires a register wider than one tile
 * (n > 12 complex128, n > 13 complex64), returns QV_ERR_ARGUMENT otherwise. */
int qv_shift_js(qv_handle handle, const qv_circuits* base, int64_t n_shift, const int64_t* gate_index,
                const qv_results* results, double* out);

/* Last error of this handle (empty string if none) and the index of the
 * circuit it belongs to (-1 if it is not specific to one circuit). */
const char* qv_last_error(qv_handle handle);
int64_t qv_last_error_circuit(qv_handle handle);

/* Execution statistics of the last qv_execute call on this handle:
 * [0] kernel launches, [1] full state sweeps executed (passes x states),
 * [2] sweeps a schedule without prefix sharing would run, [3] unique states simulated,
 * [4] algorithmic HBM bytes moved by pass kernels, [5] device ms of pass kernels
 * (CUDA events on the executor stream), [6] passes per circuit, [7] tile bits k,
 * [8] device ms of the call (first to last kernel), [9] host->device bytes,
 * [10] device->host bytes, [11] algorithmic flops of pass kernels
 * (28 per amplitude pair per fused 2x2 matrix), [12] TMA pass launches,
 * [13] read-only Pauli sweeps, [14] / [15] device ms / bytes of TMA passes,
 * [16] host wall ms of the whole call, [17] host wall ms before its first
 * kernel (validation, fusion, dedup, planning, copies).  n_stats <= 18. */
int qv_last_stats(qv_handle handle, double* stats, int32_t n_stats);

/* Library version string, e.g. "qvb200 0.1 sm_100a". */
const char* qv_version(void);

/* Number of visible CUDA devices (0 if none / no driver).  The virtual-QPU
 * pool maps vQPU b to device b mod qv_device_count() (pool.py:88-138). */
int qv_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* QVB200_H */
