"""qvb200 — B200-native state-vector executor behind the virtual-QPU plugin
surface of arXiv 2406.03466 (reference package `qvirt`).

The public names mirror `qvirt/__init__.py` so code written against the
reference switches by changing the import; `B200Backend` replaces
`StatevectorBackend` as the default accelerator.  Numerics run in
libqvb200.so (hand-written sm_100a CUDA behind a C ABI, include/qvb200.h).
"""

from .backend import (
    MODES,
    Accelerator,
    B200Backend,
    ExecutionConfig,
    ExecutionError,
    lower_batch,
    support_indices,
)
from .ir import (
    BoundRows,
    Circuit,
    Gate,
    GateKind,
    Lowering,
    ParameterVector,
    bind,
    bind_rows,
    cnot,
    cz,
    h,
    measure_all,
    rx,
    ry,
    rz,
    x,
)
from .mcvqe import (
    McvqeAnsatzSpec,
    entangler_gates,
    mcvqe_ansatz,
    mcvqe_ansatz_template,
    mcvqe_energy,
    mcvqe_execution_count,
    mcvqe_gradient,
    mcvqe_gradient_batch,
    mcvqe_parameter_count,
    mcvqe_raw_ansatz,
    random_angles,
    random_cis_amplitudes,
    w_state_prep,
)
from .observables import (
    AiemCoefficients,
    Observable,
    PauliTerm,
    aiem_hamiltonian,
    combine,
    expectation_from_counts,
    measurable_term_count,
    measurement_basis_circuit,
    pauli,
    random_aiem_coefficients,
    term_masks,
)
from .qcl import (
    DdclSpec,
    ddcl_batch,
    ddcl_circuit,
    ddcl_circuit_template,
    ddcl_distribution,
    ddcl_forward_losses,
    ddcl_execution_count,
    ddcl_gradient,
    ddcl_parameter_count,
    js_divergence,
    random_target_distribution,
)
from .results import ChildResult, ResultBuffer, deserialize, dump_buffer, load_buffer, merge, serialize
from .shift import SHIFT, SHIFT_TAGS, GradientReport, central_difference, shift_table, shifted_batch, shifted_circuits
from .vqpu import (Block, VqpuPoolConfig, consolidate, execute_parallel, execute_row_values, execute_values,
                   partition)

__version__ = "0.1.0"
