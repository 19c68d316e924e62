"""B200-native gate-application hot path of qHiPSTER (arXiv:1601.07195).

Drop-in for the register + gate-application API of the reference package
``svsim`` (pkg/src/svsim/__init__.py): the same names and signatures, with
the state vector resident in GPU memory and every gate a hand-written sm_100a
kernel in ``libsvb200.so`` called through a C ABI (include/svb200.h).  Gates
on global qubits exchange halves with the partner GPU over NVLink inside one
fused kernel (``NvlinkFabric`` is the ``transport``).  There is no CPU path.
"""

from __future__ import annotations

from ._lib import LIB_PATH, NativeError, launch_count
from .circuits import (
    Circuit,
    GateOp,
    build_iqft,
    build_qft,
    hadamard,
    pauli_x,
    pauli_y,
    pauli_z,
    per_target_sweep,
    phase_r,
    phase_shift,
    random_circuit,
    random_unitary,
    rotation_x,
    rotation_y,
    rotation_z,
)
from .core import (
    max_abs_diff,
    ALIGNMENT,
    AMP_BYTES,
    Layout,
    LocalState,
    aligned_zeros,
    global_norm_sq,
    init_basis_state,
    init_random_state,
    probability_of_bit,
    state_from_global,
)
from .distributed import (
    CONTROL_TAG,
    DEFAULT_CHUNK_BYTES,
    GATHER_MAX_QUBITS,
    ComputesHalf,
    CudaExecutor,
    ExchangePlan,
    GateAction,
    InprocFabric,
    NvlinkFabric,
    ScratchPool,
    apply_controlled_distributed,
    apply_global,
    apply_op,
    apply_single_distributed,
    execute_action,
    gather_full_state,
    make_exchange_plan,
    plan_gate,
    is_diagonal,
)
from .circuitfile import parse_circuit_file, parse_circuit_text
from .engine import CircuitGraph, GateRecord, run_circuit, run_circuit_inproc, run_pipelined
from .passes import Pass, execute_pass, plan_passes
from .remap import QubitMap, Swap, plan_remapped, restore_map, run_circuit_remapped, swap_global
from .errors import CircuitParseError, FusionContractError, LayoutError, ResourceError, TransportError
from .fusion import (
    FusedBlockRun,
    FusionConfig,
    FusionPlan,
    PassThrough,
    default_block_exponent,
    execute_plan,
    gpu_block_exponent,
    plan_fusion,
    run_fused,
)
from .kernels import (
    SERIAL,
    UNITARITY_TOL,
    GateMatrix,
    ParallelLevel,
    ThreadPolicy,
    apply_block,
    apply_controlled_local,
    apply_controlled_raw,
    apply_single_local,
    apply_single_raw,
)
from .perfmodel import (
    BoundCase,
    MachineParams,
    achieved_bandwidth,
    b200_params,
    classify_case,
    link_bytes_per_direction,
    lower_bound_seconds,
    traffic_bytes,
)

Transport = NvlinkFabric  # the reference's transport slot is filled by the NVLink fabric

__all__ = [name for name in dir() if not name.startswith("_")]
