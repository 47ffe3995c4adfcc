"""B200-native FlashSchNet MD step behind the flashcg API.

Mirrors the hot-path surface of the reference package `flashcg`
(/root/reference/pkg/src/flashcg/__init__.py): neighbour lists and CSR
layouts, segment_reduce, flash_energy_forces, the batched Langevin
integrator and run_simulation.  All per-step compute runs in libfcg.so
(hand-written sm_100a CUDA behind the C ABI in include/fcg.h); the Python
modules only prepare inputs, move buffers and write outputs.
"""

from .schnet import (
    EnergyForces,
    PipelineMode,
    TrafficReport,
    flash_energy_forces,
    io_model_base,
    io_model_flash,
    segment_reduce,
    traffic_report,
)
from .langevin import (
    KB,
    GpuReplicaForces,
    RunResult,
    SimConfig,
    SimState,
    SimulationBlowupError,
    integrate,
    kinetic_temperature,
    make_step_rng,
    run_simulation,
    throughput_report,
)
from .modelparams import BlockParams, ConfigError, ModelConfig, ModelParams, RbfSpec, init_params
from .csr import (
    CsrLayout,
    NeighborList,
    build_neighbors_bruteforce,
    build_neighbors_cells,
    group_by_destination,
    group_by_source,
)
from .prior import PriorSpec
from ._lib import CapacityError
from .inputs import SystemSpec, generate_system

__all__ = [
    "BlockParams", "CapacityError", "ConfigError", "CsrLayout", "EnergyForces", "GpuReplicaForces", "KB",
    "ModelConfig", "ModelParams", "NeighborList", "PipelineMode", "PriorSpec", "RbfSpec",
    "RunResult", "SimConfig", "SimState", "SimulationBlowupError", "SystemSpec",
    "TrafficReport", "traffic_report", "build_neighbors_bruteforce", "build_neighbors_cells",
    "flash_energy_forces", "generate_system", "group_by_destination", "group_by_source",
    "init_params", "integrate", "io_model_base", "io_model_flash", "kinetic_temperature",
    "make_step_rng", "run_simulation", "segment_reduce", "throughput_report",
]

__version__ = "0.1.0"
