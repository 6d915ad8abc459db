"""B200-native D2Q37 thermal lattice Boltzmann step (arXiv 1703.00185).

Drop-in for the hot path of the reference package ``thermolb``
(/root/reference/pkg/src/thermolb/__init__.py:3-26): the lattice, kernel,
runtime and run APIs keep their names; the compute is hand-written sm_100a
CUDA in libtlb.so (include/tlb.h), driven through ctypes.  The analytic
planner (paper Eqs. 10-19) and the snapshot writers (``io``) are restated
for the SURVEY §8(f) rows; the CLI and the CPU micro-benchmarks are out of
scope.
"""

from .errors import (AllocationError, ConfigurationError, ContractViolation,
                     DeadlockError, DegenerateStateError, DeviceError,
                     DomainError, ProtocolError, ThermoLBError,
                     UnsupportedCaseError)
from .geometry import (AOS, COLUMN, SOA, LatticeGeometry, MacroFields, PopulationField,
                       allocate_field, site_index, swap_buffers)
from .kernels import (WALL_ROWS, PhysicsParams, apply_shift, bc, collide,
                      count_negative, equilibrium, moments, propagate,
                      propagate_collide_fused)
from .planner import (BandwidthTable, CostModelInput, Prediction, brent_bound,
                      comm_time_2d, optimal_grid, predict_1d, predict_1d_overlap,
                      predict_2d, predict_2d_overlap, scaling_curve,
                      surface_over_volume)
from .runtime import (DistFabric, Fabric, RankWorker, TileAssignment,
                      boundary_bytes_per_site, decompose, face_plans)
from .sim import RunResult, SimConfig, run
from .velocity_set import VelocitySet, build_velocity_set

__all__ = [
    "AOS", "COLUMN", "SOA", "LatticeGeometry", "MacroFields", "PopulationField",
    "allocate_field", "site_index", "swap_buffers",
    "PhysicsParams", "apply_shift", "bc", "collide", "equilibrium", "moments",
    "propagate", "propagate_collide_fused", "count_negative", "WALL_ROWS",
    "RankWorker", "TileAssignment", "decompose", "face_plans",
    "boundary_bytes_per_site", "Fabric", "DistFabric",
    "RunResult", "SimConfig", "run",
    "BandwidthTable", "CostModelInput", "Prediction", "brent_bound", "optimal_grid",
    "predict_1d", "predict_1d_overlap", "predict_2d", "predict_2d_overlap",
    "scaling_curve", "comm_time_2d", "surface_over_volume",
    "VelocitySet", "build_velocity_set",
    "ThermoLBError", "ConfigurationError", "ContractViolation", "DomainError",
    "DegenerateStateError", "AllocationError", "ProtocolError", "DeadlockError",
    "UnsupportedCaseError", "DeviceError",
]

__version__ = "0.1.0"
