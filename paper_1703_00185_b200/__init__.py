"""B200-native D2Q37 thermal lattice Boltzmann step (arXiv 1703.00185).

Drop-in for the hot path of the reference package ``thermolb``
(/root/reference/pkg/src/thermolb/__init__.py:3-26): the lattice, kernel,
runtime and run APIs keep their names; the compute is hand-written sm_100a
CUDA in libtlb.so (include/tlb.h), driven through ctypes.  The reference's
analytic planner, CLI, IO and CPU micro-benchmarks are out of scope
(SURVEY.md §2 rows 9-12).
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
    "VelocitySet", "build_velocity_set",
    "ThermoLBError", "ConfigurationError", "ContractViolation", "DomainError",
    "DegenerateStateError", "AllocationError", "ProtocolError", "DeadlockError",
    "UnsupportedCaseError", "DeviceError",
]

__version__ = "0.1.0"
