"""B200-native D2Q37 thermal lattice Boltzmann step (arXiv 1703.00185).

A drop-in for the hot path of the reference package ``thermolb``: the
public names of its lattice, kernel, runtime, run and planner modules are
re-exported here unchanged, plus the B200 additions (column layout, NCCL /
NVLink-peer ``DistFabric``, ``count_negative``, ``DeviceError``).  All
compute runs in libtlb.so (hand-written sm_100a CUDA, C ABI in
include/tlb.h) through ctypes; there is no CPU fallback.  Out of scope: the
reference's CLI and its CPU micro-benchmarks.
"""

from importlib import import_module

# module -> public names re-exported at package level
_PUBLIC = {
    "errors": "ThermoLBError ConfigurationError ContractViolation DomainError "
              "DegenerateStateError AllocationError ProtocolError DeadlockError "
              "UnsupportedCaseError DeviceError",
    "velocity_set": "VelocitySet build_velocity_set",
    "geometry": "SOA AOS COLUMN LatticeGeometry PopulationField MacroFields "
                "allocate_field swap_buffers site_index",
    "kernels": "PhysicsParams moments equilibrium apply_shift collide propagate bc "
               "propagate_collide_fused count_negative WALL_ROWS",
    "runtime": "TileAssignment decompose face_plans boundary_bytes_per_site "
               "RankWorker Fabric DistFabric",
    "sim": "SimConfig RunResult run",
    "planner": "BandwidthTable CostModelInput Prediction surface_over_volume "
               "comm_time_2d optimal_grid predict_1d predict_2d predict_1d_overlap "
               "predict_2d_overlap brent_bound scaling_curve",
}

__all__ = []
for _mod, _names in _PUBLIC.items():
    _m = import_module(f".{_mod}", __name__)
    for _n in _names.split():
        globals()[_n] = getattr(_m, _n)
        __all__.append(_n)
from . import init, io  # noqa: E402  (submodules: presets, snapshot writers)

del _mod, _names, _m, _n
__version__ = "0.1.0"
