"""B200-native ESP long-range (k-space) path — drop-in for the mesh pipeline
of ``prolate_ewald`` (arXiv 2601.00161).

The k-space path and the near-field pair sum (realspace.py) live in
``libesp_b200.so`` (hand-written sm_100a CUDA + cuFFT,
C ABI in include/esp_b200.h); this package is the host-side mirror of the
reference's Python API for that path.  There is no CPU fallback: device
functions raise if the library or a GPU is missing.
"""

from .cells import CellType, infer_cell_type
from .errors import (CellError, DomainError, EspCudaError, GeometryError, InputError, MeshError,
                     ParameterError, PlanningError, PswfError, RealspaceError,
                     SingularPairError)
from .kernel import (SplitKernel, background_correction, background_integral, eval_phi0,
                     far_field, far_field_hat, fn_weight, near_field, pressure_kernel_hat,
                     self_energy)
from .mesh import (GridField, GridSpec, ModeWorkspace, TransformProvider, forward_density,
                   local_pressure, long_range_energy, long_range_forces,
                   long_range_pressure, plan_grid, spread_charges)
from .plan import EspPlan, cell_tables
from .pswf import (PswfBasis, WindowTable, build_pswf, eval_psi0, solve_bandwidth,
                   tabulate_window)
from .solver import (CoulombSolver, EnergyBreakdown, EwaldParameters, KSpaceResult,
                     KSpaceSolver, evaluate_system, kinetic_pressure)
from .particles import read_particles, write_particles
from .realspace import (NearFieldPlan, PairTable, ShortRangeResult, build_cell_list,
                        build_pair_table, short_range)
from .system import Cell, NeighborList, ParticleSystem, check_cutoff, minimum_image

__version__ = "0.1.0"

__all__ = [
    "Cell", "CellError", "CellType", "CoulombSolver", "DomainError", "EnergyBreakdown",
    "EspCudaError", "EspPlan", "EwaldParameters", "GridField", "GridSpec", "KSpaceResult",
    "KSpaceSolver", "MeshError", "ModeWorkspace", "ParameterError", "ParticleSystem",
    "PlanningError", "PswfBasis", "PswfError", "SplitKernel", "TransformProvider",
    "WindowTable", "background_correction", "build_pswf", "cell_tables", "check_cutoff",
    "eval_psi0", "evaluate_system", "far_field_hat", "forward_density", "infer_cell_type",
    "local_pressure", "long_range_energy", "long_range_forces", "long_range_pressure",
    "plan_grid", "self_energy", "solve_bandwidth", "spread_charges", "tabulate_window",
    "GeometryError", "RealspaceError", "SingularPairError", "far_field", "fn_weight",
    "near_field", "NearFieldPlan", "PairTable", "ShortRangeResult", "build_pair_table",
    "short_range", "NeighborList", "minimum_image", "build_cell_list", "read_particles",
    "write_particles", "InputError", "eval_phi0", "pressure_kernel_hat", "background_integral",
    "kinetic_pressure",
]
