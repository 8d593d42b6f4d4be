"""B200-native classical Ewald summation (arXiv 1708.01135 electrostatics).

Drop-in for the Ewald entry points of the reference package ``ewaldmd``:
the same names, argument layout and exceptions, computed by hand-written
sm_100a fp64 CUDA kernels behind a C-ABI (``include/ewald_b200.h``).
See DESIGN.md.
"""

from .core import (
    NEUTRALITY_TOL,
    BoxTooSmallError,
    CoincidentParticlesError,
    ContractViolationError,
    CutoffTooLargeError,
    EwaldmdError,
    GlobalAccumulator,
    KSpaceEmptyError,
    LatticeError,
    NeutralityError,
    OracleSizeError,
    ParticleSet,
    SimulationBox,
    create_particle_set,
    minimum_image,
    set_error_types,
    total_charge,
    wrap_position,
)
from .ewald import (
    BALANCE_CONSTANT,
    EwaldEnergies,
    EwaldParams,
    EwaldSolver,
    ReciprocalSpace,
    choose_parameters,
    compute_rho_hat,
    enumerate_kvectors,
    long_range_energy_forces,
    self_energy,
    total_coulomb,
)

__all__ = [
    "NEUTRALITY_TOL", "BoxTooSmallError", "CoincidentParticlesError",
    "ContractViolationError", "CutoffTooLargeError", "EwaldmdError",
    "GlobalAccumulator", "KSpaceEmptyError", "LatticeError",
    "NeutralityError", "OracleSizeError", "ParticleSet", "SimulationBox",
    "create_particle_set", "minimum_image", "set_error_types", "total_charge",
    "wrap_position",
    "BALANCE_CONSTANT", "EwaldEnergies", "EwaldParams", "EwaldSolver",
    "ReciprocalSpace", "choose_parameters", "compute_rho_hat",
    "enumerate_kvectors", "long_range_energy_forces", "self_energy",
    "total_coulomb",
]
