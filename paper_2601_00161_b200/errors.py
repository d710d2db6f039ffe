"""Exception classes with the reference's names and meanings.

PlanningError, MeshError   <- prolate_ewald/mesh.py:25-30
ParameterError             <- prolate_ewald/evaluate.py:247
PswfError, DomainError     <- prolate_ewald/pswf.py:33-38
CellError, GeometryError   <- prolate_ewald/system.py:12-17
RealspaceError, SingularPairError <- prolate_ewald/realspace.py:15-21
InputError                 <- prolate_ewald/cli.py:46-47
"""


class PlanningError(Exception):
    """A grid invariant cannot be satisfied; the message names it."""


class MeshError(Exception):
    """Wrong field space, unknown differentiation mode, or call order."""


class ParameterError(Exception):
    """Invalid solver parameters or a cell that does not match the solver."""


class PswfError(Exception):
    """Construction or evaluation failure in the prolate machinery."""


class DomainError(PswfError):
    """Argument outside the domain of the requested evaluation."""


class CellError(Exception):
    """Invalid cell matrix or particle arrays."""


class GeometryError(CellError):
    """Cutoff too large for the cell, or other geometric safety violation."""


class RealspaceError(Exception):
    """Near-field (pair sum) failure."""


class SingularPairError(RealspaceError):
    """Coincident particles; physical configurations never need them."""


class InputError(Exception):
    """Malformed input file; the message carries path:line[:column] (cli.py:46-47)."""


class EspCudaError(RuntimeError):
    """CUDA / cuFFT failure inside the B200 library."""
