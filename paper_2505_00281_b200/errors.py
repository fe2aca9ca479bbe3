"""Exception classes of the reference, same names and meaning.

ofrr/projection.py:24-29 (OverflowDiagnostic, EmptyPencilError), ofrr/basis.py:41-42
(EmptyBasisError), ofrr/smallsolve.py:20-25 (ConvergenceError).
"""


class OverflowDiagnostic(RuntimeError):
    """A projected matrix (or a MatVec / restart block) picked up non-finite entries."""


class EmptyPencilError(RuntimeError):
    """The mass matrix retained no eigenvalues above the nullspace cutoff."""


class EmptyBasisError(RuntimeError):
    """Every candidate column was dropped."""


class ConvergenceError(RuntimeError):
    """Jacobi iteration failed to reach its off-diagonal tolerance."""

    def __init__(self, msg: str, off_norm: float):
        super().__init__(f"{msg} (remaining off-norm {off_norm:.3e})")
        self.off_norm = off_norm
