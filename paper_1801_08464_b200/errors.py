"""Exception types of the reference's solver path, raised by the GPU path.

When the reference package (``ncpflow``) is importable these subclass its own
classes, so ``except ncpflow.mgr.ZeroFDiagonal`` keeps working after the
switch; otherwise they are standalone with the same names and bases
(mgr.py:41-44, amg.py:27-28, sparse.py:18-28, newton.py:27-31).
"""
from __future__ import annotations

try:  # pragma: no cover - only where the reference is installed
    from ncpflow import amg as _ramg, ilu as _rilu, mgr as _rmgr, newton as _rnewton, sparse as _rsparse
    _BASES = dict(zero=(_rmgr.ZeroFDiagonal,), amg=(_ramg.AmgSetupError,),
                  dim=(_rsparse.DimensionMismatch,), sing=(_rsparse.SingularMatrixError,),
                  lsf=(_rnewton.LinearSolveFailure,), piv=(_rilu.ZeroPivot,))
except Exception:  # noqa: BLE001
    _BASES = dict(zero=(RuntimeError,), amg=(RuntimeError,), dim=(ValueError,), sing=(RuntimeError,),
                  lsf=(RuntimeError,), piv=(RuntimeError,))


class ZeroFDiagonal(*_BASES["zero"]):
    def __init__(self, row):
        RuntimeError.__init__(self, f"zero diagonal in A_ff at fine row {row}")
        self.row = row


class AmgSetupError(*_BASES["amg"]):
    pass


class DimensionMismatch(*_BASES["dim"]):
    pass


class SingularMatrixError(*_BASES["sing"]):
    def __init__(self, row, pivot=0.0, msg=None):
        RuntimeError.__init__(self, msg or f"singular matrix: pivot {pivot:.3e} at elimination step {row}")
        self.row = row
        self.pivot = pivot


class LinearSolveFailure(*_BASES["lsf"]):
    pass


class ZeroPivot(*_BASES["piv"]):
    """ILU zero pivot (ilu.py:24-27)."""

    def __init__(self, row):
        RuntimeError.__init__(self, f"zero pivot encountered at row {row}")
        self.row = row


class UnsupportedOnGpu(NotImplementedError):
    pass


class CudaError(RuntimeError):
    pass


def from_status(st: int, msg: str, row: int):
    if st == 1:
        return ZeroFDiagonal(row)
    if st == 2:
        return AmgSetupError(msg)
    if st == 3:
        return DimensionMismatch(msg)
    if st == 4:
        return ValueError(msg)
    if st == 6:
        return SingularMatrixError(row, 0.0, msg)
    if st == 7:
        return UnsupportedOnGpu(msg)
    if st == 8:
        return ZeroPivot(row)
    return CudaError(f"libmgrgpu CUDA failure: {msg}")
