"""B200-native MGR-preconditioned GMRES (fp64) for block-sparse NCP Jacobians.

Drop-in GPU path for the reference package's (``ncpflow``) linear-solver hot
path: ``setup_from_matrix`` / ``mgr_apply`` / ``build_rp`` (ncpflow/mgr.py),
``amg_setup`` / ``amg_vcycle`` / ``amg_apply`` (ncpflow/amg.py), ``gmres``
(ncpflow/krylov.py) and ``GmresSolver`` (ncpflow/linsolve.py).  All compute
runs in hand-written sm_100a CUDA kernels behind the C-ABI declared in
``include/mgrgpu.h``; this package is the ctypes host side.  There is no CPU
fallback: using any solver entry point without the built CUDA library (or
without a GPU) raises ``RuntimeError``.
"""
__version__ = "0.1.0"
