"""Host-side checks (no GPU): C-ABI exports, generator, option schema, errors,
and that the product path fails loudly instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_1801_08464_b200 import _lib, errors, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mgrgpu.h")).read()
    return sorted(set(re.findall(r"\b(mg_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        getattr(lib, s)  # raises AttributeError when missing
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if l.strip()}
    assert set(syms) <= exported
    assert set(_lib.EXPORTED) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.Context(0)


def test_error_mapping():
    e = errors.from_status(1, "x", 7)
    assert isinstance(e, errors.ZeroFDiagonal) and e.row == 7
    assert isinstance(errors.from_status(2, "m", -1), errors.AmgSetupError)
    assert isinstance(errors.from_status(3, "m", -1), errors.DimensionMismatch)
    assert isinstance(errors.from_status(3, "m", -1), ValueError)
    assert isinstance(errors.from_status(4, "m", -1), ValueError)
    assert isinstance(errors.from_status(6, "m", 3), errors.SingularMatrixError)
    assert isinstance(errors.from_status(7, "m", -1), NotImplementedError)


def test_option_schema_validation():
    from paper_1801_08464_b200.amg import AmgOptions, as_options
    from paper_1801_08464_b200.krylov import GmresOptions
    from paper_1801_08464_b200.mgr import FRelax, MgrLevelSpec, RpKind
    with pytest.raises(ValueError):
        AmgOptions(strength_theta=1.0)
    with pytest.raises(ValueError):
        AmgOptions(pre_sweeps=-1)
    with pytest.raises(ValueError):
        FRelax("sor")
    with pytest.raises(ValueError):
        FRelax(sweeps=0)
    with pytest.raises(ValueError):
        GmresOptions(rel_tol=0.0)
    with pytest.raises(ValueError):
        GmresOptions(restart=0)
    assert as_options(AmgOptions(interpolation="classical")).interpolation == "classical"
    assert MgrLevelSpec().rp is RpKind.INJECTIVE
    c = AmgOptions(max_elmts=3, seed=5).to_c()
    assert c.max_elmts == 3 and c.seed == 5


def test_reference_option_objects_accepted(ncpflow):
    """The reference's own schema objects are valid inputs (drop-in)."""
    from ncpflow.amg import AmgOptions as RAmg
    from paper_1801_08464_b200.amg import as_options
    from paper_1801_08464_b200.mgr import _rp_code
    import ncpflow.mgr as rmgr
    o = as_options(RAmg(pre_sweeps=2, post_sweeps=2, strength_theta=0.3))
    assert (o.pre_sweeps, o.post_sweeps, o.strength_theta) == (2, 2, 0.3)
    assert _rp_code(rmgr.RpKind.NONINJECTIVE) == 1


@pytest.mark.parametrize("cfg,nnzb,n", [(1, 20224, 8192), (2, 1810432, 524288)])
def test_generator_sizes(cfg, nnzb, n):
    s = synth.make_config(cfg)
    assert s.nnzb == nnzb and s.n == n


def test_generator_readings():
    s = synth.make_config(1)
    assert abs(s.gas.mean() - 0.38) < 0.02          # disc r = 0.35*64 -> ~38% gas, ~62% absent
    s3 = synth.make_config(3, 32)
    assert abs((~s3.gas).mean() - 0.30) < 0.03      # interface z < 0.3E + ...
    s4 = synth.make_config(4, 24)
    assert abs((~s4.gas).mean() - 0.50) < 0.03      # sphere r = 0.4924E
    # gas-absent S rows: only A_sp(i,i) = -0.01 (b=2) / A_srho(i,i) = 1 (b=3)
    brow = np.repeat(np.arange(s.n_cells), np.diff(s.rowptr))
    absent = ~s.gas[brow]
    diag = s.col == brow
    assert np.all(s.vals[absent & ~diag][:, 1, :] == 0.0)
    assert np.all(s.vals[absent & diag][:, 1, 0] == -0.01)
    assert np.all(s.vals[absent & diag][:, 1, 1] == 0.0)
    brow4 = np.repeat(np.arange(s4.n_cells), np.diff(s4.rowptr))
    d4 = s4.vals[(s4.col == brow4) & ~s4.gas[brow4]]
    np.testing.assert_array_equal(d4[:, 1, :], np.tile([0.0, 0.0, 1.0], (d4.shape[0], 1)))
    # determinism
    t = synth.make_config(2, 8, seed=3)
    u = synth.make_config(2, 8, seed=3)
    np.testing.assert_array_equal(t.vals, u.vals)
    np.testing.assert_array_equal(t.rhs, u.rhs)


def test_variable_major_layout_matches_cell_major():
    s = synth.make_config(2, 6)
    a_cell = synth.to_scalar_csr(s, "cell")
    a_var = synth.to_scalar_csr(s, "var")
    N, b = s.n_cells, s.b
    perm = (np.arange(s.n) % b) * N + np.arange(s.n) // b   # cell-major index -> var-major index
    np.testing.assert_array_equal(a_var[perm][:, perm].toarray(), a_cell.toarray())


def test_pipeline_defaults_mirrored_in_the_oracle():
    """The synthetic pipeline's DESIGN decisions are the same on both sides of every
    parity test: MGR sweep order per block size and the default R/P kind."""
    from oracle import pipeline as opipe
    from paper_1801_08464_b200 import pipeline as gpipe
    for b in (1, 2, 3):
        assert gpipe.default_post_smoothing(b) == opipe.default_post_smoothing(b)
    assert gpipe.default_post_smoothing(2) and not gpipe.default_post_smoothing(3)
    for b, ncell in ((2, 8), (3, 8)):
        pg = gpipe.default_plan(b, ncell)
        po = opipe.default_plan(b, ncell)
        assert [s.rp.value for _, s in pg] == [s.rp.value for _, s in po]
        assert len(pg) == b - 1
