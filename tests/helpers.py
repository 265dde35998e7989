"""Shared test helpers (seeded inputs, CSR comparisons)."""
import numpy as np
import scipy.sparse as sp


def rand_csr(rng, n, m, density, diag=0.0):
    a = sp.random(n, m, density=density, random_state=np.random.RandomState(rng.integers(1 << 31)),
                  data_rvs=lambda k: rng.standard_normal(k)).tocsr()
    if diag:
        a = (a + sp.identity(n) * diag).tocsr() if n == m else a
    a.sort_indices()
    return a


def poisson1d(n):
    e = np.ones(n)
    return sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1]).tocsr()


def poisson2d(m):
    e = np.ones(m)
    t = sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1])
    i = sp.identity(m)
    return (sp.kron(t, i) + sp.kron(i, t)).tocsr()


def poisson3d(m, zf=1.0):
    e = np.ones(m)
    t = sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1])
    i = sp.identity(m)
    return (sp.kron(sp.kron(t, i), i) * zf + sp.kron(sp.kron(i, t), i) + sp.kron(sp.kron(i, i), t)).tocsr()


def csr_parts(m):
    m = m.tocsr()
    m.sort_indices()
    return np.asarray(m.indptr, dtype=np.int64), np.asarray(m.indices, dtype=np.int64), np.asarray(m.data)


def assert_same_pattern(got, want):
    gi, gj, _ = csr_parts(got)
    wi, wj, _ = csr_parts(want)
    assert got.shape == want.shape
    np.testing.assert_array_equal(gi, wi)
    np.testing.assert_array_equal(gj, wj)


def assert_bitwise(got, want):
    assert_same_pattern(got, want)
    _, _, gv = csr_parts(got)
    _, _, wv = csr_parts(want)
    np.testing.assert_array_equal(gv.view(np.int64), wv.view(np.int64))


def assert_close_csr(got, want, rtol=1e-12):
    assert_same_pattern(got, want)
    _, _, gv = csr_parts(got)
    _, _, wv = csr_parts(want)
    scale = max(np.abs(wv).max(initial=0.0), 1e-300)
    assert np.max(np.abs(gv - wv), initial=0.0) <= rtol * scale


def relerr(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
