"""CPU unit tests of the CUDA path's per-point arithmetic: the kernels' __host__ __device__
eigen-decomposition and regularisation (gsicp_internal.cuh), compiled for the host
(libgsicp_hostmath.so), against the oracle's Jacobi + regularisation on the hard spectra
(nearly repeated, line-like, plane-like, degenerate) at the parity tolerance."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def hm():
    from paper_2403_12550_b200 import _build

    _build.build()
    L = C.CDLL(_build.HOSTMATH)
    L.gsicp_host_regularize.restype = C.c_uint
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def host_eig(L, C6):
    C6 = np.ascontiguousarray(C6, np.float64)
    lam, V = np.zeros(3), np.zeros(9)
    L.gsicp_host_eig3(_p(C6), _p(lam), _p(V))
    return lam, V.reshape(3, 3)  # rows are eigenvectors


def host_reg(L, C6, mode, eps=1e-3):
    C6 = np.ascontiguousarray(C6, np.float64)
    out, lm = np.zeros(6), np.zeros(1)
    fl = L.gsicp_host_regularize(_p(C6), mode, C.c_double(eps), _p(out), _p(lm))
    return out, fl, lm[0]


def spectra(rng, n):
    for t in range(n):
        Q = np.linalg.qr(rng.normal(size=(3, 3)))[0]
        lam = 10.0 ** rng.uniform(-9, -1, 3)
        kind = t % 5
        if kind == 1:
            lam[1] = lam[2] * (1 + rng.uniform(-1e-7, 1e-7))  # line-like pair
            lam[0] = lam[1] * 10 ** rng.uniform(2, 6)
        elif kind == 2:
            lam[0] = lam[1] * (1 + rng.uniform(-1e-7, 1e-7))  # plane-like pair
            lam[2] = lam[1] * 10 ** rng.uniform(-6, -2)
        elif kind == 3:
            lam[:] = lam[0] * (1 + rng.uniform(-1e-9, 1e-9, 3))  # isotropic
        A = Q @ np.diag(lam) @ Q.T
        yield np.array([A[0, 0], A[0, 1], A[0, 2], A[1, 1], A[1, 2], A[2, 2]])


def test_eig_matches_jacobi(hm):
    rng = np.random.default_rng(30)
    for C6 in spectra(rng, 3000):
        lam, V = host_eig(hm, C6)
        lo, _ = oracle.eigen(C6)
        assert np.abs(lam - lo).max() <= 1e-13 * lo[0]
        A = np.array([[C6[0], C6[1], C6[2]], [C6[1], C6[3], C6[4]], [C6[2], C6[4], C6[5]]])
        assert np.abs((V.T * lam) @ V - A).max() <= 1e-13 * lo[0]
        assert np.abs(V @ V.T - np.eye(3)).max() <= 1e-13


@pytest.mark.parametrize("mode", [oracle.NONE, oracle.PLANE, oracle.ELLIPSE])
def test_regularize_matches_oracle(hm, mode):
    rng = np.random.default_rng(31 + mode)
    for C6 in spectra(rng, 3000):
        out, fl, lm = host_reg(hm, C6, mode)
        ref, rfl = oracle.regularize(C6, mode, 1e-3)
        lo, _ = oracle.eigen(C6)
        assert fl == rfl
        if mode == oracle.PLANE and (lo[1] - lo[2]) < 1e-3 * lo[0]:
            continue  # normal ill-defined: only the trace is pinned
        err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
        assert err <= 1e-6, (C6, out, ref)


def test_degenerate_and_exact_cases(hm):
    # exactly collinear moments (the C1 k=5 case that broke a pure trigonometric solver)
    C6 = np.array([0.01881856, 0, 0, 0, 0, 0])
    out, fl, _ = host_reg(hm, C6, oracle.ELLIPSE)
    np.testing.assert_allclose(out, [1, 0, 0, 1e-3, 0, 1e-3], atol=1e-15)
    assert fl == oracle.FLAG_DEGENERATE
    out, fl, _ = host_reg(hm, np.zeros(6), oracle.ELLIPSE)
    np.testing.assert_array_equal(out, [1, 0, 0, 1, 0, 1])
    out, fl, _ = host_reg(hm, np.zeros(6), oracle.NONE)
    np.testing.assert_allclose(out, [1e-6, 0, 0, 1e-6, 0, 1e-6], rtol=1e-12)
    out, fl, lm = host_reg(hm, np.array([9.0, 0, 0, 4, 0, 1]), oracle.ELLIPSE)
    np.testing.assert_allclose(out, [2.25, 0, 0, 1, 0, 0.25], atol=1e-15)
    assert lm == pytest.approx(4.0, rel=1e-15)


def test_keyframe_policy():
    """P:213 (proportion of correspondences below the threshold) and P:264-265 (forced at the
    30th frame since the last keyframe)."""
    import paper_2403_12550_b200 as g

    assert g.is_keyframe(0.80, 1, min_fitness=0.9)
    assert not g.is_keyframe(0.95, 1, min_fitness=0.9)
    assert not g.is_keyframe(0.9, 29, min_fitness=0.9, max_gap=30)  # threshold is strict
    assert g.is_keyframe(1.0, 30, min_fitness=0.9, max_gap=30)
