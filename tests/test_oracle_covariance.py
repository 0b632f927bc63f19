"""Pins of the oracle's O3 (covariance), O4 (eigen), O5 (regularisation), O6 (map -> target)
and O12 (scale aligning), CPU only.  Library cross-checks (numpy.cov, numpy.linalg.eigh),
SPEC's worked examples, closed forms and invariants.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
MODES = {"none": oracle.NONE, "plane": oracle.PLANE, "ellipse": oracle.ELLIPSE}


def pack(A):
    return np.array([A[0, 0], A[0, 1], A[0, 2], A[1, 1], A[1, 2], A[2, 2]])


def unpack(c):
    return np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]], dtype=np.float64)


def rand_spd(rng, spread=3.0):
    Q = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    lam = 10.0 ** rng.uniform(-spread, 0, 3)
    return Q @ np.diag(lam) @ Q.T


def test_covariance_matches_numpy_cov():
    rng = np.random.default_rng(10)
    P = rng.normal(size=(200, 3)).astype(np.float32) * [1.0, 0.3, 0.01] + [5.0, -2.0, 3.0]
    P = P.astype(np.float32)
    for _ in range(20):
        nbr = rng.choice(200, 20, replace=False).astype(np.int32)
        c = oracle.covariance(P, nbr)
        ref = np.cov(P[nbr].astype(np.float64).T, bias=True)
        np.testing.assert_allclose(unpack(c), ref, rtol=1e-12, atol=1e-15)


def test_eigen_matches_lapack():
    rng = np.random.default_rng(11)
    for _ in range(200):
        A = rand_spd(rng, spread=rng.uniform(0, 8))
        lam, V = oracle.eigen(pack(A))
        w, U = np.linalg.eigh(A)
        np.testing.assert_allclose(lam, w[::-1], rtol=1e-12, atol=1e-15 * w.max())
        np.testing.assert_allclose(V @ np.diag(lam) @ V.T, A, rtol=0, atol=1e-13 * np.abs(A).max())
        np.testing.assert_allclose(V.T @ V, np.eye(3), atol=1e-13)


@pytest.mark.parametrize("ex", GOLD["decompose"])
def test_decompose_spec_examples(ex):
    C = np.array(ex["C"], float) if "C" in ex else np.outer(ex["v"], ex["v"])
    lam, V = oracle.eigen(pack(C))
    np.testing.assert_allclose(lam, np.square(ex["S"]), atol=1e-14 * max(lam))
    if "v" in ex:  # principal axis along v
        assert abs(abs(V[:, 0] @ np.array(ex["v"])) / 2.0 - 1.0) < 1e-12


@pytest.mark.parametrize("ex", GOLD["regularize"])
def test_regularize_spec_examples(ex):
    out, fl = oracle.regularize(pack(np.array(ex["C"], float)), MODES[ex["mode"]], ex["eps"])
    np.testing.assert_allclose(unpack(out), np.array(ex["out"]), atol=1e-14)
    assert fl == 0


def test_ellipse_is_c_over_lambda_mid_and_preserves_axes():
    """Eq. 4 with C = R Lambda^2 R^T gives C' = C / s_1^2 = C / lambda_mid when
    the eps floor does not bite; middle scale is 1; eigenvectors preserved."""
    rng = np.random.default_rng(12)
    for _ in range(200):
        A = rand_spd(rng, spread=2.5)
        w, U = np.linalg.eigh(A)
        if w[0] / w[1] < 2e-3:
            continue
        out, fl = oracle.regularize(pack(A), oracle.ELLIPSE, 1e-3)
        np.testing.assert_allclose(unpack(out), A / w[1], rtol=1e-10, atol=1e-12 * w[2] / w[1])
        w2, U2 = np.linalg.eigh(unpack(out))
        assert abs(w2[1] - 1.0) < 1e-10
        assert np.all(np.abs(np.abs(np.sum(U * U2, 0)) - 1) < 1e-8)


def test_ellipse_floor_and_plane_spectrum():
    rng = np.random.default_rng(13)
    Q = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    A = Q @ np.diag([5.0, 2.0, 1e-7]) @ Q.T  # lambda0 / lambda1 = 5e-8 < eps
    out, _ = oracle.regularize(pack(A), oracle.ELLIPSE, 1e-3)
    np.testing.assert_allclose(np.linalg.eigvalsh(unpack(out)), [1e-3, 1.0, 2.5], rtol=1e-9)
    out, _ = oracle.regularize(pack(A), oracle.PLANE, 1e-3)
    w, U = np.linalg.eigh(unpack(out))
    np.testing.assert_allclose(w, [1e-3, 1.0, 1.0], rtol=1e-9)
    assert abs(abs(U[:, 0] @ Q[:, 2]) - 1) < 1e-9  # normal = smallest-eigenvalue axis


def test_psd_on_random_vectors():
    """v^T C v >= 0 for 100 random v per matrix, all modes."""
    rng = np.random.default_rng(14)
    for _ in range(50):
        A = rand_spd(rng, spread=6)
        for m in MODES.values():
            C = unpack(oracle.regularize(pack(A), m, 1e-3)[0])
            v = rng.normal(size=(100, 3))
            assert np.all(np.einsum("ij,jk,ik->i", v, C, v) >= 0)


def test_degenerate_coincident_and_collinear():
    # S:67 coincident points -> floor * I (NONE), I + flag (ELLIPSE, Q8)
    P = np.tile(np.float32([[1.0, 2.0, 3.0]]), (25, 1))
    r = oracle.covariances(P, k=20, mode=oracle.NONE)
    np.testing.assert_allclose(unpack(r["cov"][0]), 1e-6 * np.eye(3), rtol=1e-6)
    r = oracle.covariances(P, k=20, mode=oracle.ELLIPSE)
    np.testing.assert_allclose(unpack(r["cov"][0]), np.eye(3))
    assert r["flags"][0] & oracle.FLAG_DEGENERATE
    # S:69 collinear -> two eigenvalues at floor, principal axis along the line
    d = np.array([1.0, 2.0, 2.0]) / 3.0
    P = (np.arange(30)[:, None] * 0.01 * d).astype(np.float32)
    r = oracle.covariances(P, k=20, mode=oracle.NONE)
    w, U = np.linalg.eigh(unpack(r["cov"][10]).astype(np.float64))
    np.testing.assert_allclose(w[:2], [1e-6, 1e-6], rtol=1e-3)
    assert abs(abs(U[:, 2] @ d) - 1) < 1e-6
    r = oracle.covariances(P, k=20, mode=oracle.ELLIPSE)
    w, U = np.linalg.eigh(unpack(r["cov"][10]).astype(np.float64))
    np.testing.assert_allclose(w, [1e-3, 1e-3, 1.0], rtol=0, atol=1e-7)  # binary32 storage
    assert r["flags"][10] & oracle.FLAG_DEGENERATE


def test_planar_patch_normal_and_noise_variance():
    """BJ pin: planar patches yield the normal as the smallest eigenvector with the eps-regularised
    spectrum; lambda_min <= 1e-3 lambda_max on a regular planar grid."""
    rng = np.random.default_rng(15)
    n = np.array([0.3, -0.4, 0.866])
    n /= np.linalg.norm(n)
    t1 = np.cross(n, [1.0, 0, 0]); t1 /= np.linalg.norm(t1)
    t2 = np.cross(n, t1)
    g = np.stack(np.meshgrid(np.arange(30), np.arange(30)), -1).reshape(-1, 2) * 0.01
    P = (g[:, :1] * t1 + g[:, 1:] * t2 + [1.0, 2.0, 3.0]).astype(np.float32)
    r = oracle.covariances(P, k=20, mode=oracle.ELLIPSE)
    i = 15 * 30 + 15
    lam, V = oracle.eigen(r["raw"][i])
    assert lam[2] <= 1e-3 * lam[0]
    assert abs(abs(V[:, 2] @ n) - 1) < 1e-5
    w = np.linalg.eigvalsh(unpack(r["cov"][i]).astype(np.float64))
    np.testing.assert_allclose(w[0], 1e-3, rtol=0, atol=1e-7)  # eps-regularised normal variance (binary32)
    # with normal noise sigma, lambda_0 ~ sigma^2 (statistical, many points)
    sig = 2e-3
    P2 = (g[:, :1] * t1 + g[:, 1:] * t2 + rng.normal(0, sig, (900, 1)) * n).astype(np.float32)
    C = oracle.covariance(P2, np.arange(900, dtype=np.int32))
    lam, V = oracle.eigen(C)
    assert abs(lam[2] / sig ** 2 - 1) < 0.15 and abs(abs(V[:, 2] @ n) - 1) < 1e-3


@pytest.mark.parametrize("mode", [oracle.NONE, oracle.PLANE, oracle.ELLIPSE])
def test_target_from_map_roundtrip(mode):
    """a Gaussian built from the eigen-decomposition (R, sqrt(lambda)) of C gives the same
    target covariance as regularising C directly (to binary32 storage precision)."""
    rng = np.random.default_rng(16)
    As = [rand_spd(rng, spread=2.5) for _ in range(300)]
    Rs, S = [], []
    for A in As:
        w, U = np.linalg.eigh(A)
        perm = rng.permutation(3)  # scale axis order is arbitrary in a 3DGS map
        U = U[:, perm]
        if np.linalg.det(U) < 0:
            U[:, 0] *= -1
        Rs.append(U); S.append(np.sqrt(w[perm]))
    q = synth.quat_from_rotmat(np.array(Rs)) * rng.uniform(0.5, 2.0, (300, 1))  # unnormalised on purpose
    S = np.array(S)
    cov, fl = oracle.target_from_map(q.astype(np.float32), S.astype(np.float32), mode)
    cov_log, _ = oracle.target_from_map(q.astype(np.float32), np.log(S).astype(np.float32), mode,
                                        scales_are_log=True)
    for i, A in enumerate(As):
        Af = Rs[i] @ np.diag(S[i] ** 2) @ Rs[i].T  # == A up to rounding; inputs were rounded to binary32
        ref, _ = oracle.regularize(pack(Af), mode, 1e-3)
        np.testing.assert_allclose(cov[i], ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())
        np.testing.assert_allclose(cov_log[i], ref, rtol=1e-5, atol=1e-5 * np.abs(ref).max())


@pytest.mark.parametrize("ex", GOLD["scale_align"])
def test_scale_align_spec_examples(ex):
    np.testing.assert_allclose(oracle.scale_align(ex["scales"], ex["z"], ex["p"]), ex["out"], rtol=1e-15)
    with pytest.raises(ValueError):
        oracle.scale_align(ex["scales"], 0.0, ex["p"])


# ------------------------------------------------------------------ N4 voxel downsampling (R31)
def test_voxel_spec_examples():
    """SPEC S:58-60 worked examples."""
    p, c = oracle.voxel_downsample(np.array([[0.3, -0.2, 1.5]], np.float32), 0.1)
    np.testing.assert_array_equal(p, np.float32([[0.3, -0.2, 1.5]]))
    assert c.tolist() == [1]
    p, c = oracle.voxel_downsample(np.array([[0, 0, 0], [0.01, 0, 0]], np.float32), 0.1)
    np.testing.assert_allclose(p, [[0.005, 0, 0]], rtol=1e-6)
    assert c.tolist() == [2]
    p, c = oracle.voxel_downsample(np.array([[0, 0, 0], [1.0, 0, 0]], np.float32), 0.1)
    assert p.shape == (2, 3) and c.tolist() == [1, 1]


def test_voxel_brute_force_groups():
    """Brute force on a random cloud: one output per distinct floor(x/h) triple (numpy.unique),
    each the binary64 mean of its members (numpy) rounded to binary32, in the order of each voxel's
    first member; counts sum to n; output size <= input size; empty in, empty out."""
    rng = np.random.default_rng(31)
    P = (rng.normal(size=(3000, 3)) * [0.4, 0.3, 0.2] + [0.0, 0.05, 2.0]).astype(np.float32)
    P[5] = np.nan  # skipped
    for h in (0.02, 0.1, 0.37):
        pts, cnt = oracle.voxel_downsample(P, h)
        ok = np.isfinite(P).all(1)
        idx = np.nonzero(ok)[0]
        keys = np.floor(P[idx].astype(np.float64) / np.float64(np.float32(h))).astype(np.int64)
        uk, first, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
        inv = inv.reshape(-1)
        order = np.argsort(idx[first])
        assert pts.shape[0] == uk.shape[0] <= P.shape[0] and cnt.sum() == idx.size
        for j, g_ in enumerate(order):
            mem = idx[inv == g_]
            np.testing.assert_array_equal(pts[j], P[mem].astype(np.float64).mean(0).astype(np.float32))
            assert cnt[j] == mem.size
    e, ce = oracle.voxel_downsample(np.zeros((0, 3), np.float32), 0.1)
    assert e.shape == (0, 3) and ce.size == 0
