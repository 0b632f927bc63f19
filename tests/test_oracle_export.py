"""Pins of the oracle's O12' 3DGS export (ALG-12: Eq. 3-4, Lambda'' = Lambda'/z^p
P:250-255), CPU only.  Library cross-checks (scipy's quaternion -> rotation, numpy eigh), SPEC's
worked scale-aligning examples, the O5 spectrum (pinned in test_oracle_covariance.py)
and closed forms for the pose.
"""
import json
import os

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
MODES = [oracle.NONE, oracle.PLANE, oracle.ELLIPSE]


def pack(A):
    return np.array([A[0, 0], A[0, 1], A[0, 2], A[1, 1], A[1, 2], A[2, 2]])


def unpack(c):
    return np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]], dtype=np.float64)


def rot_of(q_wxyz):
    """scipy (library) quaternion -> rotation; scipy's order is xyzw."""
    w, x, y, z = q_wxyz
    return Rotation.from_quat([x, y, z, w]).as_matrix()


def gauss_cov(q, s):
    R = rot_of(q)
    return R @ np.diag(np.asarray(s) ** 2) @ R.T


def test_spd_with_known_frame_gives_that_frame_and_ellipse_scales():
    """C = R0 diag(lam) R0^T with distinct lam: the exported rotation's columns are R0's columns
    (sorted by lam descending) up to sign, det +1, w >= 0; scales = sqrt(max(lam/lam_mid, eps))."""
    rng = np.random.default_rng(70)
    for _ in range(200):
        R0 = Rotation.random(random_state=rng.integers(1 << 30)).as_matrix()
        lam = np.sort(10.0 ** rng.uniform(-4, 0, 3))[::-1] * [1.5, 1.0, 0.6]  # distinct, descending
        C = R0 @ np.diag(lam) @ R0.T
        z = float(np.float32(rng.uniform(0.3, 6.0)))  # the point is binary32
        mean, q, s, rc = oracle.export_gaussian(pack(C), np.array([0.1, -0.2, z], np.float32))
        assert rc == 0
        assert q[0] >= 0 and abs(np.linalg.norm(q) - 1) < 1e-14
        Rq = rot_of(q)
        assert np.linalg.det(Rq) > 0
        for j in range(3):
            assert abs(abs(Rq[:, j] @ R0[:, j]) - 1) < 1e-9
        ref = np.sqrt(np.maximum(lam / lam[1], 1e-3)) / z ** 1.5
        np.testing.assert_allclose(s, ref, rtol=1e-10)
        np.testing.assert_allclose(mean, [np.float32(0.1), np.float32(-0.2), np.float32(z)], rtol=0, atol=0)


@pytest.mark.parametrize("mode", MODES)
def test_reconstruction_is_the_regularised_covariance_over_z2p(mode):
    """R(q) diag(s^2) R(q)^T * z^(2p) / c^2 == O5's regularised covariance of C (every mode,
    including the degenerate cases of R8: coincident points, collinear points)."""
    rng = np.random.default_rng(71 + mode)
    cases = []
    for _ in range(150):
        Q = np.linalg.qr(rng.normal(size=(3, 3)))[0]
        cases.append(Q @ np.diag(10.0 ** rng.uniform(-5, 0, 3)) @ Q.T)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    cases.append(np.outer(d, d) * 0.04)  # collinear: lam_1 = lam_0 = 0
    cases.append(np.zeros((3, 3)))        # coincident
    cases.append(np.eye(3) * 0.01)        # isotropic: frame arbitrary, covariance unique
    for C in cases:
        z, p, c = rng.uniform(0.5, 5.0), rng.uniform(0.5, 2.0), rng.uniform(0.5, 3.0)
        _, q, s, rc = oracle.export_gaussian(pack(C), np.array([0, 0, z], np.float32), mode=mode, p=p, c=c)
        assert rc == 0
        ref, _ = oracle.regularize(pack(C), mode, 1e-3)
        got = gauss_cov(q, s) * float(np.float32(z)) ** (2 * p) / c ** 2
        np.testing.assert_allclose(pack(got), ref, rtol=0, atol=1e-11 * max(1.0, np.abs(ref).max()))
        assert s[0] >= s[1] >= s[2] >= 0


@pytest.mark.parametrize("ex", GOLD["scale_align"])
def test_spec_scale_align_examples_through_the_export(ex):
    """Lambda' = (2, 1, 0.5) (median 1) at depth z -> the printed Lambda''."""
    lam = np.array(ex["scales"]) ** 2  # C = diag(Lambda'^2), lambda_mid = 1
    _, q, s, rc = oracle.export_gaussian(pack(np.diag(lam)), np.array([0, 0, ex["z"]], np.float32), p=ex["p"])
    assert rc == 0
    np.testing.assert_allclose(s, ex["out"], rtol=1e-14)
    np.testing.assert_allclose(np.abs(rot_of(q)), np.eye(3), atol=1e-14)  # axes stay the coordinate axes


def test_pose_moves_mean_and_rotates_the_gaussian():
    """With T = [Rt | t]: mean = Rt x + t, world covariance = Rt Sigma_cam Rt^T (closed form)."""
    rng = np.random.default_rng(72)
    for _ in range(50):
        Q = np.linalg.qr(rng.normal(size=(3, 3)))[0]
        C = Q @ np.diag(10.0 ** rng.uniform(-3, 0, 3)) @ Q.T
        T = np.eye(4)
        T[:3, :3] = Rotation.random(random_state=rng.integers(1 << 30)).as_matrix()
        T[:3, 3] = rng.normal(size=3)
        x = np.array([0.3, -0.1, 2.5], np.float32)
        _, q0, s0, _ = oracle.export_gaussian(pack(C), x)
        mean, q, s, _ = oracle.export_gaussian(pack(C), x, T=T)
        np.testing.assert_allclose(mean, T[:3, :3] @ x.astype(np.float64) + T[:3, 3], rtol=0, atol=1e-14)
        np.testing.assert_allclose(s, s0, rtol=0, atol=0)
        np.testing.assert_allclose(gauss_cov(q, s), T[:3, :3] @ gauss_cov(q0, s0) @ T[:3, :3].T, atol=1e-12)


def test_nonpositive_depth_is_rejected_with_zero_scales():
    _, q, s, rc = oracle.export_gaussian(pack(np.eye(3)), np.array([0, 0, 0], np.float32))
    assert rc == -1 and np.all(s == 0) and abs(np.linalg.norm(q) - 1) < 1e-14


def test_cloud_export_matches_the_per_point_export():
    rng = np.random.default_rng(73)
    P = (rng.normal(size=(300, 3)) * [0.5, 0.3, 0.02] + [0, 0, 2.0]).astype(np.float32)
    cv = oracle.covariances(P, k=20)
    T = np.eye(4)
    T[:3, 3] = [1.0, 2.0, 3.0]
    means, quats, scales = oracle.export_gaussians(P, cv["raw"], T=T)
    for i in range(0, 300, 7):
        m, q, s, _ = oracle.export_gaussian(cv["raw"][i], P[i], T=T)
        np.testing.assert_array_equal(means[i], m)
        np.testing.assert_array_equal(quats[i], q)
        np.testing.assert_array_equal(scales[i], s)
