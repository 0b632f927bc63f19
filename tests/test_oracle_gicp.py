"""Pins of the oracle's O7-O11 (correspondences, Eq. 1 linearisation, GN solve/update/loop), CPU only.

- SPEC's mle_cost worked examples via single-pair clouds.
- Analytic Jacobian vs central finite differences of the residual d(delta) = m - (Exp(w) q + v)
  with scipy.linalg.expm (library) for Exp, on cases where Sigma has a closed form.
- Cost invariance under a common rigid transform.
- Identity alignment returns a zero update (BJ).
- Known rigid transform recovered (C1 shape, BJ).
- Point-to-point special case C^s = C^t = I/2 => M = I: the GN fixed point equals the Kabsch /
  Umeyama closed form (numpy SVD) on the final correspondences.
- Swap gives the inverse; clouds 100 m apart -> TRACKING_LOST with the init pose.
- Solver / Exp cross-checked against numpy.linalg.solve and scipy.linalg.expm.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.linalg import expm

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def skew(w):
    return np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]], dtype=np.float64)


def pack(A):
    return np.array([A[0, 0], A[0, 1], A[0, 2], A[1, 1], A[1, 2], A[2, 2]])


def rot_err(Ra, Rb):
    return math.acos(max(-1.0, min(1.0, (np.trace(Ra.T @ Rb) - 1) / 2)))


@pytest.mark.parametrize("ex", GOLD["mle_cost"])
def test_mle_cost_spec_examples(ex):
    # one source point at the origin, one target point at d; C^s = C^t = Sigma / 2, T = I
    half = pack(np.diag(ex["Sigma_diag"]) / 2.0).astype(np.float32)
    src = np.zeros((1, 3), np.float32)
    tgt = np.float32([ex["d"]])
    r = oracle.linearize(src, half[None], tgt, half[None], np.eye(4))
    assert r["n"] == 1 and r["cost"] == pytest.approx(ex["cost"], abs=1e-15)


def _numeric_jacobian(q, m, h=1e-6):
    """d(delta) = m - (Exp(w) q + v), central differences in each twist coordinate."""
    J = np.zeros((3, 6))
    for k in range(6):
        e = np.zeros(6); e[k] = h
        rp = m - (expm(skew(e[:3])) @ q + e[3:])
        rm = m - (expm(skew(-e[:3])) @ q - e[3:])
        J[:, k] = (rp - rm) / (2 * h)
    return J


def test_linearize_matches_finite_differences_point_to_point():
    rng = np.random.default_rng(20)
    n = 200
    src = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    tgt = (src + rng.normal(0, 0.01, (n, 3))).astype(np.float32)
    half = np.tile(pack(np.eye(3) / 2), (n, 1)).astype(np.float32)  # M = I
    T = np.eye(4)
    r = oracle.linearize(src, half, tgt, half, T)
    assert r["n"] == n
    H = np.zeros((6, 6)); b = np.zeros(6); cost = 0.0
    for i in range(n):
        q = src[i].astype(np.float64)
        m = tgt[r["corr"][i]].astype(np.float64)
        J = _numeric_jacobian(q, m)
        d = m - q
        H += J.T @ J; b += J.T @ d; cost += d @ d
    np.testing.assert_allclose(r["H"], H, rtol=1e-7, atol=1e-7 * np.abs(H).max())
    np.testing.assert_allclose(r["b"], b, rtol=1e-6, atol=1e-7 * np.abs(b).max())
    assert r["cost"] == pytest.approx(cost, rel=1e-12)


def test_linearize_matches_finite_differences_anisotropic():
    """Translation-only pose (R = I): Sigma = C^t + C^s is a closed form (diagonal covariances)."""
    rng = np.random.default_rng(21)
    n = 150
    src = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    t = np.array([0.003, -0.002, 0.001])
    tgt = (src + t + rng.normal(0, 0.005, (n, 3))).astype(np.float32)
    ds = rng.uniform(0.1, 2.0, (n, 3)); dt = rng.uniform(0.1, 2.0, (n, 3))
    cs = np.zeros((n, 6), np.float32); ct = np.zeros((n, 6), np.float32)
    cs[:, [0, 3, 5]] = ds; ct[:, [0, 3, 5]] = dt
    T = np.eye(4); T[:3, 3] = t
    r = oracle.linearize(src, cs, tgt, ct, T)
    H = np.zeros((6, 6)); b = np.zeros(6)
    for i in range(n):
        j = r["corr"][i]
        q = src[i].astype(np.float64) + t
        m = tgt[j].astype(np.float64)
        Minv = np.diag(1.0 / (cs[i, [0, 3, 5]].astype(np.float64) + ct[j, [0, 3, 5]].astype(np.float64)))
        J = _numeric_jacobian(q, m)
        H += J.T @ Minv @ J; b += J.T @ Minv @ (m - q)
    np.testing.assert_allclose(r["H"], H, rtol=1e-6, atol=1e-7 * np.abs(H).max())
    np.testing.assert_allclose(r["b"], b, rtol=1e-5, atol=1e-6 * np.abs(b).max())
    # H symmetric PSD
    assert np.allclose(r["H"], r["H"].T) and np.linalg.eigvalsh(r["H"]).min() > 0


def _c1_like(seed=1, n_side=(64, 48)):
    w = synth.make_c1(seed)
    K = w.K
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, 1)
    T = w.T_gt
    tgt = (xyz.astype(np.float64) @ T[:3, :3].T + T[:3, 3]).astype(np.float32)
    return xyz, tgt, T


def test_cost_invariant_under_common_rigid_transform():
    xyz, tgt, T = _c1_like()
    cs = oracle.covariances(xyz)["cov"]
    ct = oracle.covariances(tgt)["cov"]
    r0 = oracle.linearize(xyz, cs, tgt, ct, np.eye(4))
    # move the target cloud (and its covariances) by a rigid T0; evaluate at T0 * I
    T0 = np.eye(4); T0[:3, :3] = synth.rot_axis_angle([1.0, 2.0, 3.0], 0.3); T0[:3, 3] = [0.5, -0.2, 0.1]
    R0 = T0[:3, :3]
    tgt2 = (tgt.astype(np.float64) @ R0.T + T0[:3, 3]).astype(np.float32)
    C = np.array([[[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]] for c in ct.astype(np.float64)])
    ct2 = np.array([pack(R0 @ Ci @ R0.T) for Ci in C]).astype(np.float32)
    r1 = oracle.linearize(xyz, cs, tgt2, ct2, T0)
    assert r1["n"] == r0["n"]
    assert r1["cost"] == pytest.approx(r0["cost"], rel=1e-4)


def test_identity_alignment_zero_update():
    xyz, _, _ = _c1_like()
    cs = oracle.covariances(xyz)["cov"]
    r = oracle.linearize(xyz, cs, xyz, cs, np.eye(4))
    assert r["cost"] == 0.0 and np.all(r["b"] == 0.0) and r["n"] == xyz.shape[0]
    delta, ok = oracle.solve(r["H"], r["b"])
    assert ok and np.all(delta == 0.0)
    a = oracle.align(xyz, cs, xyz, cs, np.eye(4))
    assert a["status"] == oracle.OK and a["iters"] == 1
    np.testing.assert_array_equal(a["T"], np.eye(4))


def test_known_rigid_transform_recovered_c1():
    xyz, tgt, T = _c1_like()
    cs = oracle.covariances(xyz)["cov"]
    ct = oracle.covariances(tgt)["cov"]
    a = oracle.align(xyz, cs, tgt, ct, np.eye(4), max_iters=30, eps_rot=0.0, eps_trans=0.0)
    assert a["status"] == oracle.MAX_ITERS and a["iters"] == 30
    assert rot_err(a["T"][:3, :3], T[:3, :3]) < 1e-6
    assert np.linalg.norm(a["T"][:3, 3] - T[:3, 3]) < 1e-6
    assert a["fitness"] == 1.0


def _kabsch(P, Q):
    """R, t minimising sum |R p + t - q|^2 (Umeyama without scale)."""
    mp, mq = P.mean(0), Q.mean(0)
    U, S, Vt = np.linalg.svd((Q - mq).T @ (P - mp))
    D = np.diag([1, 1, np.sign(np.linalg.det(U @ Vt))])
    R = U @ D @ Vt
    return R, mq - R @ mp


def test_point_to_point_equals_kabsch():
    rng = np.random.default_rng(22)
    n = 500
    src = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    Tg = np.eye(4); Tg[:3, :3] = synth.rot_axis_angle(rng.normal(size=3), 0.1); Tg[:3, 3] = [0.05, 0.02, -0.03]
    tgt = (src.astype(np.float64) @ Tg[:3, :3].T + Tg[:3, 3] + rng.normal(0, 0.01, (n, 3))).astype(np.float32)
    half = np.tile(pack(np.eye(3) / 2), (n, 1)).astype(np.float32)
    a = oracle.align(src, half, tgt, half, np.eye(4), max_iters=100, eps_rot=1e-12, eps_trans=1e-12)
    r = oracle.linearize(src, half, tgt, half, a["T"])
    R, t = _kabsch(src.astype(np.float64), tgt[r["corr"]].astype(np.float64))
    assert np.abs(a["T"][:3, :3] - R).max() < 1e-9 and np.abs(a["T"][:3, 3] - t).max() < 1e-9


def test_swap_gives_inverse_and_lost_tracking():
    xyz, tgt, T = _c1_like()
    cs = oracle.covariances(xyz)["cov"]
    ct = oracle.covariances(tgt)["cov"]
    a = oracle.align(xyz, cs, tgt, ct, np.eye(4))
    b = oracle.align(tgt, ct, xyz, cs, np.eye(4))
    D = a["T"] @ b["T"]
    assert rot_err(D[:3, :3], np.eye(3)) < 1e-3 and np.linalg.norm(D[:3, 3]) < 1e-3
    far = (tgt + np.float32([100.0, 0, 0])).astype(np.float32)
    T0 = np.eye(4); T0[0, 3] = 0.01
    c = oracle.align(xyz, cs, far, ct, T0, max_corr_dist=0.5)
    assert c["status"] == oracle.TRACKING_LOST and c["fitness"] == 0.0
    np.testing.assert_array_equal(c["T"], T0)


def test_acceptance_random_box_clouds():
    """S:578 acceptance (reduced to 20 trials for CPU time): 500-point box-surface clouds,
    T_gt <= 10 deg / 0.1 m, recovered within 0.5 deg / 5 mm."""
    rng = np.random.default_rng(23)
    ok = 0
    trials = 20
    for _ in range(trials):
        face = rng.integers(0, 6, 500)
        p = rng.uniform(-0.5, 0.5, (500, 3))
        p[np.arange(500), face // 2] = np.where(face % 2 == 0, -0.5, 0.5)
        src = (p * [1.0, 0.8, 0.6]).astype(np.float32)
        Tg = np.eye(4)
        Tg[:3, :3] = synth.rot_axis_angle(rng.normal(size=3), math.radians(rng.uniform(0, 10)))
        Tg[:3, 3] = rng.normal(size=3); Tg[:3, 3] *= rng.uniform(0, 0.1) / np.linalg.norm(Tg[:3, 3])
        # target: an independent sample of the same box surface, moved by T_gt
        face = rng.integers(0, 6, 500)
        p = rng.uniform(-0.5, 0.5, (500, 3))
        p[np.arange(500), face // 2] = np.where(face % 2 == 0, -0.5, 0.5)
        tgt = ((p * [1.0, 0.8, 0.6]) @ Tg[:3, :3].T + Tg[:3, 3]).astype(np.float32)
        cs = oracle.covariances(src, mode=oracle.PLANE)["cov"]
        ct = oracle.covariances(tgt, mode=oracle.PLANE)["cov"]
        a = oracle.align(src, cs, tgt, ct, np.eye(4), max_corr_dist=0.5)
        ok += rot_err(a["T"][:3, :3], Tg[:3, :3]) < math.radians(0.5) and \
            np.linalg.norm(a["T"][:3, 3] - Tg[:3, 3]) < 5e-3
    assert ok >= trials - 1


def test_solve_and_exp_library_crosscheck():
    rng = np.random.default_rng(24)
    A = rng.normal(size=(6, 6)); H = A @ A.T + 0.1 * np.eye(6); b = rng.normal(size=6)
    x, ok = oracle.solve(H, b)
    assert ok
    np.testing.assert_allclose(x, -np.linalg.solve(H, b), rtol=1e-10)
    for w in (rng.normal(size=3), rng.normal(size=3) * 1e-9, np.zeros(3)):
        np.testing.assert_allclose(oracle.so3_exp(w), expm(skew(w)), atol=1e-14)
    T = np.eye(4); T[:3, :3] = synth.rot_axis_angle([0, 0, 1], 0.2); T[:3, 3] = [1, 2, 3]
    d = rng.normal(size=6) * 0.1
    Tn = oracle.update(T, d)
    E = np.eye(4); E[:3, :3] = expm(skew(d[:3])); E[:3, 3] = d[3:]
    np.testing.assert_allclose(Tn, E @ T, atol=1e-14)


def test_kdtree_linearize_equals_brute():
    xyz, tgt, T = _c1_like()
    cs = oracle.covariances(xyz)["cov"]
    ct = oracle.covariances(tgt)["cov"]
    Tp = synth.perturb_pose(T, 5)
    a = oracle.linearize(xyz, cs, tgt, ct, Tp, max_corr_dist=0.1)
    b = oracle.linearize(xyz, cs, tgt, ct, Tp, max_corr_dist=0.1, tree=oracle.KDTree(tgt))
    np.testing.assert_array_equal(a["corr"], b["corr"])
    np.testing.assert_array_equal(a["H"], b["H"])


# ------------------------------------------------------------------ Levenberg-Marquardt (R30)
@pytest.mark.parametrize("lam0", [1e-2, 1.0, 1e3])
def test_lm_first_step_closed_form(lam0):
    """The first LM step is delta = -(H + lam0 diag(H))^-1 b at T0 (numpy.linalg.solve) and the
    pose Exp(delta) T0 with Exp = scipy.linalg.expm of the twist's rotation (left update)."""
    xyz, tgt, T = _c1_like()
    cs = oracle.covariances(xyz)["cov"]
    ct = oracle.covariances(tgt)["cov"]
    T0 = np.eye(4)
    r = oracle.linearize(xyz, cs, tgt, ct, T0)
    D = r["H"] + lam0 * np.diag(np.diag(r["H"]))
    delta = np.linalg.solve(D, -r["b"])
    E = expm(skew(delta[:3]))
    ref = np.eye(4)
    ref[:3, :3] = E @ T0[:3, :3]
    ref[:3, 3] = E @ T0[:3, 3] + delta[3:]
    a = oracle.align(xyz, cs, tgt, ct, T0, max_iters=5, eps_rot=1e9, eps_trans=1e9, solver=1, lm_lambda0=lam0)
    assert a["status"] == oracle.OK and a["iters"] == 1
    np.testing.assert_allclose(a["T"], ref, rtol=0, atol=1e-12)
    assert a["n_inliers"] == r["n"] and abs(a["mean_cost"] - r["cost"] / r["n"]) <= 1e-12 * r["cost"] / r["n"]


def test_lm_identity_and_known_transform():
    """Identical clouds: one iteration, zero update.  C1 known transform: LM reaches the
    same optimum as GN (the transform, 1e-6) and the two fixed points agree to 1e-9."""
    xyz, tgt, T = _c1_like()
    cs = oracle.covariances(xyz)["cov"]
    ct = oracle.covariances(tgt)["cov"]
    a = oracle.align(xyz, cs, xyz, cs, np.eye(4), solver=1)
    assert a["status"] == oracle.OK and a["iters"] == 1
    np.testing.assert_array_equal(a["T"], np.eye(4))
    lm = oracle.align(xyz, cs, tgt, ct, np.eye(4), max_iters=60, eps_rot=1e-10, eps_trans=1e-10, solver=1)
    gn = oracle.align(xyz, cs, tgt, ct, np.eye(4), max_iters=60, eps_rot=1e-10, eps_trans=1e-10)
    assert lm["converged"] and gn["converged"]
    assert rot_err(lm["T"][:3, :3], T[:3, :3]) < 1e-6 and np.linalg.norm(lm["T"][:3, 3] - T[:3, 3]) < 1e-6
    assert rot_err(lm["T"][:3, :3], gn["T"][:3, :3]) < 1e-9 and np.abs(lm["T"][:3, 3] - gn["T"][:3, 3]).max() < 1e-9


def test_lm_point_to_point_equals_kabsch_and_best_iterate_at_cap():
    """Point-to-point (M = I): the LM fixed point is the Kabsch closed form on its final
    correspondences.  At the iteration cap LM returns its best accepted iterate: its cost is
    never above the initial pose's."""
    rng = np.random.default_rng(23)
    n = 500
    src = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    Tg = np.eye(4); Tg[:3, :3] = synth.rot_axis_angle(rng.normal(size=3), 0.3); Tg[:3, 3] = [0.1, -0.05, 0.08]
    tgt = (src.astype(np.float64) @ Tg[:3, :3].T + Tg[:3, 3] + rng.normal(0, 0.01, (n, 3))).astype(np.float32)
    half = np.tile(pack(np.eye(3) / 2), (n, 1)).astype(np.float32)
    a = oracle.align(src, half, tgt, half, np.eye(4), max_iters=200, eps_rot=1e-12, eps_trans=1e-12, solver=1)
    r = oracle.linearize(src, half, tgt, half, a["T"])
    R, t = _kabsch(src.astype(np.float64), tgt[r["corr"]].astype(np.float64))
    assert np.abs(a["T"][:3, :3] - R).max() < 1e-9 and np.abs(a["T"][:3, 3] - t).max() < 1e-9
    c0 = oracle.linearize(src, half, tgt, half, np.eye(4), max_corr_dist=0.2)["cost"]
    for cap in (1, 2, 3):
        b = oracle.align(src, half, tgt, half, np.eye(4), max_iters=cap, eps_rot=0.0, eps_trans=0.0, solver=1,
                         max_corr_dist=0.2, lm_lambda0=10.0)
        assert b["status"] == oracle.MAX_ITERS
        cb = oracle.linearize(src, half, tgt, half, b["T"], max_corr_dist=0.2)["cost"]
        assert cb <= c0


# ------------------------------------------------------------------ O7 on the binary64 query (R15)
_HALF_I = pack(np.eye(3) / 2.0).astype(np.float32)


def test_nn_uses_binary64_query_not_its_binary32_rounding():
    """q = K3(T, x) = 1 + 2^-23 - 2^-30 (x = 1 + 2^-23, t = -2^-30): exactly one of two targets
    1 and 1 + 2^-22 is nearer (distances 2^-23 - 2^-30 vs 2^-23 + 2^-30), but fl32(q) = 1 + 2^-23
    is their midpoint (a binary32 tie, which the lower index, the farther target, would win)."""
    x = np.float32([[1.0 + 2.0 ** -23, 0.0, 0.0]])
    assert float(x[0, 0]) == 1.0 + 2.0 ** -23
    tgt = np.float32([[1.0 + 2.0 ** -22, 0, 0], [1.0, 0, 0]])  # index 0 is the farther one
    T = np.eye(4)
    T[0, 3] = -(2.0 ** -30)
    r = oracle.linearize(x, _HALF_I[None], tgt, np.repeat(_HALF_I[None], 2, 0), T)
    assert r["corr"][0] == 1
    # exact rational check of the claim
    q = 1.0 + 2.0 ** -23 - 2.0 ** -30
    assert abs(q - 1.0) < abs(q - (1.0 + 2.0 ** -22))
    assert np.float32(q) == np.float32(1.0 + 2.0 ** -23)
    # the kd-tree path takes the same decision
    r2 = oracle.linearize(x, _HALF_I[None], tgt, np.repeat(_HALF_I[None], 2, 0), T, tree=oracle.KDTree(tgt))
    assert r2["corr"][0] == 1


def test_nn_equal_distance_tie_goes_to_lower_index():
    x = np.float32([[0.0, 0.0, 0.0]])
    tgt = np.float32([[0, 0.25, 0], [0.25, 0, 0], [0, 0, -0.25]])  # all at exactly 1/4
    r = oracle.linearize(x, _HALF_I[None], tgt, np.repeat(_HALF_I[None], 3, 0), np.eye(4))
    assert r["corr"][0] == 0


def test_correspondence_gate_is_strict():
    """R15: valid iff key < r^2.  A target at exactly r (0.5: key 0.25 = r^2) is rejected; one
    binary32 ulp closer is accepted."""
    x = np.zeros((1, 3), np.float32)
    for d, valid in ((0.5, False), (float(np.nextafter(np.float32(0.5), np.float32(0))), True)):
        tgt = np.float32([[d, 0, 0]])
        r = oracle.linearize(x, _HALF_I[None], tgt, _HALF_I[None], np.eye(4), max_corr_dist=0.5)
        assert (r["n"] == 1) == valid and (r["corr"][0] == 0) == valid


def test_non_pd_sigma_pair_is_skipped():
    """A pair whose Sigma = C^t + R C^s R^T is not positive definite contributes nothing."""
    x = np.float32([[0, 0, 0], [1, 0, 0]])
    tgt = np.float32([[0, 0, 0.01], [1, 0, 0.01]])
    zero = np.zeros(6, np.float32)
    r = oracle.linearize(x, np.stack([zero, _HALF_I]), tgt, np.stack([zero, _HALF_I]), np.eye(4))
    assert r["n"] == 1 and r["corr"][0] == -1 and r["corr"][1] == 1
    np.testing.assert_allclose(r["cost"], np.float64(np.float32(0.01)) ** 2, rtol=1e-12)  # M = I


def test_solve_pd_fallback():
    """A8/O9: a singular H (zero eigenvalue) is solved as H + 1e-6 tr(H)/6 I (numpy.linalg.solve);
    a negative definite H fails both attempts."""
    H = np.diag([1.0, 2.0, 3.0, 4.0, 5.0, 0.0])
    b = np.array([1.0, -1.0, 2.0, 0.5, 1.0, 0.25])
    x, ok = oracle.solve(H, b)
    assert ok
    np.testing.assert_allclose(x, np.linalg.solve(H + 1e-6 * 15.0 / 6.0 * np.eye(6), -b), rtol=1e-12)
    x, ok = oracle.solve(-np.eye(6), b)
    assert not ok


def test_linearize_bsum_is_sum_of_per_pair_b_norms():
    """bsum = sum_i |J_i^T M_i d_i| (SURVEY §8(c).5's b scale): with one valid pair it equals |b|;
    with two pairs whose contributions cancel it is the sum of the two norms while b = 0."""
    x = np.float32([[0, 0, 0]])
    r = oracle.linearize(x, _HALF_I[None], np.float32([[0.3, 0, 0]]), _HALF_I[None], np.eye(4))
    assert r["bsum"] == pytest.approx(np.linalg.norm(r["b"]), rel=1e-15)
    x2 = np.float32([[0, 0, 0], [0, 0, 0]])
    # two points at the origin matched to targets at +-0.3 x: contributions cancel
    r2 = oracle.linearize(x2[:1], _HALF_I[None], np.float32([[0.3, 0, 0]]), _HALF_I[None], np.eye(4))
    r3 = oracle.linearize(x2[:1], _HALF_I[None], np.float32([[-0.3, 0, 0]]), _HALF_I[None], np.eye(4))
    assert r2["bsum"] == pytest.approx(r3["bsum"]) and np.allclose(r2["b"] + r3["b"], 0)
