"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star, made precise in SURVEY §8(c).5 / DESIGN.md §6):
  A1 points and kNN indices (binary64 K2 order, ties by index): bit-exact;
  covariances: per-point ||dC||_F <= 1e-4 ||C||_F;
  H/b per linearisation at the same T — every GN iteration, at the pose the GPU iteration used:
  ||dH||_F <= 1e-4 ||H||_F, ||db|| <= 1e-4 * sum_i ||J_i^T M_i d_i|| (the oracle's bsum), cost rel 1e-4,
  inliers and every correspondence exact;  final pose from the same init: 1e-5 rad and 1e-5 m.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

FULL_M = 1_000_000


@pytest.fixture(scope="module")
def g():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2403_12550_b200 as g

    g.lib()
    return g


DEV = "cuda"


def t(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def rot_angle(Ra, Rb):
    return math.acos(max(-1.0, min(1.0, (np.trace(Ra.T @ Rb) - 1) / 2)))


def cov_rel_err(a, b):
    def full(c):
        return np.stack([c[:, 0], c[:, 1], c[:, 2], c[:, 1], c[:, 3], c[:, 4], c[:, 2], c[:, 4], c[:, 5]], 1)

    A, B = full(np.asarray(a, np.float64)), full(np.asarray(b, np.float64))
    return np.linalg.norm(A - B, axis=1) / np.linalg.norm(B, axis=1)


# ----------------------------------------------------------------------------------------- workloads
@pytest.fixture(scope="module")
def c1():
    return synth.make_c1(1)


@pytest.fixture(scope="module")
def replica():
    return synth.make_frame_workload(2, "replica", M=FULL_M, stride=4)


@pytest.fixture(scope="module")
def tum():
    return synth.make_frame_workload(3, "tum", M=FULL_M, stride=1, noisy=True)


def gpu_points(g, depth, K, stride):
    pos, d_n = g.backproject_downsample(t(depth), (K.fx, K.fy, K.cx, K.cy), stride=stride)
    return pos, d_n


# ----------------------------------------------------------------------------------------- A1
@pytest.mark.parametrize("case", ["c1", "replica4", "tum1", "tum4", "tum3"])
def test_backproject_bit_exact(g, c1, replica, tum, case):
    w, s = {"c1": (c1, 1), "replica4": (replica, 4), "tum1": (tum, 1), "tum4": (tum, 4), "tum3": (tum, 3)}[case]
    K = w.K
    pos, d_n = gpu_points(g, w.depth, K, s)
    n = int(d_n.item())
    oxyz, opix = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, s)
    assert n == oxyz.shape[0]
    gp = pos[:n].cpu().numpy()
    np.testing.assert_array_equal(gp[:, :3], oxyz)
    np.testing.assert_array_equal(gp[:, 3].view(np.int32), opix)


def test_backproject_edge_cases(g):
    K = (50.0, 50.0, 20.0, 15.0)
    depth = np.zeros((31, 41), np.float32)
    pos, d_n = g.backproject_downsample(t(depth), K, stride=2)
    assert int(d_n.item()) == 0
    depth[:] = np.nan
    depth[3, 4] = np.inf
    depth[10, 10] = 0.5
    depth[10, 12] = 10.5
    pos, d_n = g.backproject_downsample(t(depth), K, stride=2)
    assert int(d_n.item()) == 1 and pos[0, 2].item() == 0.5
    # pitched rows
    big = torch.zeros((31, 64), dtype=torch.float32, device=DEV)
    big[:, :41] = torch.rand((31, 41), device=DEV) * 3 + 0.2
    view = big[:, :41]
    pos, d_n = g.backproject_downsample(view, K, stride=3)
    oxyz, _ = oracle.backproject(view.cpu().numpy(), *K, 3)
    n = int(d_n.item())
    np.testing.assert_array_equal(pos[:n, :3].cpu().numpy(), oxyz)


# ----------------------------------------------------------------------------------------- A2-A4
def _cov_check(g, xyz_np, pos, d_n, k=20, mode=oracle.ELLIPSE, cell0=0.01, levels=5, sample=None, brute_max=60000,
               image=None):
    """image = (H, W, stride, K): run the image-window path (gsicp_covariances_image) instead."""
    n = xyz_np.shape[0]
    knn = torch.full((pos.shape[0], k), -7, dtype=torch.int32, device=DEV)
    if image is None:
        cl = g.covariances(pos, d_n, k=k, mode=mode, eps_var=1e-3, cell0=cell0, levels=levels, knn_idx=knn)
    else:
        H, W, s, K = image
        cl = g.covariances_image(pos, d_n, H, W, s, (K.fx, K.fy, K.cx, K.cy), k=k, mode=mode, eps_var=1e-3,
                                 cell0=cell0, levels=levels, knn_idx=knn)
    gk = knn[:n].cpu().numpy()
    gc = cl.cov6()[:n].cpu().numpy()
    gf = cl.flags()[:n].cpu().numpy()
    if sample is None:
        ok = oracle.knn_brute(xyz_np, k) if n <= brute_max else oracle.KDTree(xyz_np).knn(xyz_np, k)
        np.testing.assert_array_equal(gk, ok)
        ref = oracle.covariances(xyz_np, k=k, mode=mode, brute_max=brute_max)
        idx = np.arange(n)
    else:
        idx = np.random.default_rng(7).choice(n, size=min(sample, n), replace=False).astype(np.int32)
        ok = oracle.knn_brute(xyz_np, k, queries=idx) if n * len(idx) <= 4e9 else \
            oracle.KDTree(xyz_np).knn(xyz_np[idx], k)
        np.testing.assert_array_equal(gk[idx], ok)
        ref = None
    if ref is not None:
        err = cov_rel_err(gc, ref["cov"])
        if mode == oracle.PLANE:
            lam = np.array([oracle.eigen(c)[0] for c in ref["raw"]])
            good = (lam[:, 1] - lam[:, 2]) >= 1e-3 * lam[:, 0]
            assert good.mean() > 0.5
            assert err[good].max() <= 1e-4, err[good].max()
        else:
            assert err.max() <= 1e-4, (err.max(), np.argmax(err))
        np.testing.assert_array_equal(gf, ref["flags"])
    else:  # sampled: covariances from the oracle's own neighbour sets
        for j, i in enumerate(idx):
            C = oracle.covariance(xyz_np, ok[j])
            R, fl = oracle.regularize(C, mode, 1e-3)
            e = cov_rel_err(gc[i:i + 1], R.astype(np.float32)[None])[0]
            assert e <= 1e-4 and gf[i] == fl, (i, e)
    return cl


def test_knn_cov_c1(g, c1):
    K = c1.K
    pos, d_n = gpu_points(g, c1.depth, K, 1)
    xyz, _ = oracle.backproject(c1.depth, K.fx, K.fy, K.cx, K.cy, 1)
    for k in (1, 5, 20, 32):
        _cov_check(g, xyz, pos, d_n, k=k, cell0=0.05, levels=3)


@pytest.mark.parametrize("mode", [oracle.NONE, oracle.PLANE, oracle.ELLIPSE])
def test_knn_cov_replica_full(g, replica, mode):
    K = replica.K
    pos, d_n = gpu_points(g, replica.depth, K, 4)
    xyz, _ = oracle.backproject(replica.depth, K.fx, K.fy, K.cx, K.cy, 4)
    _cov_check(g, xyz, pos, d_n, mode=mode, cell0=0.005, levels=6)


def test_knn_cov_tum_full_resolution(g, tum):
    K = tum.K
    pos, d_n = gpu_points(g, tum.depth, K, 1)
    xyz, _ = oracle.backproject(tum.depth, K.fx, K.fy, K.cx, K.cy, 1)
    _cov_check(g, xyz, pos, d_n, cell0=0.004, levels=6)


@pytest.mark.parametrize("levels,cell0", [(1, 0.02), (1, 0.2), (3, 0.003), (8, 0.001), (1, 0.0), (4, 0.0)])
def test_knn_cov_grid_params_do_not_change_results(g, replica, levels, cell0):
    K = replica.K
    pos, d_n = gpu_points(g, replica.depth, K, 4)
    xyz, _ = oracle.backproject(replica.depth, K.fx, K.fy, K.cx, K.cy, 4)
    _cov_check(g, xyz, pos, d_n, cell0=cell0, levels=levels, sample=3000)


# ----------------------------------------------------------------------------------------- A3/A4 image window
@pytest.mark.parametrize("case", ["c1", "replica4", "tum1", "tum3", "tum4"])
def test_knn_cov_image_window(g, c1, replica, tum, case):
    """gsicp_covariances_image == the oracle's brute-force kNN (bit-exact) and covariances."""
    w, s = {"c1": (c1, 1), "replica4": (replica, 4), "tum1": (tum, 1), "tum3": (tum, 3), "tum4": (tum, 4)}[case]
    K = w.K
    H, W = w.depth.shape
    pos, d_n = gpu_points(g, w.depth, K, s)
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, s)
    ks = (1, 5, 20, 32) if case == "c1" else (20,)
    for k in ks:
        _cov_check(g, xyz, pos, d_n, k=k, cell0=3.0 * s / K.fx, levels=4, image=(H, W, s, K),
                   sample=4000 if case == "tum1" else None)


def test_knn_cov_image_window_modes_and_ties(g, replica):
    """PLANE / NONE modes, and a fronto-parallel wall (tie-heavy lattice), through the image path."""
    K = replica.K
    H, W = replica.depth.shape
    pos, d_n = gpu_points(g, replica.depth, K, 4)
    xyz, _ = oracle.backproject(replica.depth, K.fx, K.fy, K.cx, K.cy, 4)
    for mode in (oracle.NONE, oracle.PLANE):
        _cov_check(g, xyz, pos, d_n, mode=mode, cell0=0.02, levels=4, image=(H, W, 4, K))
    wall = np.full((96, 128), 2.0, np.float32)
    wall[40:60, 50:90] = np.nan  # a hole
    Kw = synth.Intrinsics(W=128, H=96, fx=64.0, fy=64.0, cx=63.5, cy=47.5)
    pos, d_n = gpu_points(g, wall, Kw, 1)
    xyz, _ = oracle.backproject(wall, Kw.fx, Kw.fy, Kw.cx, Kw.cy, 1)
    _cov_check(g, xyz, pos, d_n, cell0=0.1, levels=3, image=(96, 128, 1, Kw))


@pytest.mark.parametrize("path", ["image", "hash"])
def test_knn_cov_fronto_parallel_wall_replica(g, path):
    """SURVEY hard part 1 at full size: the 1200x680 stride-4 fronto-parallel wall at 2 m (51k points
    on an exact lattice: binary32 keys pick another k=20 set than exact kNN on ~4% of queries).
    Every kNN list bit-exact against the oracle's binary64 (K2, index) order, covariances 1e-4."""
    K = synth.REPLICA
    depth = synth.fronto_parallel_wall(K, hole=(300, 380, 500, 700))
    pos, d_n = gpu_points(g, depth, K, 4)
    xyz, _ = oracle.backproject(depth, K.fx, K.fy, K.cx, K.cy, 4)
    image = (K.H, K.W, 4, K) if path == "image" else None
    _cov_check(g, xyz, pos, d_n, cell0=0.02, levels=3, image=image)


def test_knn_cov_image_window_non_frame_cloud(g):
    """A cloud whose pixel ids are not a lattice of the image is detected and searched by the hash."""
    rng = np.random.default_rng(11)
    n = 3000
    xyz = rng.normal(size=(n, 3)).astype(np.float32) + np.float32([0, 0, 4])
    pos = torch.zeros((n, 4), dtype=torch.float32, device=DEV)
    pos[:, :3] = t(xyz)
    pos[:, 3] = t(np.zeros(n, np.int32).view(np.float32))  # every point claims pixel 0
    d_n = torch.tensor([n], dtype=torch.int32, device=DEV)
    K = synth.make_c1(1).K
    _cov_check(g, xyz, pos, d_n, cell0=0.3, levels=3, image=(48, 64, 1, K))
    # the same through a CUDA graph: the hash tail is then the body of a conditional node that
    # the device switches on (every query needs the hash here); results identical to eager
    Kt = (K.fx, K.fy, K.cx, K.cy)
    ws = g._ws(g.lib().gsicp_covariances_image_workspace_size(n, 3, 48, 64, 1), DEV)
    knn_e = torch.full((n, 20), -7, dtype=torch.int32, device=DEV)
    ce = g.covariances_image(pos, d_n, 48, 64, 1, Kt, 20, cell0=0.3, levels=3, knn_idx=knn_e, ws=ws)
    ca_e, cb_e = ce.cov_a.clone(), ce.cov_b.clone()
    knn_g = torch.full((n, 20), -7, dtype=torch.int32, device=DEV)
    ca_g, cb_g = torch.zeros_like(ca_e), torch.zeros_like(cb_e)
    st = torch.cuda.Stream()
    fg = g.FrameGraph()
    with fg.capture(st):
        g.covariances_image(pos, d_n, 48, 64, 1, Kt, 20, cell0=0.3, levels=3, cov_a=ca_g, cov_b=cb_g, knn_idx=knn_g,
                            ws=ws, stream=st)
    fg.replay(st)
    st.synchronize()
    assert torch.equal(knn_g, knn_e) and torch.equal(ca_g, ca_e) and torch.equal(cb_g, cb_e)


def test_knn_cov_ragged_and_low_support(g):
    rng = np.random.default_rng(9)
    for n, cap in ((5, 64), (19, 19), (20, 1000), (1000, 1037), (4097, 5000)):
        xyz = rng.normal(size=(n, 3)).astype(np.float32)
        pos = torch.zeros((cap, 4), dtype=torch.float32, device=DEV)
        pos[:n, :3] = t(xyz)
        d_n = torch.tensor([n], dtype=torch.int32, device=DEV)
        cl = _cov_check(g, xyz, pos, d_n, cell0=0.3, levels=2)
        fl = cl.flags()[:n].cpu().numpy()
        assert bool((fl & oracle.FLAG_LOW_SUPPORT).all()) == (n < 20)


def test_knn_cov_degenerate_clouds(g):
    # coincident points, collinear points, planar lattice with exact ties
    pts = [np.tile(np.float32([[0.5, -1.0, 2.0]]), (40, 1)),
           (np.arange(60)[:, None] * 0.01 * np.array([[1.0, 2.0, 2.0]]) / 3.0).astype(np.float32),
           np.concatenate([np.stack(np.meshgrid(np.arange(30), np.arange(30)), -1).reshape(-1, 2) * 0.01,
                           np.full((900, 1), 1.0)], 1).astype(np.float32)]
    for xyz in pts:
        n = xyz.shape[0]
        pos = torch.zeros((n, 4), dtype=torch.float32, device=DEV)
        pos[:, :3] = t(xyz)
        d_n = torch.tensor([n], dtype=torch.int32, device=DEV)
        for mode in (oracle.NONE, oracle.ELLIPSE):
            _cov_check(g, xyz, pos, d_n, mode=mode, cell0=0.02, levels=2)


def test_knn_cov_brick_edge_cases(g):
    """The brick kernel's corner paths against the oracle (every query, bit-exact lists): a
    brick holding more points than one 32-lane round (a 70-point blob: a lone brick over several
    rounds) and one holding more than its query list (600 points in one cell), a staging
    overflow (a 27-brick neighbourhood beyond the 448-candidate buffer), isolated points with fewer
    than k points in their 27 bricks, and exact-distance ties on a lattice crossing brick faces."""
    rng = np.random.default_rng(77)
    plane = np.concatenate([rng.uniform(-0.3, 0.3, (6000, 2)), np.zeros((6000, 1))], 1)
    blob = rng.normal(0.0, 0.002, (600, 3)) + np.array([0.05, 0.05, 0.0])
    blob2 = rng.normal(0.0, 0.0015, (70, 3)) + np.array([-0.2, 0.1, 0.5])  # one brick, several rounds
    far = rng.uniform(-2.0, 2.0, (40, 3)) + np.array([0.0, 0.0, 3.0])
    lat = np.concatenate([np.stack(np.meshgrid(np.arange(12), np.arange(12)), -1).reshape(-1, 2) * 0.01 + 0.4,
                          np.full((144, 1), 0.2)], 1)
    xyz = np.concatenate([plane, blob, blob2, far, lat]).astype(np.float32)
    n = xyz.shape[0]
    pos = torch.zeros((n, 4), dtype=torch.float32, device=DEV)
    pos[:, :3] = t(xyz)
    d_n = torch.tensor([n], dtype=torch.int32, device=DEV)
    for cell0, levels in ((0.02, 3), (0.04, 2)):
        _cov_check(g, xyz, pos, d_n, mode=oracle.ELLIPSE, cell0=cell0, levels=levels)


@pytest.mark.parametrize("cell,levels,sample", [(2.5, 1, 300), (3.4, 3, 100_000), (6.5, 1, 300)])
def test_knn_cov_map_c4_sampled(g, cell, levels, sample):
    """C4-style: kNN covariance of a 4e6-point map (sampled queries vs the oracle's exact kd-tree /
    brute force); levels=1 is the warp search of every point, (3.4, 3) the bench configuration."""
    scene = synth.make_scene(1004)
    means, _, _, ell = synth.sample_map(scene, 4_000_000, 4004)
    pos = torch.zeros((means.shape[0], 4), dtype=torch.float32, device=DEV)
    pos[:, :3] = t(means)
    d_n = torch.tensor([means.shape[0]], dtype=torch.int32, device=DEV)
    _cov_check(g, means, pos, d_n, cell0=cell * ell, levels=levels, sample=sample)


def test_knn_cov_map_two_phase_full(g):
    """A 3e5-point map (above the two-phase grid build's 2^18 capacity threshold: level 0 from the
    randomly ordered points, levels 1-2 from level 0's cell-ordered records, their alloc over the
    created-cell list) at the bench's brick grid (3.4 spacings x 3 levels): EVERY query's neighbour
    list and covariance against the oracle (the floating outliers reach the coarse levels)."""
    scene = synth.make_scene(1004)
    means, _, _, ell = synth.sample_map(scene, 300_000, 4104)
    assert means.shape[0] >= 1 << 18
    pos = torch.zeros((means.shape[0], 4), dtype=torch.float32, device=DEV)
    pos[:, :3] = t(means)
    d_n = torch.tensor([means.shape[0]], dtype=torch.int32, device=DEV)
    _cov_check(g, means, pos, d_n, cell0=3.4 * ell, levels=3)


# ----------------------------------------------------------------------------------------- A5
@pytest.mark.parametrize("mode,log", [(oracle.ELLIPSE, False), (oracle.PLANE, False), (oracle.NONE, True)])
def test_build_target_covariances(g, mode, log):
    scene = synth.make_scene(1005)
    means, quats, scales, ell = synth.sample_map(scene, 200_000, 4005)
    if log:
        scales = np.log(scales).astype(np.float32)
    tgt = g.build_target(t(means), t(quats), t(scales), scales_are_log=log, mode=mode, eps_var=1e-3)
    M = means.shape[0]
    pos, ca, cb = tgt.arrays()  # cell-ordered views into the target workspace
    order = pos[:, 3].contiguous().view(torch.int32).long().cpu().numpy()
    assert np.array_equal(np.sort(order), np.arange(M))
    inv = np.empty(M, np.int64)
    inv[order] = np.arange(M)
    np.testing.assert_array_equal(pos[:, :3].cpu().numpy()[inv], means)
    gc = torch.cat([ca, cb[:, :2]], 1).cpu().numpy()[inv]
    gf = cb[:, 3].contiguous().view(torch.int32).cpu().numpy()[inv]
    ref, fl = oracle.target_from_map(quats, scales, mode, scales_are_log=log)
    err = cov_rel_err(gc, ref)
    assert err.max() <= 1e-4, err.max()
    np.testing.assert_array_equal(gf, fl)


# ----------------------------------------------------------------------------------------- A6-A9
@pytest.fixture(scope="module")
def c1_setup(g, c1):
    K = c1.K
    xyz, _ = oracle.backproject(c1.depth, K.fx, K.fy, K.cx, K.cy, 1)
    T = c1.T_gt
    txyz = (xyz.astype(np.float64) @ T[:3, :3].T + T[:3, 3]).astype(np.float32)
    pos, d_n = gpu_points(g, c1.depth, K, 1)
    src = g.covariances(pos, d_n, cell0=0.0, levels=3)  # automatic cell sizes
    tc = g.Cloud.from_points(t(txyz))
    tcl = g.covariances(tc.pos, tc.d_n, cell0=0.0, levels=3)
    tgt = g.build_target_cloud(tcl)
    ocs = oracle.covariances(xyz)["cov"]
    oct_ = oracle.covariances(txyz)["cov"]
    return dict(xyz=xyz, txyz=txyz, src=src, tgt=tgt, ocs=ocs, oct=oct_, T=T)


@pytest.fixture(scope="module")
def replica_setup(g, replica):
    w = replica
    K = w.K
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, 4)
    pos, d_n = gpu_points(g, w.depth, K, 4)
    src = g.covariances(pos, d_n, cell0=0.005, levels=6)
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    ocs = oracle.covariances(xyz)["cov"]
    oct_, _ = oracle.target_from_map(w.quats, w.scales)
    tree = oracle.KDTree(w.means)
    return dict(xyz=xyz, txyz=w.means, src=src, tgt=tgt, ocs=ocs, oct=oct_, tree=tree, w=w)


def _lin_check(g, S, T, r):
    corr = torch.full((S["src"].cap,), -9, dtype=torch.int32, device=DEV)
    lg = g.linearize(S["src"], S["tgt"], T, r, corr_out=corr)
    lo = oracle.linearize(S["xyz"], S["ocs"], S["txyz"], S["oct"], T, r, tree=S.get("tree"))
    n = S["xyz"].shape[0]
    np.testing.assert_array_equal(corr[:n].cpu().numpy(), lo["corr"])
    assert lg["n"] == lo["n"]
    assert np.linalg.norm(lg["H"] - lo["H"]) <= 1e-4 * np.linalg.norm(lo["H"])
    assert abs(lg["cost"] - lo["cost"]) <= 1e-4 * max(lo["cost"], 1e-300)
    # b -> 0 at the optimum: SURVEY §8(c).5 scales its tolerance by sum_i |J_i^T M_i d_i|
    assert np.linalg.norm(lg["b"] - lo["b"]) <= 1e-4 * lo["bsum"], (lg["b"], lo["b"], lo["bsum"])
    return lg, lo


def _iter_parity(S, iters, r, label=""):
    """Per-iteration parity: each GN iteration the GPU ran, re-linearised by the
    oracle at the pose T_it that iteration used: every correspondence and the inlier count exact,
    H / b / cost within 1e-4."""
    assert len(iters) >= 1
    n = S["xyz"].shape[0]
    for k, it in enumerate(iters):
        lo = oracle.linearize(S["xyz"], S["ocs"], S["txyz"], S["oct"], it["T"], r, tree=S.get("tree"))
        np.testing.assert_array_equal(it["corr"][:n], lo["corr"], err_msg=f"{label} iteration {k}")
        assert it["n"] == lo["n"], (label, k)
        assert np.linalg.norm(it["H"] - lo["H"]) <= 1e-4 * np.linalg.norm(lo["H"]), (label, k)
        assert abs(it["cost"] - lo["cost"]) <= 1e-4 * max(lo["cost"], 1e-300), (label, k)
        assert np.linalg.norm(it["b"] - lo["b"]) <= 1e-4 * lo["bsum"], (label, k, it["b"], lo["b"])
    return len(iters)


def test_linearize_c1(g, c1_setup):
    S = c1_setup
    for T in (np.eye(4), S["T"], synth.perturb_pose(S["T"], 11, 3.0, 0.05)):
        _lin_check(g, S, T, math.inf)
        _lin_check(g, S, T, 0.05)


def test_linearize_replica_full(g, replica_setup):
    S = replica_setup
    w = S["w"]
    for T in (w.T_init, w.T_gt, synth.perturb_pose(w.T_gt, 12, 4.0, 0.08)):
        _lin_check(g, S, T, 0.1)


def test_align_c1_pose(g, c1_setup):
    S = c1_setup
    p = g.align_params(max_iters=30, max_corr_dist=math.inf, eps_rot=0.0, eps_trans=0.0)
    Tg, st = g.align(S["src"], S["tgt"], np.eye(4), p)
    ref = oracle.align(S["xyz"], S["ocs"], S["txyz"], S["oct"], np.eye(4), max_iters=30, eps_rot=0.0, eps_trans=0.0)
    assert st["status"] == g.WARN_MAX_ITERS and st["iters"] == 30
    assert rot_angle(Tg[:3, :3], ref["T"][:3, :3]) <= 1e-5
    assert np.linalg.norm(Tg[:3, 3] - ref["T"][:3, 3]) <= 1e-5
    # and the known transform is recovered (C1 pin)
    assert rot_angle(Tg[:3, :3], S["T"][:3, :3]) <= 1e-5 and np.linalg.norm(Tg[:3, 3] - S["T"][:3, 3]) <= 1e-5
    assert st["fitness"] == ref["fitness"] == 1.0


def test_align_replica_pose(g, replica_setup):
    S = replica_setup
    w = S["w"]
    p = g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6)
    Tg, st = g.align(S["src"], S["tgt"], w.T_init, p)
    ref = oracle.align(S["xyz"], S["ocs"], S["txyz"], S["oct"], w.T_init, max_iters=30, max_corr_dist=0.1,
                       use_tree=True)
    assert st["status"] == ref["status"] == g.OK
    assert rot_angle(Tg[:3, :3], ref["T"][:3, :3]) <= 1e-5
    assert np.linalg.norm(Tg[:3, 3] - ref["T"][:3, 3]) <= 1e-5
    assert st["n_inliers"] == ref["n_inliers"]
    assert abs(st["iters"] - ref["iters"]) <= 1


def test_align_tum_noisy_pose_and_linearize(g, tum):
    """C3: TUM-shaped noisy frame (stride 4) vs the 1e6 map.  Per-linearisation parity at the
    initial pose, and the final pose from the same init after a fixed number of GN iterations
    (on noisy depth the 1e-6 convergence test is not reached: both run to the cap)."""
    w = tum
    K = w.K
    s = 4
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, s)
    pos, d_n = gpu_points(g, w.depth, K, s)
    src = g.covariances(pos, d_n, cell0=3.0 * s / K.fx, levels=4)
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    S = dict(xyz=xyz, txyz=w.means, src=src, tgt=tgt, ocs=oracle.covariances(xyz)["cov"],
             oct=oracle.target_from_map(w.quats, w.scales)[0], tree=oracle.KDTree(w.means))
    _lin_check(g, S, w.T_init, 0.1)
    for iters in (3, 8):
        p = g.align_params(max_iters=iters, max_corr_dist=0.1, eps_rot=0.0, eps_trans=0.0)
        Tg, st = g.align(src, tgt, w.T_init, p)
        ref = oracle.align(xyz, S["ocs"], w.means, S["oct"], w.T_init, max_iters=iters, max_corr_dist=0.1,
                           eps_rot=0.0, eps_trans=0.0, use_tree=True, tree=S["tree"])
        assert rot_angle(Tg[:3, :3], ref["T"][:3, :3]) <= 1e-5, iters
        assert np.linalg.norm(Tg[:3, 3] - ref["T"][:3, 3]) <= 1e-5, iters
        assert st["n_inliers"] == ref["n_inliers"] and st["iters"] == ref["iters"] == iters


def test_align_per_iteration_c1(g, c1_setup):
    S = c1_setup
    p = g.align_params(max_iters=30, max_corr_dist=math.inf, eps_rot=0.0, eps_trans=0.0)
    with g.AlignIterations(30, S["src"].cap) as rec:
        g.align(S["src"], S["tgt"], np.eye(4), p)
    torch.cuda.synchronize()
    assert _iter_parity(S, rec.iterations(), math.inf, "c1") == 30


def test_align_per_iteration_bench_frame(g, replica, replica_setup):
    """The bench's own path: Tracker (A1 -> image-window A2-A4 -> seeded A6-A9, one graph replay)
    on the Replica workload frame vs the 1e6 map, every iteration against the oracle."""
    w, S = replica, replica_setup
    K = w.K
    H, W = w.depth.shape
    tr = g.Tracker(H, W, (K.fx, K.fy, K.cx, K.cy), stride=4)
    with g.AlignIterations(30, tr.cap) as rec:
        Tg, st = tr.track(t(w.depth), S["tgt"], w.T_init)
    torch.cuda.synchronize()
    it = rec.iterations()
    assert len(it) == st["iters"] >= 2
    np.testing.assert_array_equal(it[0]["T"], w.T_init)
    _iter_parity(S, it, 0.1, "bench")
    ref = oracle.align(S["xyz"], S["ocs"], S["txyz"], S["oct"], w.T_init, max_iters=30, max_corr_dist=0.1,
                       tree=S["tree"])
    assert rot_angle(Tg[:3, :3], ref["T"][:3, :3]) <= 1e-5 and np.linalg.norm(Tg[:3, 3] - ref["T"][:3, 3]) <= 1e-5
    assert st["n_inliers"] == ref["n_inliers"] and abs(st["iters"] - ref["iters"]) <= 1


@pytest.mark.parametrize("stride,iters", [(4, 8), (1, 5)])
def test_align_per_iteration_tum(g, tum, stride, iters):
    """C3: noisy TUM-shaped frame vs the 1e6 map; stride 1 (~205k points) exercises the
    non-resident path (more points than the co-resident grid's threads)."""
    w = tum
    K = w.K
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, stride)
    pos, d_n = gpu_points(g, w.depth, K, stride)
    src = g.covariances(pos, d_n, cell0=3.0 * stride / K.fx, levels=4)
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    S = dict(xyz=xyz, txyz=w.means, src=src, tgt=tgt, ocs=oracle.covariances(xyz)["cov"],
             oct=oracle.target_from_map(w.quats, w.scales)[0], tree=oracle.KDTree(w.means))
    if stride == 1:
        assert xyz.shape[0] > 148 * 384  # beyond one resident point per thread
    p = g.align_params(max_iters=iters, max_corr_dist=0.1, eps_rot=0.0, eps_trans=0.0)
    with g.AlignIterations(iters, src.cap) as rec:
        g.align(src, tgt, w.T_init, p)
    torch.cuda.synchronize()
    assert _iter_parity(S, rec.iterations(), 0.1, f"tum s={stride}") == iters


def test_align_per_iteration_c2_tracker(g):
    """C2 as bench.py times it: the Replica-shaped frame vs a 1e5-Gaussian map through the Tracker
    (one graph replay), every GN iteration against the oracle, then the final pose."""
    w = synth.make_frame_workload(2, "replica", M=100_000, stride=4)
    K = w.K
    H, W = w.depth.shape
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, 4)
    S = dict(xyz=xyz, txyz=w.means, ocs=oracle.covariances(xyz)["cov"],
             oct=oracle.target_from_map(w.quats, w.scales)[0], tree=oracle.KDTree(w.means))
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    prm = g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6)
    tr = g.Tracker(H, W, (K.fx, K.fy, K.cx, K.cy), stride=4, params=prm)
    with g.AlignIterations(30, tr.cap) as rec:
        Tg, st = tr.track(t(w.depth), tgt, w.T_init)
    torch.cuda.synchronize()
    it = rec.iterations()
    assert len(it) == st["iters"] >= 2
    _iter_parity(S, it, 0.1, "c2")
    ref = oracle.align(xyz, S["ocs"], w.means, S["oct"], w.T_init, max_iters=30, max_corr_dist=0.1, tree=S["tree"])
    assert rot_angle(Tg[:3, :3], ref["T"][:3, :3]) <= 1e-5 and np.linalg.norm(Tg[:3, 3] - ref["T"][:3, 3]) <= 1e-5
    assert st["n_inliers"] == ref["n_inliers"] and abs(st["iters"] - ref["iters"]) <= 1


@pytest.mark.parametrize("stride", [4, 1])
def test_align_per_iteration_tum_tracker(g, tum, stride):
    """C3 through the bench's own path (Tracker: A1 -> image-window A2-A4 -> seeded A6-A9, one
    graph replay; stride 1 takes the flat GN loop with seeds): every iteration of the first 8
    against the oracle at the pose the GPU iteration used."""
    w = tum
    K = w.K
    H, W = w.depth.shape
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, stride)
    S = dict(xyz=xyz, txyz=w.means, ocs=oracle.covariances(xyz)["cov"],
             oct=oracle.target_from_map(w.quats, w.scales)[0], tree=oracle.KDTree(w.means))
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    iters = 8
    tr = g.Tracker(H, W, (K.fx, K.fy, K.cx, K.cy), stride=stride,
                   params=g.align_params(max_iters=iters, max_corr_dist=0.1, eps_rot=0.0, eps_trans=0.0))
    if stride == 1:
        assert tr.cap > 148 * 384  # the flat GN loop
    with g.AlignIterations(iters, tr.cap) as rec:
        tr.track(t(w.depth), tgt, w.T_init)
    torch.cuda.synchronize()
    it = rec.iterations()
    np.testing.assert_array_equal(it[0]["T"], w.T_init)
    assert _iter_parity(S, it, 0.1, f"tum tracker s={stride}") == iters


@pytest.mark.parametrize("B", [3, 8])
def test_align_per_iteration_batch_frame(g, replica_setup, B):
    """N2: frame 0 of a B-frame batch (the others: perturbed poses of the same frame); B = 3 runs
    k_align_batch, B = 8 the flat loop over the frames."""
    S = replica_setup
    w = S["w"]
    src = S["src"]
    inits = [w.T_init] + [synth.perturb_pose(w.T_gt, 31 + b) for b in range(B - 1)]
    d_T = t(np.stack([np.ascontiguousarray(T, np.float64).reshape(16) for T in inits]))
    d_stats = torch.zeros((B, 32), dtype=torch.uint8, device=DEV)
    ws = [g.align_workspace(src.cap) for _ in range(B)]
    p = g.align_params(max_iters=30, max_corr_dist=0.1)
    with g.AlignIterations(30, src.cap) as rec:
        g.align_batch_async([src] * B, S["tgt"], d_T, d_stats, p, wss=ws)
    torch.cuda.synchronize()
    it = rec.iterations()
    np.testing.assert_array_equal(it[0]["T"], w.T_init)
    _iter_parity(S, it, 0.1, "batch frame 0")


def test_align_deterministic(g, replica_setup):
    S = replica_setup
    w = S["w"]
    outs = [g.align(S["src"], S["tgt"], w.T_init)[0] for _ in range(3)]
    for o in outs[1:]:
        np.testing.assert_array_equal(o, outs[0])


def _align_dev(g, S, T, ws, seed_T=None, params=None):
    params = params or g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6)
    d_T = torch.from_numpy(np.ascontiguousarray(T, dtype=np.float64).reshape(-1)).to(DEV)
    d_stats = torch.zeros(32, dtype=torch.uint8, device=DEV)
    if seed_T is not None:
        d_seed = torch.from_numpy(np.ascontiguousarray(seed_T, dtype=np.float64).reshape(-1)).to(DEV)
        g.align_seed(S["src"], S["tgt"], d_seed, params, ws)
    g.align_async(S["src"], S["tgt"], d_T, d_stats, params, ws)
    torch.cuda.synchronize()
    return d_T.cpu().numpy().reshape(4, 4), g.decode_stats(d_stats)


def test_align_seed_identical(g, replica_setup):
    """Iteration-0 correspondences computed ahead (gsicp_align_seed) give bit-identical results;
    seeds at another pose, or for another workspace, are ignored."""
    S = replica_setup
    w = S["w"]
    ws = g.align_workspace(S["src"].cap, DEV)
    ws2 = g.align_workspace(S["src"].cap, DEV)
    T_ref, st_ref = _align_dev(g, S, w.T_init, ws)
    T_s, st_s = _align_dev(g, S, w.T_init, ws, seed_T=w.T_init)
    np.testing.assert_array_equal(T_s, T_ref)
    assert st_s == st_ref
    other = synth.perturb_pose(w.T_init, 31, 2.0, 0.03)
    T_o, st_o = _align_dev(g, S, w.T_init, ws, seed_T=other)  # stale pose: ignored
    np.testing.assert_array_equal(T_o, T_ref)
    assert st_o == st_ref
    # seed into ws2, align on ws: the seed is not consumed there (and ws2's is dropped)
    d_seed = torch.from_numpy(w.T_init.reshape(-1).copy()).to(DEV)
    g.align_seed(S["src"], S["tgt"], d_seed, None, ws2)
    T_w, st_w = _align_dev(g, S, w.T_init, ws)
    np.testing.assert_array_equal(T_w, T_ref)
    # linearize after a seed at the same pose: same H / b / correspondences as without
    T = synth.perturb_pose(w.T_gt, 12, 4.0, 0.08)
    lg0 = g.linearize(S["src"], S["tgt"], T, 0.1, ws=ws)
    d_seed = torch.from_numpy(np.ascontiguousarray(T).reshape(-1).copy()).to(DEV)
    g.align_seed(S["src"], S["tgt"], d_seed, None, ws)
    lg1 = g.linearize(S["src"], S["tgt"], T, 0.1, ws=ws)
    np.testing.assert_array_equal(lg1["H"], lg0["H"])
    assert lg1["n"] == lg0["n"]


def test_align_errors(g, c1_setup):
    S = c1_setup
    # disjoint clouds 100 m apart -> TRACKING_LOST with the init pose
    T0 = np.eye(4)
    T0[0, 3] = 100.0
    Tg, st = g.align(S["src"], S["tgt"], T0, g.align_params(max_corr_dist=0.5))
    assert st["status"] == g.ERR_TRACKING_LOST and st["fitness"] == 0.0
    np.testing.assert_array_equal(Tg, T0)
    # empty frame -> DEGENERATE_FRAME
    empty = g.Cloud.empty(64)
    Tg, st = g.align(empty, S["tgt"], np.eye(4))
    assert st["status"] == g.ERR_DEGENERATE_FRAME


def test_tracker_host_frames_and_sampled_rows(g, replica, tum):
    """A1 from only the sampled rows == A1 from the full image (bit-exact), and track_host()
    (sampled-row upload + graph replay) returns the same pose as track() on the device image."""
    for w, s in ((replica, 4), (tum, 3), (tum, 1)):
        H, W = w.depth.shape
        K = (w.K.fx, w.K.fy, w.K.cx, w.K.cy)
        full, n_full = g.backproject_downsample(t(w.depth), K, stride=s)
        rows = torch.empty(((H + s - 1) // s, W), dtype=torch.float32, device=DEV)
        g.upload_sampled_rows(rows, torch.from_numpy(w.depth).pin_memory(), s)
        part, n_part = g.backproject_sampled_rows(rows, H, W, K, stride=s)
        n = int(n_full.item())
        assert n == int(n_part.item())
        assert torch.equal(full[:n], part[:n])
        # the lattice map written by A1: output index of every sampled pixel, -1 where invalid
        for src, rs in ((t(w.depth), False), (rows, True)):
            pos_l, n_l, lat = g.backproject_lattice(src, H, W, K, stride=s, rows_sampled=rs)
            assert torch.equal(pos_l[:n], full[:n])
            Ws = (W + s - 1) // s
            pix = full[:n, 3].cpu().numpy().view(np.int32)
            expect = np.full(lat.shape[0], -1, np.int32)
            expect[(pix // W) // s * Ws + (pix % W) // s] = np.arange(n, dtype=np.int32)
            np.testing.assert_array_equal(lat.cpu().numpy(), expect)
    w = replica
    tr = g.Tracker(w.K.H, w.K.W, (w.K.fx, w.K.fy, w.K.cx, w.K.cy), stride=4)
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    T_dev, st_dev = tr.track(t(w.depth), tgt, w.T_init)
    host = torch.from_numpy(w.depth).pin_memory()
    for _ in range(2):
        T_host, st_host = tr.track_host(host, tgt, w.T_init)
        np.testing.assert_array_equal(T_host, T_dev)
        assert st_host["iters"] == st_dev["iters"] and st_host["fitness"] == st_dev["fitness"]
    assert tr.upload_bytes() == ((w.K.H + 3) // 4) * w.K.W * 4
    # the streaming call (double-buffered uploads overlapping compute) returns the same poses
    res = tr.track_host_stream([host] * 5, tgt, w.T_init)
    for T_s, st_s in res:
        np.testing.assert_array_equal(T_s, T_dev)
        assert st_s["iters"] == st_dev["iters"]


def test_tracker_graph_capture(g, replica):
    """The whole frame (A1 -> A4 -> A6-A9) captured in one CUDA graph and replayed."""
    w = replica
    tr = g.Tracker(w.K.H, w.K.W, (w.K.fx, w.K.fy, w.K.cx, w.K.cy), stride=4)
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    depth = t(w.depth)
    T_ref, st_ref = tr.track(depth, tgt, w.T_init)
    s = torch.cuda.Stream()
    T0 = torch.from_numpy(w.T_init.reshape(-1).copy()).to(DEV)
    with torch.cuda.stream(s):
        tr.d_T.copy_(T0)
        tr.step_async(depth, tgt)  # warm
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        tr.step_async(depth, tgt)
    for _ in range(2):
        tr.d_T.copy_(T0)
        graph.replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(tr.d_T.cpu().numpy().reshape(4, 4), T_ref)
        assert g.decode_stats(tr.d_stats)["iters"] == st_ref["iters"]


def test_tracker_graph_capture_large_cloud(g, tum):
    """A stride-1 TUM frame (205k points: more than the persistent align grid holds, so the GN loop
    runs as the flat kernels, inside the captured graph the body of a conditional WHILE node): the
    replayed graph equals the direct (eager, one launch per iteration) call bit for bit, and the
    iteration count and inlier count agree."""
    w = tum
    tr = g.Tracker(w.K.H, w.K.W, (w.K.fx, w.K.fy, w.K.cx, w.K.cy), stride=1,
                   params=g.align_params(max_iters=12, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6))
    tgt = g.build_target(t(w.means), t(w.quats), t(w.scales))
    depth = t(w.depth)
    T_ref, st_ref = tr.track(depth, tgt, w.T_init)  # (the Tracker's own frame graph)
    assert tr.cloud.n() > 148 * 384  # (the flat path)
    tr.preprocess(depth)
    T_e, st_e = g.align(tr.cloud, tgt, w.T_init, tr.params, tr.ws_align)  # eager, unseeded
    np.testing.assert_array_equal(T_e, T_ref)
    assert st_e["iters"] == st_ref["iters"] and st_e["n_inliers"] == st_ref["n_inliers"]
    s = torch.cuda.Stream()
    T0 = torch.from_numpy(w.T_init.reshape(-1).copy()).to(DEV)
    with torch.cuda.stream(s):
        tr.d_T.copy_(T0)
        tr.step_async(depth, tgt)  # warm
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        tr.step_async(depth, tgt)
    for _ in range(2):
        tr.d_T.copy_(T0)
        graph.replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(tr.d_T.cpu().numpy().reshape(4, 4), T_ref)
        st = g.decode_stats(tr.d_stats)
        assert st["iters"] == st_ref["iters"] and st["n_inliers"] == st_ref["n_inliers"]


# ----------------------------------------------------------------------------------------- C5
def test_sequence_tracking(g):
    """C5-style: a 30 Hz synthetic sequence tracked with the device-side constant-velocity init
    (one graph replay per frame): every frame converges and the trajectory error stays small."""
    seq = synth.make_sequence(0, 40, "replica", M=300_000)
    rows = synth.render_sequence_rows(seq, DEV)
    tgt = g.build_target(t(seq.means), t(seq.quats), t(seq.scales))
    K = seq.K
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride,
                   params=g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6))
    T_est, ms = g.track_sequence(tr, tgt, rows, seq.T_gt[0])
    err = synth.trajectory_error(T_est, seq.T_gt[1:])
    assert err["ate_rmse_m"] < 5e-3 and err["rot_max_deg"] < 0.5, err
    # frames 1..6 against the oracle, each from the constant-velocity prediction of the GPU's
    # previous poses (zero velocity before frame 1)
    oct_, _ = oracle.target_from_map(seq.quats, seq.scales)
    tree = oracle.KDTree(seq.means)
    prev2, prev1 = seq.T_gt[0], seq.T_gt[0]
    for f in range(1, 7):
        init = prev1 @ np.linalg.inv(prev2) @ prev1
        depth = np.full((K.H, K.W), np.nan, np.float32)
        depth[::seq.stride] = rows[f].cpu().numpy()
        xyz, _ = oracle.backproject(depth, K.fx, K.fy, K.cx, K.cy, seq.stride)
        res = oracle.align(xyz, oracle.covariances(xyz)["cov"], seq.means, oct_, init, max_iters=30,
                           max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6, tree=tree)
        Tg = T_est[f - 1]
        assert rot_angle(Tg[:3, :3], res["T"][:3, :3]) <= 1e-5 and np.abs(Tg[:3, 3] - res["T"][:3, 3]).max() <= 1e-5, f
        prev2, prev1 = prev1, Tg
    assert g.decode_stats(tr.d_stats)["status"] in (g.OK, g.WARN_MAX_ITERS)
    # the device-side prediction equals the constant-velocity formula on the host
    hist = torch.from_numpy(np.concatenate([seq.T_gt[3].reshape(-1), seq.T_gt[4].reshape(-1)])).to(DEV)
    out = torch.zeros(16, dtype=torch.float64, device=DEV)
    g.pose_predict(hist, out)
    A, B = seq.T_gt[3], seq.T_gt[4]
    P = out.cpu().numpy().reshape(4, 4)
    np.testing.assert_allclose(P, B @ np.linalg.inv(A) @ B, atol=1e-12)
    np.testing.assert_allclose(P[:3, :3] @ P[:3, :3].T, np.eye(3), atol=1e-14)


# ----------------------------------------------------------------------------------------- A4 export
def _quat_rot(q):
    """(n,4) wxyz -> (n,3,3) rotation matrices (the textbook formula, binary64)."""
    q = np.asarray(q, np.float64)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1),
                     np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1),
                     np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)], 1)


@pytest.mark.parametrize("case,mode", [("c1", oracle.ELLIPSE), ("replica4", oracle.ELLIPSE),
                                       ("replica4", oracle.PLANE), ("replica4", oracle.NONE)])
def test_export_gaussians(g, c1, replica, case, mode):
    """gsicp_export_gaussians (ALG-12) vs the oracle's O12' on the same frame and pose:
    means bit-exact (K3, rounded to binary32); the exported world covariance R diag(s^2) R^T within
    1e-4 (the covariance tolerance); the variances within 1e-4 of the largest; unit quaternions
    with w >= 0; where the spectrum has clear gaps, the same axes up to sign.  ELLIPSE round trip:
    build_target of the export gives the source covariance rotated into the world."""
    w, s = {"c1": (c1, 1), "replica4": (replica, 4)}[case]
    K = w.K
    H, W = w.depth.shape
    pos, d_n = gpu_points(g, w.depth, K, s)
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, s)
    n = xyz.shape[0]
    cl = g.covariances_image(pos, d_n, H, W, s, (K.fx, K.fy, K.cx, K.cy), k=20, mode=mode, eps_var=1e-3,
                             cell0=3.0 * s / K.fx, levels=4)
    rng = np.random.default_rng(80)
    a = rng.normal(size=3)
    a /= np.linalg.norm(a)  # 0.5 rad about a random unit axis (Rodrigues)
    Kx = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    T = np.eye(4)
    T[:3, :3] = np.eye(3) + math.sin(0.5) * Kx + (1 - math.cos(0.5)) * Kx @ Kx
    T[:3, 3] = [0.3, -1.2, 2.0]
    p, c = 1.5, 0.7
    gm, gq, gs, d_m = g.export_gaussians(cl.pos, cl.d_n, cl.cov_a, cl.cov_b, T=t(T), p=p, c=c)
    assert int(d_m.item()) == n
    gm, gq, gs = gm[:n].cpu().numpy(), gq[:n].cpu().numpy(), gs[:n].cpu().numpy()
    ref = oracle.covariances(xyz, k=20, mode=mode)
    om, oq, os_ = oracle.export_gaussians(xyz, ref["raw"], T=T, mode=mode, p=p, c=c)
    np.testing.assert_array_equal(gm, om.astype(np.float32))
    assert np.abs(np.linalg.norm(gq.astype(np.float64), axis=1) - 1).max() < 1e-6
    assert (gq[:, 0] >= 0).all()
    Rg, Ro = _quat_rot(gq), _quat_rot(oq)
    Sg = Rg @ (gs.astype(np.float64)[:, :, None] ** 2 * np.transpose(Rg, (0, 2, 1)))
    So = Ro @ (os_[:, :, None] ** 2 * np.transpose(Ro, (0, 2, 1)))
    err = np.linalg.norm(Sg - So, axis=(1, 2)) / np.linalg.norm(So, axis=(1, 2))
    assert err.max() <= 1e-4, (err.max(), np.argmax(err))
    vg, vo = gs.astype(np.float64) ** 2, os_ ** 2
    assert (np.abs(vg - vo) <= 1e-4 * vo[:, :1]).all()
    assert (gs[:, 0] >= gs[:, 1]).all() and (gs[:, 1] >= gs[:, 2]).all()
    # an axis is unique (up to sign) where its variance is separated from its neighbours' (PLANE:
    # only the normal, the other two share variance 1)
    g01 = vo[:, 0] - vo[:, 1] > 1e-2 * vo[:, 0]
    g12 = vo[:, 1] - vo[:, 2] > 1e-2 * vo[:, 0]
    dots = np.abs(np.einsum("nrj,nrj->nj", Rg, Ro))
    for j, sep in enumerate((g01, g01 & g12, g12)):
        if mode != oracle.PLANE or j == 2:
            assert sep.mean() > 0.5, (j, sep.mean())
        if sep.any():
            assert dots[sep, j].min() >= 1 - 1e-6, (j, dots[sep, j].min())
    if mode == oracle.ELLIPSE:
        tgt = g.build_target(t(gm), t(gq), t(gs), mode=mode, eps_var=1e-3)
        tpos, ca, cb = tgt.arrays()
        order = tpos[:, 3].contiguous().view(torch.int32).long().cpu().numpy()
        inv = np.empty(n, np.int64)
        inv[order] = np.arange(n)
        tc = torch.cat([ca, cb[:, :2]], 1).cpu().numpy()[inv]
        R = T[:3, :3]
        cam = cl.cov6()[:n].cpu().numpy().astype(np.float64)
        full = cam[:, [0, 1, 2, 1, 3, 4, 2, 4, 5]].reshape(-1, 3, 3)
        wc = R @ full @ R.T
        wc6 = wc[:, [0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2]]
        e2 = cov_rel_err(tc, wc6)
        assert e2.max() <= 1e-4, e2.max()


def test_export_overlap_filter(g, replica_setup):
    """Overlap filter (R28): with the correspondences of a linearisation, only the points
    without a map correspondence are exported, compacted in index order — the same rows as the
    oracle's export of the points its own O7 leaves unmatched at the same pose (bit-exact means)."""
    S = replica_setup
    src, tgt, xyz = S["src"], S["tgt"], S["xyz"]
    n = xyz.shape[0]
    T = synth.perturb_pose(S["w"].T_gt, 13, 2.0, 0.03)
    oraw = oracle.covariances(xyz)["raw"]
    for r in (0.01, 0.03, 1e3):
        corr = torch.full((src.cap,), -9, dtype=torch.int32, device=DEV)
        g.linearize(src, tgt, T, r, corr_out=corr)
        gm, gq, gs, d_m = g.export_gaussians(src.pos, src.d_n, src.cov_a, src.cov_b, T=t(T), corr=corr)
        m = int(d_m.item())
        lin = oracle.linearize(xyz, S["ocs"], S["txyz"], S["oct"], T, r, tree=S["tree"])
        keep = np.nonzero(lin["corr"] < 0)[0]
        assert m == keep.size, (r, m, keep.size, n)
        if r > 1.0:
            assert m == 0
            continue
        assert m < n and (m > 0 or r > 0.01), (r, m)
        if m == 0:
            continue
        om, oq, os_ = oracle.export_gaussians(xyz[keep], oraw[keep], T=T)
        np.testing.assert_array_equal(gm[:m].cpu().numpy(), om.astype(np.float32))
        Rg, Ro = _quat_rot(gq[:m].cpu().numpy()), _quat_rot(oq)
        gsn = gs[:m].cpu().numpy().astype(np.float64)
        Sg = Rg @ (gsn[:, :, None] ** 2 * np.transpose(Rg, (0, 2, 1)))
        So = Ro @ (os_[:, :, None] ** 2 * np.transpose(Ro, (0, 2, 1)))
        err = np.linalg.norm(Sg - So, axis=(1, 2)) / np.linalg.norm(So, axis=(1, 2))
        assert err.max() <= 1e-4, err.max()


def _half_room_map(seq, rows):
    K = seq.K
    d = rows[0].cpu().numpy()
    v, u = np.nonzero(np.isfinite(d) & (d > 0.1) & (d < 10))
    z = d[v, u]
    P0 = np.stack([(u - K.cx) * z / K.fx, (v * seq.stride - K.cy) * z / K.fy, z], 1) @ seq.T_gt[0][:3, :3].T \
        + seq.T_gt[0][:3, 3]
    return seq.means[:, 0] < np.median(P0[:, 0])


def test_sequence_map_growth(g):
    """N1: half of the room removed from the map; with keyframe
    insertion (device decision + conditional insertion inside the per-frame graph, no host round
    trip) the first frame becomes a keyframe, inserts exactly its unmatched points, and the
    following frames are fully matched; without it the fitness stays ~0.5.  Tracking stays exact
    (ATE < 1 mm) either way."""
    seq = synth.make_sequence(1, 40, "replica", M=300_000)
    rows = synth.render_sequence_rows(seq, DEV)
    K = seq.K
    keep = _half_room_map(seq, rows)
    M0 = int(keep.sum())
    prm = g.align_params(max_iters=30, max_corr_dist=0.1)
    for grow in (False, True):
        tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, keep_corr=True, params=prm)
        gm = g.GaussianMap(t(seq.means[keep]), t(seq.quats[keep]), t(seq.scales[keep]), capacity=M0 + 4 * tr.cap,
                           max_insert=tr.cap)
        if grow:  # frame 1 alone (same constant-velocity init: zero velocity): its unmatched points
            tr1 = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, keep_corr=True, params=prm)
            tr1.rows.copy_(rows[1])
            T1, st1 = tr1.track_rows(gm.tgt, seq.T_gt[0])
            unmatched = int((tr1.corr[:tr1.cloud.n()] < 0).sum().item())
            assert st1["fitness"] < 0.95 and unmatched == tr1.cloud.n() - st1["n_inliers"]
        T_est, kfs, added, fit, _ = g.track_sequence_mapping(tr, gm, rows, seq.T_gt[0],
                                                             min_fitness=0.95 if grow else -1.0,
                                                             max_gap=30 if grow else 10 ** 9)
        err = synth.trajectory_error(T_est, seq.T_gt[1:])
        assert err["ate_rmse_m"] < 1e-3 and err["rot_max_deg"] < 0.05, err
        if grow:
            assert kfs[0] == 1 and added[0] == unmatched and gm.M == M0 + sum(added)
            assert fit[-10:].min() > 0.99, fit
        else:
            assert kfs == [] and gm.M == M0 and fit[-10:].max() < 0.7, fit


def test_map_incremental_equals_rebuild(g):
    """N1 incremental target maintenance: after several insertions the map's target equals a
    from-scratch gsicp_build_target of the same rows — identical 16-NN neighbour sets for every
    row, covariances bitwise, and an align against either target returns the same pose."""
    seq = synth.make_sequence(2, 12, "replica", M=300_000)
    rows = synth.render_sequence_rows(seq, DEV)
    K = seq.K
    keep = _half_room_map(seq, rows)
    M0 = int(keep.sum())
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, keep_corr=True)
    gm = g.GaussianMap(t(seq.means[keep]), t(seq.quats[keep]), t(seq.scales[keep]), capacity=M0 + 6 * tr.cap,
                       max_insert=tr.cap)
    for i, filt in ((1, True), (5, True), (9, False)):  # two overlap-filtered keyframes and an unfiltered one
        tr.rows.copy_(rows[i])
        T, st = tr.track_rows(gm.tgt, seq.T_gt[i])
        gm.insert(tr.cloud, tr.d_T, tr.corr if filt else None)
    torch.cuda.synchronize()
    M = gm.M
    assert M > M0 + tr.cloud.n()
    ref = g.build_target(gm.means[:M].contiguous(), gm.quats[:M].contiguous(), gm.scales[:M].contiguous(),
                         cell=gm.cell)
    a_inc = [x[:M] for x in gm.tgt.arrays()]
    a_ref = ref.arrays()

    def by_row(arr):
        pos, ca, cb = (x.cpu().numpy() for x in arr)
        r = pos[:, 3].view(np.int32)
        out = [np.empty_like(pos), np.empty_like(ca), np.empty_like(cb)]
        for o, x in zip(out, (pos, ca, cb)):
            o[r] = x
        return out
    inc, rf = by_row(a_inc), by_row(a_ref)
    for x, y in zip(inc, rf):
        np.testing.assert_array_equal(x, y)
    np.testing.assert_array_equal(gm.tgt.graph_rows(M), ref.graph_rows(M))
    tr2 = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride)
    tr2.rows.copy_(rows[10])
    Ta, sa = tr2.track_rows(gm.tgt, seq.T_gt[10])
    Tb, sb = tr2.track_rows(ref, seq.T_gt[10])
    np.testing.assert_array_equal(Ta, Tb)
    assert sa["n_inliers"] == sb["n_inliers"]


@pytest.mark.parametrize("B", [4, 8])
def test_align_batch(g, B):
    """N2: B frames of a sequence in one BatchTracker step (concurrent A1-A4 streams + one
    k_align_batch launch for B = 4, the flat loop over the frames for B = 8) give the poses
    single-frame tracking gives (same algorithm; only the grouping of the H/b partial sums differs)
    and, for a frame checked against the oracle from the same initial pose, the oracle's pose
    within 1e-5 rad / 1e-5 m."""
    seq = synth.make_sequence(2, B + 1, "replica", M=300_000)
    rows = synth.render_sequence_rows(seq, DEV)
    K = seq.K
    prm = g.align_params(max_iters=30, max_corr_dist=0.1)
    tgt = g.build_target(t(seq.means), t(seq.quats), t(seq.scales))
    init = np.stack([synth.perturb_pose(seq.T_gt[1 + b], 20 + b, 2.0, 0.03) for b in range(B)])
    bt = g.BatchTracker(B, K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    bt.rows.copy_(rows[1:1 + B])
    Tb, stb = bt.track_rows(tgt, init)
    Tb2, _ = bt.track_rows(tgt, init)  # deterministic replay
    np.testing.assert_array_equal(Tb, Tb2)
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    for b in range(B):
        tr.rows.copy_(rows[1 + b])
        Ts, sts = tr.track_rows(tgt, init[b])
        assert rot_angle(Tb[b][:3, :3], Ts[:3, :3]) < 1e-6 and np.abs(Tb[b][:3, 3] - Ts[:3, 3]).max() < 1e-6
        assert stb[b]["n_inliers"] == sts["n_inliers"] and stb[b]["status"] == sts["status"]
        assert rot_angle(Tb[b][:3, :3], seq.T_gt[1 + b][:3, :3]) < math.radians(0.05)
    # oracle for frame 0 of the batch, from the same initial pose
    d = rows[1].cpu().numpy()
    depth = np.full((K.H, K.W), np.nan, np.float32)
    depth[::seq.stride] = d
    xyz, _ = oracle.backproject(depth, K.fx, K.fy, K.cx, K.cy, seq.stride)
    ocs = oracle.covariances(xyz)["cov"]
    oct_, _ = oracle.target_from_map(seq.quats, seq.scales)
    res = oracle.align(xyz, ocs, seq.means, oct_, init[0], max_iters=30, max_corr_dist=0.1)
    assert rot_angle(Tb[0][:3, :3], res["T"][:3, :3]) < 1e-5 and np.abs(Tb[0][:3, 3] - res["T"][:3, 3]).max() < 1e-5


def test_align_batch_bench_config_all_frames(g):
    """N2 at the configuration bench.py times: 8 distinct frames of a Replica-shaped sequence vs its
    1e6-Gaussian map (frames 1..8, initial poses perturbed with seeds 500 + b, the bench's GN
    parameters) in one BatchTracker step through the flat GN loop; EVERY frame's pose against the
    oracle from the same initial pose."""
    B = 8
    seq = synth.make_sequence(0, B + 1, "replica", M=1_000_000)
    rows = synth.render_sequence_rows(seq, DEV)
    K = seq.K
    prm = g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6)
    tgt = g.build_target(t(seq.means), t(seq.quats), t(seq.scales))
    init = np.stack([synth.perturb_pose(seq.T_gt[1 + b], 500 + b, 2.0, 0.03) for b in range(B)])
    bt = g.BatchTracker(B, K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    bt.rows.copy_(rows[1:1 + B])
    Tb, stb = bt.track_rows(tgt, init)
    oct_, _ = oracle.target_from_map(seq.quats, seq.scales)
    tree = oracle.KDTree(seq.means)
    for b in range(B):
        depth = np.full((K.H, K.W), np.nan, np.float32)
        depth[::seq.stride] = rows[1 + b].cpu().numpy()
        xyz, _ = oracle.backproject(depth, K.fx, K.fy, K.cx, K.cy, seq.stride)
        ocs = oracle.covariances(xyz)["cov"]
        res = oracle.align(xyz, ocs, seq.means, oct_, init[b], max_iters=30, max_corr_dist=0.1, eps_rot=1e-6,
                           eps_trans=1e-6, tree=tree)
        assert rot_angle(Tb[b][:3, :3], res["T"][:3, :3]) <= 1e-5, b
        assert np.abs(Tb[b][:3, 3] - res["T"][:3, 3]).max() <= 1e-5, b
        assert stb[b]["n_inliers"] == res["n_inliers"] and abs(stb[b]["iters"] - res["iters"]) <= 1, b


def test_align_batch_single_and_ragged(g):
    """B = 1 runs the same blocks and summation as the single-frame kernel: bitwise-identical pose
    and stats.  A ragged batch (one frame with a third of its depth missing, so fewer points) gives
    every frame its single-frame pose."""
    seq = synth.make_sequence(3, 4, "replica", M=300_000)
    rows = synth.render_sequence_rows(seq, DEV)
    K = seq.K
    prm = g.align_params(max_iters=30, max_corr_dist=0.1)
    tgt = g.build_target(t(seq.means), t(seq.quats), t(seq.scales))
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    init1 = synth.perturb_pose(seq.T_gt[1], 40, 2.0, 0.03)
    tr.rows.copy_(rows[1])
    Ts, sts = tr.track_rows(tgt, init1)
    b1 = g.BatchTracker(1, K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    b1.rows.copy_(rows[1:2])
    Tb, stb = b1.track_rows(tgt, init1[None])
    np.testing.assert_array_equal(Tb[0], Ts)
    assert stb[0] == sts
    rr = rows[1:4].clone()
    rr[2, : rr.shape[1] // 3] = 0.0  # invalid depth: a third fewer points in frame 3
    init = np.stack([synth.perturb_pose(seq.T_gt[1 + b], 41 + b, 2.0, 0.03) for b in range(3)])
    b3 = g.BatchTracker(3, K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    b3.rows.copy_(rr)
    Tb3, st3 = b3.track_rows(tgt, init)
    ns = [tr_.cloud.n() for tr_ in b3.trs]
    assert ns[2] < 0.75 * ns[0], ns
    for b in range(3):
        tr.rows.copy_(rr[b])
        Ts, sts = tr.track_rows(tgt, init[b])
        assert tr.cloud.n() == ns[b]
        assert rot_angle(Tb3[b][:3, :3], Ts[:3, :3]) < 1e-6 and np.abs(Tb3[b][:3, 3] - Ts[:3, 3]).max() < 1e-6
        assert st3[b]["n_inliers"] == sts["n_inliers"]


@pytest.mark.parametrize("lam0", [1e-4, 1.0])
def test_align_lm_pose(g, c1_setup, replica_setup, lam0):
    """Levenberg-Marquardt (R30) through the C ABI vs the oracle's LM from the same initial pose:
    C1 (30 fixed iterations, known transform) and the Replica frame vs the 1e6 map (converged);
    the pose within 1e-5 rad / 1e-5 m.  A large initial damping takes more iterations but reaches
    the same pose."""
    S = c1_setup
    p = g.align_params(max_iters=30, max_corr_dist=math.inf, eps_rot=0.0, eps_trans=0.0, solver=g.SOLVER_LM,
                       lm_lambda0=lam0)
    Tg, st = g.align(S["src"], S["tgt"], np.eye(4), p)
    ref = oracle.align(S["xyz"], S["ocs"], S["txyz"], S["oct"], np.eye(4), max_iters=30, eps_rot=0.0, eps_trans=0.0,
                       solver=1, lm_lambda0=lam0)
    assert st["status"] == ref["status"] == g.WARN_MAX_ITERS
    assert rot_angle(Tg[:3, :3], ref["T"][:3, :3]) <= 1e-5 and np.linalg.norm(Tg[:3, 3] - ref["T"][:3, 3]) <= 1e-5
    assert rot_angle(Tg[:3, :3], S["T"][:3, :3]) <= 1e-5 and np.linalg.norm(Tg[:3, 3] - S["T"][:3, 3]) <= 1e-5
    R = replica_setup
    w = R["w"]
    p = g.align_params(max_iters=30, max_corr_dist=0.1, solver=g.SOLVER_LM, lm_lambda0=lam0)
    Tg, st = g.align(R["src"], R["tgt"], w.T_init, p)
    ref = oracle.align(R["xyz"], R["ocs"], R["txyz"], R["oct"], w.T_init, max_iters=30, max_corr_dist=0.1,
                       use_tree=True, tree=R["tree"], solver=1, lm_lambda0=lam0)
    assert st["status"] == ref["status"] == g.OK, (st, ref["status"], ref["iters"])
    assert rot_angle(Tg[:3, :3], ref["T"][:3, :3]) <= 1e-5 and np.linalg.norm(Tg[:3, 3] - ref["T"][:3, 3]) <= 1e-5
    assert abs(st["iters"] - ref["iters"]) <= 1 and st["n_inliers"] == ref["n_inliers"]
    gn, _ = g.align(R["src"], R["tgt"], w.T_init, g.align_params(max_iters=30, max_corr_dist=0.1))
    assert rot_angle(Tg[:3, :3], gn[:3, :3]) <= 1e-5 and np.linalg.norm(Tg[:3, 3] - gn[:3, 3]) <= 1e-5


def test_align_flat_path_matches_persistent_and_oracle(g, replica_setup):
    """The flat GN loop (chosen for clouds whose capacity exceeds the persistent grid) on the
    Replica frame copied into a 120k-capacity cloud: GN and LM poses equal the persistent kernel's
    within 1e-6 (as the frame batches: only the grouping of the H/b sums differs, and both stop
    at an update below eps = 1e-6; measured 2e-8 rad), the same iteration and inlier counts,
    and the oracle's LM pose within 1e-5 rad / 1e-5 m."""
    R = replica_setup
    w = R["w"]
    src = R["src"]
    n = src.n()
    big = g.Cloud.empty(120_000)
    for a, b in ((big.pos, src.pos), (big.cov_a, src.cov_a), (big.cov_b, src.cov_b)):
        a[:n] = b[:n]
    big.d_n.copy_(src.d_n)
    assert big.cap > 148 * 384
    for solver in (g.SOLVER_GN, g.SOLVER_LM):
        p = g.align_params(max_iters=30, max_corr_dist=0.1, solver=solver)
        Tp, stp = g.align(src, R["tgt"], w.T_init, p)
        Tf, stf = g.align(big, R["tgt"], w.T_init, p)
        assert rot_angle(Tf[:3, :3], Tp[:3, :3]) < 1e-6 and np.abs(Tf[:3, 3] - Tp[:3, 3]).max() < 1e-6
        assert stf["iters"] == stp["iters"] and stf["n_inliers"] == stp["n_inliers"] and stf["status"] == stp["status"]
    ref = oracle.align(R["xyz"], R["ocs"], R["txyz"], R["oct"], w.T_init, max_iters=30, max_corr_dist=0.1,
                       use_tree=True, tree=R["tree"], solver=1, lm_lambda0=1e-4)
    assert rot_angle(Tf[:3, :3], ref["T"][:3, :3]) <= 1e-5 and np.linalg.norm(Tf[:3, 3] - ref["T"][:3, 3]) <= 1e-5


@pytest.mark.parametrize("h", [0.01, 0.03, 0.1])
def test_voxel_downsample(g, replica, tum, h):
    """N4 (R31) vs the oracle on a Replica frame (stride 1, ~800k points) and the noisy
    TUM frame: the same voxels in the same order (first member), counts exact, centroids equal
    (binary64 sums of one voxel's members are exact, so bit-equal in practice; checked to 1 ulp);
    then A2-A4 on the voxel cloud (general-cloud hash path) == the oracle (kNN bit-exact)."""
    for w in (replica, tum):
        K = w.K
        pos, d_n = gpu_points(g, w.depth, K, 1)
        xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, 1)
        out, d_m = g.voxel_downsample(pos, d_n, h)
        m = int(d_m.item())
        op, oc = oracle.voxel_downsample(xyz, h)
        assert m == op.shape[0] and 0 < m <= xyz.shape[0]
        gp = out[:m].cpu().numpy()
        np.testing.assert_array_equal(gp[:, 3].view(np.int32), oc)
        np.testing.assert_allclose(gp[:, :3], op, rtol=1.2e-7, atol=0)
        assert (gp[:, :3] == op).mean() > 0.999
    if h == 0.03:  # the voxel cloud through A2-A4 (hash path)
        cl = g.Cloud.from_points(out[:m, :3].contiguous())
        _cov_check(g, gp[:, :3].copy(), cl.pos, cl.d_n, cell0=2 * h, levels=1)


def test_align_batch_lm(g):
    """The LM solver in the batched kernel (k_align_batch<true>): each frame's pose equals
    single-frame LM tracking's (1e-6)."""
    seq = synth.make_sequence(4, 4, "replica", M=300_000)
    rows = synth.render_sequence_rows(seq, DEV)
    K = seq.K
    prm = g.align_params(max_iters=30, max_corr_dist=0.1, solver=g.SOLVER_LM, lm_lambda0=1e-2)
    tgt = g.build_target(t(seq.means), t(seq.quats), t(seq.scales))
    init = np.stack([synth.perturb_pose(seq.T_gt[1 + b], 60 + b, 2.0, 0.03) for b in range(3)])
    bt = g.BatchTracker(3, K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    bt.rows.copy_(rows[1:4])
    Tb, stb = bt.track_rows(tgt, init)
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
    for b in range(3):
        tr.rows.copy_(rows[1 + b])
        Ts, sts = tr.track_rows(tgt, init[b])
        assert rot_angle(Tb[b][:3, :3], Ts[:3, :3]) < 1e-6 and np.abs(Tb[b][:3, 3] - Ts[:3, 3]).max() < 1e-6
        assert stb[b]["status"] == sts["status"] == g.OK
        assert rot_angle(Tb[b][:3, :3], seq.T_gt[1 + b][:3, :3]) < math.radians(0.05)


def test_gaussian_map_capacity_and_unfiltered_insert(g, c1):
    """GaussianMap: an unfiltered insertion (corr None) appends every point at the pose (means ==
    K3 of the oracle); an insertion beyond the capacity drops the excess rows on the device and
    counts them (no out-of-bounds write, the map unchanged)."""
    K = c1.K
    pos, d_n = gpu_points(g, c1.depth, K, 1)
    xyz, _ = oracle.backproject(c1.depth, K.fx, K.fy, K.cx, K.cy, 1)
    n = xyz.shape[0]
    cl = g.covariances(pos, d_n, cell0=0.0, levels=3)
    m0 = np.zeros((10, 3), np.float32)
    q0 = np.tile(np.float32([1, 0, 0, 0]), (10, 1))
    s0 = np.full((10, 3), 0.01, np.float32)
    gm = g.GaussianMap(t(m0), t(q0), t(s0), capacity=10 + n, max_insert=n, cell=0.05)
    T = np.eye(4)
    T[:3, 3] = [0.5, -0.25, 1.0]
    gm.insert(cl, t(T), None)
    assert gm.M == 10 + n and int(gm.d_M[1].item()) == n
    om, _, _ = oracle.export_gaussians(xyz, oracle.covariances(xyz)["raw"], T=T)
    np.testing.assert_array_equal(gm.means[10:10 + n].cpu().numpy(), om.astype(np.float32))
    gm.insert(cl, t(T), None)  # 10 + 2n > capacity: all n rows dropped
    assert gm.M == 10 + n and int(gm.d_M[4].item()) == n
    np.testing.assert_array_equal(gm.means[10:10 + n].cpu().numpy(), om.astype(np.float32))
