"""ctypes binding of the CPU ORACLE (oracle/oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module.  The product path (paper_2403_12550_b200) never imports it.
Every function here is argument marshalling; the arithmetic is in oracle.c, where each
function cites the PAPER.md / SPEC.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NONE, PLANE, ELLIPSE = 0, 1, 2
FLAG_LOW_SUPPORT, FLAG_DEGENERATE = 1, 2
OK, DEGENERATE_FRAME, TRACKING_LOST, MAX_ITERS = 0, 4, 5, 6


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, -O2 -ffp-contract=off, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i, f, d = C.c_int, C.c_float, C.c_double
        L.ora_backproject.argtypes = [P, i, i, i, f, f, f, f, i, f, f, P, P, i]
        L.ora_backproject.restype = i
        L.ora_knn_brute.argtypes = [P, i, P, i, i, P, P]
        L.ora_kdtree_build.argtypes = [P, i]
        L.ora_kdtree_build.restype = P
        L.ora_kdtree_free.argtypes = [P]
        L.ora_kdtree_knn.argtypes = [P, P, i, i, P, P]
        L.ora_kdtree_nn_d.argtypes = [P, P, i, P, P]
        L.ora_covariance.argtypes = [P, P, i, P]
        L.ora_eigen_jacobi.argtypes = [P, P, P]
        L.ora_regularize_eig.argtypes = [P, P, i, d, P]
        L.ora_regularize_eig.restype = i
        L.ora_regularize.argtypes = [P, i, d, P]
        L.ora_regularize.restype = i
        L.ora_covariances.argtypes = [P, i, i, i, d, i, P, P, P, P]
        L.ora_target_from_map.argtypes = [P, P, i, i, i, d, P, P]
        L.ora_linearize.argtypes = [P, P, i, P, P, i, P, P, f, P, P, P, P]
        L.ora_linearize.restype = i
        L.ora_linearize_ex.argtypes = [P, P, i, P, P, i, P, P, f, P, P, P, P, P]
        L.ora_linearize_ex.restype = i
        L.ora_solve.argtypes = [P, P, P]
        L.ora_solve.restype = i
        L.ora_so3_exp.argtypes = [P, P]
        L.ora_update.argtypes = [P, P]
        L.ora_align.argtypes = [P, P, i, P, P, i, i, P, P, i, f, d, d, i, P, P]
        L.ora_align.restype = i
        L.ora_align2.argtypes = [P, P, i, P, P, i, i, P, P, i, f, d, d, i, i, d, P, P]
        L.ora_align2.restype = i
        L.ora_voxel_downsample.argtypes = [P, i, f, P, P]
        L.ora_voxel_downsample.restype = i
        L.ora_num_threads.restype = i
        L.ora_set_threads.argtypes = [i]
        L.ora_set_threads.restype = None
        L.ora_scale_align.argtypes = [P, d, d, d, P]
        L.ora_scale_align.restype = i
        L.ora_export_gaussian.argtypes = [P, P, P, i, d, d, d, P, P, P]
        L.ora_export_gaussian.restype = i
        L.ora_export_gaussians.argtypes = [P, P, i, P, i, d, d, d, P, P, P]
        L.ora_export_gaussians.restype = None
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f32(a, shape_last=None):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def num_threads() -> int:
    return lib().ora_num_threads()


def set_threads(n: int) -> None:
    lib().ora_set_threads(int(n))


def backproject(depth, fx, fy, cx, cy, stride=1, zmin=0.1, zmax=10.0):
    """O1 -> (xyz (n,3) f32, pix (n,) int32)."""
    depth = _f32(depth)
    H, W = depth.shape
    cap = ((H + stride - 1) // stride) * ((W + stride - 1) // stride)
    xyz = np.empty((max(cap, 1), 3), np.float32)
    pix = np.empty(max(cap, 1), np.int32)
    n = lib().ora_backproject(_p(depth), H, W, W, fx, fy, cx, cy, stride, zmin, zmax, _p(xyz), _p(pix), cap)
    assert n >= 0
    return xyz[:n].copy(), pix[:n].copy()


def knn_brute(xyz, k, queries=None, return_keys=False):
    """O2 brute-force kNN by the binary64 K2 key, ties by index.  queries: indices into xyz
    (default all).  -> idx (nq,k) int32 [, keys (nq,k) float64]"""
    xyz = _f32(xyz)
    n = xyz.shape[0]
    q = np.arange(n, dtype=np.int32) if queries is None else np.ascontiguousarray(queries, np.int32)
    out = np.empty((q.shape[0], k), np.int32)
    keys = np.empty((q.shape[0], k), np.float64)
    lib().ora_knn_brute(_p(xyz), n, _p(q), q.shape[0], k, _p(out), _p(keys))
    return (out, keys) if return_keys else out


class KDTree:
    """Exact kd-tree over binary32 points with the (K2 key, idx) order of knn_brute."""

    def __init__(self, xyz):
        self.xyz = _f32(xyz)
        self.n = self.xyz.shape[0]
        self._t = lib().ora_kdtree_build(_p(self.xyz), self.n)

    def knn(self, q, k, return_keys=False):
        q = _f32(q).reshape(-1, 3)
        out = np.empty((q.shape[0], k), np.int32)
        keys = np.empty((q.shape[0], k), np.float64)
        lib().ora_kdtree_knn(C.c_void_p(self._t), _p(q), q.shape[0], k, _p(out), _p(keys))
        return (out, keys) if return_keys else out

    def nn(self, q):
        """1-NN of binary64 queries (n,3) by (K2, idx) -> (idx (n,) int32, key (n,) float64)."""
        q = np.ascontiguousarray(np.asarray(q, np.float64).reshape(-1, 3))
        out = np.empty(q.shape[0], np.int32)
        keys = np.empty(q.shape[0], np.float64)
        lib().ora_kdtree_nn_d(C.c_void_p(self._t), _p(q), q.shape[0], _p(out), _p(keys))
        return out, keys

    def __del__(self):
        if getattr(self, "_t", None):
            lib().ora_kdtree_free(C.c_void_p(self._t))
            self._t = None


def covariance(xyz, nbr):
    """O3 for one neighbour list -> packed (6,) f64 (c00,c01,c02,c11,c12,c22)."""
    xyz = _f32(xyz)
    nbr = np.ascontiguousarray(nbr, np.int32)
    C6 = np.empty(6)
    lib().ora_covariance(_p(xyz), _p(nbr), nbr.shape[0], _p(C6))
    return C6


def eigen(C6):
    """O4 Jacobi -> (lam (3,) descending, V (3,3) with V[:, j] the eigenvector of lam[j])."""
    C6 = np.ascontiguousarray(C6, np.float64)
    lam = np.empty(3)
    Vc = np.empty(9)
    lib().ora_eigen_jacobi(_p(C6), _p(lam), _p(Vc))
    return lam, Vc.reshape(3, 3).T.copy()


def regularize(C6, mode, eps=1e-3):
    """O5 -> (packed (6,) f64, flags)."""
    C6 = np.ascontiguousarray(C6, np.float64)
    out = np.empty(6)
    fl = lib().ora_regularize(_p(C6), mode, eps, _p(out))
    return out, fl


def regularize_eig(lam, V, mode, eps=1e-3):
    lam = np.ascontiguousarray(lam, np.float64)
    Vc = np.ascontiguousarray(np.asarray(V, np.float64).T)
    out = np.empty(6)
    fl = lib().ora_regularize_eig(_p(lam), _p(Vc), mode, eps, _p(out))
    return out, fl


def covariances(xyz, k=20, mode=ELLIPSE, eps=1e-3, brute_max=60000):
    """A2-A4 composed -> dict(cov (n,6) f32, raw (n,6) f64, lam_mid (n,) f64, flags (n,) i32)."""
    xyz = _f32(xyz)
    n = xyz.shape[0]
    cov = np.empty((n, 6), np.float32)
    raw = np.empty((n, 6))
    lm = np.empty(n)
    fl = np.empty(n, np.int32)
    lib().ora_covariances(_p(xyz), n, k, mode, eps, brute_max, _p(cov), _p(raw), _p(lm), _p(fl))
    return dict(cov=cov, raw=raw, lam_mid=lm, flags=fl)


def target_from_map(quats, scales, mode=ELLIPSE, eps=1e-3, scales_are_log=False):
    """O6 -> (cov (M,6) f32, flags (M,) i32)."""
    quats = _f32(quats)
    scales = _f32(scales)
    M = quats.shape[0]
    cov = np.empty((M, 6), np.float32)
    fl = np.empty(M, np.int32)
    lib().ora_target_from_map(_p(quats), _p(scales), int(scales_are_log), M, mode, eps, _p(cov), _p(fl))
    return cov, fl


def linearize(src_xyz, src_cov, tgt_xyz, tgt_cov, T, max_corr_dist=np.inf, tree: KDTree | None = None):
    """O7+O8 -> dict(H (6,6), b (6,), cost, n, corr (n,) int32, bsum = sum_i |J_i^T M_i d_i|)."""
    src_xyz, src_cov, tgt_xyz, tgt_cov = map(_f32, (src_xyz, src_cov, tgt_xyz, tgt_cov))
    T = np.ascontiguousarray(T, np.float64)
    H = np.empty((6, 6))
    b = np.empty(6)
    cost = np.empty(1)
    bsum = np.empty(1)
    corr = np.empty(src_xyz.shape[0], np.int32)
    t = C.c_void_p(tree._t) if tree is not None else None
    n = lib().ora_linearize_ex(_p(src_xyz), _p(src_cov), src_xyz.shape[0], _p(tgt_xyz), _p(tgt_cov),
                               tgt_xyz.shape[0], t, _p(T), float(max_corr_dist), _p(H), _p(b), _p(cost), _p(corr),
                               _p(bsum))
    return dict(H=H, b=b, cost=float(cost[0]), n=n, corr=corr, bsum=float(bsum[0]))


def solve(H, b):
    H = np.ascontiguousarray(H, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    x = np.empty(6)
    ok = lib().ora_solve(_p(H), _p(b), _p(x))
    return x, bool(ok)


def so3_exp(w):
    w = np.ascontiguousarray(w, np.float64)
    R = np.empty(9)
    lib().ora_so3_exp(_p(w), _p(R))
    return R.reshape(3, 3)


def update(T, delta):
    T = np.array(T, np.float64, order="C")
    delta = np.ascontiguousarray(delta, np.float64)
    lib().ora_update(_p(T), _p(delta))
    return T


def align(src_xyz, src_cov, tgt_xyz, tgt_cov, T0, max_iters=30, max_corr_dist=np.inf, eps_rot=1e-6,
          eps_trans=1e-6, min_pairs=50, use_tree=None, tree: KDTree | None = None, solver=0, lm_lambda0=1e-4):
    """O10/O11 -> dict(T, fitness, mean_cost, n_inliers, iters, converged, status).
    tree: optional prebuilt KDTree over tgt_xyz (else one is built per call if use_tree).
    solver 0 = Gauss-Newton, 1 = Levenberg-Marquardt (R30) with initial damping lm_lambda0."""
    src_xyz, src_cov, tgt_xyz, tgt_cov = map(_f32, (src_xyz, src_cov, tgt_xyz, tgt_cov))
    if use_tree is None:
        use_tree = src_xyz.shape[0] * tgt_xyz.shape[0] > 10_000_000
    T0 = np.ascontiguousarray(T0, np.float64)
    T = np.empty((4, 4))
    st = np.empty(6)
    status = lib().ora_align2(_p(src_xyz), _p(src_cov), src_xyz.shape[0], _p(tgt_xyz), _p(tgt_cov),
                              tgt_xyz.shape[0], int(use_tree),
                              C.c_void_p(tree._t) if tree is not None else None, _p(T0), max_iters,
                              float(max_corr_dist), eps_rot, eps_trans, min_pairs, int(solver), float(lm_lambda0),
                              _p(T), _p(st))
    return dict(T=T, fitness=st[0], mean_cost=st[1], n_inliers=int(st[2]), iters=int(st[3]),
                converged=bool(st[4]), status=int(status))


def scale_align(scales, z, p=1.5, c=1.0):
    """O12 -> (3,) f64 scales c * scales / z^p."""
    s = np.ascontiguousarray(scales, np.float64)
    out = np.empty(3)
    rc = lib().ora_scale_align(_p(s), float(z), float(p), float(c), _p(out))
    if rc != 0:
        raise ValueError("scale_align: z must be > 0")
    return out


def export_gaussian(C6, p_cam, T=None, mode=ELLIPSE, eps=1e-3, p=1.5, c=1.0):
    """O12' one point -> (mean (3,), quat wxyz (4,), scales (3,), rc) in binary64."""
    C6 = np.ascontiguousarray(C6, np.float64)
    pc = _f32(p_cam)
    Tm = None if T is None else np.ascontiguousarray(T, np.float64)
    mean, quat, sc = np.empty(3), np.empty(4), np.empty(3)
    rc = lib().ora_export_gaussian(_p(C6), _p(pc), _p(Tm), mode, eps, p, c, _p(mean), _p(quat), _p(sc))
    return mean, quat, sc, rc


def export_gaussians(xyz, raw, T=None, mode=ELLIPSE, eps=1e-3, p=1.5, c=1.0):
    """O12' over a cloud (raw covariances from covariances()['raw']) -> (means, quats, scales) f64."""
    xyz = _f32(xyz)
    raw = np.ascontiguousarray(raw, np.float64)
    n = xyz.shape[0]
    Tm = None if T is None else np.ascontiguousarray(T, np.float64)
    means, quats, sc = np.empty((n, 3)), np.empty((n, 4)), np.empty((n, 3))
    lib().ora_export_gaussians(_p(xyz), _p(raw), n, _p(Tm), mode, eps, p, c, _p(means), _p(quats), _p(sc))
    return means, quats, sc


def voxel_downsample(xyz, voxel):
    """N4 (R31) -> (points (m,3) f32 ordered by each voxel's first member, counts (m,) i32)."""
    xyz = _f32(xyz)
    n = xyz.shape[0]
    out = np.empty((max(n, 1), 3), np.float32)
    cnt = np.empty(max(n, 1), np.int32)
    m = lib().ora_voxel_downsample(_p(xyz), n, float(voxel), _p(out), _p(cnt))
    return out[:m].copy(), cnt[:m].copy()
