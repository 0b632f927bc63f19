"""Seeded synthetic workloads for the G-ICP tracking hot path.

This module only *generates inputs*: depth frames ray-cast from an analytic room,
3DGS-like map Gaussians sampled on the room's surfaces, and camera poses.  It holds
none of the method's arithmetic (no back-projection, kNN, covariance, regularisation,
correspondence or Gauss-Newton code) and is imported by both the oracle-side tests
and the CUDA-side tests/bench, so that both see identical input bytes.

Shapes follow the paper's workloads (Replica 1200x680 synthetic,
TUM 640x480 real with holes) as made concrete in SURVEY.md §8(d).1.
Seeds: scene 1000+cfg, pose 2000+cfg, noise 3000+cfg, map 4000+cfg (PCG64).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Intrinsics", "REPLICA", "TUM", "TINY", "Scene", "make_scene", "raycast_depth",
    "tum_noise", "sample_map", "camera_pose", "perturb_pose", "rot_axis_angle",
    "make_frame_workload", "make_c1", "quat_from_rotmat", "raycast_depth_torch", "lissajous_trajectory",
    "make_sequence", "Sequence", "render_sequence_rows", "trajectory_error", "fronto_parallel_wall",
]


@dataclasses.dataclass(frozen=True)
class Intrinsics:
    W: int
    H: int
    fx: float
    fy: float
    cx: float
    cy: float


# Replica export used by dense-SLAM work (1200x680, f=600); TUM fr1 (640x480); tiny C1 (same 90 deg HFOV).
REPLICA = Intrinsics(1200, 680, 600.0, 600.0, 599.5, 339.5)
TUM = Intrinsics(640, 480, 517.3, 516.5, 318.6, 255.3)
TINY = Intrinsics(64, 48, 32.0, 32.0, 31.5, 23.5)


@dataclasses.dataclass
class Scene:
    room: np.ndarray           # (3,) extents, room is [0,Lx]x[0,Ly]x[0,Lz], z up
    boxes: np.ndarray          # (nb, 7): cx, cy, cz, hx, hy, hz, yaw
    spheres: np.ndarray        # (ns, 4): cx, cy, cz, r
    cylinders: np.ndarray      # (nc, 5): cx, cy, r, z0, h   (vertical axis)


def make_scene(seed: int, room=(6.0, 5.0, 3.0), n_boxes=12, n_spheres=6, n_cyl=4) -> Scene:
    """Axis-aligned room seen from inside with interior objects."""
    rng = np.random.default_rng(seed)
    L = np.asarray(room, dtype=np.float64)
    boxes = []
    for _ in range(n_boxes):
        e = rng.uniform(0.2, 1.2, size=3)
        e[2] = min(e[2], 0.8 * L[2])
        c = np.array([rng.uniform(0.3, L[0] - 0.3), rng.uniform(0.3, L[1] - 0.3), e[2] / 2])
        boxes.append([*c, *(e / 2), rng.uniform(0, np.pi)])
    spheres = []
    for _ in range(n_spheres):
        r = rng.uniform(0.1, 0.4)
        spheres.append([rng.uniform(r + 0.2, L[0] - r - 0.2), rng.uniform(r + 0.2, L[1] - r - 0.2),
                        rng.uniform(r, L[2] - r - 0.3), r])
    cyls = []
    for _ in range(n_cyl):
        r = rng.uniform(0.05, 0.3)
        cyls.append([rng.uniform(r + 0.2, L[0] - r - 0.2), rng.uniform(r + 0.2, L[1] - r - 0.2), r, 0.0,
                     min(rng.uniform(0.5, 2.0), L[2] - 0.1)])
    return Scene(L, np.array(boxes, dtype=np.float64).reshape(-1, 7),
                 np.array(spheres, dtype=np.float64).reshape(-1, 4),
                 np.array(cyls, dtype=np.float64).reshape(-1, 5))


def _rot_z(yaw):
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _ray_hits(scene: Scene, o: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Smallest positive ray parameter t for rays o + t d (d per ray, o shared). inf on miss."""
    n = d.shape[0]
    big = np.inf
    with np.errstate(divide="ignore", invalid="ignore"):
        # room interior: exit distance
        inv = 1.0 / d
        t1 = (0.0 - o[None, :]) * inv
        t2 = (scene.room[None, :] - o[None, :]) * inv
        tfar = np.min(np.maximum(t1, t2), axis=1)
        best = np.where(tfar > 0, tfar, big)
        for b in scene.boxes:
            Rz = _rot_z(b[6])
            ol = Rz.T @ (o - b[:3])
            dl = d @ Rz  # (Rz^T d)^T
            invl = 1.0 / dl
            h = b[3:6]
            ta = (-h[None, :] - ol[None, :]) * invl
            tb = (h[None, :] - ol[None, :]) * invl
            tn = np.max(np.minimum(ta, tb), axis=1)
            tf = np.min(np.maximum(ta, tb), axis=1)
            hit = (tn <= tf) & (tn > 1e-6)
            best = np.where(hit & (tn < best), tn, best)
        for s in scene.spheres:
            oc = o - s[:3]
            a = np.einsum("ij,ij->i", d, d)
            bq = d @ oc
            c = oc @ oc - s[3] ** 2
            disc = bq * bq - a * c
            t = (-bq - np.sqrt(np.maximum(disc, 0))) / a
            hit = (disc >= 0) & (t > 1e-6)
            best = np.where(hit & (t < best), t, best)
        for cy in scene.cylinders:
            ox, oy = o[0] - cy[0], o[1] - cy[1]
            a = d[:, 0] ** 2 + d[:, 1] ** 2
            bq = ox * d[:, 0] + oy * d[:, 1]
            c = ox * ox + oy * oy - cy[2] ** 2
            disc = bq * bq - a * c
            t = (-bq - np.sqrt(np.maximum(disc, 0))) / a
            z = o[2] + t * d[:, 2]
            hit = (disc >= 0) & (t > 1e-6) & (z >= cy[3]) & (z <= cy[3] + cy[4])
            best = np.where(hit & (t < best), t, best)
            # top cap
            tc = (cy[3] + cy[4] - o[2]) / d[:, 2]
            px, py = ox + tc * d[:, 0], oy + tc * d[:, 1]
            hit = (tc > 1e-6) & (px * px + py * py <= cy[2] ** 2)
            best = np.where(hit & (tc < best), tc, best)
    return best


def raycast_depth(scene: Scene, K: Intrinsics, T_wc: np.ndarray) -> np.ndarray:
    """z-depth image (H, W) float32 in metres of the scene seen from camera pose T_wc
    (camera->world, OpenCV camera axes: x right, y down, z forward)."""
    u, v = np.meshgrid(np.arange(K.W, dtype=np.float64), np.arange(K.H, dtype=np.float64))
    dc = np.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, np.ones_like(u)], axis=-1).reshape(-1, 3)
    R, t = T_wc[:3, :3], T_wc[:3, 3]
    dw = dc @ R.T
    tt = _ray_hits(scene, t, dw)  # ray parameter along a direction with unit camera-z => z-depth
    depth = np.where(np.isfinite(tt), tt, 0.0).reshape(K.H, K.W)
    return depth.astype(np.float32)


def tum_noise(depth: np.ndarray, seed: int) -> np.ndarray:
    """Kinect-like degradation: axial noise sigma(z)=0.0012+0.0019(z-0.4)^2,
    quantisation to 1/5000 m, elliptical holes (~10%), depth-edge dropout, dropout ramp beyond 4 m."""
    rng = np.random.default_rng(seed)
    H, W = depth.shape
    z = depth.astype(np.float64)
    valid = z > 0
    sig = 0.0012 + 0.0019 * (z - 0.4) ** 2
    zn = z + rng.standard_normal(z.shape) * sig
    zn = np.round(zn * 5000.0) / 5000.0
    gy, gx = np.gradient(z)
    edge = np.maximum(np.abs(gx), np.abs(gy)) > 0.1
    holes = np.zeros_like(valid)
    vv, uu = np.mgrid[0:H, 0:W]
    target = 0.10 * H * W
    while holes.sum() < target:
        cu, cv = rng.uniform(0, W), rng.uniform(0, H)
        a, b = rng.uniform(0.02, 0.08) * W, rng.uniform(0.02, 0.08) * H
        th = rng.uniform(0, np.pi)
        du, dv = uu - cu, vv - cv
        x = du * math.cos(th) + dv * math.sin(th)
        y = -du * math.sin(th) + dv * math.cos(th)
        holes |= (x / a) ** 2 + (y / b) ** 2 <= 1.0
    ramp = np.clip((z - 4.0) / 4.0, 0.0, 1.0)
    drop = rng.uniform(size=z.shape) < ramp
    keep = valid & ~edge & ~holes & ~drop & (zn > 0)
    return np.where(keep, zn, 0.0).astype(np.float32)


def _unit(v):
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def quat_from_rotmat(R: np.ndarray) -> np.ndarray:
    """wxyz unit quaternions (w >= 0) for a stack of rotation matrices (N,3,3)."""
    R = np.asarray(R, dtype=np.float64)
    tr = R[:, 0, 0] + R[:, 1, 1] + R[:, 2, 2]
    q = np.empty((R.shape[0], 4))
    w = np.sqrt(np.maximum(0.0, 1.0 + tr)) / 2
    x = np.sqrt(np.maximum(0.0, 1.0 + R[:, 0, 0] - R[:, 1, 1] - R[:, 2, 2])) / 2
    y = np.sqrt(np.maximum(0.0, 1.0 - R[:, 0, 0] + R[:, 1, 1] - R[:, 2, 2])) / 2
    z = np.sqrt(np.maximum(0.0, 1.0 - R[:, 0, 0] - R[:, 1, 1] + R[:, 2, 2])) / 2
    x = np.copysign(x, R[:, 2, 1] - R[:, 1, 2])
    y = np.copysign(y, R[:, 0, 2] - R[:, 2, 0])
    z = np.copysign(z, R[:, 1, 0] - R[:, 0, 1])
    q[:, 0], q[:, 1], q[:, 2], q[:, 3] = w, x, y, z
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _surfaces(scene: Scene):
    """List of (area, sampler) where sampler(rng, n) -> (points (n,3), normals (n,3))."""
    L = scene.room
    out = []

    def rect(origin, e1, e2, normal):
        origin, e1, e2, normal = map(np.asarray, (origin, e1, e2, normal))
        area = np.linalg.norm(e1) * np.linalg.norm(e2)

        def f(rng, n):
            a, b = rng.uniform(size=(2, n, 1))
            return origin + a * e1 + b * e2, np.broadcast_to(normal, (n, 3)).copy()
        return area, f

    # room faces (normals point inward)
    out.append(rect([0, 0, 0], [L[0], 0, 0], [0, L[1], 0], [0, 0, 1]))
    out.append(rect([0, 0, L[2]], [L[0], 0, 0], [0, L[1], 0], [0, 0, -1]))
    out.append(rect([0, 0, 0], [L[0], 0, 0], [0, 0, L[2]], [0, 1, 0]))
    out.append(rect([0, L[1], 0], [L[0], 0, 0], [0, 0, L[2]], [0, -1, 0]))
    out.append(rect([0, 0, 0], [0, L[1], 0], [0, 0, L[2]], [1, 0, 0]))
    out.append(rect([L[0], 0, 0], [0, L[1], 0], [0, 0, L[2]], [-1, 0, 0]))
    for b in scene.boxes:
        Rz = _rot_z(b[6])
        c, h = b[:3], b[3:6]
        for ax in range(3):
            for sgn in (-1.0, 1.0):
                if ax == 2 and sgn < 0:
                    continue  # bottom face rests on the floor
                o1, o2 = [i for i in range(3) if i != ax]
                nrm = np.zeros(3); nrm[ax] = sgn
                e1 = np.zeros(3); e1[o1] = 2 * h[o1]
                e2 = np.zeros(3); e2[o2] = 2 * h[o2]
                corner = -h.copy(); corner[ax] = sgn * h[ax]
                out.append(rect(c + Rz @ corner, Rz @ e1, Rz @ e2, Rz @ nrm))
    for s in scene.spheres:
        def fs(rng, n, s=s):
            nrm = _unit(rng.standard_normal((n, 3)))
            return s[:3] + s[3] * nrm, nrm
        out.append((4 * np.pi * s[3] ** 2, fs))
    for cy in scene.cylinders:
        def fc(rng, n, cy=cy):
            th = rng.uniform(0, 2 * np.pi, n)
            zz = rng.uniform(cy[3], cy[3] + cy[4], n)
            nrm = np.stack([np.cos(th), np.sin(th), np.zeros(n)], 1)
            return np.stack([cy[0] + cy[2] * nrm[:, 0], cy[1] + cy[2] * nrm[:, 1], zz], 1), nrm

        def ft(rng, n, cy=cy):
            r = cy[2] * np.sqrt(rng.uniform(size=n))
            th = rng.uniform(0, 2 * np.pi, n)
            p = np.stack([cy[0] + r * np.cos(th), cy[1] + r * np.sin(th), np.full(n, cy[3] + cy[4])], 1)
            return p, np.broadcast_to(np.array([0.0, 0.0, 1.0]), (n, 3)).copy()
        out.append((2 * np.pi * cy[2] * cy[4], fc))
        out.append((np.pi * cy[2] ** 2, ft))
    return out


def sample_map(scene: Scene, M: int, seed: int, outlier_frac: float = 0.01):
    """3DGS-like map of M Gaussians on the scene surfaces.

    Returns (means (M,3) f32, quats_wxyz (M,4) f32, scales (M,3) f32 linear, spacing l).
    Scales are ordered along the rotation's columns (t1, t2, n)."""
    rng = np.random.default_rng(seed)
    surf = _surfaces(scene)
    areas = np.array([a for a, _ in surf])
    A = areas.sum()
    ell = math.sqrt(A / M)
    n_out = int(round(outlier_frac * M))
    n_surf = M - n_out
    counts = rng.multinomial(n_surf, areas / A)
    pts, nrms = [], []
    for (a, f), c in zip(surf, counts):
        if c:
            p, nn = f(rng, int(c))
            pts.append(p); nrms.append(nn)
    P = np.concatenate(pts)
    N = _unit(np.concatenate(nrms))
    P = P + N * rng.normal(0.0, 0.001, size=(P.shape[0], 1))
    # tangent frame with random in-plane angle
    ref = np.where(np.abs(N[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]), np.array([[1.0, 0.0, 0.0]]))
    t1 = _unit(np.cross(ref, N))
    t2 = np.cross(N, t1)
    th = rng.uniform(0, 2 * np.pi, size=(P.shape[0], 1))
    a1 = np.cos(th) * t1 + np.sin(th) * t2
    a2 = np.cross(N, a1)
    R = np.stack([a1, a2, N], axis=2)  # columns
    line = rng.uniform(size=P.shape[0]) < 0.1
    S = np.empty((P.shape[0], 3))
    S[:, 0] = np.where(line, rng.uniform(1.0, 3.0, P.shape[0]), rng.uniform(0.5, 1.5, P.shape[0])) * ell
    S[:, 1] = np.where(line, rng.uniform(0.05, 0.2, P.shape[0]), rng.uniform(0.5, 1.5, P.shape[0])) * ell
    S[:, 2] = rng.uniform(0.05, 0.2, P.shape[0]) * ell
    # floating outliers
    Po = rng.uniform(size=(n_out, 3)) * scene.room
    Ro = np.linalg.qr(rng.standard_normal((n_out, 3, 3)))[0]
    Ro[np.linalg.det(Ro) < 0, :, 2] *= -1
    So = rng.uniform(0.3, 1.5, size=(n_out, 3)) * ell
    means = np.concatenate([P, Po])
    Rall = np.concatenate([R, Ro])
    scales = np.concatenate([S, So])
    perm = rng.permutation(M)
    q = quat_from_rotmat(Rall[perm])
    return (means[perm].astype(np.float32), q.astype(np.float32), scales[perm].astype(np.float32), ell)


def rot_axis_angle(axis, angle) -> np.ndarray:
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    Kx = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(angle) * Kx + (1 - math.cos(angle)) * (Kx @ Kx)


def _clearance(scene: Scene, p: np.ndarray) -> float:
    d = min(p.min(), (scene.room - p).min())
    for b in scene.boxes:
        d = min(d, np.linalg.norm(p - b[:3]) - np.linalg.norm(b[3:6]))
    for s in scene.spheres:
        d = min(d, np.linalg.norm(p - s[:3]) - s[3])
    for c in scene.cylinders:
        d = min(d, math.hypot(p[0] - c[0], p[1] - c[1]) - c[2])
    return d


def camera_pose(scene: Scene, seed: int) -> np.ndarray:
    """Camera-to-world 4x4 pose inside free space (>=0.5 m clearance), looking at a wall point."""
    rng = np.random.default_rng(seed)
    L = scene.room
    for _ in range(10000):
        p = np.array([rng.uniform(0.6, L[0] - 0.6), rng.uniform(0.6, L[1] - 0.6), rng.uniform(0.8, L[2] - 0.6)])
        if _clearance(scene, p) >= 0.5:
            break
    tgt = np.array([rng.uniform(0, L[0]), rng.uniform(0, L[1]), rng.uniform(0.2, L[2] - 0.2)])
    face = rng.integers(4)
    tgt[face // 2] = 0.0 if face % 2 == 0 else L[face // 2]
    zc = _unit(tgt - p)
    xc = _unit(np.cross(zc, np.array([0.0, 0.0, 1.0])))
    yc = np.cross(zc, xc)
    T = np.eye(4)
    T[:3, :3] = np.stack([xc, yc, zc], axis=1)
    T[:3, 3] = p
    return T


def perturb_pose(T: np.ndarray, seed: int, max_deg=2.0, max_trans=0.03) -> np.ndarray:
    """T o D: perturb T in the camera frame by a rotation U[0,max_deg] deg about a random axis and a
    translation of norm U[0,max_trans] (typical 30 Hz inter-frame motion)."""
    rng = np.random.default_rng(seed)
    ax = _unit(rng.standard_normal(3))
    R = rot_axis_angle(ax, math.radians(rng.uniform(0, max_deg)))
    tv = _unit(rng.standard_normal(3)) * rng.uniform(0, max_trans)
    D = np.eye(4); D[:3, :3] = R; D[:3, 3] = tv
    return T @ D


@dataclasses.dataclass
class FrameWorkload:
    K: Intrinsics
    depth: np.ndarray       # (H, W) f32 metres, 0 = invalid
    T_gt: np.ndarray        # camera -> world
    T_init: np.ndarray
    means: np.ndarray       # map
    quats: np.ndarray
    scales: np.ndarray
    ell: float
    stride: int


def make_frame_workload(cfg: int, shape: str = "replica", M: int = 1_000_000, stride: int = 4,
                        noisy: bool = False) -> FrameWorkload:
    """One frame + its map (configs C2-C4 of BASELINE.json)."""
    if shape == "replica":
        K, room, nb, ns, nc = REPLICA, (6.0, 5.0, 3.0), 12, 6, 4
    elif shape == "tum":
        K, room, nb, ns, nc = TUM, (8.0, 8.0, 3.0), 16, 6, 6
    else:
        raise ValueError(shape)
    scene = make_scene(1000 + cfg, room, nb, ns, nc)
    T = camera_pose(scene, 2000 + cfg)
    depth = raycast_depth(scene, K, T)
    if noisy:
        depth = tum_noise(depth, 3000 + cfg)
    means, quats, scales, ell = sample_map(scene, M, 4000 + cfg)
    T0 = perturb_pose(T, 2100 + cfg)
    return FrameWorkload(K, depth, T, T0, means, quats, scales, ell, stride)


@dataclasses.dataclass
class C1Workload:
    K: Intrinsics
    depth: np.ndarray
    T_gt: np.ndarray


def make_c1(cfg: int = 1) -> C1Workload:
    """C1 (BASELINE.json configs[0]): 64x48 frame of the Replica-shaped room; the target is the same
    cloud under T_gt = 8 deg about a random axis + (0.05,-0.08,0.03) m; init = identity."""
    scene = make_scene(1000 + cfg)
    T = camera_pose(scene, 2000 + cfg)
    depth = raycast_depth(scene, TINY, T)
    rng = np.random.default_rng(2200 + cfg)
    Tg = np.eye(4)
    Tg[:3, :3] = rot_axis_angle(rng.standard_normal(3), math.radians(8.0))
    Tg[:3, 3] = [0.05, -0.08, 0.03]
    return C1Workload(TINY, depth, Tg)


def fronto_parallel_wall(K: Intrinsics = REPLICA, z: float = 2.0, hole=None) -> np.ndarray:
    """Depth of a wall parallel to the image plane at distance z (the tie-heavy case of SURVEY
    hard part 1: back-projected stride lattices give many equal squared distances).  hole =
    (v0, v1, u0, u1) pixels set invalid (NaN)."""
    depth = np.full((K.H, K.W), z, np.float32)
    if hole is not None:
        v0, v1, u0, u1 = hole
        depth[v0:v1, u0:u1] = np.nan
    return depth


# ------------------------------------------------------------------------------------------ C5
def raycast_depth_torch(scene: Scene, K: Intrinsics, T_wc, device="cuda"):
    """raycast_depth on the GPU (torch, binary64): the same analytic z-depth, for generating long
    sequences (C5) quickly.  Returns a (H, W) float32 tensor on `device`."""
    import torch

    f64 = torch.float64
    u, v = torch.meshgrid(torch.arange(K.W, dtype=f64, device=device), torch.arange(K.H, dtype=f64, device=device),
                          indexing="xy")
    dc = torch.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, torch.ones_like(u)], dim=-1).reshape(-1, 3)
    T = torch.as_tensor(np.asarray(T_wc), dtype=f64, device=device)
    R, o = T[:3, :3], T[:3, 3]
    d = dc @ R.T
    inf = torch.tensor(float("inf"), dtype=f64, device=device)
    room = torch.as_tensor(scene.room, dtype=f64, device=device)
    inv = 1.0 / d
    t1 = (0.0 - o[None, :]) * inv
    t2 = (room[None, :] - o[None, :]) * inv
    tfar = torch.max(t1, t2).min(dim=1).values
    best = torch.where(tfar > 0, tfar, inf)
    for b in scene.boxes:
        Rz = torch.as_tensor(_rot_z(b[6]), dtype=f64, device=device)
        c = torch.as_tensor(b[:3], dtype=f64, device=device)
        h = torch.as_tensor(b[3:6], dtype=f64, device=device)
        ol = Rz.T @ (o - c)
        dl = d @ Rz
        invl = 1.0 / dl
        ta = (-h[None, :] - ol[None, :]) * invl
        tb = (h[None, :] - ol[None, :]) * invl
        tn = torch.min(ta, tb).max(dim=1).values
        tf = torch.max(ta, tb).min(dim=1).values
        hit = (tn <= tf) & (tn > 1e-6)
        best = torch.where(hit & (tn < best), tn, best)
    for s in scene.spheres:
        oc = o - torch.as_tensor(s[:3], dtype=f64, device=device)
        a = (d * d).sum(dim=1)
        bq = d @ oc
        c = oc @ oc - s[3] ** 2
        disc = bq * bq - a * c
        t = (-bq - torch.sqrt(torch.clamp(disc, min=0))) / a
        hit = (disc >= 0) & (t > 1e-6)
        best = torch.where(hit & (t < best), t, best)
    for cy in scene.cylinders:
        ox, oy = o[0] - cy[0], o[1] - cy[1]
        a = d[:, 0] ** 2 + d[:, 1] ** 2
        bq = ox * d[:, 0] + oy * d[:, 1]
        c = ox * ox + oy * oy - cy[2] ** 2
        disc = bq * bq - a * c
        t = (-bq - torch.sqrt(torch.clamp(disc, min=0))) / a
        z = o[2] + t * d[:, 2]
        hit = (disc >= 0) & (t > 1e-6) & (z >= cy[3]) & (z <= cy[3] + cy[4])
        best = torch.where(hit & (t < best), t, best)
        tc = (cy[3] + cy[4] - o[2]) / d[:, 2]
        px, py = ox + tc * d[:, 0], oy + tc * d[:, 1]
        hit = (tc > 1e-6) & (px * px + py * py <= cy[2] ** 2)
        best = torch.where(hit & (tc < best), tc, best)
    depth = torch.where(torch.isfinite(best), best, torch.zeros_like(best)).reshape(K.H, K.W)
    return depth.to(torch.float32)


@dataclasses.dataclass
class Sequence:
    K: Intrinsics
    scene: Scene
    T_gt: np.ndarray        # (n, 4, 4) camera -> world at 30 Hz
    means: np.ndarray       # the map of the room
    quats: np.ndarray
    scales: np.ndarray
    ell: float
    stride: int


def lissajous_trajectory(scene: Scene, seed: int, n: int, fps: float = 30.0, vmax: float = 0.5,
                         wmax_deg: float = 30.0) -> np.ndarray:
    """Camera poses (n, 4, 4) along a Lissajous path inside the room's free space (>= 0.5 m from
    walls and objects), looking at a slowly moving point on the walls; speed <= vmax m/s, view
    rotation <= wmax_deg deg/s.  Parameters are redrawn until both hold."""
    rng = np.random.default_rng(seed)
    L = scene.room
    ts = np.arange(n) / fps
    for _attempt in range(1000):
        c = np.array([rng.uniform(0.35, 0.65) * L[0], rng.uniform(0.35, 0.65) * L[1], min(1.5, L[2] / 2)])
        A = np.array([0.25 * L[0], 0.25 * L[1], 0.15 * L[2]]) * rng.uniform(0.3, 1.0, 3)
        w = rng.uniform(0.1, 0.3, 3) * 2 * np.pi / 10.0  # rad/s (periods of tens of seconds)
        ph = rng.uniform(0, 2 * np.pi, 3)
        w = w * min(1.0, vmax / max(np.linalg.norm(A * w), 1e-9))  # |p'| <= |A w| <= vmax
        P = c[None, :] + A[None, :] * np.sin(w[None, :] * ts[:, None] + ph[None, :])
        if min(_clearance(scene, p) for p in P) < 0.5:
            continue
        look_c = np.array([L[0] / 2, L[1] / 2, L[2] / 2])
        look_A = np.array([0.45 * L[0], 0.45 * L[1], 0.2 * L[2]])
        look_w = rng.uniform(0.05, 0.15, 3) * 2 * np.pi / 10.0
        look_ph = rng.uniform(0, 2 * np.pi, 3)
        T = np.zeros((n, 4, 4))
        for i in range(n):
            tgt = look_c + look_A * np.sin(look_w * ts[i] + look_ph)
            zc = _unit(tgt - P[i])
            xc = _unit(np.cross(zc, np.array([0.0, 0.0, 1.0])))
            yc = np.cross(zc, xc)
            T[i] = np.eye(4)
            T[i, :3, :3] = np.stack([xc, yc, zc], axis=1)
            T[i, :3, 3] = P[i]
        rate = 0.0
        for i in range(1, n):
            Rrel = T[i - 1, :3, :3].T @ T[i, :3, :3]
            rate = max(rate, math.degrees(math.acos(max(-1.0, min(1.0, (np.trace(Rrel) - 1) / 2)))) * fps)
        if rate <= wmax_deg:
            return T
    raise RuntimeError("no admissible Lissajous path found")


def make_sequence(seq: int, n_frames: int, shape: str = "replica", M: int = 1_000_000, stride: int = 4) -> Sequence:
    """C5: sequence `seq` (scene seed 100+seq) — a room, its M-Gaussian map and an n-frame 30 Hz
    trajectory.  Frames are rendered on demand (raycast_depth_torch)."""
    if shape == "replica":
        K, room, nb, ns, nc = REPLICA, (6.0, 5.0, 3.0), 12, 6, 4
    elif shape == "tum":
        K, room, nb, ns, nc = TUM, (8.0, 8.0, 3.0), 16, 6, 6
    else:
        raise ValueError(shape)
    scene = make_scene(100 + seq, room, nb, ns, nc)
    T = lissajous_trajectory(scene, 200 + seq, n_frames)
    means, quats, scales, ell = sample_map(scene, M, 400 + seq)
    return Sequence(K, scene, T, means, quats, scales, ell, stride)


def render_sequence_rows(seq: Sequence, device="cuda"):
    """All frames' sampled depth rows (n, ceil(H/s), W) float32 on `device` (GPU ray casting)."""
    import torch

    K, s = seq.K, seq.stride
    rows = torch.empty((seq.T_gt.shape[0], (K.H + s - 1) // s, K.W), dtype=torch.float32, device=device)
    for i in range(seq.T_gt.shape[0]):
        rows[i] = raycast_depth_torch(seq.scene, K, seq.T_gt[i], device=device)[::s]
    return rows


def trajectory_error(T_est: np.ndarray, T_gt: np.ndarray) -> dict:
    """Absolute trajectory error of camera poses (no alignment: both start from the frame-0 pose)."""
    dt = np.linalg.norm(T_est[:, :3, 3] - T_gt[:, :3, 3], axis=1)
    ang = [math.degrees(math.acos(max(-1.0, min(1.0, (np.trace(A[:3, :3].T @ B[:3, :3]) - 1) / 2))))
           for A, B in zip(T_est, T_gt)]
    return {"ate_rmse_m": float(np.sqrt(np.mean(dt ** 2))), "trans_max_m": float(dt.max()),
            "rot_max_deg": float(max(ang))}
