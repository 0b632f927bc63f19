"""paper_2403_12550_b200 — B200-native G-ICP tracking hot path of GS-ICP SLAM (arXiv 2403.12550).

Thin ctypes binding of libgsicp.so (C ABI: include/gsicp.h).  This module only marshals
arguments (torch CUDA tensors -> device pointers, the current torch stream -> cudaStream_t);
every step of the path runs in the library's sm_100a kernels.  There is no CPU fallback:
if the library or a CUDA device is missing, every call raises.

Public API (names follow include/gsicp.h):
    backproject_downsample, covariances, build_target, build_target_cloud,
    align, align_async, linearize, Cloud, Target, Tracker
"""
from __future__ import annotations

import contextlib
import ctypes as C
import dataclasses
import math
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgsicp.so")

OK, ERR_INVALID_ARGUMENT, ERR_WORKSPACE_TOO_SMALL, ERR_CUDA = 0, 1, 2, 3
ERR_DEGENERATE_FRAME, ERR_TRACKING_LOST, WARN_MAX_ITERS, WARN_LOW_SUPPORT = 4, 5, 6, 7
REG_NONE, REG_PLANE, REG_ELLIPSE = 0, 1, 2
FLAG_LOW_SUPPORT, FLAG_DEGENERATE = 1, 2


class GsicpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"gsicp status {status}: {msg}")
        self.status = status


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float)]


class _Cloud(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("cov_a", C.c_void_p), ("cov_b", C.c_void_p), ("d_n", C.c_void_p),
                ("cap", C.c_int32)]


class _Target(C.Structure):
    _fields_ = [("pos", C.c_void_p), ("cov_a", C.c_void_p), ("cov_b", C.c_void_p), ("table", C.c_void_p),
                ("bbox", C.c_void_p), ("dense", C.c_void_p), ("dense_hdr", C.c_void_p), ("nbr", C.c_void_p),
                ("nbr_key", C.c_void_p),
                ("table_mask", C.c_uint32), ("cell", C.c_float), ("M", C.c_int32)]


class AlignParams(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("max_corr_dist", C.c_float), ("eps_rot", C.c_double),
                ("eps_trans", C.c_double), ("min_pairs", C.c_int32), ("solver", C.c_int32),
                ("lm_lambda0", C.c_double)]


class AlignStats(C.Structure):
    _fields_ = [("fitness", C.c_double), ("mean_cost", C.c_double), ("n_inliers", C.c_int32),
                ("iters", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load libgsicp.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built; run __graft_entry__.build() or python -m "
                               f"paper_2403_12550_b200._build")
        L = C.CDLL(LIB_PATH)
        P, i32, f32, f64, sz = C.c_void_p, C.c_int32, C.c_float, C.c_double, C.c_size_t
        L.gsicp_backproject_workspace_size.argtypes = [i32, i32, i32]
        L.gsicp_backproject_workspace_size.restype = sz
        L.gsicp_backproject_downsample.argtypes = [P, i32, i32, i32, Intrinsics, i32, f32, f32, P, i32, P, P, sz, P]
        L.gsicp_backproject_sampled_rows.argtypes = [P, i32, i32, i32, Intrinsics, i32, f32, f32, P, i32, P, P, sz, P]
        L.gsicp_upload_sampled_rows.argtypes = [P, P, i32, i32, i32, i32, P]
        L.gsicp_backproject_lattice.argtypes = [P, i32, i32, i32, i32, Intrinsics, i32, f32, f32, P, i32, P, P, P,
                                                sz, P]
        L.gsicp_covariances_workspace_size.argtypes = [i32, i32]
        L.gsicp_covariances_workspace_size.restype = sz
        L.gsicp_covariances.argtypes = [P, P, i32, i32, i32, f32, f32, i32, P, P, P, P, sz, P]
        L.gsicp_covariances_image_workspace_size.argtypes = [i32, i32, i32, i32, i32]
        L.gsicp_covariances_image_workspace_size.restype = sz
        L.gsicp_covariances_image.argtypes = [P, P, i32, i32, i32, i32, Intrinsics, i32, i32, f32, f32, i32, P, P, P,
                                              P, P, sz, P, P]
        L.gsicp_build_target_workspace_size.argtypes = [i32]
        L.gsicp_build_target_workspace_size.restype = sz
        L.gsicp_build_target.argtypes = [P, P, P, i32, i32, i32, f32, f32, C.POINTER(_Target), P, sz, P]
        L.gsicp_build_target_cloud.argtypes = [C.POINTER(_Cloud), i32, f32, C.POINTER(_Target), P, sz, P]
        L.gsicp_align_workspace_size.argtypes = [i32]
        L.gsicp_align_workspace_size.restype = sz
        L.gsicp_align.argtypes = [C.POINTER(_Cloud), C.POINTER(_Target), P, C.POINTER(AlignParams), P,
                                  C.POINTER(AlignStats), P, sz, P]
        L.gsicp_align_async.argtypes = [C.POINTER(_Cloud), C.POINTER(_Target), P, C.POINTER(AlignParams), P, P, P,
                                        sz, P]
        L.gsicp_align_seed.argtypes = [C.POINTER(_Cloud), C.POINTER(_Target), P, C.POINTER(AlignParams), P, sz, P]
        L.gsicp_linearize.argtypes = [C.POINTER(_Cloud), C.POINTER(_Target), P, f32, P, P, P, P, P, P, sz, P]
        L.gsicp_status_string.argtypes = [i32]
        L.gsicp_status_string.restype = C.c_char_p
        L.gsicp_last_error.restype = C.c_char_p
        L.gsicp_kernel_launch_count.restype = C.c_uint64
        L.gsicp_abi_version.restype = i32
        L.gsicp_debug_knn_counters.argtypes = [P]
        L.gsicp_debug_knn_counters.restype = None
        L.gsicp_debug_align_timeline.argtypes = [P, C.c_int64]
        L.gsicp_debug_align_timeline.restype = None
        L.gsicp_debug_align_counters.argtypes = [P]
        L.gsicp_debug_align_counters.restype = None
        L.gsicp_debug_align_iterations.argtypes = [P, P, i32]
        L.gsicp_debug_align_iterations.restype = None
        L.gsicp_pose_predict.argtypes = [P, P, P]
        L.gsicp_pose_push.argtypes = [P, P, P, P, i32, P]
        L.gsicp_export_gaussians.argtypes = [P, P, P, P, i32, P, C.c_double, C.c_double, P, P, P, P, P, P, sz, P]
        L.gsicp_align_batch_async.argtypes = [P, i32, P, P, P, P, P, P, sz, P]
        L.gsicp_align_batch_async.restype = i32
        L.gsicp_align_batch_max.argtypes = []
        L.gsicp_align_batch_max.restype = i32
        L.gsicp_voxel_downsample_workspace_size.argtypes = [i32]
        L.gsicp_voxel_downsample_workspace_size.restype = sz
        L.gsicp_voxel_downsample.argtypes = [P, P, i32, f32, P, P, P, sz, P]
        L.gsicp_voxel_downsample.restype = i32
        L.gsicp_export_workspace_size.argtypes = [i32]
        L.gsicp_export_workspace_size.restype = sz
        L.gsicp_map_workspace_size.argtypes = [i32, i32]
        L.gsicp_map_workspace_size.restype = sz
        L.gsicp_map_init.argtypes = [P, P, P, i32, i32, i32, i32, i32, f32, f32, P, P, sz, P]
        L.gsicp_map_insert.argtypes = [P, P, P, P, C.c_double, C.c_double, P, P]
        L.gsicp_keyframe_decide.argtypes = [P, P, f32, i32, P]
        for name in ("gsicp_map_init", "gsicp_map_insert", "gsicp_keyframe_decide"):
            getattr(L, name).restype = i32
        for name in ("gsicp_pose_predict", "gsicp_pose_push", "gsicp_export_gaussians"):
            getattr(L, name).restype = i32
        L.gsicp_graph_instantiate.argtypes = [P, C.POINTER(C.c_void_p)]
        L.gsicp_graph_launch.argtypes = [P, P]
        L.gsicp_graph_destroy.argtypes = [P]
        for name in ("gsicp_graph_instantiate", "gsicp_graph_launch", "gsicp_graph_destroy"):
            getattr(L, name).restype = i32
        L.gsicp_debug_kernel_timer.argtypes = [i32]
        L.gsicp_debug_kernel_timer.restype = None
        L.gsicp_debug_kernel_time.argtypes = [i32, C.POINTER(C.c_float)]
        L.gsicp_debug_kernel_time.restype = i32
        for name in ("gsicp_backproject_downsample", "gsicp_backproject_sampled_rows", "gsicp_upload_sampled_rows",
                     "gsicp_backproject_lattice",
                     "gsicp_covariances", "gsicp_covariances_image", "gsicp_build_target",
                     "gsicp_build_target_cloud", "gsicp_align", "gsicp_align_async", "gsicp_align_seed",
                     "gsicp_linearize"):
            getattr(L, name).restype = i32
        _lib = L
    return _lib


EXPORTED = [
    "gsicp_backproject_workspace_size", "gsicp_backproject_downsample", "gsicp_backproject_sampled_rows",
    "gsicp_upload_sampled_rows", "gsicp_backproject_lattice", "gsicp_covariances_workspace_size",
    "gsicp_covariances", "gsicp_covariances_image_workspace_size", "gsicp_covariances_image",
    "gsicp_build_target_workspace_size", "gsicp_build_target", "gsicp_build_target_cloud",
    "gsicp_align_workspace_size", "gsicp_align", "gsicp_align_async", "gsicp_align_seed", "gsicp_linearize",
    "gsicp_status_string",
    "gsicp_last_error", "gsicp_kernel_launch_count", "gsicp_abi_version", "gsicp_debug_knn_counters",
    "gsicp_debug_align_timeline", "gsicp_debug_align_counters", "gsicp_debug_align_iterations",
    "gsicp_debug_kernel_timer",
    "gsicp_debug_kernel_time", "gsicp_graph_instantiate", "gsicp_graph_launch", "gsicp_graph_destroy",
    "gsicp_pose_predict", "gsicp_pose_push", "gsicp_export_workspace_size", "gsicp_export_gaussians",
    "gsicp_align_batch_max", "gsicp_align_batch_async", "gsicp_voxel_downsample_workspace_size",
    "gsicp_voxel_downsample", "gsicp_map_workspace_size", "gsicp_map_init", "gsicp_map_insert",
    "gsicp_keyframe_decide",
]

KT_KNN_SEARCH, KT_ALIGN, KT_SEED, KT_BP, KT_COVS, KT_WIDE, KT_TAIL = 0, 1, 2, 3, 4, 5, 6


def debug_kernel_timer(enable):
    """Diagnostic: the hot kernels record CUDA events around their launches (see gsicp.h)."""
    lib().gsicp_debug_kernel_timer(int(enable))


def debug_kernel_time(kernel: int) -> float | None:
    """Elapsed ms of the last recorded launch of `kernel` (KT_*), after a synchronize."""
    ms = C.c_float()
    return float(ms.value) if lib().gsicp_debug_kernel_time(kernel, C.byref(ms)) else None


def debug_align_counters(out: torch.Tensor | None):
    """Diagnostic: while set, align/linearize write (queued searches, reuses, graph certificates, iterations)
    per resident source point into `out` ((cap, 4) int32 CUDA tensor); None switches it off."""
    lib().gsicp_debug_align_counters(_ptr(out) if out is not None else None)


class AlignIterations:
    """Diagnostic (per-iteration parity): while active, align launches record every GN iteration's
    pose T_it and reduced Eq. 1 terms, and each point's correspondence (gsicp_debug_align_iterations).
    Usage: with AlignIterations(max_iters, src_cap) as rec: ... ; rec.iterations() after a sync."""

    REC = 48

    def __init__(self, max_iters: int, cap: int, device="cuda"):
        self.max_iters, self.cap = int(max_iters), int(cap)
        self.rec = torch.full((self.max_iters, self.REC), float("nan"), dtype=torch.float64, device=device)
        self.corr = torch.full((self.max_iters, self.cap), -3, dtype=torch.int32, device=device)

    def __enter__(self):
        lib().gsicp_debug_align_iterations(_ptr(self.rec), _ptr(self.corr), self.max_iters)
        return self

    def __exit__(self, *exc):
        lib().gsicp_debug_align_iterations(None, None, 0)
        return False

    def iterations(self, n_points: int | None = None) -> list[dict]:
        """[{T (4,4), H (6,6), b (6,), cost, n, corr (n_points,)}] for the iterations that ran."""
        rec = self.rec.cpu().numpy()
        corr = self.corr.cpu().numpy()
        out = []
        for it in range(self.max_iters):
            r = rec[it]
            if np.isnan(r[0]):
                break
            T = np.eye(4)
            T[:3, :] = r[:12].reshape(3, 4)
            H = np.zeros((6, 6))
            k = 12
            for a_ in range(6):
                for b_ in range(a_, 6):
                    H[a_, b_] = H[b_, a_] = r[k]
                    k += 1
            out.append(dict(T=T, H=H, b=r[33:39].copy(), cost=float(r[39]), n=int(r[40]),
                            corr=corr[it, :(n_points if n_points is not None else self.cap)].copy()))
        return out


def debug_align_timeline(out: torch.Tensor | None):
    """Diagnostic: while set, align/linearize launches record globaltimer stamps into `out`
    ((N,) int64 CUDA tensor), layout in include/gsicp.h; None switches it off."""
    lib().gsicp_debug_align_timeline(_ptr(out) if out is not None else None, out.numel() if out is not None else 0)


def debug_knn_counters(out: torch.Tensor | None):
    """Diagnostic: while set, covariances() also writes (level, probes, candidates, insertions)
    per query into `out` ((cap, 4) int32 CUDA tensor); None switches it off."""
    lib().gsicp_debug_knn_counters(_ptr(out) if out is not None else None)


# align outcomes that are results, not errors (the stats carry the status)
_ALIGN_ALLOW = (OK, WARN_MAX_ITERS, ERR_TRACKING_LOST, ERR_DEGENERATE_FRAME)


def _check(st: int, allow=(OK,)):
    if st not in allow:
        detail = lib().gsicp_last_error().decode()
        raise GsicpError(st, f"{lib().gsicp_status_string(st).decode()} {detail}")
    return st


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ws(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def launch_count() -> int:
    """Kernels libgsicp launched from this thread so far."""
    return int(lib().gsicp_kernel_launch_count())


@dataclasses.dataclass
class Cloud:
    """Gaussian cloud G = {X, C} as SoA float4 tensors on one device."""
    pos: torch.Tensor          # (cap, 4) f32: x, y, z, payload bits
    cov_a: torch.Tensor        # (cap, 4) f32: c00, c01, c02, c11
    cov_b: torch.Tensor        # (cap, 4) f32: c12, c22, lam_mid, flags bits
    d_n: torch.Tensor          # (1,) int32 valid count

    @property
    def cap(self) -> int:
        return int(self.pos.shape[0])

    def c_struct(self) -> _Cloud:
        return _Cloud(_ptr(self.pos), _ptr(self.cov_a), _ptr(self.cov_b), _ptr(self.d_n), self.cap)

    def n(self) -> int:
        return int(self.d_n.item())

    def cov6(self) -> torch.Tensor:
        """(cap, 6) packed symmetric covariances (c00, c01, c02, c11, c12, c22)."""
        return torch.cat([self.cov_a, self.cov_b[:, :2]], dim=1)

    def flags(self) -> torch.Tensor:
        return self.cov_b[:, 3].contiguous().view(torch.int32)

    @staticmethod
    def empty(cap: int, device="cuda") -> "Cloud":
        z = lambda: torch.zeros((cap, 4), dtype=torch.float32, device=device)
        return Cloud(z(), z(), z(), torch.zeros(1, dtype=torch.int32, device=device))

    @staticmethod
    def from_points(xyz: torch.Tensor, cov6: torch.Tensor | None = None) -> "Cloud":
        """Pack (n, 3) points (and optional (n, 6) covariances) into the SoA float4 layout."""
        n = xyz.shape[0]
        dev = xyz.device
        c = Cloud.empty(n, dev)
        c.pos[:, :3] = xyz
        c.pos[:, 3] = torch.arange(n, device=dev, dtype=torch.int32).view(torch.float32)
        if cov6 is not None:
            c.cov_a[:] = cov6[:, :4]
            c.cov_b[:, :2] = cov6[:, 4:6]
        c.d_n.fill_(n)
        return c


def _check_depth(depth: torch.Tensor, what: str = "depth"):
    """A depth image handed to the library: a 2-D float32 CUDA tensor with unit column stride (the
    row pitch is passed on); anything else would be misread, so it is rejected here."""
    if not isinstance(depth, torch.Tensor) or not depth.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")
    if depth.dtype != torch.float32:
        raise ValueError(f"{what} must be float32 metres (got {depth.dtype})")
    if depth.dim() != 2 or depth.stride(1) != 1 or depth.stride(0) < depth.shape[1]:
        raise ValueError(f"{what} must be a 2-D row-major view with unit column stride")


def backproject_downsample(depth: torch.Tensor, K, stride: int = 4, z_min: float = 0.1, z_max: float = 10.0,
                           pos_out: torch.Tensor | None = None, d_n: torch.Tensor | None = None,
                           ws: torch.Tensor | None = None, stream=None):
    """A1.  depth: (H, W) f32 metres on the GPU.  Returns (pos (cap, 4), d_n (1,))."""
    _check_depth(depth)
    H, W = depth.shape
    pitch = depth.stride(0)
    cap = ((H + stride - 1) // stride) * ((W + stride - 1) // stride)
    dev = depth.device
    if pos_out is None:
        pos_out = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    if d_n is None:
        d_n = torch.zeros(1, dtype=torch.int32, device=dev)
    need = lib().gsicp_backproject_workspace_size(H, W, stride)
    if ws is None:
        ws = _ws(need, dev)
    Kc = K if isinstance(K, Intrinsics) else Intrinsics(*K)
    _check(lib().gsicp_backproject_downsample(C.c_void_p(depth.data_ptr()), H, W, pitch, Kc, stride, z_min, z_max,
                                              _ptr(pos_out), pos_out.shape[0], _ptr(d_n), _ptr(ws), ws.numel(),
                                              _stream(stream)))
    return pos_out, d_n


def backproject_sampled_rows(rows: torch.Tensor, H: int, W: int, K, stride: int = 4, z_min: float = 0.1,
                             z_max: float = 10.0, pos_out: torch.Tensor | None = None,
                             d_n: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    """A1 from only the sampled rows (rows[r] = image row r*stride): same output as
    backproject_downsample on the full (H, W) image."""
    _check_depth(rows, "rows")
    if rows.shape != ((H + stride - 1) // stride, W):
        raise ValueError(f"rows must be ({(H + stride - 1) // stride}, {W})")
    pitch = rows.stride(0)
    cap = ((H + stride - 1) // stride) * ((W + stride - 1) // stride)
    dev = rows.device
    if pos_out is None:
        pos_out = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    if d_n is None:
        d_n = torch.zeros(1, dtype=torch.int32, device=dev)
    if ws is None:
        ws = _ws(lib().gsicp_backproject_workspace_size(H, W, stride), dev)
    Kc = K if isinstance(K, Intrinsics) else Intrinsics(*K)
    _check(lib().gsicp_backproject_sampled_rows(C.c_void_p(rows.data_ptr()), H, W, pitch, Kc, stride, z_min, z_max,
                                                _ptr(pos_out), pos_out.shape[0], _ptr(d_n), _ptr(ws), ws.numel(),
                                                _stream(stream)))
    return pos_out, d_n


def backproject_lattice(depth: torch.Tensor, H: int, W: int, K, stride: int = 4, rows_sampled: bool = False,
                        z_min: float = 0.1, z_max: float = 10.0, pos_out: torch.Tensor | None = None,
                        d_n: torch.Tensor | None = None, lattice: torch.Tensor | None = None,
                        ws: torch.Tensor | None = None, stream=None):
    """A1 (from the full image, or from its sampled rows) that also writes the lattice map
    (output index of every sampled pixel, -1 if invalid).  Returns (pos, d_n, lattice)."""
    _check_depth(depth)
    if depth.shape != (((H + stride - 1) // stride, W) if rows_sampled else (H, W)):
        raise ValueError(f"depth shape {tuple(depth.shape)} does not match H={H}, W={W}, stride={stride}")
    pitch = depth.stride(0)
    Hs, Ws = (H + stride - 1) // stride, (W + stride - 1) // stride
    dev = depth.device
    if pos_out is None:
        pos_out = torch.empty((Hs * Ws, 4), dtype=torch.float32, device=dev)
    if d_n is None:
        d_n = torch.zeros(1, dtype=torch.int32, device=dev)
    if lattice is None:
        lattice = torch.empty(Hs * Ws, dtype=torch.int32, device=dev)
    if ws is None:
        ws = _ws(lib().gsicp_backproject_workspace_size(H, W, stride), dev)
    Kc = K if isinstance(K, Intrinsics) else Intrinsics(*K)
    _check(lib().gsicp_backproject_lattice(C.c_void_p(depth.data_ptr()), 1 if rows_sampled else 0, H, W, pitch, Kc,
                                           stride, z_min, z_max, _ptr(pos_out), pos_out.shape[0], _ptr(d_n),
                                           _ptr(lattice), _ptr(ws), ws.numel(), _stream(stream)))
    return pos_out, d_n, lattice


def upload_sampled_rows(dst_rows: torch.Tensor, depth_host: torch.Tensor, stride: int, stream=None):
    """Copy rows 0, s, 2s, ... of a (pinned) host depth image into dst_rows (device), async."""
    H, W = depth_host.shape
    assert dst_rows.is_cuda and dst_rows.is_contiguous() and dst_rows.shape == ((H + stride - 1) // stride, W)
    assert not depth_host.is_cuda and depth_host.dtype == torch.float32
    _check(lib().gsicp_upload_sampled_rows(_ptr(dst_rows), C.c_void_p(depth_host.data_ptr()), H, W,
                                           depth_host.stride(0), stride, _stream(stream)))


def covariances(pos: torch.Tensor, d_n: torch.Tensor, k: int = 20, mode: int = REG_ELLIPSE, eps_var: float = 1e-3,
                cell0: float = 0.0, levels: int = 1, cov_a=None, cov_b=None, knn_idx: torch.Tensor | None = None,
                ws=None, stream=None):
    """A2-A4 (Eq. 3-4).  cell0 <= 0: automatic cell size (blocking).  Returns a Cloud sharing `pos`."""
    cap = pos.shape[0]
    dev = pos.device
    if cov_a is None:
        cov_a = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    if cov_b is None:
        cov_b = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    need = lib().gsicp_covariances_workspace_size(cap, levels)
    if ws is None:
        ws = _ws(need, dev)
    _check(lib().gsicp_covariances(_ptr(pos), _ptr(d_n), cap, k, mode, eps_var, cell0, levels, _ptr(cov_a),
                                   _ptr(cov_b), _ptr(knn_idx), _ptr(ws), ws.numel(), _stream(stream)))
    return Cloud(pos, cov_a, cov_b, d_n)


def covariances_image(pos: torch.Tensor, d_n: torch.Tensor, H: int, W: int, stride: int, K, k: int = 20,
                      mode: int = REG_ELLIPSE, eps_var: float = 1e-3, cell0: float = 0.01, levels: int = 1,
                      cov_a=None, cov_b=None, knn_idx: torch.Tensor | None = None, ws=None, stream=None,
                      lattice: torch.Tensor | None = None, window_done: torch.cuda.Event | None = None):
    """A2-A4 for a depth-frame cloud from backproject_downsample(H, W, stride, K): the
    image-window kNN (same result as covariances()).  `lattice`: the map backproject_lattice
    wrote for these points (else built here).  Returns a Cloud sharing `pos`."""
    cap = pos.shape[0]
    dev = pos.device
    if cov_a is None:
        cov_a = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    if cov_b is None:
        cov_b = torch.empty((cap, 4), dtype=torch.float32, device=dev)
    need = lib().gsicp_covariances_image_workspace_size(cap, levels, H, W, stride)
    if ws is None:
        ws = _ws(need, dev)
    Kc = K if isinstance(K, Intrinsics) else Intrinsics(*K)
    _check(lib().gsicp_covariances_image(_ptr(pos), _ptr(d_n), cap, H, W, stride, Kc, k, mode, eps_var, cell0, levels,
                                         _ptr(cov_a), _ptr(cov_b), _ptr(knn_idx), _ptr(lattice), _ptr(ws), ws.numel(),
                                         _stream(stream),
                                         C.c_void_p(window_done.cuda_event) if window_done is not None else None))
    return Cloud(pos, cov_a, cov_b, d_n)


@dataclasses.dataclass
class Target:
    """Target Gaussians G^t: hashed copy living in `ws` (keep this object alive)."""
    ws: torch.Tensor
    st: _Target
    keepalive: tuple = ()

    @property
    def M(self) -> int:
        return int(self.st.M)

    @property
    def cell(self) -> float:
        return float(self.st.cell)

    def graph_rows(self, n: int | None = None) -> np.ndarray:
        """Diagnostic: the exact 16-NN graph by input row — (n, 16) int64, row r's neighbour rows
        sorted ascending (-1 padded), for the first n slots' rows (default all M)."""
        n = self.M if n is None else n
        base = self.ws.data_ptr()
        pos = self.arrays()[0][:n]
        rows = pos[:, 3].contiguous().view(torch.int32).long().cpu().numpy()
        off = self.st.nbr - base
        nbr = self.ws[off:off + 4 * 16 * n].view(torch.int32).view(n, 16).long().cpu().numpy()
        out = np.full((n, 16), -1, np.int64)
        nb = np.where(nbr >= 0, rows[np.clip(nbr, 0, n - 1)], -1)
        nb.sort(axis=1)
        out[rows] = nb
        return out

    def arrays(self):
        """(pos, cov_a, cov_b) as (M, 4) float32 views into the workspace, in cell order;
        pos[:, 3] holds the original index bits."""
        base = self.ws.data_ptr()
        out = []
        for p in (self.st.pos, self.st.cov_a, self.st.cov_b):
            off = p - base
            out.append(self.ws[off:off + 16 * self.M].view(torch.float32).view(self.M, 4))
        return tuple(out)


def build_target(means: torch.Tensor, quats_wxyz: torch.Tensor, scales: torch.Tensor, scales_are_log: bool = False,
                 mode: int = REG_ELLIPSE, eps_var: float = 1e-3, cell: float = 0.0, stream=None) -> Target:
    """A5."""
    M = means.shape[0]
    need = lib().gsicp_build_target_workspace_size(M)
    ws = _ws(need, means.device)
    st = _Target()
    _check(lib().gsicp_build_target(_ptr(means), _ptr(quats_wxyz), _ptr(scales), int(scales_are_log), M, mode, eps_var,
                                    cell, C.byref(st), _ptr(ws), ws.numel(), _stream(stream)))
    return Target(ws, st, (means, quats_wxyz, scales))


def build_target_cloud(cloud: Cloud, cell: float = 0.0, M: int | None = None, stream=None) -> Target:
    """A5 for a cloud that carries covariances; cell <= 0: automatic (blocking)."""
    M = cloud.cap if M is None else M
    need = lib().gsicp_build_target_workspace_size(M)
    ws = _ws(need, cloud.pos.device)
    st = _Target()
    cs = cloud.c_struct()
    _check(lib().gsicp_build_target_cloud(C.byref(cs), M, cell, C.byref(st), _ptr(ws), ws.numel(), _stream(stream)))
    return Target(ws, st, (cloud,))


SOLVER_GN, SOLVER_LM = 0, 1


def align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6, min_pairs=50, solver=SOLVER_GN,
                 lm_lambda0=1e-4) -> AlignParams:
    """A6-A9 parameters; solver SOLVER_LM selects Levenberg-Marquardt (R30) with initial damping
    lm_lambda0."""
    return AlignParams(max_iters, max_corr_dist, eps_rot, eps_trans, min_pairs, solver, lm_lambda0)


def align_workspace(cap: int, device="cuda") -> torch.Tensor:
    return _ws(lib().gsicp_align_workspace_size(cap), device)


def align(src: Cloud, tgt: Target, init_T, params: AlignParams | None = None, ws: torch.Tensor | None = None,
          stream=None, allow=None):
    """A6-A9 (Eq. 1).  Blocking; returns (T (4,4) float64 numpy, stats dict)."""
    params = params or align_params()
    ws = ws if ws is not None else align_workspace(src.cap, src.pos.device)
    T0 = np.ascontiguousarray(init_T, dtype=np.float64)
    Tout = np.empty((4, 4), dtype=np.float64)
    stats = AlignStats()
    cs = src.c_struct()
    st = lib().gsicp_align(C.byref(cs), C.byref(tgt.st), T0.ctypes.data_as(C.c_void_p), C.byref(params),
                           Tout.ctypes.data_as(C.c_void_p), C.byref(stats), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, allow or _ALIGN_ALLOW)
    return Tout, stats.as_dict()


def align_async(src: Cloud, tgt: Target, d_T: torch.Tensor, d_stats: torch.Tensor, params: AlignParams | None = None,
                ws: torch.Tensor | None = None, corr_out: torch.Tensor | None = None, stream=None):
    """Graph-capturable A6-A9: d_T (16,) float64 on the device is read and updated in place,
    d_stats (32,) uint8 receives gsicp_align_stats."""
    params = params or align_params()
    ws = ws if ws is not None else align_workspace(src.cap, src.pos.device)
    cs = src.c_struct()
    _check(lib().gsicp_align_async(C.byref(cs), C.byref(tgt.st), _ptr(d_T), C.byref(params), _ptr(d_stats),
                                   _ptr(corr_out), _ptr(ws), ws.numel(), _stream(stream)))


def align_batch_async(srcs: list, tgt: Target, d_T: torch.Tensor, d_stats: torch.Tensor,
                      params: AlignParams | None = None, wss: list | None = None, corr_outs: list | None = None,
                      stream=None):
    """N2: B frames against one target in one launch.  d_T (B, 16) float64 and d_stats
    (B, sizeof(gsicp_align_stats)) uint8 on the device, read / written per frame; wss: B distinct
    align workspaces."""
    B = len(srcs)
    params = params or align_params()
    wss = wss if wss is not None else [align_workspace(c.cap, c.pos.device) for c in srcs]
    cs = (_Cloud * B)(*[c.c_struct() for c in srcs])
    ws_arr = (C.c_void_p * B)(*[_ptr(w) for w in wss])
    corr_arr = (C.c_void_p * B)(*[_ptr(c) for c in corr_outs]) if corr_outs is not None else None
    _check(lib().gsicp_align_batch_async(cs, B, C.byref(tgt.st), _ptr(d_T), C.byref(params), _ptr(d_stats), corr_arr,
                                         ws_arr, min(w.numel() for w in wss), _stream(stream)))


def align_seed(src: Cloud, tgt: Target, d_T: torch.Tensor, params: AlignParams | None = None,
               ws: torch.Tensor | None = None, stream=None):
    """Iteration-0 correspondences at the device pose d_T into the align workspace `ws` (reads
    only src.pos / src.d_n: may overlap the covariance stage on another stream).  Consumed by the
    next align call on `ws` from this thread if it starts at the same pose."""
    params = params or align_params()
    cs = src.c_struct()
    _check(lib().gsicp_align_seed(C.byref(cs), C.byref(tgt.st), _ptr(d_T), C.byref(params), _ptr(ws), ws.numel(),
                                  _stream(stream)))


def decode_stats(d_stats: torch.Tensor) -> dict:
    raw = d_stats.cpu().numpy().tobytes()
    st = AlignStats.from_buffer_copy(raw[:C.sizeof(AlignStats)])
    return st.as_dict()


def linearize(src: Cloud, tgt: Target, T, max_corr_dist: float = math.inf, corr_out: torch.Tensor | None = None,
              ws: torch.Tensor | None = None, stream=None):
    """One linearisation of Eq. 1 at pose T -> dict(H, b, cost, n)."""
    ws = ws if ws is not None else align_workspace(src.cap, src.pos.device)
    T = np.ascontiguousarray(T, dtype=np.float64)
    H = np.empty((6, 6))
    b = np.empty(6)
    cost = C.c_double()
    n = C.c_int32()
    cs = src.c_struct()
    _check(lib().gsicp_linearize(C.byref(cs), C.byref(tgt.st), T.ctypes.data_as(C.c_void_p), max_corr_dist,
                                 H.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p), C.byref(cost),
                                 C.byref(n), _ptr(corr_out), _ptr(ws), ws.numel(), _stream(stream)))
    return dict(H=H, b=b, cost=cost.value, n=n.value)


def pose_predict(hist: torch.Tensor, T_out: torch.Tensor, stream=None):
    """T_out = constant-velocity extrapolation of hist = (T_{t-2}, T_{t-1}) (device, double[32])."""
    _check(lib().gsicp_pose_predict(_ptr(hist), _ptr(T_out), _stream(stream)))


def pose_push(hist: torch.Tensor, T: torch.Tensor, traj: torch.Tensor | None = None,
              counter: torch.Tensor | None = None, stream=None):
    """hist <- (T_{t-1}, T); traj[counter++] = T if given (device tensors)."""
    cap = traj.shape[0] if traj is not None else 0
    _check(lib().gsicp_pose_push(_ptr(hist), _ptr(T), _ptr(traj), _ptr(counter), cap, _stream(stream)))


def voxel_downsample(pos: torch.Tensor, d_n: torch.Tensor, voxel: float, out: torch.Tensor | None = None,
                     stream=None):
    """N4 (R31): -> (pos_out (cap, 4) float32, d_m (1,) int32): rows [0, d_m) are the voxel
    centroids in the order of each voxel's first member, w = member count (int bits)."""
    cap = pos.shape[0]
    out = out if out is not None else torch.empty((cap, 4), dtype=torch.float32, device=pos.device)
    d_m = torch.zeros(1, dtype=torch.int32, device=pos.device)
    ws = _ws(lib().gsicp_voxel_downsample_workspace_size(cap), pos.device)
    _check(lib().gsicp_voxel_downsample(_ptr(pos), _ptr(d_n), cap, float(voxel), _ptr(out), _ptr(d_m), _ptr(ws),
                                        ws.numel(), _stream(stream)))
    return out, d_m


def export_gaussians(pos: torch.Tensor, d_n: torch.Tensor, cov_a: torch.Tensor, cov_b: torch.Tensor,
                     T: torch.Tensor | None = None, p: float = 1.5, c: float = 1.0, corr: torch.Tensor | None = None,
                     out=None, stream=None):
    """A4 export (ALG-12): the cloud's points as 3DGS Gaussians in the world frame of
    the device pose T (float64 4x4, None = identity) -> (means (cap,3), quats wxyz (cap,4),
    scales (cap,3), d_m (1,) int32) float32 device tensors, rows [0, d_m) written — the layout
    build_target reads.  corr (int32, from align/linearize): export only the points without a map
    correspondence (the overlap filter), compacted in index order."""
    cap = pos.shape[0]
    dev = pos.device
    if out is None:
        out = (torch.empty((cap, 3), dtype=torch.float32, device=dev),
               torch.empty((cap, 4), dtype=torch.float32, device=dev),
               torch.empty((cap, 3), dtype=torch.float32, device=dev))
    means, quats, scales = out
    d_m = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = _ws(lib().gsicp_export_workspace_size(cap), dev) if corr is not None else None
    _check(lib().gsicp_export_gaussians(_ptr(pos), _ptr(cov_a), _ptr(cov_b), _ptr(d_n), cap, _ptr(T), float(p),
                                        float(c), _ptr(corr), _ptr(means), _ptr(quats), _ptr(scales), _ptr(d_m),
                                        _ptr(ws), ws.numel() if ws is not None else 0, _stream(stream)))
    return means, quats, scales, d_m


class FrameGraph:
    """A stream capture instantiated with per-node launch priorities (gsicp_graph_instantiate):
    the critical-path kernels run high, the side-stream work low.  Usage:
        fg = FrameGraph(); with fg.capture(stream): ...; fg.replay(stream)"""

    def __init__(self):
        self._g = torch.cuda.CUDAGraph(keep_graph=True)
        self._exec = C.c_void_p()

    @contextlib.contextmanager
    def capture(self, stream):
        with torch.cuda.graph(self._g, stream=stream):
            yield
        _check(lib().gsicp_graph_instantiate(C.c_void_p(self._g.raw_cuda_graph()), C.byref(self._exec)))

    def replay(self, stream=None):
        _check(lib().gsicp_graph_launch(self._exec, _stream(stream)))

    def __del__(self):
        try:
            if self._exec:
                lib().gsicp_graph_destroy(self._exec)
        except Exception:
            pass


class Tracker:
    """Per-frame tracking pipeline with preallocated buffers: A1 -> A2-A4 -> A6-A9 against a
    prebuilt target.  Public per-frame calls: `track()` (depth already on the device) and
    `track_host()` (depth in host memory: only the sampled rows are uploaded); both replay the
    frame from a CUDA graph captured on first use.  `step_async()` is the graph-capturable frame."""

    def __init__(self, H: int, W: int, K, stride: int = 4, k: int = 20, mode: int = REG_ELLIPSE,
                 eps_var: float = 1e-3, z_min: float = 0.1, z_max: float = 10.0, cell0: float | None = None,
                 levels: int = 4, params: AlignParams | None = None, device="cuda", keep_corr: bool = False):
        self.H, self.W, self.stride, self.k, self.mode, self.eps = H, W, stride, k, mode, eps_var
        self.K = K if isinstance(K, Intrinsics) else Intrinsics(*K)
        self.z_min, self.z_max = z_min, z_max
        self.cap = ((H + stride - 1) // stride) * ((W + stride - 1) // stride)
        # finest cell ~ 3 x the point spacing at 1 m depth (performance knob only: results are exact)
        self.cell0 = cell0 if cell0 is not None else max(3.0 * stride / self.K.fx, 1e-3)
        self.levels = levels
        self.params = params or align_params()
        self.device = torch.device(device)
        self.cloud = Cloud.empty(self.cap, self.device)
        self.rows = torch.empty(((H + stride - 1) // stride, W), dtype=torch.float32, device=self.device)
        self.lattice = torch.empty(self.cap, dtype=torch.int32, device=self.device)
        self.ws_bp = _ws(lib().gsicp_backproject_workspace_size(H, W, stride), self.device)
        self.ws_cov = _ws(lib().gsicp_covariances_image_workspace_size(self.cap, levels, H, W, stride), self.device)
        self.ws_align = align_workspace(self.cap, self.device)
        self.d_T = torch.zeros(16, dtype=torch.float64, device=self.device)
        self.d_stats = torch.zeros(C.sizeof(AlignStats), dtype=torch.uint8, device=self.device)
        # final correspondences (the overlap filter of keyframe insertion needs them; 4 B/point/iteration)
        self.corr = torch.full((self.cap,), -1, dtype=torch.int32, device=self.device) if keep_corr else None
        self._side = torch.cuda.Stream(self.device)
        self._fork = torch.cuda.Event()
        self._join = torch.cuda.Event()
        self._fork.record(torch.cuda.current_stream(self.device))  # creates the event (handle passed to C)
        self._graphs = {}
        self._depth = None  # staging buffer of track()
        self._T_host = torch.zeros(16, dtype=torch.float64).pin_memory()
        self._T_out = torch.zeros(16, dtype=torch.float64).pin_memory()
        self._st_out = torch.zeros(C.sizeof(AlignStats), dtype=torch.uint8).pin_memory()

    def preprocess(self, depth: torch.Tensor, stream=None):
        self._backproject(depth, stream)
        self._covariances(stream)

    def _backproject(self, depth, stream, rows=None):
        """A1 from `depth`, or from a sampled-row buffer (`rows`, default self.rows) when depth is
        None; also writes the lattice map the image-window kNN uses."""
        src = depth if depth is not None else (rows if rows is not None else self.rows)
        backproject_lattice(src, self.H, self.W, self.K, self.stride, depth is None, self.z_min, self.z_max,
                            self.cloud.pos, self.cloud.d_n, self.lattice, self.ws_bp, stream)

    def _covariances(self, stream, window_done=None):
        covariances_image(self.cloud.pos, self.cloud.d_n, self.H, self.W, self.stride, self.K, self.k, self.mode,
                          self.eps, self.cell0, self.levels, self.cloud.cov_a, self.cloud.cov_b, None, self.ws_cov,
                          stream, self.lattice, window_done)

    def step_async(self, depth: torch.Tensor | None, tgt: Target, stream=None, events=None, rows=None):
        """Whole frame, device-resident pose in self.d_T (set it before), no host sync.
        A1 on `stream` (from `depth`, or from the sampled-row buffer `self.rows` when depth is
        None); then the iteration-0 correspondences (gsicp_align_seed) on a side stream
        concurrently with A2-A4; joined before A6-A9.  `events` (optional, 4 CUDA events) are
        recorded on `stream` around A1 / A2-A4 / A6-A9."""
        s0 = stream if stream is not None else torch.cuda.current_stream(self.device)
        if events:
            events[0].record(s0)
        self._backproject(depth, s0, rows)
        if events:
            events[1].record(s0)
        # the iteration-0 correspondences need only the points: on a side stream, forked right
        # after A1 (measured: forking after the window kernel — the SM-heavy part of A2-A4 — speeds
        # that kernel up but the ~55-80 us seed pass then ends after A2-A4 and delays A6-A9)
        self._fork.record(s0)
        self._covariances(s0)
        self._side.wait_event(self._fork)
        align_seed(self.cloud, tgt, self.d_T, self.params, self.ws_align, self._side)
        self._join.record(self._side)
        s0.wait_event(self._join)
        if events:
            events[2].record(s0)
        align_async(self.cloud, tgt, self.d_T, self.d_stats, self.params, self.ws_align, self.corr, s0)
        if events:
            events[3].record(s0)

    def _graph(self, key, depth, tgt, rows=None):
        """The whole frame (step_async) captured once per (input, target), replayed after."""
        hit = self._graphs.get(key)
        if hit is not None:
            return hit[0]
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        self.step_async(depth, tgt, s, rows=rows)  # one run outside the capture (lazy library state)
        s.synchronize()
        g = FrameGraph()
        with g.capture(s):
            self.step_async(depth, tgt, s, rows=rows)
        self._graphs[key] = (g, depth, tgt, rows)  # keep the captured buffers alive
        return g

    def _run(self, key, depth, tgt, init_T, stream, upload=None):
        s0 = stream if stream is not None else torch.cuda.current_stream(self.device)
        g = self._graph(key, depth, tgt)
        self._T_host.numpy()[:] = np.ascontiguousarray(init_T, dtype=np.float64).reshape(16)
        with torch.cuda.stream(s0):
            self.d_T.copy_(self._T_host, non_blocking=True)
            if upload is not None:
                upload(s0)
            g.replay(s0)
            self._T_out.copy_(self.d_T, non_blocking=True)
            self._st_out.copy_(self.d_stats, non_blocking=True)
        s0.synchronize()
        stats = AlignStats.from_buffer_copy(self._st_out.numpy().tobytes()[:C.sizeof(AlignStats)]).as_dict()
        _check(stats["status"], _ALIGN_ALLOW)
        return self._T_out.numpy().reshape(4, 4).copy(), stats

    def track(self, depth: torch.Tensor, tgt: Target, init_T, stream=None):
        """Whole frame from a device depth image: host pose in, (T, stats) out (blocking).  The
        image is copied into the tracker's staging buffer on the stream, so one graph per target
        serves every caller tensor (no per-address graphs, nothing of the caller's retained)."""
        _check_depth(depth)
        if tuple(depth.shape) != (self.H, self.W):
            raise ValueError(f"depth must be ({self.H}, {self.W})")
        if self._depth is None:
            self._depth = torch.zeros((self.H, self.W), dtype=torch.float32, device=self.device)
        up = lambda s0: self._depth.copy_(depth, non_blocking=True)  # noqa: E731
        return self._run(("dev", id(tgt)), self._depth, tgt, init_T, stream, up)

    def track_host(self, depth_host: torch.Tensor, tgt: Target, init_T, stream=None):
        """Whole frame from a host depth image (pinned for an asynchronous copy): uploads only the
        rows A1 reads (every stride-th), then as track().  Returns (T, stats)."""
        key = ("rows", id(tgt))
        up = lambda s0: upload_sampled_rows(self.rows, depth_host, self.stride, s0)  # noqa: E731
        return self._run(key, None, tgt, init_T, stream, up)

    def track_rows(self, tgt: Target, init_T, stream=None):
        """Whole frame from the sampled rows already in self.rows (device): (T, stats), blocking."""
        return self._run(("rows", id(tgt)), None, tgt, init_T, stream)

    def drop_graphs(self):
        """Forget the captured frame graphs (and the targets they keep alive), e.g. after the map
        was rebuilt."""
        self._graphs.clear()

    def sequence_graph(self, tgt: Target, hist: torch.Tensor, traj: torch.Tensor, counter: torch.Tensor):
        """A graph for sequence tracking (C5): pose_predict(hist) -> the frame from self.rows ->
        pose_push(hist, traj).  Replay it once per frame after writing the frame's sampled rows
        into self.rows; no host round trip between frames."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        fg = FrameGraph()

        def frame():
            pose_predict(hist, self.d_T, s)
            self.step_async(None, tgt, s)
            pose_push(hist, self.d_T, traj, counter, s)
        with torch.cuda.stream(s):
            h0, c0 = hist.clone(), counter.clone()
            frame()  # one run outside the capture (lazy library state); state restored after
            s.synchronize()
            hist.copy_(h0)
            counter.copy_(c0)
            s.synchronize()
        with fg.capture(s):
            frame()
        torch.cuda.current_stream(self.device).wait_stream(s)
        return fg

    def track_host_stream(self, frames, tgt: Target, init_T, stream=None):
        """Track a stream of host depth frames (each pinned (H, W) float32; init_T: one pose for all
        frames, or one per frame).  The sampled-row upload of frame t+1 runs on a copy stream
        into the other of two row buffers while frame t computes; each frame's pose and stats are
        read back asynchronously.  Returns [(T, stats)] in order (blocks once, at the end)."""
        s0 = stream if stream is not None else torch.cuda.current_stream(self.device)
        if not hasattr(self, "_rows2"):
            self._rows2 = [self.rows, torch.empty_like(self.rows)]
            self._cp = torch.cuda.Stream(self.device)
            self._ev_up = [torch.cuda.Event(), torch.cuda.Event()]
            self._ev_done = [torch.cuda.Event(), torch.cuda.Event()]
        graphs = [self._graph(("rows", id(tgt), b), None, tgt, self._rows2[b]) for b in range(2)]
        n = len(frames)
        inits = [init_T] * n if np.asarray(init_T).ndim == 2 else list(init_T)
        T_host = torch.empty((n, 16), dtype=torch.float64).pin_memory()
        T_out = torch.empty((n, 16), dtype=torch.float64).pin_memory()
        st_out = torch.empty((n, C.sizeof(AlignStats)), dtype=torch.uint8).pin_memory()
        for i in range(n):
            T_host[i].numpy()[:] = np.ascontiguousarray(inits[i], dtype=np.float64).reshape(16)
        for b in range(2):
            self._ev_done[b].record(s0)
        for i, fr in enumerate(frames):
            b = i & 1
            self._cp.wait_event(self._ev_done[b])  # buffer b's previous frame has finished
            upload_sampled_rows(self._rows2[b], fr, self.stride, self._cp)
            self._ev_up[b].record(self._cp)
            s0.wait_event(self._ev_up[b])
            with torch.cuda.stream(s0):
                self.d_T.copy_(T_host[i], non_blocking=True)
                graphs[b].replay(s0)
                T_out[i].copy_(self.d_T, non_blocking=True)
                st_out[i].copy_(self.d_stats, non_blocking=True)
            self._ev_done[b].record(s0)
        s0.synchronize()
        out = []
        for i in range(n):
            stats = AlignStats.from_buffer_copy(st_out[i].numpy().tobytes()[:C.sizeof(AlignStats)]).as_dict()
            _check(stats["status"], _ALIGN_ALLOW)
            out.append((T_out[i].numpy().reshape(4, 4).copy(), stats))
        return out

    def upload_bytes(self) -> int:
        """Bytes track_host() copies host -> device per frame (the sampled rows)."""
        return self.rows.numel() * 4


def track_sequence(tr: Tracker, tgt: Target, frames_rows: torch.Tensor, T0, flush: torch.Tensor | None = None,
                   warmup: int = 3):
    """Sequence tracking (C5): frames_rows (n, ceil(H/s), W) — each frame's sampled depth rows on
    the device; T0 — the pose of frame 0.  Frames 1..n-1 are tracked in order, each with the
    constant-velocity initial pose computed on the device, one graph replay per frame and no host
    round trip.  `flush` (optional device tensor) is zeroed between frames outside the timed
    events (L2 flush).  Returns (T_est (n-1, 4, 4) numpy, per-frame device ms (n-1,) numpy)."""
    dev = tr.device
    n = frames_rows.shape[0]
    T0t = torch.from_numpy(np.ascontiguousarray(T0, dtype=np.float64).reshape(-1)).to(dev)
    hist = torch.cat([T0t, T0t])  # zero velocity before frame 1
    traj = torch.zeros((max(n - 1, 1), 16), dtype=torch.float64, device=dev)
    counter = torch.zeros(1, dtype=torch.int32, device=dev)
    fg = tr.sequence_graph(tgt, hist, traj, counter)
    stream = torch.cuda.current_stream(dev)
    for i in range(1, 1 + min(warmup, n - 1)):  # warm-up, then restart from frame 1
        tr.rows.copy_(frames_rows[i])
        fg.replay(stream)
    torch.cuda.synchronize()
    hist.copy_(torch.cat([T0t, T0t]))
    counter.zero_()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n - 1)]
    for i in range(1, n):
        if flush is not None:
            flush.zero_()
        ev[i - 1][0].record(stream)
        tr.rows.copy_(frames_rows[i])
        fg.replay(stream)
        ev[i - 1][1].record(stream)
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    return traj[: n - 1].cpu().numpy().reshape(-1, 4, 4), ms


# ----------------------------------------------------------------------------------------------
# N1: keyframes and map growth (P:209-214 keyframe selection by the correspondence proportion,
# P:237 only non-overlapping Gaussians, P:250-255 scale aligning, P:262-266 forced keyframe)
def is_keyframe(fitness: float, since_last: int, min_fitness: float = 0.95, max_gap: int = 30) -> bool:
    """a frame whose proportion of correspondences with the map (the align fitness, R19)
    falls below the threshold is a keyframe; if none qualified for max_gap frames since
    the last keyframe, this one is.  The paper gives no threshold value (R29: a parameter)."""
    return fitness < min_fitness or since_last >= max_gap


class _Map(C.Structure):
    _fields_ = [("target", _Target), ("means", C.c_void_p), ("quats", C.c_void_p), ("scales", C.c_void_p),
                ("d_M", C.c_void_p), ("capacity", C.c_int32), ("max_insert", C.c_int32), ("mode", C.c_int32),
                ("cell", C.c_float), ("eps_var", C.c_float), ("ws", C.c_void_p)]


class GaussianMap:
    """N1: a device-resident growing 3DGS map for tracking (gsicp_map_*): the library owns rows
    [0, M) of means / quats wxyz / scales (linear) for `capacity` rows and the G-ICP target over
    them, maintained INCREMENTALLY on insertion (only the affected 16-NN lists are recomputed; the
    target views never move, so frame graphs captured against `tgt` stay valid as the map grows).
    Counts live on the device: insert() can sit inside a CUDA graph, switched by a device flag."""

    def __init__(self, means: torch.Tensor, quats: torch.Tensor, scales: torch.Tensor, capacity: int,
                 max_insert: int | None = None, mode: int = REG_ELLIPSE, eps_var: float = 1e-3, cell: float = 0.0,
                 scales_are_log: bool = False, stream=None):
        M0 = means.shape[0]
        if capacity < M0:
            raise ValueError("capacity < initial map size")
        dev = means.device
        self.capacity = int(capacity)
        self.max_insert = int(max_insert if max_insert is not None else min(capacity, 1 << 20))
        need = lib().gsicp_map_workspace_size(self.capacity, self.max_insert)
        if need == 0:
            raise ValueError("bad map capacity / max_insert")
        self.ws = _ws(need, dev)
        self.st = _Map()
        m, q, sc = (x.contiguous() for x in (means, quats, scales))
        _check(lib().gsicp_map_init(_ptr(m), _ptr(q), _ptr(sc), int(scales_are_log), M0, self.capacity,
                                    self.max_insert, mode, eps_var, cell, C.byref(self.st), _ptr(self.ws),
                                    self.ws.numel(), _stream(stream)))
        self.tgt = Target(self.ws, self.st.target, (self,))
        self.cell = float(self.st.cell)
        base = self.ws.data_ptr()

        def view(ptr, cols, dtype=torch.float32):
            off = ptr - base
            return self.ws[off:off + 4 * cols * self.capacity].view(dtype).view(self.capacity, cols)
        self.means, self.quats, self.scales = view(self.st.means, 3), view(self.st.quats, 4), view(self.st.scales, 3)
        off = self.st.d_M - base
        self.d_M = self.ws[off:off + 32].view(torch.int32)  # [0] M, [1] last insert, [4] dropped (full)

    @property
    def M(self) -> int:
        """Current row count (reads the device counter: synchronising)."""
        return int(self.d_M[0].item())

    def insert(self, cloud: Cloud, d_T: torch.Tensor, corr: torch.Tensor | None = None, p: float = 1.5,
               c: float = 1.0, flag: torch.Tensor | None = None, stream=None):
        """Append the cloud's non-overlapping points (corr < 0; all if corr is None) as scale-aligned
        Gaussians at the device pose d_T and maintain the target (gsicp_map_insert).  flag (device
        int32): insert only if nonzero (a conditional graph node inside a capture).  Asynchronous;
        d_M[1] holds the rows added."""
        cs = cloud.c_struct()
        _check(lib().gsicp_map_insert(C.byref(self.st), C.byref(cs), _ptr(d_T), _ptr(corr), float(p), float(c),
                                      _ptr(flag), _stream(stream)))


def keyframe_decide(d_stats: torch.Tensor, state: torch.Tensor, min_fitness: float = 0.95, max_gap: int = 30,
                    stream=None):
    """Device keyframe decision (R29): state (int32[2] device) = (frames since
    the last keyframe, this frame's decision), updated from the frame's align stats."""
    _check(lib().gsicp_keyframe_decide(_ptr(d_stats), _ptr(state), float(min_fitness), int(max_gap),
                                       _stream(stream)))


def track_sequence_mapping(tr: Tracker, gmap: GaussianMap, frames_rows: torch.Tensor, T0, min_fitness: float = 0.95,
                           max_gap: int = 30, p: float = 1.5, c: float = 1.0, timed: bool = False):
    """Tracking with map growth (N1), frames 1..n-1 in order, one graph replay per frame and NO
    host round trip: constant-velocity initial pose (gsicp_pose_predict) -> the frame
    (A1-A9 from tr.rows) -> device keyframe decision (gsicp_keyframe_decide) -> a conditional
    insertion of the frame's non-overlapping points into the map with incremental target
    maintenance (gsicp_map_insert, the tracker's final correspondences as the overlap filter) ->
    pose history.  `tr` must be built with keep_corr=True.  Returns (T_est (n-1,4,4), keyframe
    frame indices, Gaussians inserted per keyframe, per-frame fitness, per-frame device ms or None)."""
    if tr.corr is None:
        raise ValueError("track_sequence_mapping needs Tracker(keep_corr=True)")
    dev = tr.device
    n = frames_rows.shape[0]
    T0t = torch.from_numpy(np.ascontiguousarray(T0, dtype=np.float64).reshape(-1)).to(dev)
    hist = torch.cat([T0t, T0t])
    traj = torch.zeros((max(n - 1, 1), 16), dtype=torch.float64, device=dev)
    counter = torch.zeros(1, dtype=torch.int32, device=dev)
    state = torch.zeros(2, dtype=torch.int32, device=dev)
    log = torch.zeros((max(n - 1, 1), 4), dtype=torch.float64, device=dev)  # fitness, keyframe, added, M
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    stats_f64 = tr.d_stats[:8].view(torch.float64)  # fitness (first field)

    def frame():
        pose_predict(hist, tr.d_T, s)
        tr.step_async(None, gmap.tgt, s)
        keyframe_decide(tr.d_stats, state, min_fitness, max_gap, s)
        gmap.insert(tr.cloud, tr.d_T, tr.corr, p=p, c=c, flag=state[1:], stream=s)
        rec = torch.stack([stats_f64[0], state[1].double(), gmap.d_M[1].double() * state[1].double(),
                           gmap.d_M[0].double()]).view(1, 4)
        log.index_copy_(0, counter.long().clamp(max=log.shape[0] - 1), rec)
        pose_push(hist, tr.d_T, traj, counter, s)

    with torch.cuda.stream(s):
        tr.rows.copy_(frames_rows[min(1, n - 1)])
        tr.step_async(None, gmap.tgt, s)  # one frame outside the capture (lazy library state), no insertion
        s.synchronize()
        fg = FrameGraph()
        with fg.capture(s):
            frame()
    torch.cuda.current_stream(dev).wait_stream(s)
    stream = torch.cuda.current_stream(dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n - 1)] \
        if timed else None
    for i in range(1, n):
        tr.rows.copy_(frames_rows[i])
        if ev:
            ev[i - 1][0].record(stream)
        fg.replay(stream)
        if ev:
            ev[i - 1][1].record(stream)
    torch.cuda.synchronize()
    L = log[: n - 1].cpu().numpy()
    kfs = [i + 1 for i in range(n - 1) if L[i, 1] > 0]
    added = [int(L[i, 2]) for i in range(n - 1) if L[i, 1] > 0]
    ms = np.array([a.elapsed_time(b) for a, b in ev]) if ev else None
    return traj[: n - 1].cpu().numpy().reshape(-1, 4, 4), kfs, added, L[:, 0].copy(), ms


class BatchTracker:
    """N2 throughput mode: B independent frames per step against one target.  Each frame's A1 and
    A2-A4 run on a stream of its own (concurrently), then one batched GN loop runs the B frames
    side by side (gsicp_align_batch_async: k_align_batch, or the flat loop for B >= FLAT_MIN_B);
    the whole step is one graph replay.  Frames are written into self.rows[b] (sampled depth
    rows, as Tracker.rows)."""

    FLAT_MIN_B = 6  # (GSICP_FLAT_BATCH in align.cu)

    def __init__(self, B: int, H: int, W: int, K, stride: int = 4, params: AlignParams | None = None,
                 device="cuda", seeds: bool | None = None, **kw):
        if not 1 <= B <= int(lib().gsicp_align_batch_max()):
            raise ValueError(f"B must be in [1, {lib().gsicp_align_batch_max()}]")
        self.B = B
        # iteration-0 seeds per frame (gsicp_align_seed): None = only for batches below the flat
        # loop's size (the flat loop spreads the iteration-0 hard queries over the GPU itself)
        self.seeds = (B < self.FLAT_MIN_B) if seeds is None else bool(seeds)
        self.params = params or align_params()
        self.device = torch.device(device)
        self.trs = [Tracker(H, W, K, stride=stride, params=self.params, device=device, **kw) for _ in range(B)]
        self.rows = torch.empty((B,) + tuple(self.trs[0].rows.shape), dtype=torch.float32, device=self.device)
        self.d_T = torch.zeros((B, 16), dtype=torch.float64, device=self.device)
        self.d_stats = torch.zeros((B, C.sizeof(AlignStats)), dtype=torch.uint8, device=self.device)
        self._streams = [torch.cuda.Stream(self.device) for _ in range(B)]
        self._fork = torch.cuda.Event()
        self._joins = [torch.cuda.Event() for _ in range(B)]
        self._graphs = {}
        self._T_host = torch.zeros((B, 16), dtype=torch.float64).pin_memory()
        self._T_out = torch.zeros((B, 16), dtype=torch.float64).pin_memory()
        self._st_out = torch.zeros((B, C.sizeof(AlignStats)), dtype=torch.uint8).pin_memory()

    def step_async(self, tgt: Target, stream=None):
        s0 = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._fork.record(s0)
        for b, tr in enumerate(self.trs):
            sb = self._streams[b]
            sb.wait_event(self._fork)
            tr._backproject(None, sb, self.rows[b])
            # iteration-0 correspondences at the frame's pose (needs only the points), then A2-A4;
            # the frames' streams run concurrently
            if self.seeds:
                align_seed(tr.cloud, tgt, self.d_T[b], self.params, tr.ws_align, sb)
            tr._covariances(sb)
            self._joins[b].record(sb)
            s0.wait_event(self._joins[b])
        align_batch_async([tr.cloud for tr in self.trs], tgt, self.d_T, self.d_stats, self.params,
                          [tr.ws_align for tr in self.trs], None, s0)

    def graph(self, tgt: Target):
        hit = self._graphs.get(id(tgt))
        if hit is not None:
            return hit[0]
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            T0 = self.d_T.clone()
            self.step_async(tgt, s)  # one run outside the capture (lazy library state)
            self.d_T.copy_(T0)
        s.synchronize()
        g = FrameGraph()
        with g.capture(s):
            self.step_async(tgt, s)
        self._graphs[id(tgt)] = (g, tgt)
        return g

    def track_rows(self, tgt: Target, init_T, stream=None):
        """The B frames in self.rows from the B initial poses init_T (B, 4, 4): (T (B, 4, 4),
        [stats] * B), blocking."""
        s0 = stream if stream is not None else torch.cuda.current_stream(self.device)
        g = self.graph(tgt)
        self._T_host.numpy()[:] = np.ascontiguousarray(init_T, dtype=np.float64).reshape(self.B, 16)
        with torch.cuda.stream(s0):
            self.d_T.copy_(self._T_host, non_blocking=True)
            g.replay(s0)
            self._T_out.copy_(self.d_T, non_blocking=True)
            self._st_out.copy_(self.d_stats, non_blocking=True)
        s0.synchronize()
        raw = self._st_out.numpy()
        stats = [AlignStats.from_buffer_copy(raw[b].tobytes()[:C.sizeof(AlignStats)]).as_dict() for b in range(self.B)]
        for st in stats:
            _check(st["status"], _ALIGN_ALLOW)
        return self._T_out.numpy().reshape(self.B, 4, 4).copy(), stats
