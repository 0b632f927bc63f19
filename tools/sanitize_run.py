"""Workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): C1 and the Replica
bench frame through every entry point of the hot path, eagerly (no graphs, so each kernel launch
is checked on its own).  python tools/sanitize_run.py [c1|map|replica|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def frame(depth, K, stride, tgt, T0, label):
    dev = torch.device("cuda")
    d = torch.from_numpy(depth).to(dev)
    Kt = (K.fx, K.fy, K.cx, K.cy)
    H, W = depth.shape
    pos, d_n = g.backproject_downsample(d, Kt, stride=stride)
    knn = torch.empty((pos.shape[0], 20), dtype=torch.int32, device=dev)
    cl = g.covariances(pos, d_n, k=20, cell0=0.0, levels=4, knn_idx=knn)  # hash path (auto cell)
    ci = g.covariances_image(pos, d_n, H, W, stride, Kt, 20, cell0=3.0 * stride / K.fx, levels=4, knn_idx=knn)
    p = g.align_params(max_iters=8, max_corr_dist=0.1 if tgt is not None else float("inf"))
    if tgt is None:
        tgt = g.build_target_cloud(cl)
    dT = torch.from_numpy(np.ascontiguousarray(T0, np.float64).reshape(-1)).to(dev)
    ws = g.align_workspace(ci.cap)
    g.align_seed(ci, tgt, dT, p, ws)
    T, st = g.align(ci, tgt, T0, p, ws)
    g.linearize(ci, tgt, T, 0.1)
    corr = torch.full((ci.cap,), -1, dtype=torch.int32, device=dev)
    d_stats = torch.zeros(32, dtype=torch.uint8, device=dev)
    g.align_async(ci, tgt, dT, d_stats, p, ws, corr)
    g.export_gaussians(ci.pos, ci.d_n, ci.cov_a, ci.cov_b, T=dT, corr=corr)
    g.voxel_downsample(pos, d_n, 0.05)
    B = 2
    dTb = dT.repeat(B)
    g.align_batch_async([ci] * B, tgt, dTb.view(B, 16), torch.zeros((B, 32), dtype=torch.uint8, device=dev), p)
    # frame batch through the flat loop (B >= 6) and one large-capacity cloud (the flat loop)
    B = 6
    g.align_batch_async([ci] * B, tgt, dT.repeat(B).view(B, 16), torch.zeros((B, 32), dtype=torch.uint8, device=dev), p)
    big = g.Cloud.empty(60_000)
    n = int(ci.d_n.item())
    for a_, b_ in ((big.pos, ci.pos), (big.cov_a, ci.cov_a), (big.cov_b, ci.cov_b)):
        a_[:n] = b_[:n]
    big.d_n.copy_(ci.d_n)
    g.align(big, tgt, T0, p)
    tr = g.Tracker(H, W, Kt, stride=stride)
    tr.track(d, tgt, T0)
    torch.cuda.synchronize()
    print(f"{label}: n={int(d_n.item())} iters={st['iters']} status={st['status']}")


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("c1", "all"):
        w = synth.make_c1(1)
        frame(w.depth, w.K, 1, None, np.eye(4), "c1")
    if which in ("map", "all"):  # the brick kNN over a map-shaped cloud with floating outliers
        dev = torch.device("cuda")  # (3e5 points: above kTwoPhaseMin, the two-phase grid build)
        scene = synth.make_scene(1004)
        means, _, _, ell = synth.sample_map(scene, 300_000, 4004)
        c = g.Cloud.from_points(torch.from_numpy(means).to(dev))
        g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, 3.4 * ell, 3, c.cov_a, c.cov_b)
        torch.cuda.synchronize()
        print("map: n=300000")
    if which in ("replica", "all"):
        w = synth.make_frame_workload(2, "replica", M=200_000, stride=4)
        dev = torch.device("cuda")
        tgt = g.build_target(*(torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales)))
        frame(w.depth, w.K, 4, tgt, w.T_init, "replica")


if __name__ == "__main__":
    main()
