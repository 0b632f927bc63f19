"""GPU diagnostic: per-query work distribution of the kNN-covariance kernel (levels, cells probed,
candidates, insertions) on the bench frame and the C4 map, plus timings for a sweep of grid knobs.
Run under gpurun:  python tools/knn_diag.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def dist(name, x):
    q = np.percentile(x, [50, 90, 99, 99.9, 100])
    print(f"  {name:10s} mean {x.mean():8.1f}  p50 {q[0]:7.0f} p90 {q[1]:7.0f} p99 {q[2]:7.0f} p99.9 {q[3]:7.0f} max {q[4]:7.0f}")


def run(pos, d_n, cell0, levels, label, reps=5):
    cap = pos.shape[0]
    ws = g._ws(g.lib().gsicp_covariances_workspace_size(cap, levels), pos.device)
    ca = torch.empty((cap, 4), device=pos.device)
    cb = torch.empty((cap, 4), device=pos.device)
    dbg = torch.zeros((cap, 4), dtype=torch.int32, device=pos.device)
    g.debug_knn_counters(dbg)
    g.covariances(pos, d_n, 20, g.REG_ELLIPSE, 1e-3, cell0, levels, ca, cb, None, ws)
    g.debug_knn_counters(None)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.covariances(pos, d_n, 20, g.REG_ELLIPSE, 1e-3, cell0, levels, ca, cb, None, ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    n = int(d_n.item())
    d = dbg[:n].cpu().numpy()
    print(f"{label}: cell0={cell0:.4f} levels={levels}  median {np.median(ts):.3f} ms")
    lv = d[:, 0]
    print("  tile level hist", np.bincount(lv[lv < 16], minlength=levels).tolist(),
          " queue (warp search) level hist", np.bincount(lv[lv >= 16] - 16, minlength=levels).tolist(),
          f" queue frac {np.mean(lv >= 16):.4f}")
    dist("probes", d[:, 1])
    dist("cands", d[:, 2])
    dist("inserts", d[:, 3])


def main():
    w = synth.make_frame_workload(2, "replica", M=1000, stride=4)
    K = w.K
    pos, d_n = g.backproject_downsample(torch.from_numpy(w.depth).cuda(), (K.fx, K.fy, K.cx, K.cy), stride=4)
    for cell0, levels in ((0.02, 4), (0.01, 5)):
        run(pos, d_n, cell0, levels, "replica s=4")
    scene = synth.make_scene(1004)
    means, _, _, ell = synth.sample_map(scene, 4_000_000, 4004)
    c4 = g.Cloud.from_points(torch.from_numpy(means).cuda())
    for cm, levels in ((3.0, 3), (2.0, 3)):
        run(c4.pos, c4.d_n, cm * ell, levels, "C4 4e6 map", reps=3)


if __name__ == "__main__":
    main()
