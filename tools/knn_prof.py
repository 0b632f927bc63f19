"""Profiling target: gsicp_covariances on the bench frame (after an L2 flush), 3 times.
python tools/knn_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2403_12550_b200 as g
import synth


def c4():
    scene = synth.make_scene(1004)
    means, _, _, ell = synth.sample_map(scene, 4_000_000, 4004)
    c = g.Cloud.from_points(torch.from_numpy(means).cuda())
    ws = g._ws(g.lib().gsicp_covariances_workspace_size(c.cap, 3), c.pos.device)
    for _ in range(3):
        g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, 3.0 * ell, 3, c.cov_a, c.cov_b, None, ws)
    torch.cuda.synchronize()


def main():
    if "c4" in sys.argv:
        return c4()
    w = synth.make_frame_workload(2, "replica", M=1000, stride=4)
    K = w.K
    dev = torch.device("cuda")
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=4, device=dev)
    depth = torch.from_numpy(w.depth).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(3):
        flush.zero_()
        tr.preprocess(depth)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
