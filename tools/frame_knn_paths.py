"""A2-A4 of depth frames: the image-window path (covariances_image) vs the general brick path
(covariances with a grid) — time and, with debug counters, how many queries the brick kernel
finished.  python tools/frame_knn_paths.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def main():
    dev = torch.device("cuda")
    cases = [("replica s4", synth.make_frame_workload(2, "replica", M=100_000, stride=4), 4),
             ("tum s4", synth.make_frame_workload(3, "tum", M=100_000, stride=4, noisy=True), 4),
             ("tum s1", synth.make_frame_workload(3, "tum", M=100_000, stride=1, noisy=True), 1)]
    for name, w, s in cases:
        K = w.K
        Kt = (K.fx, K.fy, K.cx, K.cy)
        pos, d_n = g.backproject_downsample(torch.from_numpy(w.depth).to(dev), Kt, stride=s)
        n = int(d_n.item())
        cap = pos.shape[0]
        wsi = g._ws(g.lib().gsicp_covariances_image_workspace_size(cap, 4, K.H, K.W, s), dev)
        ti = timeit(lambda: g.covariances_image(pos, d_n, K.H, K.W, s, Kt, 20, cell0=3.0 * s / K.fx, levels=4, ws=wsi))
        sp = float(np.median(w.depth[w.depth > 0])) * s / K.fx  # typical spacing
        for cm, lv in ((3.4, 3), (4.5, 3), (2.5, 4)):
            wsb = g._ws(g.lib().gsicp_covariances_workspace_size(cap, lv), dev)
            tb = timeit(lambda: g.covariances(pos, d_n, 20, g.REG_ELLIPSE, 1e-3, cm * sp, lv, ws=wsb))
            dbg = torch.zeros((cap, 4), dtype=torch.int32, device=dev)
            g.debug_knn_counters(dbg)
            g.covariances(pos, d_n, 20, g.REG_ELLIPSE, 1e-3, cm * sp, lv, ws=wsb)
            g.debug_knn_counters(None)
            torch.cuda.synchronize()
            brick = (dbg[:n, 0] == -7).float().mean().item()
            print(f"{name}: n={n} image path {ti:7.1f} us | brick cell {cm} sp x {lv} levels {tb:7.1f} us, brick-finished {brick:.3f}")


if __name__ == "__main__":
    main()
