"""C4 diagnostic: which path finished each query of the 4e6-point map kNN-cov (brick kernel vs the
warp-search fallback) and the kernel timer span of the brick stage.  python tools/c4_diag.py [cell] [levels]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    cm = float(sys.argv[1]) if len(sys.argv) > 1 else 3.4
    lv = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    scene = synth.make_scene(1004)
    means, _, _, ell = synth.sample_map(scene, 4_000_000, 4004)
    c = g.Cloud.from_points(torch.from_numpy(means).cuda())
    ws = g._ws(g.lib().gsicp_covariances_workspace_size(c.cap, lv), c.pos.device)
    dbg = torch.zeros((c.cap, 4), dtype=torch.int32, device="cuda")
    g.debug_knn_counters(dbg)
    g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, cm * ell, lv, c.cov_a, c.cov_b, None, ws)
    g.debug_knn_counters(None)
    torch.cuda.synchronize()
    d = dbg.cpu().numpy()
    brick = d[:, 0] == -7
    print(f"cell {cm} ell levels {lv}: brick-finished {brick.mean():.4f}, fallback {1 - brick.mean():.4f}; "
          f"staged candidates per query (brick) mean {d[brick, 1].mean():.0f} max {d[brick, 1].max()}, "
          f"m mean {d[brick, 2].mean():.1f}")
    w = d[brick, 3]
    print(f"  lanes/round mean {(w & 255).mean():.1f}  bricks/group mean {((w >> 8) & 255).mean():.2f}  events/round mean {(w >> 16).mean():.2f}")
    fb8 = d[:, 0] == -8
    if fb8.any():
        print("  brick failures by reason (1 staging overflow, 2 tie overflow, 3 m<k, 4 list>32, 5 band>tau, 6 certificate):",
              np.bincount(d[fb8, 1], minlength=7)[1:], " staged mean", d[fb8, 2].mean())
    fb = ~brick
    if fb.any():
        print(f"  fallback: level mean {d[fb, 0].mean():.2f}, probes mean {d[fb, 1].mean():.0f}, cands mean {d[fb, 2].mean():.0f}")
    g.debug_kernel_timer(1)
    for _ in range(3):
        g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, cm * ell, lv, c.cov_a, c.cov_b, None, ws)
    torch.cuda.synchronize()
    print(f"  brick stage (list + kernel) {g.debug_kernel_time(g.KT_KNN_SEARCH):.3f} ms")
    g.debug_kernel_timer(0)


if __name__ == "__main__":
    main()
