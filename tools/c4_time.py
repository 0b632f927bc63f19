"""C4 kNN-cov timing (4e6-point map, bench grid settings) and the per-stage launch split."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    scene = synth.make_scene(1004)
    means, _, _, ell = synth.sample_map(scene, 4_000_000, 4004)
    c = g.Cloud.from_points(torch.from_numpy(means).cuda())
    cases = ((3.4, 3), (3.7, 3), (3.7, 2), (4.0, 3), (3.4, 2))
    if len(sys.argv) > 1:  # "1": only the bench configuration (profiling)
        cases = cases[:int(sys.argv[1])]
    for cm, lv in cases:
        ws = g._ws(g.lib().gsicp_covariances_workspace_size(c.cap, lv), c.pos.device)
        for _ in range(2):
            g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, cm * ell, lv, c.cov_a, c.cov_b, None, ws)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, cm * ell, lv, c.cov_a, c.cov_b, None, ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"cell {cm} ell, levels {lv}: {np.median(ts):.3f} ms  ({4.0 / (np.median(ts) / 1000):.0f} Mpts/s)")
        del ws


if __name__ == "__main__":
    main()
