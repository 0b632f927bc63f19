"""C3 stride-1 frame through the flat GN path: per iteration, how each point's correspondence was
proven (motion-bounded reuse, neighbourhood set, graph certificate) or queued for the warp search.
python tools/c3_flat_diag.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    dev = torch.device("cuda")
    w = synth.make_frame_workload(3, "tum", M=1_000_000, stride=1, noisy=True)
    K = w.K
    tgt = g.build_target(torch.from_numpy(w.means).to(dev), torch.from_numpy(w.quats).to(dev),
                         torch.from_numpy(w.scales).to(dev))
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=1,
                   params=g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6))
    tr.preprocess(torch.from_numpy(w.depth).to(dev))
    n = tr.cloud.n()
    cnt = torch.zeros((tr.cap, 4), dtype=torch.int32, device=dev)
    g.debug_align_counters(cnt)
    T, st = g.align(tr.cloud, tgt, w.T_init, tr.params, tr.ws_align)
    g.debug_align_counters(None)
    c = cnt[:n].cpu().numpy().astype(np.int64) & 0xffffffff
    print(st, "n", n)
    for it in range(min(st["iters"], 30)):
        b = 1 << it
        q, r, s_, gr = ((c[:, k] & b) != 0 for k in range(4))
        print(f"it {it:2d}: queued {q.mean():.4f} reuse {r.mean():.4f} set {s_.mean():.4f} graph {gr.mean():.4f}")


if __name__ == "__main__":
    main()
