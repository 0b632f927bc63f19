"""Profiling target: one gsicp_align_seed on the bench frame vs the 1e6 map after an L2 flush
(run under ncu).  python tools/seed_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    w = synth.make_frame_workload(2, "replica", M=1_000_000, stride=4)
    K = w.K
    dev = torch.device("cuda")
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=4, device=dev)
    depth = torch.from_numpy(w.depth).to(dev)
    tgt = g.build_target(*(torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales)))
    tr.d_T.copy_(torch.from_numpy(w.T_init.reshape(-1).copy()).to(dev))
    tr.preprocess(depth)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    for _ in range(3):
        flush.zero_()
        g.align_seed(tr.cloud, tgt, tr.d_T, tr.params, tr.ws_align)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
