"""Profiling target: gsicp_covariances on the bench frame (after an L2 flush), 3 times.
python tools/knn_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2403_12550_b200 as g
import synth


def main():
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
