"""C3 stride-1 frame (205k points) vs the 1e6 map: one eager align (the flat GN path), for the
ncu launch list of its per-iteration kernels.  python tools/c3_flat_prof.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    for _ in range(2):
        T, st = g.align(tr.cloud, tgt, w.T_init, tr.params, tr.ws_align)
    torch.cuda.synchronize()
    print(st)


if __name__ == "__main__":
    main()
