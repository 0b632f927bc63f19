"""N2 throughput probe: BatchTracker steps (B Replica-shaped frames vs a 1e6-Gaussian map, one
graph replay per step, L2 flushed between steps) for several B; prints aligns/s and ms/step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    Bs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16").split(",")]
    seq = synth.make_sequence(0, 17, "replica", M=1_000_000)
    rows = synth.render_sequence_rows(seq, "cuda")
    K = seq.K
    tgt = g.build_target(torch.from_numpy(seq.means).cuda(), torch.from_numpy(seq.quats).cuda(),
                         torch.from_numpy(seq.scales).cuda())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    prm = g.align_params(max_iters=30, max_corr_dist=0.1)
    for B in Bs:
        bt = g.BatchTracker(B, K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=prm)
        bt.rows.copy_(rows[1:1 + B])
        init = np.stack([synth.perturb_pose(seq.T_gt[1 + b], 30 + b, 2.0, 0.03) for b in range(B)])
        Tb, st = bt.track_rows(tgt, init)
        gr = bt.graph(tgt)
        Th = torch.from_numpy(init.reshape(B, 16)).cuda()
        s = torch.cuda.current_stream()
        ts = []
        for rep in range(23):
            flush.zero_()
            bt.d_T.copy_(Th)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            gr.replay(s)
            e1.record(s)
            torch.cuda.synchronize()
            if rep >= 3:
                ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        err = max(np.abs(Tb[b][:3, 3] - seq.T_gt[1 + b][:3, 3]).max() for b in range(B))
        its = [s_["iters"] for s_ in st]
        print(f"B={B:2d}: {ms:.3f} ms/step, {B / ms * 1000:.0f} aligns/s, iters {its}, max trans err {err:.1e}")


if __name__ == "__main__":
    main()
