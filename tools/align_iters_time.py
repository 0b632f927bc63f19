"""Per-iteration cost of the persistent align kernel on the bench frame: k_align timed (CUDA events,
seeded as the Tracker does, L2 flushed before each run) with max_iters = 1..N, so the increments
are the real (uninstrumented) iteration times.  python tools/align_iters_time.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    w = synth.make_frame_workload(2, "replica", M=1_000_000, stride=4)
    K = w.K
    dev = torch.device("cuda")
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=4, device=dev)
    tr.preprocess(torch.from_numpy(w.depth).to(dev))
    tgt = g.build_target(*(torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales)))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    dT = torch.from_numpy(np.ascontiguousarray(w.T_init).reshape(-1)).to(dev)
    prev = 0.0
    d_stats = torch.zeros(32, dtype=torch.uint8, device=dev)
    dT0 = dT.clone()
    for mi in range(1, 9):
        p = g.align_params(max_iters=mi, eps_rot=0.0, eps_trans=0.0)
        ts = []
        for rep in range(12):
            flush.fill_(rep & 255)
            dT.copy_(dT0)
            g.align_seed(tr.cloud, tgt, dT, p, tr.ws_align)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.align_async(tr.cloud, tgt, dT, d_stats, p, tr.ws_align)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 2:
                ts.append(e0.elapsed_time(e1) * 1e3)
        t = float(np.median(ts))
        st = g.decode_stats(d_stats)
        print(f"max_iters {mi}: {t:7.1f} us  (+{t - prev:5.1f})  iters {st['iters']}")
        prev = t


if __name__ == "__main__":
    main()
