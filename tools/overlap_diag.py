"""GPU diagnostic: A2-A4 alone, the iteration-0 seed alone, both overlapped, and the align
kernel with / without seeds (bench frame vs the 1e6 map).  python tools/overlap_diag.py"""
import os
import statistics
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
    T0 = torch.from_numpy(w.T_init.reshape(-1).copy()).to(dev)
    tr.d_T.copy_(T0)
    tr.preprocess(depth)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    s0 = torch.cuda.current_stream()
    side = torch.cuda.Stream()

    def cov():
        g.covariances(tr.cloud.pos, tr.cloud.d_n, tr.k, tr.mode, tr.eps, tr.cell0, tr.levels, tr.cloud.cov_a,
                      tr.cloud.cov_b, None, tr.ws_cov)

    def seed(stream=None):
        g.align_seed(tr.cloud, tgt, tr.d_T, tr.params, tr.ws_align, stream)

    def both():
        ev = torch.cuda.Event()
        ev.record(s0)
        side.wait_event(ev)
        seed(side)
        j = torch.cuda.Event()
        j.record(side)
        cov()
        s0.wait_event(j)

    def align():
        tr.d_T.copy_(T0)
        g.align_async(tr.cloud, tgt, tr.d_T, tr.d_stats, tr.params, tr.ws_align)

    def seeded_align():
        tr.d_T.copy_(T0)
        seed()
        g.align_async(tr.cloud, tgt, tr.d_T, tr.d_stats, tr.params, tr.ws_align)

    def timeit(fn, reps=30):
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        return statistics.median(ts)

    for name, fn in (("A2-A4 covariances", cov), ("seed", seed), ("cov || seed", both), ("align (no seed)", align),
                     ("seed + align (serial)", seeded_align)):
        fn()
        print(f"{name:24s} {timeit(fn):8.1f} us")


if __name__ == "__main__":
    main()
