"""C3 diagnostic: a TUM-shaped noisy frame vs a 1e6-Gaussian map through the Tracker (graph replay),
per-stage kernel-timer spans, GN iterations, and the image-window certification split."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    dev = torch.device("cuda")
    for s in (4, 2, 1):
        w = synth.make_frame_workload(3, "tum", M=1_000_000, stride=s, noisy=True)
        K = w.K
        tgt = g.build_target(torch.from_numpy(w.means).to(dev), torch.from_numpy(w.quats).to(dev),
                             torch.from_numpy(w.scales).to(dev))
        tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=s,
                       params=g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6))
        depth = torch.from_numpy(w.depth).to(dev)
        T0 = torch.from_numpy(w.T_init.reshape(-1).copy()).to(dev)
        st = torch.cuda.Stream()
        g.debug_kernel_timer(2)
        with torch.cuda.stream(st):
            tr.d_T.copy_(T0)
            tr.step_async(depth, tgt, st)
        st.synchronize()
        fg = g.FrameGraph()
        with fg.capture(st):
            tr.step_async(depth, tgt, st)
        g.debug_kernel_timer(0)
        ts, spans = [], []
        for _ in range(10):
            with torch.cuda.stream(st):
                tr.d_T.copy_(T0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fg.replay(st)
            e1.record(st)
            st.synchronize()
            ts.append(e0.elapsed_time(e1))
            spans.append([g.debug_kernel_time(k) for k in range(7)])
        sp = np.nanmean(np.array([[x if x is not None else np.nan for x in r] for r in spans]), 0)
        names = ["window", "align", "seed", "A1", "A2-A4", "wide+brute", "tail"]
        print(f"stride {s}: n={tr.cloud.n()} frame {np.median(ts) * 1000:.1f} us, iters {g.decode_stats(tr.d_stats)['iters']}  " +
              " ".join(f"{nm}={v * 1000:.1f}" for nm, v in zip(names, sp)))


if __name__ == "__main__":
    main()
