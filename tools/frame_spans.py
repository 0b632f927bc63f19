"""Stage spans of the bench frame (Replica-shaped, stride 4, vs the 1e6-Gaussian map) inside the
captured frame graph: kernel-timer events around A1, A2-A4 (window / wide+brute / hash tail), the
seed pass (side stream) and A6-A9, L2 flushed between replays.  python tools/frame_spans.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    dev = torch.device("cuda")
    w = synth.make_frame_workload(2, "replica", M=1_000_000, stride=4)
    K = w.K
    tgt = g.build_target(*(torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales)))
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=4,
                   params=g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6))
    depth = torch.from_numpy(w.depth).to(dev)
    T0 = torch.from_numpy(w.T_init.reshape(-1).copy()).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
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
    for _ in range(30):
        with torch.cuda.stream(st):
            flush.zero_()
            tr.d_T.copy_(T0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fg.replay(st)
        e1.record(st)
        st.synchronize()
        ts.append(e0.elapsed_time(e1))
        spans.append([g.debug_kernel_time(k) for k in range(7)])
    sp = np.nanmedian(np.array([[x if x is not None else np.nan for x in r] for r in spans[5:]]), 0)
    names = ["window", "align", "seed", "A1", "A2-A4", "wide+brute", "tail"]
    print(f"frame {np.median(ts[5:]) * 1000:.1f} us, iters {g.decode_stats(tr.d_stats)['iters']}  " +
          " ".join(f"{nm}={v * 1000:.1f}" for nm, v in zip(names, sp)))


if __name__ == "__main__":
    main()
