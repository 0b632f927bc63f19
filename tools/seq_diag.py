"""GPU diagnostic for C5 sequence tracking: per-frame errors with (a) ground-truth init through
track(), (b) host-side constant-velocity init through track(), (c) the device-chained graph."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def err(A, B):
    c = (np.trace(A[:3, :3].T @ B[:3, :3]) - 1) / 2
    return np.linalg.norm(A[:3, 3] - B[:3, 3]), math.degrees(math.acos(max(-1.0, min(1.0, c))))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    dev = torch.device("cuda")
    seq = synth.make_sequence(0, n, "replica", M=300_000)
    rows = synth.render_sequence_rows(seq, dev)
    tgt = g.build_target(torch.from_numpy(seq.means).to(dev), torch.from_numpy(seq.quats).to(dev),
                         torch.from_numpy(seq.scales).to(dev))
    K = seq.K
    params = g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6)
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=params)
    depth_full = [synth.raycast_depth_torch(seq.scene, K, seq.T_gt[i], device=dev) for i in range(n)]
    print("frame | gt-init err (m, deg) iters fit | cv-init err iters fit | motion (m, deg)")
    Tprev2, Tprev = seq.T_gt[0], seq.T_gt[0]
    for i in range(1, n if os.environ.get("HOST", "1") == "1" else 1):
        Tg, st = tr.track(depth_full[i], tgt, seq.T_gt[i])
        e1 = err(Tg, seq.T_gt[i])
        init = Tprev @ np.linalg.inv(Tprev2) @ Tprev
        Tc, st2 = tr.track(depth_full[i], tgt, init)
        e2 = err(Tc, seq.T_gt[i])
        mo = err(seq.T_gt[i - 1], seq.T_gt[i])
        print(f"{i:4d} | {e1[0]:.2e} {e1[1]:.3f} {st['iters']:2d} {st['fitness']:.3f} | {e2[0]:.2e} {e2[1]:.3f} "
              f"{st2['iters']:2d} {st2['fitness']:.3f} st={st2['status']} | {mo[0]:.4f} {mo[1]:.3f}")
        Tprev2, Tprev = Tprev, Tc
    T_est, ms = g.track_sequence(tr, tgt, rows, seq.T_gt[0], warmup=int(os.environ.get("WARM", "3")))
    for i in range(n - 1):
        e = err(T_est[i], seq.T_gt[i + 1])
        print(f"graph frame {i + 1}: err {e[0]:.2e} m {e[1]:.3f} deg  {ms[i]:.3f} ms")


if __name__ == "__main__":
    main()
