"""Diagnostic: device-chained sequence frames one at a time (host sync after each): predicted pose,
estimate and stats per frame."""
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


rng = np.random.default_rng(0)
for _ in range(2):
    A = np.eye(4); A[:3, :3] = synth.rot_axis_angle(rng.standard_normal(3), 0.7); A[:3, 3] = rng.standard_normal(3)
    B = np.eye(4); B[:3, :3] = synth.rot_axis_angle(rng.standard_normal(3), 1.1); B[:3, 3] = rng.standard_normal(3)
    hist = torch.from_numpy(np.concatenate([A.reshape(-1), B.reshape(-1)])).cuda()
    out = torch.zeros(16, dtype=torch.float64, device="cuda")
    g.pose_predict(hist, out)
    print("predict max diff", np.abs(out.cpu().numpy().reshape(4, 4) - B @ np.linalg.inv(A) @ B).max())

n = 40
dev = torch.device("cuda")
seq = synth.make_sequence(0, n, "replica", M=300_000)
rows = synth.render_sequence_rows(seq, dev)
tgt = g.build_target(torch.from_numpy(seq.means).to(dev), torch.from_numpy(seq.quats).to(dev),
                     torch.from_numpy(seq.scales).to(dev))
K = seq.K
params = g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6)
tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, params=params)
T0 = torch.from_numpy(seq.T_gt[0].reshape(-1).copy()).to(dev)
hist = torch.cat([T0, T0])
traj = torch.zeros((n, 16), dtype=torch.float64, device=dev)
counter = torch.zeros(1, dtype=torch.int32, device=dev)
fg = tr.sequence_graph(tgt, hist, traj, counter)
pred = torch.zeros(16, dtype=torch.float64, device=dev)
for i in range(1, n):
    g.pose_predict(hist, pred)
    h = hist.cpu().numpy().reshape(2, 4, 4)
    tr.rows.copy_(rows[i])
    fg.replay()
    torch.cuda.synchronize()
    st = g.decode_stats(tr.d_stats)
    est = tr.d_T.cpu().numpy().reshape(4, 4)
    p = pred.cpu().numpy().reshape(4, 4)
    ep, ee = err(p, seq.T_gt[i]), err(est, seq.T_gt[i])
    hp = h[1] @ np.linalg.inv(h[0]) @ h[1]
    print(f"{i:3d} pred err {ep[0]:.2e} {ep[1]:.3f} | est err {ee[0]:.2e} {ee[1]:.4f} | iters {st['iters']} "
          f"fit {st['fitness']:.3f} cost {st['mean_cost']:.3e} conv {st['converged']} | pred-hostpred {np.abs(p - hp).max():.1e}")
