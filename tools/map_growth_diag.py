"""N1 diagnostic: track a synthetic sequence against a map with a region removed, with and
without keyframe insertion (GaussianMap / track_sequence_mapping); prints fitness, keyframes,
inserted counts, ATE and the rebuild cost."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    n_frames = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 300_000
    seq = synth.make_sequence(1, n_frames, "replica", M=M)
    rows = synth.render_sequence_rows(seq, "cuda")
    K = seq.K
    L = seq.scene.room
    def world_pts(i):
        d = rows[i].cpu().numpy()
        v, u = np.nonzero(np.isfinite(d) & (d > 0.1) & (d < 10))
        z = d[v, u]
        P = np.stack([(u - K.cx) * z / K.fx, (v * seq.stride - K.cy) * z / K.fy, z], 1)
        return P @ seq.T_gt[i][:3, :3].T + seq.T_gt[i][:3, 3]

    P0, P1 = world_pts(0), world_pts(n_frames - 1)
    ax = int(np.argmax(np.abs(np.median(P1, 0) - np.median(P0, 0))))
    sgn = 1.0 if np.median(P1[:, ax]) > np.median(P0[:, ax]) else -1.0
    print("axis", ax, "first-frame median", np.median(P0, 0), "last-frame median", np.median(P1, 0))
    for q in (0.5, 0.8):
        cut = np.quantile(sgn * P0[:, ax], q)  # keep the part of the room the first frame sees
        keep = sgn * seq.means[:, ax] < cut
        print(f"cut {'+-'[sgn < 0]}x{ax} < {cut:.2f}: map {keep.sum()} of {len(keep)}")
        for grow in (False, True):
            tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, keep_corr=True,
                           params=g.align_params(max_iters=30, max_corr_dist=0.1))
            gm = g.GaussianMap(torch.from_numpy(seq.means[keep]).cuda(), torch.from_numpy(seq.quats[keep]).cuda(),
                               torch.from_numpy(seq.scales[keep]).cuda(), capacity=int(keep.sum()) + 40 * tr.cap)
            t0 = time.time()
            T_est, kfs, added, st = g.track_sequence_mapping(tr, gm, rows, seq.T_gt[0],
                                                             min_fitness=0.95 if grow else -1.0,
                                                             max_gap=30 if grow else 10 ** 9)
            dt = time.time() - t0
            err = synth.trajectory_error(T_est, seq.T_gt[1:])
            fit = np.array([s["fitness"] for s in st])
            print(f"  grow={grow}: ATE {err['ate_rmse_m']:.2e} m, rot max {err['rot_max_deg']:.3f} deg, "
                  f"fitness mean {fit.mean():.3f} min {fit.min():.3f} last10 {fit[-10:].mean():.3f}, "
                  f"keyframes {kfs} added {added}, map {gm.M}, wall {dt:.1f} s")
    # rebuild cost at 1e6
    means, quats, scales, _ = synth.sample_map(synth.make_scene(1006), 1_000_000, 4006)
    gm = g.GaussianMap(torch.from_numpy(means).cuda(), torch.from_numpy(quats).cuda(), torch.from_numpy(scales).cuda(),
                       capacity=1_100_000)
    for _ in range(2):
        gm.rebuild()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gm.rebuild()
    e1.record()
    torch.cuda.synchronize()
    print(f"target rebuild at M=1e6: {e0.elapsed_time(e1) / 5:.2f} ms")


if __name__ == "__main__":
    main()
