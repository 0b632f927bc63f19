"""N1 diagnostic: (1) a synthetic sequence tracked against a map with part of the room removed,
with and without keyframe insertion (device decision + conditional incremental insertion inside
the per-frame graph: track_sequence_mapping); (2) the cost of one keyframe insertion into a
1e6-Gaussian map (incremental target maintenance) against a from-scratch gsicp_build_target.
python tools/map_growth_diag.py [n_frames] [M]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    n_frames = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 300_000
    seq = synth.make_sequence(1, n_frames, "replica", M=M)
    rows = synth.render_sequence_rows(seq, "cuda")
    K = seq.K
    d = rows[0].cpu().numpy()
    v, u = np.nonzero(np.isfinite(d) & (d > 0.1) & (d < 10))
    z = d[v, u]
    P0 = np.stack([(u - K.cx) * z / K.fx, (v * seq.stride - K.cy) * z / K.fy, z], 1) @ seq.T_gt[0][:3, :3].T \
        + seq.T_gt[0][:3, 3]
    keep = seq.means[:, 0] < np.median(P0[:, 0])
    print(f"map {keep.sum()} of {len(keep)} Gaussians (half of what frame 0 sees removed)")
    for grow in (False, True):
        tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=seq.stride, keep_corr=True,
                       params=g.align_params(max_iters=30, max_corr_dist=0.1))
        gm = g.GaussianMap(torch.from_numpy(seq.means[keep]).cuda(), torch.from_numpy(seq.quats[keep]).cuda(),
                           torch.from_numpy(seq.scales[keep]).cuda(), capacity=int(keep.sum()) + 40 * tr.cap,
                           max_insert=tr.cap)
        T_est, kfs, added, fit, ms = g.track_sequence_mapping(tr, gm, rows, seq.T_gt[0],
                                                              min_fitness=0.95 if grow else -1.0,
                                                              max_gap=30 if grow else 10 ** 9, timed=True)
        err = synth.trajectory_error(T_est, seq.T_gt[1:])
        kf_ms = [ms[i - 1] for i in kfs]
        print(f"  grow={grow}: ATE {err['ate_rmse_m']:.2e} m, rot max {err['rot_max_deg']:.3f} deg, fitness mean "
              f"{fit.mean():.3f} min {fit.min():.3f} last10 {fit[-10:].mean():.3f}, keyframes {kfs} added {added}, "
              f"map {gm.M}; frame ms median {np.median(ms):.3f}, keyframe frames {np.round(kf_ms, 3).tolist()}")
    # one insertion into a 1e6 map vs a from-scratch build
    w = synth.make_frame_workload(2, "replica", M=1_000_000, stride=4)
    dev = torch.device("cuda")
    means, quats, scales = (torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales))
    tr = g.Tracker(w.K.H, w.K.W, (w.K.fx, w.K.fy, w.K.cx, w.K.cy), stride=4, keep_corr=True)
    gm = g.GaussianMap(means, quats, scales, capacity=1_000_000 + 64 * tr.cap, max_insert=tr.cap)
    T, st = tr.track(torch.from_numpy(w.depth).to(dev), gm.tgt, w.T_init)
    corr = tr.corr.clone()
    corr[: tr.cloud.n() // 4] = -1  # a quarter of the frame unmatched (new surface)
    ms_ins = timed(lambda: gm.insert(tr.cloud, tr.d_T, corr), reps=10)
    M1 = gm.M
    ms_full = timed(lambda: g.build_target(gm.means[:M1], gm.quats[:M1], gm.scales[:M1], cell=gm.cell), reps=3)
    print(f"insertion of {int(gm.d_M[1].item())} Gaussians into a {M1 / 1e6:.2f}e6 map: {ms_ins:.3f} ms "
          f"(incremental); from-scratch gsicp_build_target of the same rows: {ms_full:.3f} ms")


if __name__ == "__main__":
    main()
