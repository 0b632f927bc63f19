"""Timing of the auxiliary rows: A4' export (51k-point Replica frame, with and without the overlap
filter), N4 voxel downsampling (Replica frame at stride 1, ~800k points), N1 insertion + target
rebuild.  Device time by CUDA events, L2 flushed before each repetition; algorithmic bytes / time
against the measured HBM copy bandwidth."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def timed(fn, reps=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs", 6547.8))
    w = synth.make_frame_workload(2, "replica", M=1_000_000, stride=4)
    K = w.K
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=4, keep_corr=True)
    tgt = g.build_target(torch.from_numpy(w.means).cuda(), torch.from_numpy(w.quats).cuda(),
                         torch.from_numpy(w.scales).cuda())
    depth = torch.from_numpy(w.depth).cuda()
    T, st = tr.track(depth, tgt, w.T_init)
    n = tr.cloud.n()
    cl = tr.cloud
    out = (torch.empty((cl.cap, 3), device="cuda"), torch.empty((cl.cap, 4), device="cuda"),
           torch.empty((cl.cap, 3), device="cuda"))
    ms = timed(lambda: g.export_gaussians(cl.pos, cl.d_n, cl.cov_a, cl.cov_b, T=tr.d_T, out=out))
    by = n * (48 + 40)
    print(f"export {n} pts: {ms * 1000:.1f} us, {by / ms / 1e6:.0f} GB/s ({by / ms / 1e6 / hbm:.1%} of {hbm:.0f})")
    corr = tr.corr.clone()
    corr[: n // 2] = -1  # half the frame unmatched
    ms = timed(lambda: g.export_gaussians(cl.pos, cl.d_n, cl.cov_a, cl.cov_b, T=tr.d_T, corr=corr, out=out))
    print(f"export with overlap filter (half kept): {ms * 1000:.1f} us")
    pos1, d1 = g.backproject_downsample(depth, (K.fx, K.fy, K.cx, K.cy), stride=1)
    n1 = int(d1.item())
    for h in (0.01, 0.03):
        vo = torch.empty_like(pos1)
        ms = timed(lambda: g.voxel_downsample(pos1, d1, h, out=vo))
        _, dm = g.voxel_downsample(pos1, d1, h, out=vo)
        m = int(dm.item())
        by = n1 * 16 + m * 16
        print(f"voxel h={h}: {n1} -> {m} pts, {ms * 1000:.1f} us, algorithmic {by / ms / 1e6:.0f} GB/s")
    M = w.means.shape[0]
    ms = timed(lambda: g.build_target(torch.from_numpy(w.means).cuda(), torch.from_numpy(w.quats).cuda(),
                                      torch.from_numpy(w.scales).cuda()), reps=5)
    print(f"target build M={M}: {ms:.2f} ms")


if __name__ == "__main__":
    main()
