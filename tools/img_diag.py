"""GPU diagnostic: image-window kNN-cov on the bench frame (and a TUM frame): how many queries the
window certifies (debug level -1) vs the hash-search queue, and timings vs the hash path.
python tools/img_diag.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def run(w, s, label):
    K = w.K
    H, W = w.depth.shape
    Kt = (K.fx, K.fy, K.cx, K.cy)
    pos, d_n = g.backproject_downsample(torch.from_numpy(w.depth).cuda(), Kt, stride=s)
    n = int(d_n.item())
    cap = pos.shape[0]
    cell0, levels = 3.0 * s / K.fx, 4
    ws_i = g._ws(g.lib().gsicp_covariances_image_workspace_size(cap, levels, H, W, s), pos.device)
    ws_h = g._ws(g.lib().gsicp_covariances_workspace_size(cap, levels), pos.device)
    dbg = torch.zeros((cap, 4), dtype=torch.int32, device=pos.device)
    g.debug_knn_counters(dbg)
    g.covariances_image(pos, d_n, H, W, s, Kt, 20, g.REG_ELLIPSE, 1e-3, cell0, levels, ws=ws_i)
    g.debug_knn_counters(None)
    torch.cuda.synchronize()
    d = dbg[:n].cpu().numpy()
    win = d[:, 0] == -1
    wide = d[:, 0] == -3
    ti = timeit(lambda: g.covariances_image(pos, d_n, H, W, s, Kt, 20, g.REG_ELLIPSE, 1e-3, cell0, levels, ws=ws_i))
    th = timeit(lambda: g.covariances(pos, d_n, 20, g.REG_ELLIPSE, 1e-3, cell0, levels, ws=ws_h))
    brute = d[:, 0] == -6
    print(f"{label}: n={n} window-certified {win.mean():.4f}, wide {int(wide.sum())}, brute {int(brute.sum())}, hash {int((~win & ~wide & ~brute).sum())}  "
          f"image path {ti * 1000:.1f} us  hash path {th * 1000:.1f} us")
    req = d[(d[:, 0] == -1) | (d[:, 0] == -2), 1] / 100.0  # projection extent of the k-th ball, in lattice pixels
    if req.size:
        qs = np.percentile(req, [50, 75, 90, 95, 99])
        need = np.ceil(req - 1.0 + 1e-9)
        print("  k-ball extent (lattice px) p50/75/90/95/99:", np.round(qs, 2).tolist(),
              " certified share by window M:", {M: round(float(np.mean(need <= M)), 3) for M in (3, 4, 5, 6, 8, 10)})
    for code, name in ((-4, "wide cert fail"), (-5, "wide m>64 / no b*"), (-6, "brute force")):
        sel = d[:, 0] == code
        if sel.any():
            print(f"  {name}: {int(sel.sum())}  field1 p50/max {np.percentile(d[sel, 1], 50):.0f}/{d[sel, 1].max()}"
                  f"  m p50/max {np.percentile(d[sel, 2], 50):.0f}/{d[sel, 2].max()}")
    if win.any():
        m = d[win, 2]
        print(f"  m (candidates at or below b*): mean {m.mean():.1f} p90 {np.percentile(m, 90):.0f} max {m.max()}")


def main():
    run(synth.make_frame_workload(2, "replica", M=1000, stride=4), 4, "replica s=4")
    tum = synth.make_frame_workload(3, "tum", M=1000, stride=1, noisy=True)
    for s in (1, 4):
        run(tum, s, f"tum s={s}")


if __name__ == "__main__":
    main()
