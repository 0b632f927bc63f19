"""GPU diagnostic: per-iteration timeline of the persistent G-ICP kernel (block barrier arrivals)
for the bench frame vs the 1e6 map, over a sweep of target cell sizes.
Run under gpurun:  python tools/align_diag.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    shape = sys.argv[1] if len(sys.argv) > 1 else "replica"
    stride = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    w = (synth.make_frame_workload(2, "replica", M=1_000_000, stride=stride) if shape == "replica"
         else synth.make_frame_workload(3, "tum", M=1_000_000, stride=stride, noisy=True))
    K = w.K
    dev = torch.device("cuda")
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=stride, device=dev)
    depth = torch.from_numpy(w.depth).to(dev)
    tr.preprocess(depth)
    means, quats, scales = (torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales))
    tl = torch.zeros(1 << 16, dtype=torch.int64, device=dev)
    cases = [("1e6", means, quats, scales, 0.0)]
    seeded = os.environ.get("SEEDED", "1") == "1"
    for name, mm, qq, ss, cell in cases:
        print(f"map {name}")
        tgt = g.build_target(mm, qq, ss, cell=cell)
        for _ in range(3):
            T, st = g.align(tr.cloud, tgt, w.T_init, tr.params, tr.ws_align)
        cnt = torch.zeros((tr.cap, 4), dtype=torch.int32, device=dev)
        g.debug_align_counters(cnt)
        T, st = g.align(tr.cloud, tgt, w.T_init, tr.params, tr.ws_align)
        g.debug_align_counters(None)
        c = cnt[:tr.cloud.n()].cpu().numpy().astype(np.int64) & 0xffffffff
        n_it = int(c[:, 3].max())
        Gb = torch.cuda.get_device_properties(0).multi_processor_count
        for it in range(n_it):
            bit = 1 << it
            q, r, gr = ((c[:, k] & bit) != 0 for k in range(3))
            fast = ~(q | r | gr)
            P = -(-c.shape[0] // Gb)  # k_align's chunk of points per block
            pb = lambda m: np.bincount(np.arange(len(m))[m] // P, minlength=Gb)
            print(f"  it {it}: queued {q.mean():.4f} reuse {r.mean():.4f} graph {gr.mean():.4f} other {fast.mean():.4f} | "
                  f"per block max: queued {pb(q).max()} graph {pb(gr).max()} other {pb(fast).max()}")
        tl.zero_()
        dT = torch.from_numpy(np.ascontiguousarray(w.T_init).reshape(-1)).to(dev)
        if seeded:  # iteration-0 correspondences ahead, as the Tracker does
            g.align_seed(tr.cloud, tgt, dT, tr.params, tr.ws_align)
            torch.cuda.synchronize()
        g.debug_align_timeline(tl)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        T, st = g.align(tr.cloud, tgt, w.T_init, tr.params, tr.ws_align)
        e1.record()
        g.debug_align_timeline(None)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t = tl.cpu().numpy()
        Gn = torch.cuda.get_device_properties(0).multi_processor_count  # k_align: the full co-resident grid
        t0 = t[0]
        print(f"cell={tgt.cell * 100:.2f} cm  iters={st['iters']} total {ms * 1000:.1f} us (event)")
        prev = t0
        max_iters = tr.params.max_iters
        ph0 = 1 + max_iters * (Gn + 1)
        names = ["A", "B", "blkred+barrier", "finalred", "solve"]
        for it in range(st["iters"] + 1):
            rec = 1 + it * (Gn + 1)
            arr = t[rec:rec + Gn]
            pas = t[rec + Gn]
            if pas == 0:
                break
            a = (arr - prev) / 1000.0
            ph = t[ph0 + it * 8: ph0 + it * 8 + 6]
            phs = " ".join(f"{nm}={(ph[j + 1] - ph[j]) / 1000.0:.1f}" for j, nm in enumerate(names))
            print(f"  it {it}: arrivals min {a.min():7.1f} p50 {np.median(a):7.1f} max {a.max():7.1f} us; "
                  f"release {(pas - prev) / 1000.0:7.1f} us | block0 phases(us) {phs}")
            sb = 1 + max_iters * (Gn + 9) + it * 8
            c = t[sb:sb + 8]
            print(f"      warp0 cycles: k3+own={c[1] - c[0]} warm={c[2] - c[1]} search={c[3] - c[2]} "
                  f"rest={c[5] - c[3]} empty_best={c[4]} | B start->{c[6] - c[5]} pair={c[7] - c[6]}")
            wb = 1 + max_iters * (Gn + 17) + it * 12 * 2
            wl = t[wb:wb + 24].reshape(12, 2)
            names_p = ["reuse", "graph", "fast", "queued", "seeded"]
            print("      block0 warps: slowest lane cycles (path) " +
                  " ".join(f"{int(c)}({names_p[int(k)] if 0 <= k < 5 else '?'})" for c, k in wl))
            prev = pas


if __name__ == "__main__":
    main()
