import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2403_12550_b200 as g, synth
from scipy.spatial import cKDTree
w = synth.make_frame_workload(2, "replica", M=1_000_000, stride=4)
K = w.K; dev = torch.device("cuda")
tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=4, device=dev)
tr.preprocess(torch.from_numpy(w.depth).to(dev))
tgt = g.build_target(*(torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales)))
cnt = torch.zeros((tr.cap, 4), dtype=torch.int32, device=dev)
g.debug_align_counters(cnt)
T, st = g.align(tr.cloud, tgt, w.T_init, tr.params, tr.ws_align)
g.debug_align_counters(None)
c = cnt[:tr.cloud.n()].cpu().numpy().astype(np.int64) & 0xffffffff
pts = tr.cloud.pos[:tr.cloud.n(), :3].cpu().numpy().astype(np.float64)
q = pts @ T[:3, :3].T + T[:3, 3]
tree = cKDTree(w.means.astype(np.float64))
d, _ = tree.query(q, k=2)
print("iters", st)
for it in range(int(c[:, 3].max())):
    m = (c[:, 0] >> it) & 1 == 1
    if m.sum() == 0: continue
    print(f"it {it}: queued {m.sum()}  d1 pct {np.percentile(d[m,0],[0,50,100]).round(4)}  d2 pct {np.percentile(d[m,1],[0,50,100]).round(4)}  gated(d1>0.1) {(d[m,0]>0.1).sum()}")
late = ((c[:, 0] >> 3) & 1 == 1)
print("late-queued indices", np.nonzero(late)[0][:20], "all d1", d[late, 0].round(4), "d2", d[late, 1].round(4))
print("overall d1 pct", np.percentile(d[:, 0], [50, 90, 99, 99.9, 100]).round(4))
