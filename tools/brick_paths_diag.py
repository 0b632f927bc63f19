import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2403_12550_b200 as g
rng = np.random.default_rng(77)
plane = np.concatenate([rng.uniform(-0.3, 0.3, (6000, 2)), np.zeros((6000, 1))], 1)
blob = rng.normal(0.0, 0.002, (600, 3)) + np.array([0.05, 0.05, 0.0])
blob2 = rng.normal(0.0, 0.0015, (70, 3)) + np.array([-0.2, 0.1, 0.5])
far = rng.uniform(-2.0, 2.0, (40, 3)) + np.array([0.0, 0.0, 3.0])
lat = np.concatenate([np.stack(np.meshgrid(np.arange(12), np.arange(12)), -1).reshape(-1, 2) * 0.01 + 0.4, np.full((144, 1), 0.2)], 1)
xyz = np.concatenate([plane, blob, blob2, far, lat]).astype(np.float32)
n = xyz.shape[0]
pos = torch.zeros((n, 4), dtype=torch.float32, device='cuda'); pos[:, :3] = torch.from_numpy(xyz).cuda()
d_n = torch.tensor([n], dtype=torch.int32, device='cuda')
for cell0, lv in ((0.02, 3), (0.04, 2)):
    dbg = torch.zeros((n, 4), dtype=torch.int32, device='cuda')
    g.debug_knn_counters(dbg)
    g.covariances(pos, d_n, 20, g.REG_ELLIPSE, 1e-3, cell0, lv)
    g.debug_knn_counters(None); torch.cuda.synchronize()
    d = dbg.cpu().numpy()
    print(cell0, lv, "brick", (d[:, 0] == -7).sum(), "fail reasons", np.bincount(d[d[:, 0] == -8, 1], minlength=7)[1:], "blob2 brick-finished", (d[6600:6670, 0] == -7).sum())
