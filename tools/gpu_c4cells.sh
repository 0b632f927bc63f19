# C4 timing per library variant and brick size (VARIANTS="a b", CELLS="3.0 3.4 3.8")
L=paper_2403_12550_b200/libgsicp.so
cp $L /tmp/libgsicp_cur.so
for v in ${VARIANTS}; do
  cp paper_2403_12550_b200/variants/libgsicp_$v.so $L
  python - <<PY
import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2403_12550_b200 as g, synth
scene = synth.make_scene(1004)
means, _, _, ell = synth.sample_map(scene, 4_000_000, 4004)
c = g.Cloud.from_points(torch.from_numpy(means).cuda())
for cm in [float(x) for x in "${CELLS:-3.4}".split()]:
    ws = g._ws(g.lib().gsicp_covariances_workspace_size(c.cap, 3), c.pos.device)
    for _ in range(2): g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, cm * ell, 3, c.cov_a, c.cov_b, None, ws)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.covariances(c.pos, c.d_n, 20, g.REG_ELLIPSE, 1e-3, cm * ell, 3, c.cov_a, c.cov_b, None, ws); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print("$v", "cell", cm, round(float(np.median(ts)), 3), "ms", flush=True)
    del ws
PY
done
cp /tmp/libgsicp_cur.so $L
