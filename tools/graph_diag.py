"""GPU diagnostic: the bench step eager (Python -> C-ABI launches) vs replayed from one CUDA
graph, device time per step (CUDA events, L2 flushed between steps).  python tools/graph_diag.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2403_12550_b200 as g
import synth


def main():
    w = synth.make_frame_workload(2, "replica", M=1_000_000, stride=4)
    K = w.K
    dev = torch.device("cuda")
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=4, device=dev)
    depth = torch.from_numpy(w.depth).to(dev)
    tgt = g.build_target(*(torch.from_numpy(x).to(dev) for x in (w.means, w.quats, w.scales)))
    T0 = torch.from_numpy(w.T_init.reshape(-1).copy()).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream()

    def step():
        tr.d_T.copy_(T0)
        tr.step_async(depth, tgt)

    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        step()
    torch.cuda.synchronize()

    def timeit(fn, reps=50, do_flush=True):
        ts = []
        for _ in range(reps):
            if do_flush:
                flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1000)
        return statistics.median(ts)

    for flush_on in (True, False):
        print(f"L2 flush={flush_on}: eager {timeit(step, do_flush=flush_on):.1f} us  graph {timeit(graph.replay, do_flush=flush_on):.1f} us")
    # back-to-back (no sync between steps): throughput
    for name, fn in (("eager", step), ("graph", graph.replay)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"back-to-back {name}: {e0.elapsed_time(e1) * 10:.1f} us/step")


if __name__ == "__main__":
    main()
