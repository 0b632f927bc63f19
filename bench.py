#!/usr/bin/env python
"""Benchmark of the G-ICP tracking hot path (BASELINE.json metric:
"G-ICP aligns/sec (Replica frame vs 1M-Gaussian map); kNN-cov Mpts/s; HBM %").

One step = one whole frame through the hot path: back-projection +
stride-4 downsampling of a Replica-shaped 1200x680 depth frame, multi-level spatial hash +
exact kNN (k=20) covariances with ELLIPSE regularisation, and the persistent G-ICP kernel
(correspondences, H/b, on-device 6x6 solve, up to 30 GN iterations) against a prebuilt
1e6-Gaussian map target.  Inputs are synthetic (synth/), resident in HBM; L2 is flushed
between timed steps.  Multi-GPU = independent replicas (one frame stream per rank, no
collective on the data path).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--no-c4]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "G-ICP aligns/sec (Replica frame vs 1M-Gaussian map); kNN-cov Mpts/s; HBM %"
WORKLOAD = "Replica-shaped 1200x680 depth frame, stride 4 (<=51k pts), vs 1e6-Gaussian map (C2 geometry, 1M map)"
ALGO_BYTES_ALIGN = 96 + 8   # per (source point x GN iteration): src pos+cov, tgt pos+cov, corr
ALGO_BYTES_KNN = 16 + 32    # per query of the kNN-cov stage: pos in, cov out
C4_CELL, C4_LEVELS = 3.4, 3  # map kNN-cov grid: bricks of 3.4 map spacings, two coarser levels for the floating outliers


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6550.1)), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


class ClockSampler:
    """SM clock + clock-event reasons sampled through NVML every 5 ms during the timed region
    (the B200_PROFILING.md clocks line; nvidia-smi's 100 ms floor is too coarse for a region of
    ~0.1-0.5 s).  Reports the median SM clock under load, the max clock and the reasons seen."""

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.sm, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:  # NVML unavailable: report it, do not fail the bench
            self.ok = False
        return self

    def _run(self):
        nv = self.nv
        names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                 nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                 nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap",
                 nv.nvmlClocksEventReasonHwPowerBrakeSlowdown: "hw_power_brake"}
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, nm in names.items():
                    if r & bit:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join(timeout=2)
        return False

    def summary(self):
        if not self.ok or not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x: float, dist=None, device=None) -> float:
    """Max of a per-rank device-timed quantity over all ranks (the slowest replica defines the
    whole-job time); identity at world size 1."""
    if dist is None:
        return float(x)
    import torch

    on_cpu = dist.get_backend() == "gloo"
    t = torch.tensor([float(x)], dtype=torch.float64, device="cpu" if on_cpu else device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank: int, world_size: int, total_ms: float) -> float:
    """Whole-job aggregate: every rank processes `units_per_rank` independent frames (replicas,
    weak scaling); the job time is the max over ranks."""
    return world_size * units_per_rank / (total_ms / 1000.0)


def csrc_sha() -> str:
    """Hash of the CUDA sources: ties a stored ncu traffic figure to the code it was measured on."""
    import hashlib

    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2403_12550_b200", "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".inc")):
            h.update(f.encode())
            h.update(open(os.path.join(d, f), "rb").read())
    return h.hexdigest()[:16]


def pct(xs, q):
    return float(np.percentile(np.asarray(xs, dtype=np.float64), q))


def time_frame_graph(g, tr, depth, tgt, T_init, steps, warmup, flush, stream, dev):
    """A frame config timed like the headline: the whole frame (Tracker.step_async) captured in one
    graph, replayed `steps` times with L2 flushed in between, CUDA events per replay on the launch
    stream; each replay's pose compared bitwise with the first.  -> (ms list, stats, bitwise)"""
    import torch

    T0 = torch.from_numpy(np.ascontiguousarray(T_init).reshape(-1).copy()).to(dev)

    def step():
        tr.d_T.copy_(T0)
        tr.step_async(depth, tgt, torch.cuda.current_stream(dev))

    for _ in range(max(warmup, 3)):
        step()
    torch.cuda.synchronize()
    cs = torch.cuda.Stream(dev)
    fg = g.FrameGraph()
    with fg.capture(cs):
        step()
    for _ in range(max(warmup, 3)):
        fg.replay(stream)
    torch.cuda.synchronize()
    ms, poses = [], []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fg.replay(stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        poses.append(tr.d_T.cpu().numpy().copy())
    bitwise = all(np.array_equal(p_, poses[0]) for p_ in poses)
    return ms, g.decode_stats(tr.d_stats), bitwise


class CollectiveWatch:
    """Counts torch.distributed collectives issued while `active` (the timed regions): the replicas
    share nothing on the data path, so the count must stay 0."""

    def __init__(self, dist):
        self.active = False
        self.count = 0
        if dist is None:
            return
        for name in ("all_reduce", "barrier", "all_gather", "broadcast", "reduce_scatter", "all_to_all",
                     "all_gather_into_tensor", "reduce_scatter_tensor"):
            fn = getattr(dist, name, None)
            if fn is None:
                continue

            def wrap(f):
                def inner(*a, **k):
                    if self.active:
                        self.count += 1
                    return f(*a, **k)
                return inner
            setattr(dist, name, wrap(fn))


def make_workload(rank: int):
    import synth

    return synth.make_frame_workload(2 + 100 * rank, "replica", M=1_000_000, stride=4)


# ------------------------------------------------------------------------------------------- oracle
def run_oracle_frame(w):
    """One frame of the oracle (as it stands): A1, A2-A4 (brute-force kNN), A6-A9 (kd-tree NN).
    The map target's covariances (A5) are prebuilt outside, like the GPU arm's target."""
    import oracle

    K = w.K
    t0 = time.perf_counter()
    xyz, _ = oracle.backproject(w.depth, K.fx, K.fy, K.cx, K.cy, w.stride)
    cs = oracle.covariances(xyz)["cov"]
    r = oracle.align(xyz, cs, w.means, w._oracle_tcov, w.T_init, max_iters=30, max_corr_dist=0.1,
                     tree=w._oracle_tree)
    return time.perf_counter() - t0, r


def oracle_prepare(w):
    """The map side (A5 covariances and the NN index over the map means) is prebuilt, as the
    GPU arm's target is."""
    import oracle

    w._oracle_tcov, _ = oracle.target_from_map(w.quats, w.scales)
    w._oracle_tree = oracle.KDTree(w.means)


def cpu_baseline(w, min_seconds=10.0, max_frames=64):
    """The oracle as it stands on the host cores: whole frames of the bench workload until about
    min_seconds of CPU time (a bounded sample), aligns/s."""
    import oracle

    oracle.set_threads(os.cpu_count() or 1)
    oracle_prepare(w)
    secs = []
    while sum(secs) < min_seconds and len(secs) < max_frames:
        secs.append(run_oracle_frame(w)[0])
    t = sum(secs)
    return {"value": len(secs) / t, "unit": "aligns/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{len(secs)} Replica-shaped frame(s) of the bench workload (A1 + brute-force kNN-cov + GN "
                      f"with kd-tree NN over the prebuilt 1e6-map index), {t:.1f} s"}


def bench_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle

    oracle.set_threads(os.cpu_count() or 1)  # every host core (torchrun sets OMP_NUM_THREADS=1)
    w = make_workload(0)
    oracle_prepare(w)
    for _ in range(args.warmup):
        run_oracle_frame(w)
    secs = [run_oracle_frame(w)[0] for _ in range(args.steps)]
    total = sum(secs)
    value = args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "aligns/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "k": 20, "max_iters": 30, "max_corr_dist": 0.1},
        "cpu_baseline": {"value": value, "unit": "aligns/s", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": "1 frame per step (whole frame, oracle as it stands)"},
        "e2e": {"value": value, "unit": "aligns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------- GPU
def bench_gpu(args):
    import torch

    ws, rank, local = dist_env()
    # BENCH_DIST_BACKEND=gloo (testing the multi-rank path on one GPU: every rank on device
    # local % device_count, CPU reductions); the real multi-GPU run uses NCCL, one GPU per rank
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count() if backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    import paper_2403_12550_b200 as g

    watch = CollectiveWatch(dist)
    w = make_workload(rank)
    K = w.K
    depth_host = torch.from_numpy(w.depth).pin_memory()
    depth = depth_host.to(dev)
    tcell = float(os.environ.get("BENCH_TGT_CELL", "0")) * w.ell  # (diagnostic; 0 = the library's auto cell)
    tgt = g.build_target(torch.from_numpy(w.means).to(dev), torch.from_numpy(w.quats).to(dev),
                         torch.from_numpy(w.scales).to(dev), cell=tcell)
    params = g.align_params(max_iters=30, max_corr_dist=0.1, eps_rot=1e-6, eps_trans=1e-6)
    tr = g.Tracker(K.H, K.W, (K.fx, K.fy, K.cx, K.cy), stride=w.stride, params=params, device=dev)
    T0 = torch.from_numpy(w.T_init.reshape(-1).copy()).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(evs=None):
        tr.d_T.copy_(T0)
        # A1 | A2-A4 (+ iteration-0 correspondences on a side stream) | A6-A9 on the current stream
        tr.step_async(depth, tgt, torch.cuda.current_stream(dev), evs)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    n_src = tr.cloud.n()
    st = g.decode_stats(tr.d_stats)
    nev = args.steps

    # per-stage split from an eager pass (informational; events on `stream`)
    n_stage = min(nev, 20)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_stage)]
    for i in range(n_stage):
        flush.zero_()
        step(evs[i])
    torch.cuda.synchronize()
    stage = np.array([[evs[i][j].elapsed_time(evs[i][j + 1]) for j in range(3)] for i in range(n_stage)])

    # the timed step: the whole frame replayed from one CUDA graph (captured once; the kernel
    # timer's event pairs around k_knn_search / k_align / the seed pass are part of the graph)
    cap_stream = torch.cuda.Stream(dev)
    # kernel timer: the dominant kernels (level 1); BENCH_SPANS=1 adds the stage spans (level 2,
    # more event nodes in the graph: diagnostic only)
    g.debug_kernel_timer(2 if os.environ.get("BENCH_SPANS") == "1" else 1)
    step()  # creates the timer events outside the capture
    torch.cuda.synchronize()
    l0 = g.launch_count()
    graph = g.FrameGraph()  # instantiated with per-node priorities (critical path high, seeds low)
    with graph.capture(cap_stream):
        step()
    launches_per_step = g.launch_count() - l0
    g.debug_kernel_timer(False)
    for _ in range(max(args.warmup, 3)):
        graph.replay(stream)
    torch.cuda.synchronize()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
    kt = {k: [] for k in (g.KT_KNN_SEARCH, g.KT_ALIGN, g.KT_SEED, g.KT_BP, g.KT_COVS, g.KT_WIDE, g.KT_TAIL)}
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    poses = []
    watch.active = True
    with ClockSampler(local) as clk:
        for i in range(nev):
            flush.zero_()  # L2 flush (256 MB > 126 MB L2), outside the timed events
            e0[i].record(stream)
            graph.replay(stream)
            e1[i].record(stream)
            torch.cuda.synchronize()  # per-step kernel timer readout (host side, outside the events)
            for k in kt:
                kt[k].append(g.debug_kernel_time(k))
            poses.append(tr.d_T.cpu().numpy().copy())  # (outside the events) for the bitwise check
    watch.active = False
    repeat_bitwise = all(np.array_equal(p_, poses[0]) for p_ in poses)
    if dist:
        dist.barrier()
    step_ms = np.array([e0[i].elapsed_time(e1[i]) for i in range(nev)])
    total_ms = max_over_ranks(float(step_ms.sum()), dist, dev)
    value = job_throughput(nev, ws, total_ms)
    launches = launches_per_step * nev
    st = g.decode_stats(tr.d_stats)

    # e2e through the public API with host buffers: a stream of host frames (pinned) through
    # Tracker.track_host_stream — every step uploads the rows A1 reads (H2D, copy stream, double
    # buffered so it overlaps the previous frame's compute), replays the frame graph and reads the
    # pose + stats back (D2H); wall clock around the whole blocking call
    T_init = w.T_init
    tr.track_host_stream([depth_host] * max(args.warmup, 3), tgt, T_init)  # warm-up
    torch.cuda.synchronize()
    flush.zero_()
    torch.cuda.synchronize()
    watch.active = True
    t0 = time.perf_counter()
    res_e2e = tr.track_host_stream([depth_host] * nev, tgt, T_init)
    t1 = time.perf_counter()
    watch.active = False
    e2e_ms = [1000 * (t1 - t0) / nev] * nev
    Tg, st_e = res_e2e[-1]
    e2e_total = max_over_ranks(sum(e2e_ms), dist, dev)
    e2e_value = job_throughput(nev, ws, e2e_total)

    # C2 (the same frame vs a 1e5-Gaussian map) and C3 (TUM-shaped noisy frame vs the 1e6 map, at
    # stride 4 and stride 1): the other single-frame configs of BASELINE.json, timed like the headline
    configs_lines = {}
    if args.configs and rank == 0:
        import synth

        scene2 = synth.make_scene(1002)
        m2, q2, s2, _ = synth.sample_map(scene2, 100_000, 4002)
        tgt2 = g.build_target(torch.from_numpy(m2).to(dev), torch.from_numpy(q2).to(dev), torch.from_numpy(s2).to(dev))
        ms2, st2, bw2 = time_frame_graph(g, tr, depth, tgt2, w.T_init, nev, args.warmup, flush, stream, dev)
        configs_lines["c2"] = {"workload": "C2: the Replica-shaped frame (stride 4) vs a 1e5-Gaussian map",
                               "aligns_per_s": 1000.0 / float(np.mean(ms2)), "ms_p10_p50_p90": [pct(ms2, 10), pct(ms2, 50), pct(ms2, 90)],
                               "gn_iters": st2["iters"], "fitness": st2["fitness"], "repeat_bitwise": bw2}
        del tgt2
        w3 = synth.make_frame_workload(3, "tum", M=1_000_000, stride=1, noisy=True)
        K3 = w3.K
        tgt3 = g.build_target(torch.from_numpy(w3.means).to(dev), torch.from_numpy(w3.quats).to(dev),
                              torch.from_numpy(w3.scales).to(dev))
        depth3 = torch.from_numpy(w3.depth).to(dev)
        for s3 in (4, 1):
            tr3 = g.Tracker(K3.H, K3.W, (K3.fx, K3.fy, K3.cx, K3.cy), stride=s3, params=params, device=dev)
            g.debug_kernel_timer(1)
            ms3, st3, bw3 = time_frame_graph(g, tr3, depth3, tgt3, w3.T_init, max(10, nev // 3), args.warmup, flush,
                                             stream, dev)
            ka = g.debug_kernel_time(g.KT_ALIGN)
            g.debug_kernel_timer(False)
            n3 = tr3.cloud.n()
            algo3 = ALGO_BYTES_ALIGN * n3 * max(1, st3["iters"])
            configs_lines[f"c3_s{s3}"] = {
                "workload": f"C3: TUM-shaped 640x480 noisy frame, stride {s3} ({n3} pts) vs the 1e6-Gaussian map",
                "aligns_per_s": 1000.0 / float(np.mean(ms3)), "ms_p10_p50_p90": [pct(ms3, 10), pct(ms3, 50), pct(ms3, 90)],
                "gn_iters": st3["iters"], "fitness": st3["fitness"], "status": st3["status"], "repeat_bitwise": bw3,
                "k_align_ms_last": ka,
                "k_align_roofline": None if not ka else {"achieved_gbs": algo3 / (ka / 1000) / 1e9,
                                                         "frac": algo3 / (ka / 1000) / 1e9 / peaks()[0],
                                                         "algo_bytes": algo3}}
            del tr3
        del tgt3, depth3

    # C5: sequence tracking — each rank its own synthetic 30 Hz sequence (scene 100+rank), frames
    # 1..n tracked in order with the constant-velocity initial pose computed on the device, one
    # graph replay per frame (no host round trip), L2 flushed between frames; ATE vs the
    # generating trajectory.  Whole-job aligns/s = frames of all ranks / max-over-ranks time.
    seq_line = None
    sq = rows_all = tgt_s = None
    if args.seq_frames > 0 or args.batch > 0:
        import synth

        # one synthetic sequence per rank serves C5 (frames 1..seq_frames) and N2 (frames 1..B)
        sq = synth.make_sequence(rank, max(args.seq_frames, args.batch) + 1, "replica", M=1_000_000)
        rows_all = synth.render_sequence_rows(sq, dev)
        tgt_s = g.build_target(torch.from_numpy(sq.means).to(dev), torch.from_numpy(sq.quats).to(dev),
                               torch.from_numpy(sq.scales).to(dev))
        Ks = sq.K
    if args.seq_frames > 0:
        tr_s = g.Tracker(Ks.H, Ks.W, (Ks.fx, Ks.fy, Ks.cx, Ks.cy), stride=sq.stride, params=params, device=dev)
        T_est, ms_s = g.track_sequence(tr_s, tgt_s, rows_all[:args.seq_frames + 1], sq.T_gt[0], flush=flush)
        seq_total = max_over_ranks(float(ms_s.sum()), dist, dev)
        seq_line = {"workload": f"C5: {args.seq_frames}-frame Replica-shaped 30 Hz sequence per rank "
                                "(Lissajous path, 1e6-Gaussian map of its room), constant-velocity init",
                    "frames_per_rank": args.seq_frames, "aligns_per_s": job_throughput(args.seq_frames, ws, seq_total),
                    "ms_per_frame_mean": float(ms_s.mean()), **synth.trajectory_error(T_est, sq.T_gt[1:args.seq_frames + 1])}
        del tr_s

    # N2 throughput mode: B distinct frames of the rank's sequence per step (frames 1..B, each from
    # a perturbed ground-truth pose) — A1-A4 on B concurrent streams, then one batched GN launch
    # (k_align_batch, or the flat GN loop over the frames for B >= 6), one graph replay, L2 flushed
    # per step.  The align stage's span (kernel timer events in the graph) gives its algorithmic
    # bandwidth: 104 B per pair-iteration x the frames' points x their iterations.
    batch_line = None
    if args.batch > 0:
        B = args.batch
        bt = g.BatchTracker(B, Ks.H, Ks.W, (Ks.fx, Ks.fy, Ks.cx, Ks.cy), stride=sq.stride, params=params, device=dev)
        bt.rows.copy_(rows_all[1:1 + B])
        init_b = np.stack([synth.perturb_pose(sq.T_gt[1 + b], 500 + b, 2.0, 0.03) for b in range(B)])
        bt.track_rows(tgt_s, init_b)
        g.debug_kernel_timer(1)
        gb = bt.graph(tgt_s)
        Tb0 = torch.from_numpy(init_b.reshape(B, 16)).to(dev)
        sb = torch.cuda.current_stream(dev)
        bt.d_T.copy_(Tb0)  # one eager (untimed) step: what ncu captures (graph nodes behind a
        bt.step_async(tgt_s, sb)  # conditional node are not profilable)
        torch.cuda.synchronize()
        nb = max(10, min(args.steps, 50))
        evb = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nb)]
        for e0, e1 in evb:
            flush.zero_()
            bt.d_T.copy_(Tb0)
            e0.record(sb)
            gb.replay(sb)
            e1.record(sb)
        torch.cuda.synchronize()
        ka_b = g.debug_kernel_time(g.KT_ALIGN)  # the last replay's align stage
        g.debug_kernel_timer(False)
        b_total = max_over_ranks(sum(a.elapsed_time(b) for a, b in evb), dist, dev)
        Tb, stb = bt.track_rows(tgt_s, init_b)
        nb_pts = [tr.cloud.n() for tr in bt.trs]
        algo_b = ALGO_BYTES_ALIGN * sum(n_ * max(1, s_["iters"]) for n_, s_ in zip(nb_pts, stb))
        batch_line = {"workload": f"N2: {B} distinct frames of a Replica-shaped sequence per step (frames 1..{B}, "
                                  "perturbed initial poses) vs its 1e6-Gaussian map; A1-A4 on B concurrent streams, "
                                  "one batched GN launch",
                      "B": B, "aligns_per_s": job_throughput(nb * B, ws, b_total), "ms_per_step": b_total / nb,
                      "iters": [s_["iters"] for s_ in stb], "points": nb_pts,
                      "max_trans_err_m": float(max(np.abs(Tb[b][:3, 3] - sq.T_gt[1 + b][:3, 3]).max() for b in range(B))),
                      "align_ms": ka_b,
                      "align_roofline": None if not ka_b else {
                          "bound": "hbm", "achieved_gbs": algo_b / (ka_b / 1000) / 1e9,
                          "frac": algo_b / (ka_b / 1000) / 1e9 / peaks()[0], "algo_bytes": algo_b,
                          "note": "whole align stage of the step (GN loop of all B frames) timed by events around it"}}
        del bt
    del sq, rows_all, tgt_s

    # kNN-cov Mpts/s over a 4e6-point map (C4), kernel stage only
    knn_mpts = None
    if not args.no_c4 and rank == 0:
        import synth

        scene = synth.make_scene(1004)
        means4, _, _, ell4 = synth.sample_map(scene, 4_000_000, 4004)
        c4 = g.Cloud.from_points(torch.from_numpy(means4).to(dev))
        ws4 = g._ws(g.lib().gsicp_covariances_workspace_size(c4.cap, C4_LEVELS), dev)
        for _ in range(3):
            g.covariances(c4.pos, c4.d_n, 20, g.REG_ELLIPSE, 1e-3, C4_CELL * ell4, C4_LEVELS, c4.cov_a, c4.cov_b,
                          None, ws4)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        tms = []
        for _ in range(5):
            flush.zero_()
            e[0].record(stream)
            g.covariances(c4.pos, c4.d_n, 20, g.REG_ELLIPSE, 1e-3, C4_CELL * ell4, C4_LEVELS, c4.cov_a, c4.cov_b,
                          None, ws4)
            e[1].record(stream)
            torch.cuda.synchronize()
            tms.append(e[0].elapsed_time(e[1]))
        knn_mpts = 4.0 / (statistics.median(tms) / 1000.0)
        knn4_ms = statistics.median(tms)
        del c4, ws4

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0
    hbm, _, peak_kind = peaks()
    iters = max(1, st["iters"])
    mean_stage = stage.mean(0)
    names = ["A1 backproject", "A2-A4 hash+kNN-cov (+seed pass on a side stream)",
             "A6-A9 align (init+persistent GN kernel)"]
    # dominant kernel of the step, timed live (kernel timer events inside the replayed graph)
    kms = {k: float(np.mean([x for x in v if x is not None])) if any(x is not None for x in v) else None
           for k, v in kt.items()}
    cand = {"k_knn_image": (kms[g.KT_KNN_SEARCH], ALGO_BYTES_KNN * n_src),
            "k_align": (kms[g.KT_ALIGN], ALGO_BYTES_ALIGN * n_src * iters)}
    kernel = max((k for k in cand if cand[k][0] is not None), key=lambda k: cand[k][0])
    kernel_ms, algo = cand[kernel]
    achieved = algo / (kernel_ms / 1000.0) / 1e9
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        tj = json.load(open(prof))
        traffic = tj.get(kernel)
        fresh = tj.get("_csrc_sha") == csrc_sha()
        traffic_src = {"file": "profiles/ncu_traffic.json", "capture": tj.get("_capture"),
                       "same_cuda_sources": fresh,
                       "note": "ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel"
                               + ("" if fresh else "; STALE: measured on other CUDA sources")}
    line = {
        "metric": METRIC, "value": value, "unit": "aligns/s", "n_gpus": ws, "steps": nev, "warmup": args.warmup,
        "ms_per_step": total_ms / nev, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 storage + f64 math", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_src": n_src, "map_gaussians": tgt.M, "k": 20, "mode": "ellipse",
                   "max_iters": 30, "gn_iters_used": st["iters"], "max_corr_dist": 0.1, "parallelism": f"replicas{ws}",
                   "rank_workload_seeds": [2 + 100 * r for r in range(ws)],
                   "collectives_in_timed_region": watch.count,
                   "l2": "flushed between timed steps (256 MB write)"},
        "timing": "CUDA graph replay of the whole frame, CUDA events per step on the launch stream",
        "ms_p10_p50_p90": [pct(step_ms, 10), pct(step_ms, 50), pct(step_ms, 90)],
        "repeat_bitwise": repeat_bitwise,
        "stage_ms_eager": {names[j]: float(mean_stage[j]) for j in range(3)},
        "kernel_ms": {"k_knn_image (11x11 window tile)": kms[g.KT_KNN_SEARCH], "k_align": kms[g.KT_ALIGN],
                      "seed pass (k_align_seed + k_align_seed_hard, side stream)": kms[g.KT_SEED],
                      "A1 (k_bp_count + k_bp_emit)": kms[g.KT_BP],
                      "A2-A4 gsicp_covariances_image, main-stream span": kms[g.KT_COVS],
                      "wide window + brute force + hash_n": kms[g.KT_WIDE],
                      "hash join + search + epilogue": kms[g.KT_TAIL]},
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src, "peak_kind": peak_kind,
                     "algo_bytes_per_launch": algo, "kernel_ms": kernel_ms},
        "e2e": {"value": e2e_value, "unit": "aligns/s", "h2d_bytes_per_step": int(tr.upload_bytes() + 16 * 8),
                "d2h_bytes_per_step": 16 * 8 + 32,
                "path": "Tracker.track_host_stream: per frame H2D of the sampled depth rows (copy stream, double "
                        "buffered) + pose, graph replay, D2H of pose + stats; wall clock over all frames",
                "l2": "flushed once before the stream of frames (not between frames)"},
        "gpu_launches": int(launches),  # captured per frame (conditional-body kernels excluded) x steps
        "clocks": clk.summary(),
        "fitness": st["fitness"], "status": st["status"],
    }
    line.update(configs_lines)
    if seq_line is not None:
        line["sequence"] = seq_line
    if batch_line is not None:
        line["batched"] = batch_line
    if knn_mpts is not None:
        line["knn_cov_mpts_s"] = knn_mpts
        line["knn_cov_4M_ms"] = knn4_ms
        line["knn_cov_hbm_frac"] = ALGO_BYTES_KNN * 4e6 / (knn4_ms / 1000) / 1e9 / hbm
    if not args.no_cpu_baseline and ws == 1:  # rank 0 at N=1 only
        line["cpu_baseline"] = cpu_baseline(w)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--seq-frames", type=int, default=120, help="C5 sequence frames per rank (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch", type=int, default=8, help="N2 frames per batched step (0: skip)")
    ap.add_argument("--no-configs", dest="configs", action="store_false", help="skip the C2 / C3 objects")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)
    return bench_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
