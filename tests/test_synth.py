"""Input generators (synth/): the C5 sequence constraints and the GPU ray caster's agreement with
the numpy one (CPU).  synth holds none of the method's arithmetic."""
import numpy as np

import synth


def test_sequence_generator_constraints():
    """C5 input generator: collision-free (>= 0.5 m), speed <= 0.5 m/s, view rate <= 30 deg/s at
    30 Hz, deterministic per seed; the torch ray caster equals the numpy one."""
    import math

    import torch

    for s in (0, 1, 7):
        sq = synth.make_sequence(s, 150, M=1000)
        assert min(synth._clearance(sq.scene, T[:3, 3]) for T in sq.T_gt) >= 0.5
        v = np.linalg.norm(np.diff(sq.T_gt[:, :3, 3], axis=0), axis=1) * 30.0
        assert v.max() <= 0.5 + 1e-9
        for a, b in zip(sq.T_gt[:-1], sq.T_gt[1:]):
            R = a[:3, :3].T @ b[:3, :3]
            assert math.degrees(math.acos(max(-1.0, min(1.0, (np.trace(R) - 1) / 2)))) * 30.0 <= 30.0 + 1e-9
        np.testing.assert_array_equal(sq.T_gt, synth.make_sequence(s, 150, M=1000).T_gt)
    K = synth.TINY
    sq = synth.make_sequence(3, 2, M=1000)
    d_np = synth.raycast_depth(sq.scene, K, sq.T_gt[1])
    d_t = synth.raycast_depth_torch(sq.scene, K, sq.T_gt[1], device="cpu").numpy()
    np.testing.assert_array_equal(d_np, d_t)
