"""Diagnostic: f32 backward vs the oracle on one perturbed scene (per group
error, drop-in path), to separate accumulation precision from determinism."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2511_22793_b200 import GaussianCloud, ViewPose
from paper_2511_22793_b200 import rasterizer as R
for n, seed in [(1500, 5), (2000, 3), (800, 5)]:
    oc = O.round_f32(O.perturbed_scene(n, seed=seed))
    cloud = GaussianCloud(oc.positions, oc.log_scales, oc.rotations, oc.raw_opacities,
                          oc.mlp_weights, oc.mlp_dims)
    tx = O.sample_tx(11, 1)[0]
    pose = ViewPose(np.zeros(3))
    _, aux_ref = O.forward(oc, np.zeros(3), np.eye(3), tx, 180, 45)
    U = np.random.default_rng(3).normal(size=(45, 180, 2)).astype(np.float32).astype(np.float64)
    ref = O.backward(U, oc, tx, aux_ref)
    for dt in (np.float32, np.float64):
        img, aux = R.rasterize_forward(cloud, pose, tx, 180, 45, dtype=dt)
        flips = int((aux.contrib_count != aux_ref.contrib_count).sum())
        g = R.rasterize_backward(U, cloud, pose, tx, aux).arrays()
        err = {k: float(np.abs(g[k] - ref[k]).max() / max(np.abs(ref[k]).max(), 1e-30)) for k in O.GROUPS}
        worst = {k: int(np.argmax(np.abs(g[k] - ref[k]).reshape(len(g[k]), -1).max(1))) for k in O.GROUPS}
        print(n, seed, dt.__name__, 'flips', flips, {k: f"{v:.2e}" for k, v in err.items()}, worst)
