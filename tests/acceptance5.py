"""Acceptance criterion 5 of the reference (end-to-end convergence,
/root/reference/pkg/tests/test_acceptance.py:209-259): 2,000 Gaussians,
5,000 iterations at 180x45 on a seed-fixed 160-sample dataset
(128 train / 32 held out, 5 emitters); pass iff the held-out median SSIM is
>= 0.85 and improves by >= 0.30 over the initial cloud.

Run as a script (in a subprocess, because mode `reference-loop` rebinds
`rfsplat.rasterizer`):

  python tests/acceptance5.py device          # paper_2511_22793_b200.optimize.train
  python tests/acceptance5.py reference-loop  # rfsplat.optimize.train (the
                                              # reference's own loop, loss and
                                              # NumPy Adam) over the drop-in

Prints one JSON line.  The dataset comes from the reference's generator in
`reference-loop` mode and from the drop-in's (byte-identical, see
tests/test_rfsim.py) in `device` mode.
"""

import json
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path[:0] = [ROOT, HERE, os.path.join(HERE, "refsuite")]

TRAIN_W, TRAIN_H = 180, 45
N_GAUSSIANS = 2000
TRAIN_ITERS = int(os.environ.get("ACCEPT5_ITERS", 5000))


def run(mode):
    if mode == "reference-loop":
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        import refsuite_plugin  # noqa: F401  (rebinds rfsplat.rasterizer)
        from rfsplat.geometry import ViewPose
        from rfsplat.optimize import TrainConfig, render_prediction, ssim, train
        from rfsplat.rfsim import gen_dataset, load_dataset, random_scene
        from rfsplat.scene import SceneBounds, init_uniform
    else:
        from paper_2511_22793_b200 import SceneBounds, ViewPose, init_uniform
        from paper_2511_22793_b200.optimize import (TrainConfig,
                                                    render_prediction, ssim,
                                                    train)
        from paper_2511_22793_b200.rfsim import (gen_dataset, load_dataset,
                                                 random_scene)
    out = tempfile.mkdtemp(prefix="accept5_")
    scene = random_scene(11, 5, spread_range=(0.3, 0.5))
    ds = load_dataset(gen_dataset(7, 160, scene, TRAIN_W, TRAIN_H, out))
    train_set, held_out = ds[:128], ds[128:]
    pose = ViewPose(np.zeros(3))
    bounds = SceneBounds([-5, -0.2, -5], [5, 3.2, 5])
    cloud = init_uniform(bounds, N_GAUSSIANS, seed=1)
    cfg = TrainConfig(iterations=TRAIN_ITERS, seed=3, width=TRAIN_W,
                      height=TRAIN_H)

    def heldout_ssims(c):
        vals = []
        for s in held_out:
            _, pred, _ = render_prediction(c, pose, s.tx_position, cfg)
            vals.append(ssim(pred.data[:, :, 0].astype(np.float64),
                             s.spectrum.data[:, :, 0].astype(np.float64)))
        return np.array(vals)

    init_median = float(np.median(heldout_ssims(cloud)))
    t0 = time.time()
    log = train(train_set, cfg, cloud, pose)
    secs = time.time() - t0
    final_median = float(np.median(heldout_ssims(cloud)))
    ok = final_median >= 0.85 and final_median - init_median >= 0.30
    return {"mode": mode, "ok": bool(ok), "init_median": init_median,
            "final_median": final_median,
            "improvement": final_median - init_median,
            "iterations": TRAIN_ITERS, "train_seconds": secs,
            "final_loss": float(log[-1]["loss"])}


if __name__ == "__main__":
    print(json.dumps(run(sys.argv[1] if len(sys.argv) > 1 else "device")))
