"""Shared fixtures.  Tests needing a B200 are marked `@pytest.mark.gpu`."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers",
                            "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    """Load one fixture written by tests/golden/make_golden.py."""
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def golden_cloud(fx, prefix=""):
    from oracle import Cloud
    return Cloud(*(fx[prefix + k].astype(np.float64) for k in
                   ("positions", "log_scales", "rotations", "raw_opacities",
                    "mlp_weights")),
                 mlp_dims=tuple(int(v) for v in fx[prefix + "mlp_dims"]))


def golden_pose(fx):
    """(rx, W) of a fixture; cases written before poses were recorded use
    the receiver at the origin with W = I."""
    rx = np.asarray(fx["rx"], np.float64) if "rx" in fx else np.zeros(3)
    W = np.asarray(fx["rotation"], np.float64) if "rotation" in fx \
        else np.eye(3)
    return rx, W


def golden_dL(fx):
    h, w = int(fx["h"]), int(fx["w"])
    U = np.random.default_rng(int(fx["dL_seed"])).normal(size=(h, w, 2))
    assert np.isclose(U.sum(), float(fx["dL_sum"]), rtol=0, atol=1e-9)
    return U


@pytest.fixture
def origin():
    return np.zeros(3), np.eye(3)


GROUPS = ("positions", "log_scales", "rotations", "raw_opacities",
          "mlp_weights")


def group_err(g, ref):
    """Per-group normwise gradient error ||g - ref||_inf / ||ref||_inf.

    Rotations are normalised by max(||ref_rot||, ||ref_log_scales||): dL/dq
    and dL/dlog_s are both dL/dSigma contracted with Sigma-sized matrices
    (rasterizer.py:345-360), so they share a scale.  For an isotropic
    Gaussian Sigma = s^2 I does not depend on q and dL/dq is analytically 0
    -- the reference's own value is rounding noise (~1e-15 on the bench
    scene, whose Gaussians are all isotropic) and relative error against it
    is meaningless."""
    out = {}
    for k in GROUPS:
        scale = np.abs(ref[k]).max()
        if k == "rotations":
            scale = max(scale, np.abs(ref["log_scales"]).max())
        out[k] = np.abs(np.asarray(g[k]) - ref[k]).max() / max(scale, 1e-30)
    return out
