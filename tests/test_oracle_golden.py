"""Pin the CPU oracle (oracle/) against golden vectors produced by the real
reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import golden, golden_cloud, golden_dL, golden_pose

FWD_CASES = ["ka_single", "ka_two", "ka_clamp", "ka_near", "rand96_0",
             "rand96_1", "rand96_2", "f64_noexit", "seam", "seam_dup",
             "bwd4", "bwd64", "bench512", "bwd_dup", "pole", "pole64",
             "pose_rot", "pose_rot64", "pose_pole"]


def _tiles_src(aux):
    keys = sorted(aux.tiles)
    ids = [aux.prep.idx[aux.tiles[k]] for k in keys]
    ofs = np.concatenate([[0], np.cumsum([len(i) for i in ids])])
    return (np.asarray(keys, np.int64).reshape(-1, 2), ofs,
            np.concatenate(ids) if ids else np.zeros(0, np.int64))


@pytest.mark.parametrize("case", FWD_CASES)
def test_forward_matches_reference(case):
    fx = golden(case)
    cloud = golden_cloud(fx)
    RX, W = golden_pose(fx)
    dt = np.dtype(str(fx["dtype"])).type
    img, aux = O.forward(cloud, RX, W, fx["tx"], int(fx["w"]), int(fx["h"]),
                         dtype=dt, t_eps=float(fx["t_eps"]))
    # tile lists: bit-exact, per tile, in source indices
    keys, ofs, src = _tiles_src(aux)
    assert np.array_equal(keys, fx["tile_keys"])
    assert np.array_equal(ofs, fx["tile_offsets"])
    assert np.array_equal(src, fx["tile_src"])
    assert np.array_equal(aux.contrib_count, fx["count"])
    assert img.dtype == fx["img"].dtype
    # same algorithm, same numpy kernels: bit-exact in practice
    assert np.array_equal(aux.transmittance, fx["T"])
    tol = 1e-6 if dt == np.float32 else 1e-13
    scale = max(1.0, np.abs(fx["img"]).max())
    assert np.abs(img.astype(np.float64) - fx["img"]).max() <= tol * scale
    if "ref" in fx:
        ref = O.reference_render(cloud, RX, W, fx["tx"], int(fx["w"]),
                                 int(fx["h"]))
        assert np.abs(ref - fx["ref"]).max() <= 1e-13 * scale


@pytest.mark.parametrize("case", ["rand96_0", "bench512"])
def test_prepare_matches_reference(case):
    fx = golden(case)
    cloud = golden_cloud(fx)
    RX, W = golden_pose(fx)
    pr = O.prepare(cloud, RX, W, fx["tx"], int(fx["w"]), int(fx["h"]))
    assert np.array_equal(pr.idx, fx["prep_idx"])
    assert np.array_equal(pr.depth, fx["prep_depth"])
    for k in ("mean2d", "conic", "radii", "opac", "s", "d_tx", "J", "cov2d"):
        ref = fx["prep_" + k]
        got = getattr(pr, k)
        assert np.allclose(got, ref, rtol=1e-13, atol=1e-13), k


RX, W = np.zeros(3), np.eye(3)
BWD_CASES = ["rand96_0", "rand96_1", "rand96_2", "bwd4", "bwd64",
             "bench512", "bwd_dup", "pole", "pole64", "pose_rot",
             "pose_rot64", "pose_pole"]


@pytest.mark.parametrize("case", BWD_CASES)
def test_backward_matches_reference(case):
    fx = golden(case)
    cloud = golden_cloud(fx)
    RX, W = golden_pose(fx)
    dt = np.dtype(str(fx["dtype"])).type
    _, aux = O.forward(cloud, RX, W, fx["tx"], int(fx["w"]), int(fx["h"]),
                       dtype=dt, t_eps=float(fx["t_eps"]))
    g = O.backward(golden_dL(fx), cloud, fx["tx"], aux)
    for k in O.GROUPS:
        ref = fx["grad_" + k]
        scale = max(np.abs(ref).max(), 1e-30)
        assert np.abs(g[k] - ref).max() <= 1e-10 * scale, k


def test_multichannel_by_linearity():
    fx = golden("csi_f2")
    cloud = golden_cloud(fx)
    w, h = int(fx["w"]), int(fx["h"])
    img, _ = O.forward(cloud, RX, W, fx["tx"], w, h, dtype=np.float64,
                       t_eps=0.0)
    assert img.shape == (h, w, 4)
    assert np.abs(img - fx["img"]).max() <= 1e-12
    ref = O.reference_render(cloud, RX, W, fx["tx"], w, h)
    assert np.abs(ref - fx["ref"]).max() <= 1e-12


def test_loss_and_image_ops():
    fx = golden("loss")
    loss, g = O.loss_and_grad(fx["pred"], fx["gt"], 0.2)
    assert abs(loss - float(fx["loss"])) <= 1e-14
    assert np.abs(g - fx["grad"]).max() <= 1e-15
    assert abs(O.ssim(fx["pred"], fx["gt"]) - float(fx["ssim"])) <= 1e-14
    assert abs(O.psnr(fx["pred"], fx["gt"]) - float(fx["psnr"])) <= 1e-12
    assert np.array_equal(O.magnitude(fx["z"]), fx["mag"])
    assert np.abs(O.magnitude_grad(fx["z"], fx["gmag"]) - fx["mag_grad"]).max() <= 1e-15
    l3, g3 = O.loss_and_grad(fx["p3"], fx["g3"], 0.2)
    assert abs(l3 - float(fx["loss3"])) <= 1e-14
    assert np.abs(g3 - fx["grad3"]).max() <= 1e-15


def test_adam_matches_reference():
    fx = golden("adam")
    c = O.Cloud(*(fx["start_" + k].copy() for k in O.GROUPS))
    m = {k: np.zeros_like(v) for k, v in c.groups().items()}
    v = {k: np.zeros_like(a) for k, a in c.groups().items()}
    cfg = O.AdamCfg()
    for s in range(3):
        O.adam_update(c, {k: fx[f"g{s}_{k}"] for k in O.GROUPS}, m, v, s, cfg)
    for k in O.GROUPS:
        assert np.abs(c.groups()[k] - fx["end_" + k]).max() <= 1e-14, k
    steps = (0, 1, 50, 150, 299, 300, 1000, 15000, 29999, 30000, 40000)
    got = np.array([O.position_lr(s, cfg) for s in steps])
    assert np.array_equal(got, fx["position_lr"])


def test_generators_match_reference():
    fx = golden("generators")
    assert np.array_equal(O.sample_tx(3, 16), fx["tx_samples"])
    b = O.bench_scene(512)
    ref = golden_cloud(fx, "bench_")
    for k in O.GROUPS:
        assert np.array_equal(getattr(b, k), getattr(ref, k)), k


def test_nonfinite_gradient_raises():
    g = O.zero_grads(O.make_uniform([-1, 0, -1], [1, 1, 1], 3, 0))
    O.check_finite(g)
    g["positions"][0, 0] = np.nan
    with pytest.raises(FloatingPointError, match="positions"):
        O.check_finite(g)
