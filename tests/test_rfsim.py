"""Dataset side of the path: RFSI I/O, ground-truth
spectra (K9), RSSI (K10) and batched evaluation.

CPU tests pin the oracle restatements and the host-side product code (RNG
recipes, wire formats, manifests) against fixtures written by the real
reference (tests/golden/make_golden.py, case "rfsim").  GPU tests compare
the kernels with the oracle and the fixtures."""

import os

import numpy as np
import pytest

import oracle as O
from conftest import golden

FX = golden("rfsim")


def _emitters():
    return [(e[:3], complex(e[3], e[4]), e[5]) for e in FX["emitters"]]


def _scene():
    from paper_2511_22793_b200 import rfsim
    return rfsim.MultipathScene(
        [rfsim.Emitter(e[:3], complex(e[3], e[4]), float(e[5]))
         for e in FX["emitters"]], FX["rx"], float(FX["wavelength"]))


def _write_golden_dataset(d):
    with open(os.path.join(d, "index.csv"), "w", newline="") as f:
        f.write(str(FX["index_txt"]))
    with open(os.path.join(d, "manifest.txt"), "w") as f:
        f.write(str(FX["manifest_txt"]))
    for k, v in FX.items():
        if k.startswith("ds_"):
            with open(os.path.join(d, k[3:] + ".rfsi"), "wb") as f:
                f.write(v.tobytes())


# ------------------------------------------------------------- CPU: oracle
def test_oracle_ground_truth_matches_reference():
    w, h = int(FX["w"]), int(FX["h"])
    for b, tx in enumerate(FX["txs"]):
        g = O.ground_truth(_emitters(), FX["rx"], float(FX["wavelength"]), tx, w, h)
        np.testing.assert_array_equal(g, FX["gt"][b])
    g = O.ground_truth(_emitters(), FX["rx"], float(FX["wavelength"]), FX["txs"][0],
                       w, h, scale=2.5)
    np.testing.assert_array_equal(g, FX["gt_scaled"][:, :, 0])


def test_oracle_rssi_matches_reference():
    r = FX["rssi"]
    assert O.rssi(FX["img2"], 0.3, 5) == r[0]
    assert O.rssi(FX["img2"], 1.0, 2, 3.5) == r[1]
    assert O.rssi(FX["img1"], 0.05, 9) == r[2]
    assert O.rssi(np.zeros((int(FX["h"]), int(FX["w"]), 1)), 0.5, 1) == r[3] == -100.0
    np.testing.assert_array_equal(O.select_pixels(5, int(FX["w"]), int(FX["h"]), 0.3),
                                  FX["sel"])


def test_oracle_rfsi_bytes(tmp_path):
    p = tmp_path / "x.rfsi"
    O.write_rfsi(p, FX["img2"])
    assert p.read_bytes() == FX["rfsi_bytes"].tobytes()
    np.testing.assert_array_equal(O.read_rfsi(p), FX["img2"])


# ----------------------------------------------- CPU: host-side product code
def test_product_rfsi_roundtrip_is_byte_compatible(tmp_path):
    from paper_2511_22793_b200 import image
    p = tmp_path / "a.rfsi"
    image.save_rfsi(p, image.SpectrumImage(FX["img2"]))
    assert p.read_bytes() == FX["rfsi_bytes"].tobytes()
    back = image.load_rfsi(p)
    np.testing.assert_array_equal(back.data, FX["img2"])
    # batched loader (pinned buffer when CUDA exists) and writer
    import torch
    t = image.load_rfsi_batch([p, p], device="cpu")
    assert t.shape == (2,) + FX["img2"].shape and t.dtype == torch.float32
    np.testing.assert_array_equal(t[1].numpy(), FX["img2"])
    q = [tmp_path / "b0.rfsi", tmp_path / "b1.rfsi"]
    image.save_rfsi_batch(q, t)
    assert q[1].read_bytes() == FX["rfsi_bytes"].tobytes()


def test_product_rfsi_errors(tmp_path):
    from paper_2511_22793_b200 import image
    bad = tmp_path / "bad.rfsi"
    bad.write_bytes(b"XXXX" + bytes(16))
    with pytest.raises(ValueError, match="bad magic"):
        image.load_rfsi(bad)
    ver = tmp_path / "ver.rfsi"
    ver.write_bytes(FX["rfsi_bytes"].tobytes()[:4] + (2).to_bytes(4, "little")
                    + FX["rfsi_bytes"].tobytes()[8:])
    with pytest.raises(ValueError, match="unsupported RFSI version"):
        image.load_rfsi(ver)
    tr = tmp_path / "tr.rfsi"
    tr.write_bytes(FX["rfsi_bytes"].tobytes()[:-4])
    with pytest.raises(ValueError, match="truncated RFSI payload"):
        image.load_rfsi(tr)


def test_product_scene_and_samplers_match_reference():
    from paper_2511_22793_b200 import rfsim
    sc = rfsim.random_scene(11, 6)
    em = np.array([[*e.position, e.gain.real, e.gain.imag, e.angular_spread]
                   for e in sc.emitters])
    np.testing.assert_array_equal(em, FX["emitters"])
    txs = rfsim._sample_tx_positions(np.random.Generator(np.random.PCG64(7)), 4,
                                     [-4, 0, -4], [4, 2, 4], sc.rx_position, 1.0)
    np.testing.assert_array_equal(txs, FX["txs"])
    np.testing.assert_array_equal(
        rfsim._select_pixels(np.random.Generator(np.random.PCG64(5)),
                             int(FX["w"]), int(FX["h"]), 0.3), FX["sel"])
    with pytest.raises(ValueError, match="angular_spread"):
        rfsim.Emitter([0, 1, 0], 1.0, 0.0)
    with pytest.raises(ValueError, match="at least one emitter"):
        rfsim.MultipathScene([], [0, 0, 0])


def test_product_manifest_and_dataset_loading(tmp_path):
    from paper_2511_22793_b200 import rfsim
    _write_golden_dataset(tmp_path)
    m = rfsim.read_manifest(tmp_path / "manifest.txt")
    sc = rfsim.scene_from_manifest(m)
    assert len(sc.emitters) == 6 and int(m["n_samples"]) == 3
    ds = rfsim.load_dataset(tmp_path / "index.csv")
    assert [s.id for s in ds] == ["00000", "00001", "00002"]
    assert ds[0].spectrum.data.shape == (8, 24, 1)
    with pytest.raises(FileNotFoundError, match="dataset index not found"):
        rfsim.load_dataset(tmp_path / "nope.csv")


def test_eval_csv_format(tmp_path):
    from paper_2511_22793_b200 import evaluate
    rows = [{"id": "00000", "ssim": 0.5, "mse": 0.25, "psnr": 6.020599913279624},
            {"id": "00001", "ssim": 0.75, "mse": 0.0, "psnr": float("inf")}]
    evaluate.write_eval_csv(rows, tmp_path)
    assert (tmp_path / "eval_per_sample.csv").read_text().splitlines() == [
        "id,ssim,mse,psnr", "00000,0.5,0.25,6.0206", "00001,0.75,0,inf"]
    assert (tmp_path / "eval_summary.csv").read_text().splitlines()[0] == \
        "metric,mean,median"


# -------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_gpu_ground_truth_matches_reference():
    from paper_2511_22793_b200 import rfsim
    w, h = int(FX["w"]), int(FX["h"])
    g = rfsim.ground_truth_batch(_scene(), FX["txs"], w, h).cpu().numpy()
    # f64 with CUDA's acos/exp/sincos and a fixed 3-term dot (the reference
    # uses a BLAS dgemv): ulp-level differences only
    np.testing.assert_allclose(g, FX["gt"], rtol=1e-12, atol=1e-15)
    s = rfsim.ground_truth_spectrum(_scene(), FX["txs"][0], w, h, scale=2.5)
    np.testing.assert_allclose(s.data, FX["gt_scaled"], rtol=1e-12, atol=1e-15)
    g32 = rfsim.ground_truth_batch(_scene(), FX["txs"], w, h,
                                   dtype=__import__("torch").float32).cpu().numpy()
    np.testing.assert_allclose(g32, FX["gt"].astype(np.float32), rtol=1e-6)


@pytest.mark.gpu
def test_gpu_gen_dataset_matches_reference(tmp_path):
    from paper_2511_22793_b200 import rfsim
    rfsim.gen_dataset(3, 3, _scene(), 24, 8, tmp_path, batch=2)
    assert (tmp_path / "index.csv").read_text() == str(FX["index_txt"])
    ref_m = dict(l.split("=", 1) for l in str(FX["manifest_txt"]).splitlines())
    got_m = rfsim.read_manifest(tmp_path / "manifest.txt")
    assert set(got_m) == set(ref_m)
    for k in ref_m:
        if k == "normalization":
            assert abs(float(got_m[k]) / float(ref_m[k]) - 1.0) < 1e-13
        else:
            assert got_m[k] == ref_m[k], k
    for k, v in FX.items():
        if k.startswith("ds_"):
            b = (tmp_path / (k[3:] + ".rfsi")).read_bytes()
            assert b[:20] == v.tobytes()[:20]
            got = np.frombuffer(b, "<f4", offset=20)
            ref = np.frombuffer(v.tobytes(), "<f4", offset=20)
            np.testing.assert_allclose(got, ref, rtol=2e-7, atol=0)


@pytest.mark.gpu
def test_gpu_rssi_matches_reference():
    import torch
    from paper_2511_22793_b200 import SpectrumImage, rfsim
    r = FX["rssi"]
    img2 = SpectrumImage(torch.as_tensor(FX["img2"], device="cuda"))
    assert abs(rfsim.rssi_from_spectrum(img2, 0.3, 5) - r[0]) < 1e-9
    assert abs(rfsim.rssi_from_spectrum(SpectrumImage(FX["img2"]), 1.0, 2, 3.5)
               - r[1]) < 1e-9
    assert abs(rfsim.rssi_from_spectrum(SpectrumImage(FX["img1"]), 0.05, 9)
               - r[2]) < 1e-9
    z = SpectrumImage(np.zeros((int(FX["h"]), int(FX["w"]), 1)))
    assert rfsim.rssi_from_spectrum(z, 0.5, 1) == -100.0
    batch = np.stack([FX["img2"], FX["img2"] * 2.0])
    got = rfsim.rssi_batch(batch, 0.3, 5)
    ref = [O.rssi(batch[0], 0.3, 5), O.rssi(batch[1], 0.3, 5)]
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-9)
    with pytest.raises(ValueError, match="fraction"):
        rfsim.rssi_from_spectrum(img2, 0.0, 1)


@pytest.mark.gpu
def test_gpu_rssi_estimate_batch_matches_oracle():
    from paper_2511_22793_b200 import ViewPose, rfsim
    from paper_2511_22793_b200.rasterizer import rasterize_forward
    fx = golden("rand96_0")
    from conftest import golden_cloud
    import paper_2511_22793_b200.scene as S
    c = golden_cloud(fx)
    cloud = S.GaussianCloud(c.positions, c.log_scales, c.rotations,
                            c.raw_opacities, c.mlp_weights)
    txs = np.array([fx["tx"], fx["tx"] + 0.3])
    w, h = int(fx["w"]), int(fx["h"])
    got = rfsim.rssi_estimate_batch(cloud, ViewPose(np.zeros(3)), txs, 0.4, 11,
                                    w=w, h=h)
    for b in range(2):
        img, _ = rasterize_forward(cloud, ViewPose(np.zeros(3)), txs[b], w, h)
        assert abs(got[b] - O.rssi(img.data, 0.4, 11)) < 1e-6
        assert abs(rfsim.rssi_estimate(cloud, ViewPose(np.zeros(3)), txs[b], 0.4,
                                       11, w=w, h=h) - got[b]) < 1e-6


@pytest.mark.gpu
def test_gpu_batched_eval_matches_oracle(tmp_path):
    import torch
    from paper_2511_22793_b200 import ViewPose, evaluate
    from paper_2511_22793_b200.rasterizer import rasterize_forward
    from conftest import golden_cloud
    import paper_2511_22793_b200.scene as S
    fx = golden("rand96_1")
    c = golden_cloud(fx)
    cloud = S.GaussianCloud(c.positions, c.log_scales, c.rotations,
                            c.raw_opacities, c.mlp_weights)
    w, h = int(fx["w"]), int(fx["h"])
    txs = np.array([fx["tx"], fx["tx"] * 0.5 + 0.2, fx["tx"] - 0.4])
    rng = np.random.default_rng(4)
    gt = rng.random((3, h, w, 1)).astype(np.float32)
    rows = evaluate.evaluate_arrays(cloud, ViewPose(np.zeros(3)),
                                    ["a", "b", "c"], txs, gt, w, h, batch=2)
    for b, r in enumerate(rows):
        img, _ = rasterize_forward(cloud, ViewPose(np.zeros(3)), txs[b], w, h)
        pred = O.magnitude(img.data.astype(np.float64))
        ref_ssim = O.ssim(pred[:, :, 0], gt[b, :, :, 0].astype(np.float64))
        ref_mse = float(np.mean((pred - gt[b].astype(np.float64)) ** 2))
        assert abs(r["ssim"] - ref_ssim) < 1e-9
        assert abs(r["mse"] - ref_mse) < 1e-12 * max(1.0, ref_mse)
        assert abs(r["psnr"] - 10 * np.log10(1 / ref_mse)) < 1e-8
    summary = evaluate.write_eval_csv(rows, tmp_path)
    assert [s["metric"] for s in summary] == ["ssim", "mse", "psnr"]
