"""Generate golden fixtures from the REAL reference package (`rfsplat`).

Run in the build container (where `/root/reference` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `rfsplat` read-only from /root/reference/pkg/src and writes
small `.npz` files next to this script.  The fixtures are committed; nothing
on the GPU box reads /root/reference.  Each case records the reference's
inputs (cloud arrays, pose, tx, image size) and outputs.
"""

import os
import sys
import types

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from rfsplat import geometry, image, mlp, optimize, rasterizer, rfsim, scene  # noqa: E402
from rfsplat.geometry import ViewPose, pixel_to_direction  # noqa: E402
from rfsplat.rasterizer import (rasterize_backward, rasterize_forward,  # noqa: E402
                                rasterize_reference)
from rfsplat.scene import GaussianCloud, SceneBounds, init_uniform  # noqa: E402

POSE = ViewPose(np.zeros(3))


def make_cloud(n, seed, spread=4.0, scale=0.3, mlp_scale=0.3,
               min_height=0.3, max_height=3.0):
    # identical recipe to /root/reference/pkg/tests/conftest.py:15-27
    rng = np.random.default_rng(seed)
    bounds = SceneBounds([-spread, min_height, -spread],
                         [spread, max_height, spread])
    cloud = init_uniform(bounds, n, seed=seed, init_scale=scale)
    cloud.mlp_weights *= mlp_scale
    cloud.raw_opacities[:] = rng.normal(0.0, 1.0, (n, 1))
    cloud.rotations += rng.normal(0.0, 0.3, (n, 4))
    cloud.log_scales += rng.normal(0.0, 0.4, (n, 3))
    return cloud


def single(position, b2=(0.8, -0.6), raw_opacity=0.0, log_scale=np.log(0.15)):
    # tests/test_rasterizer.py:14-22
    P = scene.mlp_param_count()
    w = np.zeros((1, P))
    w[0, -2:] = b2
    return GaussianCloud(np.asarray(position, float).reshape(1, 3),
                         np.full((1, 3), log_scale),
                         np.array([[1.0, 0.0, 0.0, 0.0]]),
                         np.full((1, 1), float(raw_opacity)), w)


def cloud_dict(c):
    return {"positions": c.positions, "log_scales": c.log_scales,
            "rotations": c.rotations, "raw_opacities": c.raw_opacities,
            "mlp_weights": c.mlp_weights,
            "mlp_dims": np.asarray(c.mlp_dims, np.int64)}


def tiles_flat(aux):
    """Per-tile SOURCE-index sequences, tiles in sorted (ty, tx) order."""
    keys = sorted(aux.tiles)
    ofs = [0]
    ids = []
    for k in keys:
        ids.extend(aux.prep.idx[aux.tiles[k]].tolist())
        ofs.append(len(ids))
    return {"tile_keys": np.asarray(keys, np.int64).reshape(-1, 2),
            "tile_offsets": np.asarray(ofs, np.int64),
            "tile_src": np.asarray(ids, np.int64)}


def prep_dict(p):
    return {"prep_idx": p.idx, "prep_depth": p.depth, "prep_mean2d": p.mean2d,
            "prep_conic": p.conic, "prep_radii": p.radii, "prep_opac": p.opac,
            "prep_s": p.s, "prep_d_tx": p.d_tx, "prep_J": p.J,
            "prep_cov2d": p.cov2d}


def save(name, **arrs):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrs)
    print(f"{name}: {os.path.getsize(path) / 1024:.0f} KiB")


def fwd_case(name, cloud, tx, w, h, dtype=np.float32, t_eps=rasterizer.T_EPS,
             with_ref=True, with_prep=False, dL_seed=None, pose=POSE):
    img, aux = rasterize_forward(cloud, pose, tx, w, h, dtype=dtype,
                                 t_eps=t_eps)
    out = dict(cloud_dict(cloud), tx=np.asarray(tx, float), w=w, h=h,
               dtype=np.dtype(dtype).name, t_eps=t_eps,
               rx=pose.rx_position, rotation=pose.rotation,
               img=img.data, T=aux.transmittance, count=aux.contrib_count,
               **tiles_flat(aux))
    if with_ref:
        out["ref"] = rasterize_reference(cloud, pose, tx, w, h).data
    if with_prep:
        out.update(prep_dict(aux.prep))
    if dL_seed is not None:
        U = np.random.default_rng(dL_seed).normal(size=(h, w, 2))
        g = rasterize_backward(U, cloud, pose, tx, aux)
        out["dL_seed"] = dL_seed
        out["dL_sum"] = U.sum()
        for k, v in g.arrays().items():
            out["grad_" + k] = v
    save(name, **out)


def dup_case():
    """Backward with a seam-duplicated Gaussian (rasterizer.py:139-141):
    the reference accumulates per tile with g[rows] += ..., so only the
    later copy's row survives (numpy last-write-wins).  Smallest seed whose
    perturbed 64-Gaussian cloud has a duplicate at 180 x 45."""
    tx = [0.3, 1.2, -0.8]
    for seed in range(100, 400):
        c = make_cloud(64, seed=seed)
        _, aux = rasterize_forward(c, POSE, tx, 180, 45)
        if any(len(set(r.tolist())) < len(r) for r in aux.tiles.values()):
            print(f"bwd_dup: seed {seed}")
            fwd_case("bwd_dup", c, tx, 180, 45, with_ref=False, dL_seed=23)
            return
    raise RuntimeError("no seam duplicate found")


def rfsim_case():
    """Ground truth, RSSI, RFSI bytes and a tiny gen_dataset from the real
    rfsim / image modules (rfsim.py:65-256, image.py:64-86)."""
    import tempfile
    sc = rfsim.random_scene(11, 6)
    txs = rfsim._sample_tx_positions(np.random.Generator(np.random.PCG64(7)),
                                     4, [-4, 0, -4], [4, 2, 4], sc.rx_position,
                                     1.0)
    w, h = 40, 12
    gt = np.stack([rfsim.ground_truth_spectrum(sc, t, w, h).data[:, :, 0]
                   for t in txs])
    gt_scaled = rfsim.ground_truth_spectrum(sc, txs[0], w, h, scale=2.5).data
    em = np.array([[*e.position, e.gain.real, e.gain.imag, e.angular_spread]
                   for e in sc.emitters])
    rng = np.random.default_rng(5)
    img2 = rng.normal(size=(h, w, 2)).astype(np.float32)
    img1 = np.abs(rng.normal(size=(h, w, 1))).astype(np.float32)
    rssi = np.array([
        rfsim.rssi_from_spectrum(image.SpectrumImage(img2), 0.3, 5),
        rfsim.rssi_from_spectrum(image.SpectrumImage(img2), 1.0, 2, 3.5),
        rfsim.rssi_from_spectrum(image.SpectrumImage(img1), 0.05, 9),
        rfsim.rssi_from_spectrum(image.SpectrumImage(np.zeros((h, w, 1))), 0.5, 1)])
    sel = rfsim._select_pixels(np.random.Generator(np.random.PCG64(5)), w, h, 0.3)
    with tempfile.TemporaryDirectory() as td:
        image.save_rfsi(os.path.join(td, "x.rfsi"), image.SpectrumImage(img2))
        rfsi_bytes = np.frombuffer(open(os.path.join(td, "x.rfsi"), "rb").read(),
                                   np.uint8)
        idx = rfsim.gen_dataset(3, 3, sc, 24, 8, td)
        files = sorted(f for f in os.listdir(td) if f.startswith("sample_"))
        ds = {f"ds_{f[:-5]}": np.frombuffer(open(os.path.join(td, f), "rb").read(),
                                            np.uint8) for f in files}
        index_txt = open(idx).read()
        manifest_txt = open(os.path.join(td, "manifest.txt")).read()
    save("rfsim", emitters=em, rx=sc.rx_position, wavelength=sc.wavelength,
         txs=txs, w=w, h=h, gt=gt, gt_scaled=gt_scaled, img2=img2, img1=img1,
         rssi=rssi, sel=sel, rfsi_bytes=rfsi_bytes, index_txt=np.array(index_txt),
         manifest_txt=np.array(manifest_txt), **ds)


def rotation_matrix(axis, angle):
    """Proper rotation (Rodrigues) for the non-identity ViewPose cases."""
    a = np.asarray(axis, float) / np.linalg.norm(axis)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(angle) * K + (1 - np.cos(angle)) * K @ K


def pole_cloud():
    """Gaussians above the 89 degree pole clamp (geometry.py:98-113 and its
    derivative path 152-180) among an ordinary perturbed cloud: elevations
    89.1..89.9 degrees at several azimuths and distances, so the clamp branch
    runs in the forward Jacobian and in the backward H."""
    base = make_cloud(48, seed=41)
    els = np.deg2rad([89.1, 89.4, 89.7, 89.9, 89.8, 89.55, 89.5, 89.25])
    azs = np.deg2rad([0.0, 35.0, -120.0, 170.0, 60.0, 0.0, -45.0, 100.0])
    rs = np.array([1.5, 2.2, 1.8, 2.8, 2.0, 2.5, 1.2, 3.0])
    pos = np.stack([rs * np.cos(els) * np.sin(azs), rs * np.sin(els),
                    rs * np.cos(els) * np.cos(azs)], axis=1)
    rng = np.random.default_rng(42)
    n = len(rs)
    P = scene.mlp_param_count()
    pole = GaussianCloud(pos, np.log(0.12) + rng.normal(0, 0.3, (n, 3)),
                         np.array([1.0, 0, 0, 0]) + rng.normal(0, 0.3, (n, 4)),
                         rng.normal(0.5, 1.0, (n, 1)),
                         0.3 * rng.standard_normal((n, P)))
    return GaussianCloud(*[np.concatenate([getattr(pole, k), getattr(base, k)])
                           for k in ("positions", "log_scales", "rotations",
                                     "raw_opacities", "mlp_weights")])


def geometry_cases():
    """Pole clamp and a rotated, offset receiver pose (VERDICT r1 gaps a3/a6)."""
    pc = pole_cloud()
    fwd_case("pole", pc, [0.4, 0.3, -1.1], 360, 90, dL_seed=61)
    fwd_case("pole64", pc, [0.4, 0.3, -1.1], 180, 45, dtype=np.float64,
             dL_seed=62)
    rot = ViewPose([0.3, -0.2, 0.5],
                   rotation_matrix([0.3, 1.0, -0.4], 0.9))
    rc = make_cloud(96, seed=43)
    fwd_case("pose_rot", rc, [1.2, 0.6, -0.9], 360, 90, dL_seed=63, pose=rot)
    fwd_case("pose_rot64", rc, [1.2, 0.6, -0.9], 180, 45, dtype=np.float64,
             dL_seed=64, pose=rot)
    # rotated pose with Gaussians at the receiver-frame pole
    R = rotation_matrix([1.0, 0.2, 0.1], 0.35)
    rpos = ViewPose([0.1, 0.2, -0.3], R)
    pp = pole_cloud()
    # world position = rx + R^T p_view: the pole Gaussians stay at the pole
    pp.positions[:] = rpos.rx_position + pp.positions @ R
    fwd_case("pose_pole", pp, [0.2, 0.8, 0.9], 360, 90, dL_seed=65, pose=rpos)


def main():
    if sys.argv[1:] == ["--only", "rfsim"]:
        rfsim_case()
        return
    if sys.argv[1:] == ["--only", "bwd_dup"]:
        dup_case()
        return
    if sys.argv[1:] == ["--only", "geometry"]:
        geometry_cases()
        return
    dup_case()
    rfsim_case()
    geometry_cases()
    # --- known answers (tests/test_rasterizer.py:33-70)
    d = 2.0 * pixel_to_direction(18, 4, 36, 9)
    fwd_case("ka_single", single(d), [0.0, 0.0, 0.0], 36, 9)
    dd = pixel_to_direction(18, 4, 36, 9)
    far_near = GaussianCloud(
        *[np.concatenate([getattr(single(4.0 * dd, b2=(1.0, 0.0)), k),
                          getattr(single(2.0 * dd, b2=(1.0, 0.0)), k)])
          for k in ("positions", "log_scales", "rotations", "raw_opacities",
                    "mlp_weights")])
    fwd_case("ka_two", far_near, [0, 0, 0], 36, 9, dtype=np.float64)
    fwd_case("ka_clamp", single(d, b2=(1.0, 0.0), raw_opacity=50.0),
             [0, 0, 0], 36, 9, dtype=np.float64)
    fwd_case("ka_near", single(d, b2=(1.0, 0.0)), d, 36, 9, dtype=np.float64)

    # --- random scenes (tests/test_rasterizer.py:92-98)
    for k in range(3):
        c = make_cloud(96, seed=100 + k)
        tx = np.random.default_rng(k).uniform(-2, 2, 3)
        fwd_case(f"rand96_{k}", c, tx, 360, 90, with_prep=(k == 0),
                 dL_seed=500 + k)
    # f64, no early exit (tests/test_rasterizer.py:100-105)
    fwd_case("f64_noexit", make_cloud(64, seed=11), [1, 0.5, -1], 180, 45,
             dtype=np.float64, t_eps=0.0)
    # seam wrap (tests/test_rasterizer.py:114-123)
    ds = 2.0 * pixel_to_direction(0, 10, 360, 90)
    fwd_case("seam", single(ds, b2=(1.0, 0.0), log_scale=np.log(0.3)),
             [0, 0, 0], 360, 90, dtype=np.float64, t_eps=0.0)
    # seam duplicate quirk (rasterizer.py:139-141): search a scale whose
    # wrapped span makes the two column segments overlap
    dq = 1.0 * pixel_to_direction(355, 10, 360, 90)
    lo_ls, hi_ls = np.log(0.5), np.log(1.2)
    for _ in range(60):  # bisect the log-scale to rx = 179.25 px
        ls = 0.5 * (lo_ls + hi_ls)
        c = single(dq, b2=(1.0, 0.0), log_scale=ls)
        prep = rasterizer._Prepared(c, POSE, [1.5, 0.5, 1.0], 360, 90)
        if prep.radii[0, 0] < 179.25:
            lo_ls = ls
        else:
            hi_ls = ls
    _, aux = rasterize_forward(c, POSE, [1.5, 0.5, 1.0], 360, 90)
    if not any(len(v) > 1 for v in aux.tiles.values()):
        raise RuntimeError("duplicate-quirk scene did not reproduce")
    fwd_case("seam_dup", c, [1.5, 0.5, 1.0], 360, 90)
    # backward FD scene (tests/test_rasterizer.py:158-172), f64 forward
    fwd_case("bwd4", make_cloud(4, seed=16), [0.5, 0.2, -0.3], 24, 9,
             dtype=np.float64, with_ref=False, dL_seed=17)
    # bigger backward on an f32 forward
    fwd_case("bwd64", make_cloud(64, seed=21), [0.3, 1.2, -0.8], 180, 45,
             with_ref=False, dL_seed=22)

    # --- reference bench scene (cli.py:239-246), GSPC-rounded
    bc = init_uniform(SceneBounds([-5, -0.2, -5], [5, 3.2, 5]), 512, seed=0)
    bc.mlp_weights *= 0.3
    tmp = os.path.join("/tmp", "golden_bench.gspc")
    scene.save_checkpoint(tmp, bc)
    bc = scene.load_checkpoint(tmp)
    fwd_case("bench512", bc, [2.0, 1.0, 2.0], 360, 90, with_prep=True,
             dL_seed=9)

    # --- multi-channel (F=2) by linearity: two 5->16->2 clouds sharing
    # W1/b1 whose heads are row pairs of a 5->16->4 head
    dims4 = (5, 16, 4)
    c4 = init_uniform(SceneBounds([-4, 0.3, -4], [4, 3, 4]), 80, seed=5,
                      init_scale=0.3, mlp_dims=dims4)
    c4.mlp_weights *= 0.3
    W1, b1, W2, b2 = mlp.split_weights(c4.mlp_weights, dims4)
    tx = np.array([1.0, 0.7, -1.5])
    imgs, refs = [], []
    for f in range(2):
        w2 = W2[:, 2 * f:2 * f + 2, :].reshape(80, -1)
        wf = np.concatenate([W1.reshape(80, -1), b1, w2, b2[:, 2 * f:2 * f + 2]],
                            axis=1)
        cf = GaussianCloud(c4.positions, c4.log_scales, c4.rotations,
                           c4.raw_opacities, wf)
        im, _ = rasterize_forward(cf, POSE, tx, 180, 45, dtype=np.float64,
                                  t_eps=0.0)
        imgs.append(im.data)
        refs.append(rasterize_reference(cf, POSE, tx, 180, 45).data)
    save("csi_f2", **cloud_dict(c4), tx=tx, w=180, h=45,
         img=np.concatenate(imgs, axis=2), ref=np.concatenate(refs, axis=2))

    # --- image / loss / adam
    rng = np.random.default_rng(3)
    pred = rng.random((45, 90))
    gt = rng.random((45, 90))
    loss, g = optimize.combined_loss(pred, gt, 0.2)
    z = rng.normal(size=(9, 12, 2))
    z[0, 0] = 0.0
    gm = rng.normal(size=(9, 12))
    p3 = rng.random((20, 30, 2))
    g3 = rng.random((20, 30, 2))
    loss3, grad3 = optimize.combined_loss(p3, g3, 0.2)
    save("loss", pred=pred, gt=gt, loss=loss, grad=g,
         ssim=optimize.ssim(pred, gt), psnr=optimize.psnr(pred, gt),
         z=z, mag=image.magnitude(image.SpectrumImage(z)).data,
         gmag=gm, mag_grad=image.magnitude_backward(image.SpectrumImage(z), gm),
         p3=p3, g3=g3, loss3=loss3, grad3=grad3)

    ca = make_cloud(6, seed=31)
    cfg = optimize.TrainConfig()
    st = optimize.AdamState(ca)
    start = {k: v.copy() for k, v in ca.param_arrays().items()}
    grads_seq = []
    for step in range(3):
        gr = rasterizer.ParamGradients(**{
            k: rng.normal(size=v.shape) for k, v in ca.param_arrays().items()})
        grads_seq.append(gr.arrays())
        optimize.adam_step(ca, gr, st, step, cfg)
    out = {f"start_{k}": v for k, v in start.items()}
    out.update({f"end_{k}": v for k, v in ca.param_arrays().items()})
    for s, ga in enumerate(grads_seq):
        out.update({f"g{s}_{k}": v for k, v in ga.items()})
    out["position_lr"] = np.array([optimize.position_lr(s, cfg)
                                   for s in (0, 1, 50, 150, 299, 300, 1000,
                                             15000, 29999, 30000, 40000)])
    save("adam", **out)

    # --- seeded generators
    txs = rfsim._sample_tx_positions(np.random.Generator(np.random.PCG64(3)),
                                     16, [-4, 0, -4], [4, 2, 4],
                                     np.zeros(3), 1.0)
    save("generators", tx_samples=txs, **{"bench_" + k: v for k, v in
                                          cloud_dict(bc).items()})


if __name__ == "__main__":
    main()
