"""GPU parity at the BENCHMARKED sizes (BASELINE.json configs), against the
CPU oracle (pinned to the real reference by tests/test_oracle_golden.py).

* config 3: 50k Gaussians, 90x360 x 52 subcarriers, one TX, through the
  benchmarked lazy path (K2 -> K3 -> pass A -> live MLP -> tcgen05 pass B):
  tile lists bit-exact, image within 1e-4 normwise, flips counted;
* config 2: 16k Gaussians, 90x360, the batched train step (K2..K8): per-TX
  images, K7 loss on those images, and the summed gradient of the batch
  (deterministic reduction) against the oracle's loop-and-sum on the same
  upstream gradient (threshold-flip pixels masked, see
  test_gpu_backward.masked_dL);
* config 5: 500k Gaussians at 180x720 (full geometry, 2 subcarriers) and
  the full 256-subcarrier width on a reduced cloud;
* deterministic backward on a wide frame (720x180, a near-receiver Gaussian
  spanning more than 320 tile slots: round-1's silent truncation);
* pair-buffer overflow on the overlapped (programmatic-dependent) render
  path: grow-and-retry gives the same image.
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
from conftest import group_err

pytestmark = pytest.mark.gpu

RX, W = np.zeros(3), np.eye(3)
F32_TOL = 1e-4


def host_cloud(oc):
    from paper_2511_22793_b200 import GaussianCloud
    return GaussianCloud(oc.positions, oc.log_scales, oc.rotations,
                         oc.raw_opacities, oc.mlp_weights, oc.mlp_dims)


def normwise(a, b):
    return np.abs(np.asarray(a, np.float64) - b).max() / \
        max(np.abs(b).max(), 1e-30)


def image_parity(img, ref, cnt, ref_cnt, tol=F32_TOL):
    flip = cnt != ref_cnt
    ok = ~flip[..., None].repeat(img.shape[-1], axis=-1)
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(np.asarray(img, np.float64) - ref)
    e = err[ok].max(initial=0.0) / scale
    assert e <= tol, e
    assert flip.sum() <= max(4, flip.size // 5000), int(flip.sum())
    return e, int(flip.sum())


def tiles_equal(frame_or_aux, aux_ref):
    from paper_2511_22793_b200.rasterizer import RenderAux
    aux = frame_or_aux
    if not isinstance(aux, RenderAux):
        aux = RenderAux(frame_or_aux, None, None, None, 0, np.float32, 0, None)
    got = aux.tile_sources()
    want = {k: aux_ref.prep.idx[v] for k, v in aux_ref.tiles.items()}
    assert sorted(got) == sorted(want)
    for k in want:
        assert np.array_equal(got[k], want[k]), k
    return sum(len(v) for v in want.values())



def test_config3_full_size_forward():
    """BASELINE config 3 exactly as benched (bench.py --config c3)."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud, ViewPose
    from paper_2511_22793_b200.engine import Renderer
    oc = O.bench_scene(50000, F=52)
    tx = O.sample_tx(0, 1)
    ref, aux_ref = O.forward(oc, RX, W, tx[0], 360, 90,
                             threads=O.cpu_threads())
    dc = DeviceCloud.from_host(host_cloud(oc))
    R = Renderer()
    img, fr = R.forward(dc, ViewPose(np.zeros(3)),
                        torch.as_tensor(tx, device="cuda"), 360, 90, lazy=True)
    pairs = tiles_equal(fr, aux_ref)
    assert pairs == 496788
    e, flips = image_parity(img[0].cpu().numpy(), ref,
                            fr.contrib_count().cpu().numpy(),
                            aux_ref.contrib_count)
    print(f"config 3: {pairs} pairs bit-exact, image {e:.2e} normwise, "
          f"{flips} flips")


def test_config2_train_step_parity():
    """BASELINE config 2 (16k Gaussians, 90x360) train step, 8 TX."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud, ViewPose
    from paper_2511_22793_b200.engine import LossWorkspace, Renderer, split_flat
    w, h, B = 360, 90, 8
    oc = O.bench_scene(16000)
    txs = O.sample_tx(2, B)
    gts = (np.random.default_rng(3).random((B, h, w, 1)) * 0.05).astype(
        np.float32)
    dc = DeviceCloud.from_host(host_cloud(oc))
    pose = ViewPose(np.zeros(3))
    R = Renderer()
    txd = torch.as_tensor(txs, device="cuda")
    img, fr = R.forward(dc, pose, txd, w, h, with_backward=2, lazy=False)
    ws = LossWorkspace(B, h, w, 2, "cuda")
    gtd = torch.as_tensor(gts, device="cuda")
    dimg, stats = ws.run(img, gtd, 0, 0.2)
    img_n, dimg_n = img.cpu().numpy(), dimg.double().cpu().numpy()
    st = stats.cpu().numpy()

    def oracle_tx(b):
        ref, aux = O.forward(oc, RX, W, txs[b], w, h)
        return ref, aux

    with ThreadPoolExecutor(max_workers=min(B, O.cpu_threads())) as ex:
        fw = list(ex.map(oracle_tx, range(B)))
    # one image per TX: GPU image vs oracle, counting flips (alpha and T do
    # not depend on the TX, so the batch shares one contributor count)
    cnt = fr.contrib_count().cpu().numpy()
    flips = []
    for b in range(B):
        assert np.array_equal(fw[b][1].contrib_count, fw[0][1].contrib_count)
        image_parity(img_n[b], fw[b][0], cnt, fw[b][1].contrib_count)
        flips.append(cnt != fw[b][1].contrib_count)
        # K7 on the GPU image vs the oracle's loss of the same image
        loss, gp = O.loss_and_grad(O.magnitude(img_n[b].astype(np.float64)),
                                   gts[b].astype(np.float64), 0.2)
        assert abs(st[b, 0] - loss) <= 1e-9 * max(1.0, abs(loss))
        dz = O.magnitude_grad(img_n[b].astype(np.float64), gp[:, :, 0])
        assert np.abs(dz - dimg_n[b]).max() <= 1e-6 * np.abs(dz).max()
    # summed gradient of the batch on the same (flip-masked) upstream
    Um = np.stack([dimg_n[b] * ~flips[b][..., None] for b in range(B)])
    Ud = torch.as_tensor(Um, dtype=torch.float32, device="cuda")
    # deterministic (list walk) and atomic (compacted walk over the entries
    # each half tile used: raster_bwd_tc.cu) tensor-core backward
    gs = {det: split_flat(R.backward(dc, pose, txd, Ud, fr, deterministic=det),
                          dc.n, dc.P) for det in (True, False)}
    Uq = Um.astype(np.float32).astype(np.float64)  # what the GPU consumed

    def oracle_bwd(b):
        return O.backward(Uq[b], oc, txs[b], fw[b][1])

    with ThreadPoolExecutor(max_workers=min(B, O.cpu_threads())) as ex:
        gb = list(ex.map(oracle_bwd, range(B)))
    ref = {k: sum(x[k] for x in gb) for k in O.GROUPS}
    for det, g in gs.items():
        err = group_err({k: v.double().cpu().numpy() for k, v in g.items()}, ref)
        print(f"config 2 train step (deterministic={det}): grad errors {err}, "
              f"flips {[int(f.sum()) for f in flips]}")
        assert max(err.values()) <= 1e-4, (det, err)


@pytest.mark.parametrize("n,F,w,h", [(500000, 1, 720, 180),
                                     (8000, 256, 720, 180)])
def test_config5_geometry_and_width(n, F, w, h):
    """BASELINE config 5 (500k Gaussians, 180x720 x 256 subcarriers): the
    full geometry at 2 channels, and the full channel width on a smaller
    cloud (the full 17.6 GB cloud has no CPU oracle within test time)."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud, ViewPose
    from paper_2511_22793_b200.engine import Renderer
    oc = O.bench_scene(n, F=F)
    tx = O.sample_tx(5, 1)
    ref, aux_ref = O.forward(oc, RX, W, tx[0], w, h, threads=O.cpu_threads())
    dc = DeviceCloud.from_host(host_cloud(oc))
    img, fr = Renderer().forward(dc, ViewPose(np.zeros(3)),
                                 torch.as_tensor(tx, device="cuda"), w, h,
                                 lazy=True)
    pairs = tiles_equal(fr, aux_ref)
    e, flips = image_parity(img[0].cpu().numpy(), ref,
                            fr.contrib_count().cpu().numpy(),
                            aux_ref.contrib_count)
    print(f"config 5 slice n={n} F={F}: {pairs} pairs bit-exact, image "
          f"{e:.2e}, {flips} flips")


def test_deterministic_backward_wide_frame():
    """720x180 (540 tiles) with Gaussians next to the receiver whose
    footprints span the whole azimuth over several tile rows (> 320 tile
    slots each): the fixed-order reduction covers every slot."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud, ViewPose
    from paper_2511_22793_b200.engine import Renderer, split_flat
    w, h = 720, 180
    base = O.round_f32(O.perturbed_scene(600, seed=8))
    near = O.Cloud(np.array([[0.05, 0.35, 0.1], [-0.1, 0.5, -0.05]]),
                   np.log(np.full((2, 3), 0.45)),
                   np.array([[1.0, 0, 0, 0], [0.9, 0.1, 0.2, 0]]),
                   np.array([[-2.5], [-3.0]]),
                   0.3 * np.random.default_rng(1).standard_normal((2, 130)))
    oc = O.round_f32(O.Cloud(*[np.concatenate([getattr(near, k),
                                               getattr(base, k)])
                               for k in O.GROUPS]))
    tx = O.sample_tx(21, 1)
    _, aux_ref = O.forward(oc, RX, W, tx[0], w, h)
    spans = {}
    for key, rows in aux_ref.tiles.items():
        for r in rows:
            spans[aux_ref.prep.idx[r]] = spans.get(aux_ref.prep.idx[r], 0) + 1
    assert max(spans.get(0, 0), spans.get(1, 0)) > 320, spans.get(0)
    dc = DeviceCloud.from_host(host_cloud(oc))
    pose = ViewPose(np.zeros(3))
    R = Renderer()
    txd = torch.as_tensor(tx, device="cuda")
    img, fr = R.forward(dc, pose, txd, w, h, with_backward=2, lazy=False)
    U = np.random.default_rng(4).normal(size=(1, h, w, 2))
    flip = fr.contrib_count().cpu().numpy() != aux_ref.contrib_count
    U[0] *= ~flip[..., None]
    Ud = torch.as_tensor(U, dtype=torch.float32, device="cuda")
    det = split_flat(R.backward(dc, pose, txd, Ud, fr, deterministic=True),
                     dc.n, dc.P)
    ato = split_flat(R.backward(dc, pose, txd, Ud, fr, deterministic=False),
                     dc.n, dc.P)
    for k in O.GROUPS:
        a, b = det[k].double(), ato[k].double()
        assert (a - b).abs().max() <= 1e-5 * max(b.abs().max().item(), 1e-30), k
    ref = O.backward(U[0].astype(np.float32).astype(np.float64), oc, tx[0],
                     aux_ref)
    err = group_err({k: v.double().cpu().numpy() for k, v in det.items()}, ref)
    assert max(err.values()) <= 1e-4, err


@pytest.mark.parametrize("lazy", [True, False])
def test_pair_overflow_grow_and_retry(lazy):
    """A frame planned far too small overflows inside K2; on the overlapped
    render path pass A's CTAs are already resident while K2/K3 run and must
    see the overflow through K3's published queue and exit (ADVICE r1,
    raster_px.cu).  The engine then grows the frame and re-renders: the
    result equals a render into an ample frame, repeatedly."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud, ViewPose, _lib
    from paper_2511_22793_b200.engine import CapacityError, Renderer
    oc = O.bench_scene(6000, F=26)
    dc = DeviceCloud.from_host(host_cloud(oc))
    pose = ViewPose(np.zeros(3))
    tx = torch.as_tensor(O.sample_tx(3, 1), device="cuda")
    R = Renderer()
    good, _ = R.forward(dc, pose, tx, 360, 90, lazy=lazy)
    good = good.clone()
    for rep in range(5):
        small = R.new_frame(dc.n, 360, 90, 52, capacity=500 + 1000 * rep)
        img, fr = R.forward(dc, pose, tx, 360, 90, frame=small, lazy=lazy,
                            sync_check=False)
        torch.cuda.synchronize()
        with pytest.raises(CapacityError):
            R.check_frame(fr)
        big = R.grow(small, int(fr.counters().cpu()[_lib.CNT_PAIRS]))
        img2, fr2 = R.forward(dc, pose, tx, 360, 90, frame=big, lazy=lazy)
        assert torch.equal(img2, good)


def test_async_batch_render_deferred_check():
    """rasterize_forward_batch(sync=False), the serving-loop form the bench's
    e2e leg uses: no host sync per call; the RenderCheck read later reports
    an overflowed frame (so the image is never trusted silently), and a
    valid frame renders exactly what the synchronous call renders."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud, ViewPose
    from paper_2511_22793_b200.engine import CapacityError
    from paper_2511_22793_b200.rasterizer import (rasterize_forward_batch,
                                                  renderer)
    oc = O.bench_scene(6000, F=26)
    dc = DeviceCloud.from_host(host_cloud(oc))
    pose = ViewPose(np.zeros(3))
    txs = torch.as_tensor(O.sample_tx(4, 3), device="cuda")
    want, frame = rasterize_forward_batch(dc, pose, txs, 360, 90)
    want = want.clone()
    checks = []
    for _ in range(20):          # more than the pinned ring of 16 slots
        img, frame, chk = rasterize_forward_batch(dc, pose, txs, 360, 90,
                                                  frame=frame, sync=False)
        checks.append(chk)
    for chk in checks[-16:]:
        assert chk.ok()
    assert torch.equal(img, want)
    small = renderer().new_frame(dc.n, 360, 90, 3 * 52, capacity=1000)
    _, small, chk = rasterize_forward_batch(dc, pose, txs, 360, 90,
                                            frame=small, sync=False)
    assert not chk.ok()
    with pytest.raises(CapacityError):
        chk.raise_if_overflow()
    big = renderer().grow(small, chk.pairs_needed())
    img2, _ = rasterize_forward_batch(dc, pose, txs, 360, 90, frame=big)
    assert torch.equal(img2, want)
