"""GPU parity of the training glue: K7 loss (magnitude + L1 + SSIM with the
exact adjoint) and K8 Adam against the real reference's golden values and
the oracle, plus the batched device train step against the oracle's
loop-and-sum.  Mirrors /root/reference/pkg/tests/test_optimize.py."""

import numpy as np
import pytest

import oracle as O
from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def OPT():
    from paper_2511_22793_b200 import optimize
    return optimize


def test_combined_loss_matches_reference(OPT):
    fx = golden("loss")
    loss, g = OPT.combined_loss(fx["pred"], fx["gt"], 0.2)
    assert abs(loss - float(fx["loss"])) <= 1e-12
    assert np.abs(g - fx["grad"]).max() <= 1e-12 * np.abs(fx["grad"]).max()
    assert abs(OPT.ssim(fx["pred"], fx["gt"]) - float(fx["ssim"])) <= 1e-12
    assert abs(OPT.psnr(fx["pred"], fx["gt"]) - float(fx["psnr"])) <= 1e-9
    l3, g3 = OPT.combined_loss(fx["p3"], fx["g3"], 0.2)
    assert abs(l3 - float(fx["loss3"])) <= 1e-12
    assert np.abs(g3 - fx["grad3"]).max() <= 1e-12 * np.abs(fx["grad3"]).max()


def test_magnitude_chain(OPT):
    """K7's fused magnitude backward equals image.magnitude_backward
    composed with combined_loss (image.py:54-61)."""
    import torch
    from paper_2511_22793_b200.engine import LossWorkspace
    rng = np.random.default_rng(8)
    img = rng.normal(size=(2, 20, 30, 2)) * 0.3
    img[0, 0, 0] = 0.0
    gt = rng.random((2, 20, 30, 1)) * 0.5
    ws = LossWorkspace(2, 20, 30, 2, "cuda", dtype=torch.float64)
    dimg, stats = ws.run(torch.as_tensor(img, device="cuda"),
                         torch.as_tensor(gt, device="cuda"), 0, 0.2)
    dimg = dimg.cpu().numpy()
    for b in range(2):
        pred = O.magnitude(img[b])
        loss, gp = O.loss_and_grad(pred, gt[b], 0.2)
        want = O.magnitude_grad(img[b], gp[:, :, 0])
        assert abs(float(stats[b, 0]) - loss) <= 1e-12
        assert np.abs(dimg[b] - want).max() <= 1e-12 * np.abs(want).max()
        assert dimg[b, 0, 0].tolist() == [0.0, 0.0] if b == 0 else True


def test_adam_matches_reference(OPT):
    from paper_2511_22793_b200 import GaussianCloud
    fx = golden("adam")
    c = GaussianCloud(*(fx["start_" + k].copy() for k in O.GROUPS))
    cfg = OPT.TrainConfig()
    st = OPT.AdamState(c)
    for s in range(3):
        g = OPT.ParamGradients(**{k: fx[f"g{s}_{k}"] for k in O.GROUPS})
        OPT.adam_step(c, g, st, s, cfg)
    for k in O.GROUPS:
        ref = fx["end_" + k]
        tol = 1e-6 if k == "mlp_weights" else 1e-9
        assert np.abs(getattr(c, k) - ref).max() <= tol, k
    assert np.allclose(np.linalg.norm(c.rotations, axis=1), 1.0, atol=1e-12)


def test_adam_nonfinite_aborts(OPT):
    from paper_2511_22793_b200 import GaussianCloud
    oc = O.perturbed_scene(3, seed=2)
    c = GaussianCloud(*(getattr(oc, k).copy() for k in O.GROUPS))
    before = c.copy()
    g = OPT.ParamGradients.zeros_like(c)
    g.log_scales[1, 2] = np.inf
    with pytest.raises(FloatingPointError, match="log_scales"):
        OPT.adam_step(c, g, OPT.AdamState(c), 0, OPT.TrainConfig())
    for k in O.GROUPS:
        assert np.array_equal(getattr(c, k), getattr(before, k))


def test_position_lr(OPT):
    fx = golden("adam")
    cfg = OPT.TrainConfig()
    steps = (0, 1, 50, 150, 299, 300, 1000, 15000, 29999, 30000, 40000)
    got = np.array([OPT.position_lr(s, cfg) for s in steps])
    assert np.allclose(got, fx["position_lr"], rtol=1e-14, atol=0)


def _oracle_batch_step(oc, txs, gts, cfg, w, h, step=0):
    """Oracle: loop over TX, sum gradients, one Adam step."""
    total = {k: 0.0 for k in O.GROUPS}
    losses = []
    for tx, gt in zip(txs, gts):
        img, aux = O.forward(oc, np.zeros(3), np.eye(3), tx, w, h)
        pred = O.magnitude(img)
        loss, gp = O.loss_and_grad(pred, gt, cfg.lambda_dssim)
        losses.append(loss)
        g = O.backward(O.magnitude_grad(img, gp[:, :, 0]), oc, tx, aux)
        total = {k: total[k] + g[k] for k in O.GROUPS}
    m = {k: np.zeros_like(v) for k, v in oc.groups().items()}
    v = {k: np.zeros_like(a) for k, a in oc.groups().items()}
    nxt = oc.copy()
    O.adam_update(nxt, total, m, v, step, O.AdamCfg())
    return nxt, total, losses


def test_trainer_step_matches_oracle(OPT):
    from paper_2511_22793_b200 import GaussianCloud, ViewPose
    w, h, B = 90, 30, 4
    oc = O.round_f32(O.perturbed_scene(200, seed=7))
    txs = O.sample_tx(4, B)
    gts = np.random.default_rng(1).random((B, h, w, 1)) * 0.3
    cfg = OPT.TrainConfig(width=w, height=h, batch_tx=B)
    ref_next, ref_grad, ref_losses = _oracle_batch_step(oc, txs, gts, cfg,
                                                        w, h)
    cloud = GaussianCloud(*(getattr(oc, k).copy() for k in O.GROUPS))
    tr = OPT.Trainer(cloud, ViewPose(np.zeros(3)), cfg, txs, gts)
    stats = tr.step(np.arange(B)).cpu().numpy()
    assert tr.check()
    assert np.allclose(stats[:, 0], ref_losses, rtol=1e-5, atol=1e-7)
    grads = {k: v.double().cpu().numpy() for k, v in
             __import__("paper_2511_22793_b200.engine",
                        fromlist=["split_flat"]).split_flat(
                 tr.grad, tr.dev.n, tr.dev.P).items()}
    for k in O.GROUPS:
        err = np.abs(grads[k] - ref_grad[k]).max() / \
            max(np.abs(ref_grad[k]).max(), 1e-30)
        assert err <= 1e-4, (k, err)
    tr.sync_to_host(cloud)
    for k in O.GROUPS:
        d = np.abs(getattr(cloud, k) - getattr(ref_next, k)).max()
        assert d <= 1e-5, (k, d)


def test_trainer_graph_replay_equals_eager(OPT):
    import torch
    from paper_2511_22793_b200 import GaussianCloud, ViewPose
    w, h, B = 90, 30, 4
    oc = O.round_f32(O.perturbed_scene(150, seed=9))
    txs = O.sample_tx(8, 16)
    gts = np.random.default_rng(2).random((16, h, w, 1)) * 0.3
    cfg = OPT.TrainConfig(width=w, height=h, batch_tx=B)
    mk = lambda: GaussianCloud(*(getattr(oc, k).copy() for k in O.GROUPS))
    a = OPT.Trainer(mk(), ViewPose(np.zeros(3)), cfg, txs, gts)
    b = OPT.Trainer(mk(), ViewPose(np.zeros(3)), cfg, txs, gts)
    b.capture()
    batches = [[0, 1, 2, 3], [4, 5, 6, 7], [3, 9, 12, 15]]
    for bt in batches:
        a.step(bt)
        b.step(bt)
    torch.cuda.synchronize()
    assert a.check() and b.check()
    for k in ("positions", "mlp_weights"):
        x = getattr(a.dev, k).double().cpu().numpy()
        y = getattr(b.dev, k).double().cpu().numpy()
        assert np.abs(x - y).max() <= 1e-5 * max(1.0, np.abs(x).max())


def test_deterministic_training_is_bit_identical(OPT):
    """The reference's determinism contract (tests/test_acceptance.py:310-357:
    identical runs give bit-identical checkpoints and metrics): with
    TrainConfig(deterministic=True) the backward uses the fixed-order
    reduction and the loss statistics a fixed-order sum, so two runs (one
    eager, one CUDA-graph replay) agree bit for bit in every parameter and
    every reported loss."""
    import torch
    from paper_2511_22793_b200 import GaussianCloud, ViewPose
    w, h, B = 90, 30, 4
    oc = O.round_f32(O.perturbed_scene(400, seed=12))
    txs = O.sample_tx(13, 16)
    gts = np.random.default_rng(4).random((16, h, w, 1)) * 0.3
    cfg = OPT.TrainConfig(width=w, height=h, batch_tx=B, deterministic=True)
    mk = lambda: GaussianCloud(*(getattr(oc, k).copy() for k in O.GROUPS))
    runs = []
    for graph in (False, True):
        tr = OPT.Trainer(mk(), ViewPose(np.zeros(3)), cfg, txs, gts)
        if graph:
            tr.capture()
        losses = [tr.step(bt).cpu().numpy().copy()
                  for bt in ([0, 1, 2, 3], [4, 5, 6, 7], [3, 9, 12, 15])]
        torch.cuda.synchronize()
        assert tr.check()
        runs.append((losses, {k: getattr(tr.dev, k).cpu().numpy().copy()
                              for k in O.GROUPS}))
    for la, lb in zip(runs[0][0], runs[1][0]):
        assert np.array_equal(la, lb)
    for k in O.GROUPS:
        assert np.array_equal(runs[0][1][k], runs[1][1][k]), k
