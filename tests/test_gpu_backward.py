"""GPU parity of the backward path (K5 raster backward + K6 per-Gaussian
chain) against the real reference's gradients (golden fixtures), the CPU
oracle and central finite differences.  Mirrors
/root/reference/pkg/tests/test_rasterizer.py:157-212.

Bar (north_star): per parameter group ||g_gpu - g_ref||_inf / ||g_ref||_inf
<= 1e-4 for the fp32 path; 1e-9 for the f64 verification path."""

import numpy as np
import pytest

import oracle as O
from conftest import golden, golden_cloud, golden_dL, golden_pose, group_err

pytestmark = pytest.mark.gpu

RX, W = np.zeros(3), np.eye(3)


@pytest.fixture(scope="module")
def R():
    from paper_2511_22793_b200 import rasterizer
    return rasterizer


@pytest.fixture(scope="module")
def pose():
    from paper_2511_22793_b200 import ViewPose
    return ViewPose(np.zeros(3))


def host_cloud(oc):
    from paper_2511_22793_b200 import GaussianCloud
    return GaussianCloud(oc.positions, oc.log_scales, oc.rotations,
                         oc.raw_opacities, oc.mlp_weights, oc.mlp_dims)



def masked_dL(U, flip):
    """dL with the threshold-flip pixels zeroed.  A flip (numpy's f32 exp vs
    the device's exp2 on an alpha within an ulp of 1/255) changes only its
    own pixel's terms, and with dL = 0 there that pixel contributes nothing
    to any gradient on either side, so the comparison covers exactly the
    same set of terms instead of being skipped."""
    return U * ~flip[..., None]


BWD_GOLD = ["rand96_0", "rand96_1", "rand96_2", "bwd4", "bwd64", "bench512",
            "bwd_dup", "pole", "pole64", "pose_rot", "pose_rot64", "pose_pole"]


@pytest.mark.parametrize("case", BWD_GOLD)
def test_backward_matches_golden(case, R):
    """Against the real reference's gradients.  Flip-free renders compare
    with the golden directly; with flips, dL is zeroed on the flipped pixels
    and the reference is the oracle's backward of that dL (the oracle is
    pinned to these goldens at 1e-10, tests/test_oracle_golden.py)."""
    from paper_2511_22793_b200 import ViewPose
    fx = golden(case)
    rx, rot = golden_pose(fx)
    pose = ViewPose(rx, rot)
    oc = golden_cloud(fx)
    cloud = host_cloud(oc)
    dt = np.dtype(str(fx["dtype"])).type
    w, h, t_eps = int(fx["w"]), int(fx["h"]), float(fx["t_eps"])
    img, aux = R.rasterize_forward(cloud, pose, fx["tx"], w, h, dtype=dt,
                                   t_eps=t_eps)
    flip = aux.contrib_count != fx["count"]
    U = golden_dL(fx)
    if flip.any():
        assert flip.sum() <= max(4, flip.size // 5000), int(flip.sum())
        U = masked_dL(U, flip)
        _, aux_ref = O.forward(oc, rx, rot, fx["tx"], w, h, dtype=dt,
                               t_eps=t_eps)
        assert np.array_equal(aux_ref.contrib_count, fx["count"])
        ref = O.backward(U, oc, fx["tx"], aux_ref)
    else:
        ref = {k: fx["grad_" + k] for k in O.GROUPS}
    g = R.rasterize_backward(U, cloud, pose, fx["tx"], aux)
    err = group_err(g.arrays(), ref)
    tol = 1e-4 if dt == np.float32 else 1e-9
    assert max(err.values()) <= tol, (err, int(flip.sum()))
    assert all(v.dtype == np.float64 for v in g.arrays().values())


def test_finite_differences_f64(R, pose):
    """tests/test_rasterizer.py:158-185 through the GPU f64 path."""
    w, h = 24, 9
    oc = O.perturbed_scene(4, seed=16)
    cloud = host_cloud(oc)
    tx = np.array([0.5, 0.2, -0.3])
    rng = np.random.default_rng(17)
    U = rng.normal(size=(h, w, 2))

    def loss(c):
        img, _ = R.rasterize_forward(c, pose, tx, w, h, dtype=np.float64)
        return float(np.sum(U * img.data))

    _, aux = R.rasterize_forward(cloud, pose, tx, w, h, dtype=np.float64)
    grads = R.rasterize_backward(U, cloud, pose, tx, aux)
    step = 1e-5
    for name, arr in cloud.param_arrays().items():
        g = grads.arrays()[name]
        for fi in rng.choice(arr.size, size=min(20, arr.size), replace=False):
            idx = np.unravel_index(fi, arr.shape)
            cp, cm = cloud.copy(), cloud.copy()
            cp.param_arrays()[name][idx] += step
            cm.param_arrays()[name][idx] -= step
            fd = (loss(cp) - loss(cm)) / (2 * step)
            assert abs(g[idx] - fd) <= 1e-4 * max(1.0, abs(fd)), \
                f"{name}{idx}: analytic {g[idx]:.3e} fd {fd:.3e}"


@pytest.mark.parametrize("n,F", [(2000, 1), (800, 3)])
def test_against_oracle(n, F, R, pose):
    oc = O.round_f32(O.perturbed_scene(n, seed=3, F=F))
    tx = O.sample_tx(11, 1)[0]
    _, aux_ref = O.forward(oc, RX, W, tx, 180, 45)
    U = np.random.default_rng(5).normal(size=(45, 180, 2 * F))
    ref = O.backward(U, oc, tx, aux_ref)
    img, aux = R.rasterize_forward(host_cloud(oc), pose, tx, 180, 45)
    flip = aux.contrib_count != aux_ref.contrib_count
    if flip.any():
        U = masked_dL(U, flip)
        ref = O.backward(U, oc, tx, aux_ref)
    g = R.rasterize_backward(U, host_cloud(oc), pose, tx, aux)
    err = group_err(g.arrays(), ref)
    assert max(err.values()) <= 1e-4, err


@pytest.mark.parametrize("scene,B", [("perturbed", 4), ("perturbed", 8),
                                     ("bwd_dup", 8), ("bwd_dup", 32)])
def test_batched_backward_is_sum_of_singles(scene, B, R, pose):
    """A batch of B TX (B*C columns: the tensor-core K5 from 16 columns) gives
    the sum of the single-TX backward passes (2 columns: the CUDA-core K5),
    including the reference's seam-duplicate rule (`bwd_dup`: a Gaussian
    listed twice in a tile, only the later copy counts)."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud
    from paper_2511_22793_b200.engine import split_flat
    if scene == "bwd_dup":
        fx = golden("bwd_dup")
        oc = golden_cloud(fx)
        assert (int(fx["w"]), int(fx["h"])) == (180, 45)
    else:
        oc = O.round_f32(O.perturbed_scene(300, seed=4))
    dc = DeviceCloud.from_host(host_cloud(oc))
    txs = O.sample_tx(3, B)
    U = np.random.default_rng(6).normal(size=(B, 45, 180, 2))
    _, frame = R.rasterize_forward_batch(dc, pose, txs, 180, 45,
                                         with_backward=True)
    dL = torch.as_tensor(U, dtype=torch.float32, device="cuda")
    flat = R.rasterize_backward_batch(dL, dc, pose, txs, frame)
    got = {k: v.double().cpu().numpy()
           for k, v in split_flat(flat, dc.n, dc.P).items()}
    want = {k: 0.0 for k in O.GROUPS}
    for b in range(B):
        _, aux = R.rasterize_forward(dc, pose, txs[b], 180, 45)
        g = R.rasterize_backward(U[b], dc, pose, txs[b], aux).arrays()
        want = {k: want[k] + g[k] for k in O.GROUPS}
    err = group_err(got, want)
    assert max(err.values()) <= 1e-5, err


def test_zero_upstream_and_aux_mismatch(R, pose):
    oc = O.perturbed_scene(6, seed=19)
    c = host_cloud(oc)
    _, aux = R.rasterize_forward(c, pose, [0, 0, 0], 36, 9)
    g = R.rasterize_backward(np.zeros((9, 36, 2)), c, pose, [0, 0, 0], aux)
    for arr in g.arrays().values():
        assert not arr.any()
    other = host_cloud(O.perturbed_scene(5, seed=18))
    with pytest.raises(ValueError):
        R.rasterize_backward(np.zeros((9, 36, 2)), other, pose, [0, 0, 0], aux)
    with pytest.raises(ValueError):
        R.rasterize_backward(np.zeros((9, 36, 2)), c, pose, [1, 0, 0], aux)


def test_check_finite(R):
    oc = O.perturbed_scene(2, seed=20)
    g = R.ParamGradients.zeros_like(host_cloud(oc))
    g.check_finite()
    g.positions[0, 0] = np.nan
    with pytest.raises(FloatingPointError, match="positions"):
        g.check_finite()


@pytest.mark.parametrize("n,F,B", [(1500, 1, 1), (3000, 1, 6), (1200, 4, 2),
                                   (300, 1, 3),
                                   # Cp = B*C in [16, 64]: the tensor-core K5
                                   (2000, 1, 8), (600, 1, 24), (500, 2, 12),
                                   (800, 1, 32)])
def test_deterministic_backward(n, F, B, pose):
    """the fixed-order reduction (frame planned with
    with_backward=2) gives bit-identical gradients on every rerun, agrees
    with the atomic accumulation to f32 rounding, and with the oracle's
    loop-and-sum at the north_star bar.  Batches of 16..64 channel columns
    run the tcgen05 backward (raster_bwd_tc.cu), in both modes."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud
    from paper_2511_22793_b200.engine import Renderer, split_flat
    oc = O.round_f32(O.perturbed_scene(n, seed=5, F=F))
    dc = DeviceCloud.from_host(host_cloud(oc))
    txs = O.sample_tx(11, B)
    R = Renderer()
    tx = torch.as_tensor(txs, device="cuda")
    img, fr = R.forward(dc, pose, tx, 180, 45, with_backward=2, lazy=False)
    C = dc.mlp_dims[2]
    U = torch.as_tensor(np.random.default_rng(3).normal(size=(B, 45, 180, C)),
                        dtype=torch.float32, device="cuda")
    runs = [R.backward(dc, pose, tx, U, fr, deterministic=True).clone()
            for _ in range(3)]
    for r in runs[1:]:
        assert torch.equal(r, runs[0]), "deterministic backward not bit-stable"
    atomic = R.backward(dc, pose, tx, U, fr, deterministic=False)
    det = split_flat(runs[0], dc.n, dc.P)
    ato = split_flat(atomic, dc.n, dc.P)
    for k in O.GROUPS:
        a, b = det[k].double(), ato[k].double()
        assert (a - b).abs().max() <= 1e-5 * max(b.abs().max().item(), 1e-30), k
    # oracle: loop over TX, sum -- on flip-free renders, like the other
    # gradient parity tests (a contributor-count flip changes the gradient
    # by a whole term)
    # oracle: loop over TX, sum; dL zeroed on the batch's threshold-flip
    # pixels (a flip changes only its own pixel's terms)
    Un = U.double().cpu().numpy()
    ref = {k: 0.0 for k in O.GROUPS}
    auxs = []
    for b in range(B):
        one, fb = R.forward(dc, pose, tx[b:b + 1], 180, 45, lazy=False)
        _, aux = O.forward(oc, RX, W, txs[b], 180, 45)
        flip = fb.contrib_count().cpu().numpy() != aux.contrib_count
        Un[b] = masked_dL(Un[b], flip)
        auxs.append(aux)
    Um = torch.as_tensor(Un, dtype=torch.float32, device="cuda")
    det = split_flat(R.backward(dc, pose, tx, Um, fr, deterministic=True),
                     dc.n, dc.P)
    for b in range(B):
        g = O.backward(Un[b], oc, txs[b], auxs[b])
        for k in O.GROUPS:
            ref[k] = ref[k] + g[k]
    err = group_err({k: det[k].double().cpu().numpy() for k in O.GROUPS}, ref)
    assert max(err.values()) <= 1e-4, err


def test_dropin_backward_is_bit_reproducible(R, pose):
    """The drop-in rasterize_backward uses the deterministic reduction, so two
    runs give identical ParamGradients (the reference's CPU determinism,
    tests/test_acceptance.py:310-357)."""
    oc = O.round_f32(O.perturbed_scene(800, seed=9))
    cloud = host_cloud(oc)
    tx = np.array([0.4, 0.8, -1.3])
    U = np.random.default_rng(1).normal(size=(45, 180, 2))
    outs = []
    for _ in range(2):
        _, aux = R.rasterize_forward(cloud, pose, tx, 180, 45)
        g = R.rasterize_backward(U, cloud, pose, tx, aux)
        outs.append(g.arrays())
    for k in O.GROUPS:
        assert np.array_equal(outs[0][k], outs[1][k]), k
