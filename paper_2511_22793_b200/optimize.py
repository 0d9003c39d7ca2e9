"""Training glue on the device: loss (K7), Adam (K8) and the train step /
loop, mirroring `rfsplat.optimize` (optimize.py of the reference).

Drop-in names: TrainConfig, combined_loss, ssim, l1_loss, mse, psnr,
position_lr, AdamState, adam_step, render_prediction, train_step, train.
`Trainer` is the device-resident engine behind them: B transmitters per
step (geometry shared across the batch), gradients summed over the batch,
optional data parallelism over TX shards (NCCL all-reduce of the flat
gradient buffer), optional CUDA-graph capture of the whole step.
"""

from __future__ import annotations

import csv
import ctypes
import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from . import dp
from .engine import LossWorkspace, Renderer, split_flat
from .image import SpectrumImage
from .rasterizer import ParamGradients, rasterize_forward
from .scene import GROUPS, DeviceCloud, GaussianCloud, save_checkpoint


@dataclass
class TrainConfig:
    """Hyper-parameters (optimize.py:27-53) + batch_tx (TX per step)."""

    lambda_dssim: float = 0.2
    position_lr_init: float = 0.0016
    position_lr_final: float = 1.6e-6
    position_lr_delay_mult: float = 0.01
    position_lr_max_steps: int = 30000
    opacity_lr: float = 0.0055
    scaling_lr: float = 0.005
    rotation_lr: float = 0.001
    mlp_lr: float = 0.002
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-15
    iterations: int = 5000
    seed: int = 0
    width: int = 180
    height: int = 45
    supervision: str = "magnitude"
    deterministic: bool = False
    log_every: int = 50
    checkpoint_every: int = 0
    threads: int = 1
    dtype: str = "float32"
    batch_tx: int = 1

    def render_dtype(self):
        return np.float64 if self.dtype == "float64" else np.float32

    def adam_cstruct(self):
        c = _lib.CAdamConfig()
        c.position_lr_init = self.position_lr_init
        c.position_lr_final = self.position_lr_final
        c.position_lr_delay_mult = self.position_lr_delay_mult
        c.position_lr_max_steps = float(self.position_lr_max_steps)
        c.opacity_lr = self.opacity_lr
        c.scaling_lr = self.scaling_lr
        c.rotation_lr = self.rotation_lr
        c.mlp_lr = self.mlp_lr
        c.beta1, c.beta2, c.eps = self.adam_beta1, self.adam_beta2, self.adam_eps
        return c


def position_lr(step, cfg: TrainConfig):
    """Host copy of the schedule K8 evaluates on the device
    (optimize.py:205-213); used for logging only."""
    t = min(max(step / cfg.position_lr_max_steps, 0.0), 1.0)
    lr = math.exp((1.0 - t) * math.log(cfg.position_lr_init)
                  + t * math.log(cfg.position_lr_final))
    ramp = min(max(step / (0.01 * cfg.position_lr_max_steps), 0.0), 1.0)
    return (cfg.position_lr_delay_mult + (1.0 - cfg.position_lr_delay_mult)
            * math.sin(0.5 * math.pi * ramp)) * lr


# ------------------------------------------------------------------ loss
def _img_tensor(x):
    if isinstance(x, SpectrumImage):
        x = x.tensor if x.tensor is not None else x.data
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=torch.float64)
    return torch.as_tensor(np.asarray(x, np.float64), device="cuda")


def _loss_stats(pred, gt, lam):
    p, g = _img_tensor(pred), _img_tensor(gt)
    if p.shape != g.shape:
        raise ValueError(f"image shape mismatch: {tuple(p.shape)} vs "
                         f"{tuple(g.shape)}")
    squeeze = p.dim() == 2
    if squeeze:
        p, g = p[:, :, None], g[:, :, None]
    h, w, C = p.shape
    ws = LossWorkspace(1, h, w, C, "cuda", dtype=torch.float64)
    dimg, stats = ws.run(p.contiguous()[None], g.contiguous()[None], 1, lam)
    grad = dimg[0]
    return stats[0].cpu().numpy(), (grad[:, :, 0] if squeeze else grad)


def combined_loss(pred, gt, lam):
    """(1-lam) L1 + lam (1-SSIM) and its gradient (optimize.py:165-188);
    computed by K7 on the device in f64."""
    st, grad = _loss_stats(pred, gt, lam)
    return float(st[0]), grad.cpu().numpy()


def l1_loss(pred, gt):
    return float(_loss_stats(pred, gt, 0.0)[0][1])


def ssim(pred, gt):
    """Mean SSIM (channel-averaged for 3-D input), optimize.py:134-142."""
    return float(_loss_stats(pred, gt, 0.0)[0][2])


def mse(pred, gt):
    return float(_loss_stats(pred, gt, 0.0)[0][3])


def psnr(pred, gt):
    m = mse(pred, gt)
    return math.inf if m == 0.0 else 10.0 * math.log10(1.0 / m)


# ------------------------------------------------------------------ Adam
class AdamState:
    """Device moment buffers (flat, f32) + the device step counter."""

    def __init__(self, cloud, device="cuda"):
        n = cloud.n
        P = int(np.prod(np.shape(cloud.mlp_weights)[1:]))
        total = n * (11 + P)
        self.m = torch.zeros(total, dtype=torch.float32, device=device)
        self.v = torch.zeros(total, dtype=torch.float32, device=device)
        self.step_dev = torch.zeros(1, dtype=torch.int64, device=device)
        self.counters = torch.zeros(_lib.NUM_COUNTERS, dtype=torch.int32,
                                    device=device)
        self.step = 0
        self.n, self.P = n, P


def _run_adam(dev: DeviceCloud, grad_flat, state: AdamState, cfg, counters):
    # K8 updates the f32 weights: an f64 copy made for the f64 verification
    # path is stale from here on (rasterizer._device_cloud re-derives it)
    dev.mlp_weights64 = None
    acfg = cfg.adam_cstruct()
    check(lib().gsparc_adam_step(
        ctypes.c_void_p(dev.positions.data_ptr()),
        ctypes.c_void_p(dev.log_scales.data_ptr()),
        ctypes.c_void_p(dev.rotations.data_ptr()),
        ctypes.c_void_p(dev.raw_opacities.data_ptr()),
        ctypes.c_void_p(dev.mlp_weights.data_ptr()), dev.n, dev.P,
        ctypes.c_void_p(grad_flat.data_ptr()),
        ctypes.c_void_p(state.m.data_ptr()), ctypes.c_void_p(state.v.data_ptr()),
        ctypes.c_void_p(state.step_dev.data_ptr()),
        ctypes.c_void_p(counters.data_ptr()), ctypes.byref(acfg),
        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


def _raise_nonfinite(mask):
    for g, name in enumerate(GROUPS):
        if mask & (1 << g):
            raise FloatingPointError(f"non-finite gradient in {name}")
    if mask:
        raise ValueError("zero quaternion")


def _flat_grads(grads, n, P):
    if isinstance(grads, torch.Tensor):
        return grads.to(device="cuda", dtype=torch.float32).contiguous()
    arrs = grads.arrays()
    return torch.as_tensor(np.concatenate(
        [np.asarray(arrs[g], np.float64).reshape(-1) for g in GROUPS]),
        dtype=torch.float32, device="cuda")


def adam_step(cloud, grads, state: AdamState, step, cfg: TrainConfig):
    """In-place Adam with per-group LR and quaternion renorm
    (optimize.py:234-259).  NumPy clouds are updated in place (uploaded,
    stepped by K8, written back); DeviceClouds stay on the device."""
    host = not isinstance(cloud, DeviceCloud)
    dev = DeviceCloud.from_host(cloud) if host else cloud
    g = _flat_grads(grads, dev.n, dev.P)
    state.step_dev.fill_(int(step))
    _run_adam(dev, g, state, cfg, state.counters)
    _raise_nonfinite(int(state.counters[_lib.CNT_NONFINITE].item()))
    state.step = int(step) + 1
    if host:
        back = dev.to_host()
        for name in GROUPS:
            getattr(cloud, name)[...] = getattr(back, name)


# ------------------------------------------------------------ prediction
def magnitude(img):
    """|z| of a 2-channel image on the device (image.py:46-51)."""
    t = img.tensor if isinstance(img, SpectrumImage) and img.tensor is not None \
        else _img_tensor(img)
    if t.shape[-1] != 2:
        raise ValueError(f"magnitude needs 2 channels, got {t.shape[-1]}")
    return SpectrumImage(torch.hypot(t[..., 0].double(),
                                     t[..., 1].double())[..., None])


def render_prediction(cloud, pose, tx, cfg: TrainConfig):
    img, aux = rasterize_forward(cloud, pose, tx, cfg.width, cfg.height,
                                 dtype=cfg.render_dtype(), threads=cfg.threads)
    pred = magnitude(img) if cfg.supervision == "magnitude" else img
    return img, pred, aux


# --------------------------------------------------------------- trainer
class Trainer:
    """Device-resident batched train step.

    Per step: K2..K4 forward of B_local TX (shared geometry), K7 loss on the
    B_local images, K5+K6 backward summed over the batch, NCCL all-reduce
    (sum) across ranks when `group` spans >1 process, K8 Adam.  The global
    batch is split contiguously across ranks, so the update equals the
    single-GPU update on the same global batch."""

    def __init__(self, cloud, pose, cfg: TrainConfig, tx_all, gt_all,
                 batch_tx=None, group=None, start_step=0):
        _lib.require_cuda()
        self.cfg = cfg
        self.pose = pose
        self.dev = cloud if isinstance(cloud, DeviceCloud) else \
            DeviceCloud.from_host(cloud)
        self.h, self.w = int(cfg.height), int(cfg.width)
        self.C = self.dev.mlp_dims[2]
        self.sup = 0 if cfg.supervision == "magnitude" else 1
        B = int(batch_tx or cfg.batch_tx)
        self.group = group
        import torch.distributed as dist
        self.world = dist.get_world_size(group) if (
            dist.is_available() and dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        if B % self.world:
            raise ValueError(f"batch_tx={B} not divisible by world={self.world}")
        self.B = B
        self.Bl = B // self.world
        self.R = Renderer()
        self.tx_all = torch.as_tensor(np.asarray(tx_all, np.float64),
                                      device="cuda").reshape(-1, 3)
        gt = gt_all if isinstance(gt_all, torch.Tensor) else \
            torch.as_tensor(np.asarray(gt_all, np.float32))
        self.gt_all = gt.to(device="cuda", dtype=torch.float32).contiguous()
        Cs = 1 if self.sup == 0 else self.C
        if tuple(self.gt_all.shape[1:]) != (self.h, self.w, Cs):
            raise ValueError(f"ground truth {tuple(self.gt_all.shape)} does not "
                             f"match ({self.h}, {self.w}, {Cs})")
        self.idx = torch.zeros(self.Bl, dtype=torch.int64, device="cuda")
        self.tx = torch.empty((self.Bl, 3), dtype=torch.float64, device="cuda")
        self.gt = torch.empty((self.Bl, self.h, self.w, Cs),
                              dtype=torch.float32, device="cuda")
        self.img = torch.empty((self.Bl, self.h, self.w, self.C),
                               dtype=torch.float32, device="cuda")
        self.loss = LossWorkspace(self.Bl, self.h, self.w, self.C, "cuda")
        self.grad = torch.empty(self.dev.n * (11 + self.dev.P),
                                dtype=torch.float32, device="cuda")
        self.state = AdamState(self.dev)
        self.state.step_dev.fill_(int(start_step))
        self.step_no = int(start_step)
        # size the pair buffer with one synchronous render.  The step renders
        # with the lazy MLP: only Gaussians some pixel included need coef
        # rows (pass B, K5's compacted walk); K6 recomputes the MLP itself
        self.tx.copy_(self.tx_all[:1].expand(self.Bl, 3))
        _, self.frame = self.R.forward(self.dev, pose, self.tx, self.w, self.h,
                                       image=self.img,
                                       with_backward=2 if cfg.deterministic else 1,
                                       lazy=True)
        self.graph = None

    def _gather(self):
        torch.index_select(self.tx_all, 0, self.idx, out=self.tx)
        torch.index_select(self.gt_all, 0, self.idx, out=self.gt)

    def _compute(self):
        self.R.forward(self.dev, self.pose, self.tx, self.w, self.h,
                       frame=self.frame, image=self.img, lazy=True,
                       sync_check=False)
        dimg, _ = self.loss.run(self.img, self.gt, self.sup,
                                self.cfg.lambda_dssim)
        self.R.backward(self.dev, self.pose, self.tx, dimg, self.frame,
                        grad=self.grad, deterministic=self.cfg.deterministic)

    def _update(self):
        _run_adam(self.dev, self.grad, self.state, self.cfg,
                  self.frame.counters())

    def _allreduce(self):
        if self.world > 1:
            dp.allreduce_sum(self.grad, self.group)

    def capture(self):
        """Capture gather+forward+loss+backward(+Adam when single-rank) into a
        CUDA graph; replay with step()."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):      # warm the allocator/cudaFuncSetAttribute
                self._gather()
                self._compute()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._gather()
            self._compute()
            if self.world == 1:
                self._update()
        self.graph = g

    def set_batch(self, global_indices):
        gi = np.asarray(global_indices, np.int64).reshape(-1)
        if gi.size != self.B:
            raise ValueError(f"expected {self.B} indices, got {gi.size}")
        local = dp.shard(gi, self.rank, self.world)
        self.idx.copy_(torch.as_tensor(local), non_blocking=True)

    def step(self, global_indices=None):
        """One optimizer step on the given global batch of sample indices.
        Returns the device stats tensor [B_local, 6] (loss, l1, ssim, mse,
        channel-0 ssim, channel-0 mse).  Asynchronous: a step whose pair
        buffer overflowed is skipped by K8 (parameters, moments and the
        device step counter untouched); `check()` reports it."""
        if global_indices is not None:
            self.set_batch(global_indices)
        if self.graph is not None:
            self.graph.replay()
            if self.world > 1:
                self._allreduce()
                self._update()
        else:
            self._gather()
            self._compute()
            self._allreduce()
            self._update()
        self.step_no += 1
        return self.loss.stats

    def check(self):
        """Synchronous health check of the last step: False if its pair
        buffer overflowed (K8 skipped the update; the frame is grown and the
        graph dropped, so the caller re-runs the same batch); raises
        FloatingPointError on a non-finite gradient like the reference's
        adam_step (optimize.py:241 -> rasterizer.py:63-66)."""
        c = self.frame.counters().cpu()
        if int(c[_lib.CNT_OVERFLOW]):
            need = int(c[_lib.CNT_PAIRS])
            self.frame = self.R.grow(self.frame, need)
            self.graph = None
            return False
        _raise_nonfinite(int(c[_lib.CNT_NONFINITE]))
        return True

    def step_checked(self, global_indices, use_graph=True):
        """step() + check(), re-running the batch after a buffer grow, so
        every step applies exactly one update (the reference's semantics)."""
        for _ in range(4):
            stats = self.step(global_indices)
            if self.check():
                return stats
            self.step_no -= 1
            if use_graph:
                self.capture()
        raise RuntimeError("pair capacity could not be satisfied")

    def load_cloud(self, cloud):
        """Overwrite the device parameters from a host GaussianCloud (same
        shapes), keeping the frame, workspaces and captured graph."""
        for name in GROUPS:
            t = getattr(self.dev, name)
            t.copy_(torch.as_tensor(np.asarray(getattr(cloud, name)),
                                    dtype=t.dtype))
        self.dev.mlp_weights64 = None

    def sync_to_host(self, cloud: GaussianCloud):
        back = self.dev.to_host()
        for name in GROUPS:
            getattr(cloud, name)[...] = getattr(back, name)


def _dataset_arrays(dataset, cfg):
    txs = np.stack([np.asarray(s.tx_position, np.float64) for s in dataset])
    gts = [np.asarray(s.spectrum.data, np.float32) for s in dataset]
    gt = np.stack([g[:, :, :1] if cfg.supervision == "magnitude" else g
                   for g in gts])
    return txs, gt


def _metrics_row(step, st, wall_ms):
    """The reference's log row (optimize.py:288-295): loss and l1 over the
    supervised channels, ssim_term and psnr from channel 0."""
    m0 = float(st[5])
    return {"iteration": step, "loss": float(st[0]), "l1": float(st[1]),
            "ssim_term": 1.0 - float(st[4]),
            "psnr": math.inf if m0 == 0.0 else 10.0 * math.log10(1.0 / m0),
            "wall_ms": wall_ms}


def train_step(cloud, pose, sample, state: AdamState, step, cfg: TrainConfig):
    """One render/loss/backward/Adam iteration for one sample
    (optimize.py:273-296); returns the reference's metrics dict.

    The device trainer (frame, loss workspace, graph) is built on the first
    call and kept on `state`; later calls only refresh the parameters (a
    NumPy cloud may have been changed by the caller), the sample and the
    step, so a train_step costs one upload, one step and one write-back."""
    t0 = time.perf_counter()
    gt = _dataset_arrays([sample], cfg)[1]
    tr = getattr(state, "_trainer", None)
    key = (id(cloud), cloud.n, tuple(cloud.mlp_dims), cfg.width, cfg.height,
           cfg.supervision, cfg.deterministic)
    if tr is None or state._trainer_key != key:
        tr = Trainer(cloud, pose, cfg, [sample.tx_position], gt, batch_tx=1,
                     start_step=step)
        tr.state = state
        state._trainer, state._trainer_key = tr, key
    else:
        tr.pose = pose
        if not isinstance(cloud, DeviceCloud):
            tr.load_cloud(cloud)
        tr.tx_all.copy_(torch.as_tensor(
            np.asarray(sample.tx_position, np.float64).reshape(1, 3)))
        tr.gt_all.copy_(torch.as_tensor(gt))
    tr.cfg = cfg
    state.step_dev.fill_(int(step))
    stats = tr.step_checked([0], use_graph=False)
    st = stats[0].cpu().numpy()
    if not isinstance(cloud, DeviceCloud):
        tr.sync_to_host(cloud)
    state.step = step + 1
    return _metrics_row(step, st, (time.perf_counter() - t0) * 1e3)


def sample_stream(n_samples, cfg: TrainConfig, start_step, n_steps, batch):
    """The reference's sample order (optimize.py:314-334): iid PCG64 draws,
    or epoch shuffles in deterministic mode; `batch` draws per step."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    order = None
    pos = start_step * batch
    for _ in range(n_steps):
        out = []
        for _ in range(batch):
            if cfg.deterministic:
                if pos % n_samples == 0 or order is None:
                    order = rng.permutation(n_samples)
                out.append(int(order[pos % n_samples]))
                pos += 1
            else:
                out.append(int(rng.integers(n_samples)))
        yield out


def train(dataset, cfg: TrainConfig, cloud, pose, metrics_path=None,
          checkpoint_path=None, start_step=0, progress=None, group=None,
          use_graph=True, check_every=1):
    """Training loop (optimize.py:299-351) on the device; mutates `cloud`
    (host arrays are refreshed at checkpoints and at the end).

    check_every=1 (default) checks every step on the host like the
    reference, which applies each update and raises at once: an overflowed
    step is re-run after growing the pair buffer, a non-finite gradient
    raises FloatingPointError.  Larger values trade that for fewer host
    syncs (a skipped step is then lost, not re-run)."""
    if not dataset:
        raise ValueError("dataset is empty")
    dims = {(s.spectrum.height, s.spectrum.width) for s in dataset}
    if dims != {(cfg.height, cfg.width)}:
        raise ValueError(f"dataset image dims {dims} do not match config "
                         f"({cfg.height}, {cfg.width})")
    txs, gt = _dataset_arrays(dataset, cfg)
    tr = Trainer(cloud, pose, cfg, txs, gt, group=group,
                 start_step=start_step)
    if use_graph:
        tr.capture()
    log = []
    fh = writer = None
    if metrics_path is not None and tr.rank == 0:
        fh = open(metrics_path, "w", newline="")
        writer = csv.DictWriter(fh, fieldnames=["iteration", "loss", "l1",
                                                "ssim_term", "psnr", "wall_ms"])
        writer.writeheader()
    try:
        t0 = time.perf_counter()
        last = start_step + cfg.iterations - 1
        for k, batch in enumerate(sample_stream(len(dataset), cfg, start_step,
                                                cfg.iterations, tr.B)):
            step = start_step + k
            if check_every and (k % check_every == 0 or step == last):
                stats = tr.step_checked(batch, use_graph)
            else:
                stats = tr.step(batch)
            if step % cfg.log_every == 0 or step == last:
                st = stats.mean(dim=0).cpu().numpy()
                row = _metrics_row(step, st, (time.perf_counter() - t0) * 1e3)
                t0 = time.perf_counter()
                log.append(row)
                if writer:
                    writer.writerow({k2: f"{v:.6g}" if isinstance(v, float)
                                     else v for k2, v in row.items()})
                if progress:
                    progress(row)
            if checkpoint_path and cfg.checkpoint_every and \
                    (step + 1) % cfg.checkpoint_every == 0 and tr.rank == 0:
                save_checkpoint(checkpoint_path, tr.dev)
        if not isinstance(cloud, DeviceCloud):
            tr.sync_to_host(cloud)
        if checkpoint_path and tr.rank == 0:
            save_checkpoint(checkpoint_path, tr.dev)
    finally:
        if fh:
            fh.close()
    return log
