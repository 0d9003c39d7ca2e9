"""Drop-in replacement for `rfsplat.rasterizer` (rasterizer.py of the
reference) running on the B200 kernels.

Same names, signatures, return types and errors as the reference:
  rasterize_forward(cloud, pose, tx, w, h, dtype=np.float32, t_eps=T_EPS,
                    threads=1) -> (SpectrumImage, RenderAux)     (:187-234)
  rasterize_backward(dL_dimage, cloud, pose, tx, aux) -> ParamGradients
                                                               (:262-378)
  rasterize_reference(cloud, pose, tx, w, h, row_chunk=8)     (:237-259)
plus the batched device entry points used by training and the benchmark:
  rasterize_forward_batch / rasterize_backward_batch.

`cloud` may be the reference-style `GaussianCloud` (NumPy, uploaded per
call) or a `DeviceCloud` (authoritative on the device).  Gradients returned
to NumPy callers are f64 like the reference's.  `threads` is accepted and
ignored (the GPU is the parallelism).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import CapacityError, Renderer, dtype_code, split_flat
from .geometry import ViewPose
from .image import SpectrumImage
from .scene import GROUPS, DeviceCloud, GaussianCloud

ALPHA_MAX = 0.99
ALPHA_MIN = 1.0 / 255.0
T_EPS = 1e-4
TILE = 16

_renderer = None


def renderer():
    global _renderer
    if _renderer is None:
        _renderer = Renderer()
    return _renderer


@dataclass
class ParamGradients:
    """Gradients matching GaussianCloud.param_arrays() (rasterizer.py:39-66)."""

    positions: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    raw_opacities: np.ndarray
    mlp_weights: np.ndarray

    @classmethod
    def zeros_like(cls, cloud):
        return cls(**{k: np.zeros(np.shape(v), dtype=np.float64)
                      for k, v in cloud.param_arrays().items()})

    def arrays(self):
        return {g: getattr(self, g) for g in GROUPS}

    def check_finite(self):
        for name, arr in self.arrays().items():
            if not np.all(np.isfinite(arr)):
                raise FloatingPointError(f"non-finite gradient in {name}")


class _PrepView:
    """Lazy host view of the per-Gaussian state (the reference's _Prepared):
    idx in (radial depth, source index) order and the raster record."""

    def __init__(self, frame):
        self._frame = frame
        self._idx = None

    def _keys(self):
        return self._frame.depth_keys().cpu().numpy().view(np.uint64)

    @property
    def idx(self):
        if self._idx is None:
            k = self._keys()
            kept = np.nonzero(k != np.uint64(0xFFFFFFFFFFFFFFFF))[0]
            depth = k[kept].view(np.float64)
            self._idx = kept[np.lexsort((kept, depth))]
        return self._idx

    @property
    def depth(self):
        return self._keys()[self.idx].view(np.float64)

    def _rec(self):
        f = self._frame
        r = (f.rec64() if f.dtype_code == _lib.F64 else f.rec32()).cpu().numpy()
        return r[self.idx].astype(np.float64)

    @property
    def mean2d(self):
        return self._rec()[:, 0:2]

    @property
    def conic(self):
        return self._rec()[:, 2:5]

    @property
    def opac(self):
        return self._rec()[:, 5]

    @property
    def w(self):
        return self._frame.w

    @property
    def h(self):
        return self._frame.h


class RenderAux:
    """Forward state for the backward (rasterizer.py:148-160).  Device
    buffers live in `frame`; host views are materialised on access."""

    def __init__(self, frame, cloud_dev, pose, tx, cloud_n, dtype, t_eps,
                 txs_dev):
        self.frame = frame
        self.cloud_dev = cloud_dev
        self.pose = pose
        self.tx = tx
        self.cloud_n = cloud_n
        self.dtype = dtype
        self.t_eps = t_eps
        self.txs_dev = txs_dev
        self._tiles = None

    @property
    def transmittance(self):
        return self.frame.transmittance().cpu().numpy()

    @property
    def contrib_count(self):
        return self.frame.contrib_count().cpu().numpy()

    @property
    def prep(self):
        return _PrepView(self.frame)

    def tile_sources(self):
        """{(ty, tx): source indices in compositing order} as the GPU built
        them (the reference's prep.idx[tiles[key]])."""
        f = self.frame
        starts = f.tile_start().cpu().numpy().astype(np.int64)
        total = int(starts[-1])
        pairs = f.pairs()[:total].cpu().numpy().astype(np.int64)
        src = pairs & 0xFFFFFFFF
        out = {}
        ntx = int(f.layout.ntx)
        for t in range(int(f.layout.ntiles)):
            a, b = starts[t], starts[t + 1]
            if b > a:
                out[(t // ntx, t % ntx)] = src[a:b]
        return out

    @property
    def tiles(self):
        """{(ty, tx): rows into prep order}, like the reference's aux.tiles."""
        if self._tiles is None:
            idx = self.prep.idx
            rank = np.empty(self.cloud_n, np.int64)
            rank[idx] = np.arange(idx.size)
            self._tiles = {k: rank[v].astype(np.intp)
                           for k, v in self.tile_sources().items()}
        return self._tiles


def _device_cloud(cloud, f64):
    if isinstance(cloud, DeviceCloud):
        if f64 and cloud.mlp_weights64 is None:
            cloud.mlp_weights64 = cloud.mlp_weights.double()
        return cloud
    return DeviceCloud.from_host(cloud, with_f64_mlp=f64)


def _tx_tensor(txs):
    if isinstance(txs, torch.Tensor):
        return txs.to(device="cuda", dtype=torch.float64).reshape(-1, 3) \
            .contiguous()
    return torch.as_tensor(np.asarray(txs, np.float64).reshape(-1, 3),
                           device="cuda")


def rasterize_forward(cloud, pose: ViewPose, tx, w, h, dtype=np.float32,
                      t_eps=T_EPS, threads=1):
    """Render the 2-channel (re, im) spectrum (C = mlp_out channels in
    general); returns (SpectrumImage (h, w, C) of `dtype`, RenderAux)."""
    tx = np.asarray(tx, dtype=np.float64).reshape(3)
    dc = dtype_code(dtype)
    dev = _device_cloud(cloud, dc == _lib.F64)
    txs = _tx_tensor(tx)
    # with_backward=2: the reference's backward is deterministic (bit-identical
    # reruns, tests/test_acceptance.py:310-357), so the drop-in uses the
    # fixed-order reduction
    img, frame = renderer().forward(dev, pose, txs, int(w), int(h),
                                    t_eps=t_eps, dtype_code_=dc,
                                    with_backward=2, lazy=False)
    aux = RenderAux(frame, dev, pose, tx, dev.n, np.dtype(dtype).type,
                    t_eps, txs)
    return SpectrumImage(img[0]), aux


def rasterize_reference(cloud, pose: ViewPose, tx, w, h, row_chunk=8):
    """Brute-force semantics of the reference oracle (f64, no early exit):
    the f64 kernels with t_eps = 0, which composites every overlapping
    Gaussian exactly like rasterizer.py:237-259."""
    img, _ = rasterize_forward(cloud, pose, tx, w, h, dtype=np.float64,
                               t_eps=0.0)
    return SpectrumImage(img.tensor)


def rasterize_backward(dL_dimage, cloud, pose: ViewPose, tx,
                       aux: RenderAux) -> ParamGradients:
    """Analytic gradients of <dL, image> w.r.t. every parameter group."""
    tx = np.asarray(tx, dtype=np.float64).reshape(3)
    if aux.cloud_n != cloud.n or not np.array_equal(aux.tx, tx):
        raise ValueError("aux does not match this cloud/transmitter")
    f = aux.frame
    C = aux.cloud_dev.mlp_dims[2]
    dL = torch.as_tensor(np.asarray(dL_dimage, np.float64)
                         .reshape(1, f.h, f.w, C), dtype=f.rdtype,
                         device="cuda")
    grad = renderer().backward(aux.cloud_dev, pose, aux.txs_dev, dL, f,
                               grad_dtype_code=_lib.F64,
                               deterministic=f.with_backward == 2)
    g = {k: v.cpu().numpy() for k, v in
         split_flat(grad, aux.cloud_dev.n, aux.cloud_dev.P).items()}
    return ParamGradients(**g)


class RenderCheck:
    """Deferred validity check of an asynchronous batch render (a serving
    loop's alternative to the per-call host sync): the frame counters are
    copied to pinned host memory on the render's stream, and `ok()` /
    `raise_if_overflow()` read them once that copy has landed -- typically
    when the caller collects the image anyway."""

    RING = 16  # pinned slots per frame: a check stays readable for 16 renders

    def __init__(self, frame):
        ring = getattr(frame, "_check_ring", None)
        if ring is None:
            ring = frame._check_ring = [
                [torch.empty(_lib.NUM_COUNTERS, dtype=torch.int32,
                             pin_memory=True), torch.cuda.Event()]
                for _ in range(self.RING)]
            frame._check_next = 0
        self.host, self.event = ring[frame._check_next % self.RING]
        frame._check_next += 1
        self.frame = frame
        self.host.copy_(frame.counters(), non_blocking=True)
        self.event.record()

    def ok(self):
        self.event.synchronize()
        return not int(self.host[_lib.CNT_OVERFLOW])

    def pairs_needed(self):
        self.event.synchronize()
        return int(self.host[_lib.CNT_PAIRS])

    def raise_if_overflow(self):
        if not self.ok():
            raise CapacityError(self.pairs_needed())


def rasterize_forward_batch(cloud: DeviceCloud, pose: ViewPose, txs, w, h,
                            t_eps=T_EPS, lazy=None, with_backward=False,
                            frame=None, image=None, sync=True):
    """Render B transmitters at once: image [B, h, w, C] (f32 device tensor)
    and the frame (device aux) for rasterize_backward_batch.

    sync=True checks the frame on the host (pair-buffer overflow -> grow and
    re-render) before returning.  sync=False returns (image, frame,
    RenderCheck) without waiting for the device; if `check.ok()` is False
    the image is invalid and the caller re-renders with
    `renderer().grow(frame, check.pairs_needed())`."""
    txs = _tx_tensor(txs)
    img, frame = renderer().forward(cloud, pose, txs, int(w), int(h),
                                    frame=frame, image=image, t_eps=t_eps,
                                    lazy=lazy, with_backward=with_backward,
                                    sync_check=sync)
    if not sync:
        return img, frame, RenderCheck(frame)
    return img, frame


def rasterize_backward_batch(dL, cloud: DeviceCloud, pose: ViewPose, txs,
                             frame, grad=None, deterministic=None):
    """sum_b d<dL_b, img_b>/dparams into a flat f32 device buffer.
    deterministic (default: whether the frame was planned with
    with_backward=2) selects the fixed-order reduction."""
    if deterministic is None:
        deterministic = frame.with_backward == 2
    return renderer().backward(cloud, pose, _tx_tensor(txs), dL, frame,
                               grad=grad, deterministic=deterministic)
