"""Device render/train engine over the C ABI (include/gsparc_b200.h).

`Frame` is one caller-owned device workspace (torch uint8 buffer carved by
`gsparc_plan_frame`).  `Renderer` runs K2->K3->K1->K4 (forward) and K5->K6
(backward) on the current torch CUDA stream, batched over transmitters, with
the cloud resident on the device.  Nothing here computes on the host.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .scene import DeviceCloud

T_EPS = 1e-4

_TORCH_DT = {_lib.F32: torch.float32, _lib.F64: torch.float64}


def dtype_code(dtype):
    dt = np.dtype(dtype)
    if dt == np.float32:
        return _lib.F32
    if dt == np.float64:
        return _lib.F64
    raise ValueError(f"unsupported render dtype {dt}")


def view_cstruct(pose, w, h):
    """C view for any pose object with the reference ViewPose's fields
    (`rx_position` (3,), `rotation` (3,3); geometry.py:34-47), so
    `rfsplat.geometry.ViewPose` works unchanged."""
    v = _lib.CView()
    rx = np.asarray(pose.rx_position, np.float64).reshape(3)
    rot = np.asarray(pose.rotation, np.float64).reshape(9)
    for k in range(3):
        v.rx[k] = float(rx[k])
    for k in range(9):
        v.rotation[k] = float(rot[k])
    v.width, v.height = int(w), int(h)
    return v


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Frame:
    """Device workspace for one render configuration."""

    def __init__(self, n, w, h, channels, pair_capacity, dtype_code_,
                 with_backward, device):
        L = _lib.CLayout()
        check(lib().gsparc_plan_frame(int(n), int(w), int(h), int(channels),
                                      int(pair_capacity), int(dtype_code_),
                                      int(with_backward),
                                      ctypes.byref(L)))
        self.layout = L
        # zero-initialised once: coef rows of never-live Gaussians must be
        # finite (the tensor-core accumulation multiplies them by 0)
        self.buf = torch.zeros(int(L.total_bytes), dtype=torch.uint8,
                               device=device)
        self.n, self.w, self.h = int(n), int(w), int(h)
        self.channels = int(channels)
        self.dtype_code = int(dtype_code_)
        # 0: forward only, 1: backward (atomic accumulation), 2: backward
        # with the deterministic fixed-order reduction buffers
        self.with_backward = int(with_backward)

    @property
    def ptr(self):
        return ctypes.c_void_p(self.buf.data_ptr())

    @property
    def capacity(self):
        return int(self.layout.pair_capacity)

    def view(self, name, dtype, shape):
        off = int(getattr(self.layout, "off_" + name))
        nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        return self.buf[off:off + nbytes].view(dtype).view(*shape)

    def counters(self):
        return self.view("counters", torch.int32, (_lib.NUM_COUNTERS,))

    @property
    def rdtype(self):
        return _TORCH_DT[self.dtype_code]

    # -- aux views (device tensors) --------------------------------------
    def transmittance(self):
        return self.view("T", self.rdtype, (self.h, self.w))

    def contrib_count(self):
        return self.view("count", torch.int32, (self.h, self.w))

    def last_index(self):
        return self.view("last", torch.int32, (self.h, self.w))

    def depth_keys(self):
        return self.view("key", torch.int64, (self.n,))

    def tile_start(self):
        return self.view("tile_start", torch.int32, (self.layout.ntiles + 1,))

    def pairs(self):
        return self.view("pairs", torch.int64, (self.capacity,))

    def rec32(self):
        return self.view("rec32", torch.float32, (self.n, 8))

    def rec64(self):
        return self.view("rec64", torch.float64, (self.n, 8))

    def coef(self):
        return self.view("coef", self.rdtype, (self.n, self.channels))

    def live(self):
        return self.view("live", torch.int32, (self.n,))


class CapacityError(RuntimeError):
    pass


class Renderer:
    """Frame cache + the forward/backward pipelines on the current stream."""

    def __init__(self, device=None):
        _lib.require_cuda()
        self.device = torch.device(device or "cuda")
        self._cap = {}

    def _capacity_for(self, key, n):
        return self._cap.get(key, 24 * int(n) + 4096)

    def new_frame(self, n, w, h, channels, dtype_code_=_lib.F32,
                  with_backward=False, capacity=None):
        key = (int(n), int(w), int(h))
        cap = capacity or self._capacity_for(key, n)
        return Frame(n, w, h, channels, cap, dtype_code_, with_backward,
                     self.device)

    def grow(self, frame, needed):
        key = (frame.n, frame.w, frame.h)
        cap = int(needed * 1.25) + 1024
        self._cap[key] = max(cap, self._cap.get(key, 0))
        return Frame(frame.n, frame.w, frame.h, frame.channels, cap,
                     frame.dtype_code, frame.with_backward, self.device)

    @staticmethod
    def check_frame(frame):
        """Host-synchronising validity check (overflow of the pair buffer)."""
        c = frame.counters().cpu()
        if int(c[_lib.CNT_OVERFLOW]):
            raise CapacityError(int(c[_lib.CNT_PAIRS]))
        return c

    def forward(self, cloud: DeviceCloud, pose, txs, w, h, frame=None,
                image=None, t_eps=T_EPS, lazy=None, dtype_code_=_lib.F32,
                with_backward=False, sync_check=True):
        """Render every TX in `txs` (f64 device tensor [B,3]).
        Returns (image [B,h,w,C] device tensor, frame)."""
        B = int(txs.shape[0])
        C = cloud.mlp_dims[2]
        if frame is None:
            frame = self.new_frame(cloud.n, w, h, B * C, dtype_code_,
                                   with_backward)
        if image is None:
            image = torch.empty((B, h, w, C), dtype=frame.rdtype,
                                device=self.device)
        if lazy is None:
            lazy = C >= 16
        flags = _lib.LAZY_MLP if lazy else 0
        cc = cloud.cstruct()
        view = view_cstruct(pose, w, h)
        for _ in range(3):
            check(lib().gsparc_render_forward(
                ctypes.byref(cc), ctypes.byref(view),
                ctypes.c_void_p(txs.data_ptr()), B, float(t_eps), flags,
                frame.ptr, ctypes.byref(frame.layout),
                ctypes.c_void_p(image.data_ptr()), _stream()))
            if not sync_check:
                return image, frame
            try:
                self.check_frame(frame)
                return image, frame
            except CapacityError as e:
                frame = self.grow(frame, e.args[0])
        raise RuntimeError("pair capacity could not be satisfied")

    def backward(self, cloud: DeviceCloud, pose, txs, dL, frame, grad=None,
                 grad_dtype_code=_lib.F32, deterministic=False):
        """Gradients (summed over TX) into a flat buffer
        positions|log_scales|rotations|raw_opacities|mlp_weights."""
        if not frame.with_backward:
            raise ValueError("frame was not planned with_backward")
        if deterministic and frame.with_backward != 2:
            raise ValueError("deterministic backward needs a frame planned "
                             "with with_backward=2")
        n, P = cloud.n, cloud.P
        if grad is None:
            grad = torch.empty(n * (11 + P), dtype=_TORCH_DT[grad_dtype_code],
                               device=self.device)
        cc = cloud.cstruct()
        view = view_cstruct(pose, frame.w, frame.h)
        check(lib().gsparc_render_backward(
            ctypes.byref(cc), ctypes.byref(view),
            ctypes.c_void_p(txs.data_ptr()), int(txs.shape[0]),
            ctypes.c_void_p(dL.data_ptr()), int(bool(deterministic)),
            frame.ptr, ctypes.byref(frame.layout),
            ctypes.c_void_p(grad.data_ptr()), int(grad_dtype_code), _stream()))
        return grad


def split_flat(flat, n, P):
    """Views of the flat gradient/moment buffer per parameter group."""
    o = 0
    out = {}
    for name, k in (("positions", 3), ("log_scales", 3), ("rotations", 4),
                    ("raw_opacities", 1), ("mlp_weights", P)):
        out[name] = flat[o:o + n * k].view(n, k)
        o += n * k
    return out


class LossWorkspace:
    """Scratch + outputs for K7 (loss forward/backward).  `dtype` of the
    image / ground truth / dL tensors: torch.float32 or torch.float64."""

    def __init__(self, n_img, h, w, C, device, dtype=torch.float32):
        nbytes = int(lib().gsparc_loss_scratch_bytes(n_img, h, w, C))
        self.scratch = torch.empty(nbytes, dtype=torch.uint8, device=device)
        self.stats = torch.zeros((n_img, _lib.LOSS_STATS), dtype=torch.float64,
                                 device=device)
        self.dimg = torch.empty((n_img, h, w, C), dtype=dtype, device=device)
        self.dtype_code = _lib.F64 if dtype == torch.float64 else _lib.F32
        self.shape = (n_img, h, w, C)

    def run(self, img, gt, supervision, lam):
        n_img, h, w, C = self.shape
        check(lib().gsparc_loss_fwd_bwd(
            ctypes.c_void_p(img.data_ptr()), ctypes.c_void_p(gt.data_ptr()),
            self.dtype_code, n_img, h, w, C, int(supervision), float(lam),
            ctypes.c_void_p(self.dimg.data_ptr()),
            ctypes.c_void_p(self.stats.data_ptr()),
            ctypes.c_void_p(self.scratch.data_ptr()), self.scratch.numel(),
            _stream()))
        return self.dimg, self.stats
