"""Gaussian cloud state: the host-side value type mirrored from the reference
(`rfsplat.scene`, scene.py:46-103), seeded initialisation (scene.py:184-207),
the GSPC checkpoint format (scene.py:210-239) and the device-resident copy the
CUDA path renders from.

`GaussianCloud` keeps the reference's raw f64 NumPy arrays so reference code
(optimizer loops, tests) can hold and mutate it; `DeviceCloud` is the
authoritative device copy (f64 geometry, f32 MLP weights, optional f64 MLP
copy for the f64 verification path).  Activations are applied on the device
inside K2/K6, never here.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

GSPC_MAGIC = b"GSPC"
GSPC_VERSION = 1
DEFAULT_MLP_DIMS = (5, 16, 2)
DEFAULT_OPACITY_LOGIT = -2.0
GROUPS = ("positions", "log_scales", "rotations", "raw_opacities",
          "mlp_weights")


def mlp_param_count(dims=DEFAULT_MLP_DIMS):
    """W1 | b1 | W2 | b2 (scene.py:25-27)."""
    i, h, o = dims
    return i * h + h + h * o + o


@dataclass
class SceneBounds:
    min_corner: np.ndarray
    max_corner: np.ndarray

    def __post_init__(self):
        self.min_corner = np.asarray(self.min_corner, np.float64).reshape(3)
        self.max_corner = np.asarray(self.max_corner, np.float64).reshape(3)
        if not np.all(self.min_corner < self.max_corner):
            raise ValueError("degenerate scene bounds")

    @property
    def diagonal(self):
        return float(np.linalg.norm(self.max_corner - self.min_corner))


@dataclass
class GaussianCloud:
    """The N learnable primitives, raw parameters (scene.py:46-103)."""

    positions: np.ndarray
    log_scales: np.ndarray
    rotations: np.ndarray
    raw_opacities: np.ndarray
    mlp_weights: np.ndarray
    mlp_dims: tuple = DEFAULT_MLP_DIMS

    def __post_init__(self):
        self.mlp_dims = tuple(int(v) for v in self.mlp_dims)
        n = np.shape(self.positions)[0]
        if n == 0:
            raise ValueError("cloud must contain at least one Gaussian")
        want = {"positions": (n, 3), "log_scales": (n, 3),
                "rotations": (n, 4), "raw_opacities": (n, 1),
                "mlp_weights": (n, mlp_param_count(self.mlp_dims))}
        for name, shape in want.items():
            got = np.shape(getattr(self, name))
            if got != shape:
                raise ValueError(f"{name}: expected shape {shape}, got {got}")

    @property
    def n(self):
        return np.shape(self.positions)[0]

    def copy(self):
        return GaussianCloud(*(np.array(getattr(self, g)) for g in GROUPS),
                             mlp_dims=self.mlp_dims)

    def param_arrays(self):
        """Learnable arrays in the optimizer/gradient order."""
        return {g: getattr(self, g) for g in GROUPS}


def init_uniform(bounds: SceneBounds, n, seed, init_scale=None,
                 init_opacity_logit=DEFAULT_OPACITY_LOGIT,
                 mlp_dims=DEFAULT_MLP_DIMS):
    """Seeded uniform cloud; same PCG64 draws as the reference
    (scene.py:184-207), so both sides see identical inputs."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if init_scale is None:
        init_scale = 0.02 * bounds.diagonal
    if init_scale <= 0:
        raise ValueError("init_scale must be > 0")
    rng = np.random.Generator(np.random.PCG64(seed))
    pos = rng.uniform(bounds.min_corner, bounds.max_corner, size=(n, 3))
    ls = np.full((n, 3), np.log(init_scale))
    rot = np.zeros((n, 4))
    rot[:, 0] = 1.0
    op = np.full((n, 1), float(init_opacity_logit))
    mw = rng.standard_normal((n, mlp_param_count(mlp_dims)))
    return GaussianCloud(pos, ls, rot, op, mw, mlp_dims)


def save_checkpoint(path, cloud):
    """GSPC v1: magic, u32 version/n/i/h/o, f32-LE payload (scene.py:210-218)."""
    i, h, o = cloud.mlp_dims
    host = cloud.to_host() if isinstance(cloud, DeviceCloud) else cloud
    with open(path, "wb") as f:
        f.write(GSPC_MAGIC + struct.pack("<5I", GSPC_VERSION, host.n, i, h, o))
        for g in GROUPS:
            f.write(np.ascontiguousarray(getattr(host, g), "<f4").tobytes())


def load_checkpoint(path):
    """Inverse of save_checkpoint; ValueError on bad magic / version /
    truncation (scene.py:221-239)."""
    with open(path, "rb") as f:
        magic = f.read(4)
        if magic != GSPC_MAGIC:
            raise ValueError(f"{path}: bad magic {magic!r}, expected GSPC")
        hdr = f.read(20)
        if len(hdr) != 20:
            raise ValueError(f"{path}: truncated GSPC header")
        version, n, mi, mh, mo = struct.unpack("<5I", hdr)
        if version != GSPC_VERSION:
            raise ValueError(f"{path}: unsupported GSPC version {version}")
        dims = (mi, mh, mo)
        arrs = []
        for shape in [(n, 3), (n, 3), (n, 4), (n, 1),
                      (n, mlp_param_count(dims))]:
            cnt = shape[0] * shape[1]
            buf = f.read(4 * cnt)
            if len(buf) != 4 * cnt:
                raise ValueError(f"{path}: truncated GSPC payload")
            arrs.append(np.frombuffer(buf, "<f4").astype(np.float64)
                        .reshape(shape))
    return GaussianCloud(*arrs, mlp_dims=dims)


class DeviceCloud:
    """Device-resident cloud (torch CUDA tensors), the authoritative copy in
    train/bench mode.  Geometry in f64 (K2 needs bit-exact depth), MLP
    weights in f32 (+ optional f64 copy for the f64 verification path)."""

    def __init__(self, positions, log_scales, rotations, raw_opacities,
                 mlp_weights, mlp_dims, mlp_weights64=None):
        self.positions = positions
        self.log_scales = log_scales
        self.rotations = rotations
        self.raw_opacities = raw_opacities
        self.mlp_weights = mlp_weights
        self.mlp_weights64 = mlp_weights64
        self.mlp_dims = tuple(int(v) for v in mlp_dims)

    @property
    def n(self):
        return int(self.positions.shape[0])

    @property
    def P(self):
        return mlp_param_count(self.mlp_dims)

    @classmethod
    def from_host(cls, cloud, device="cuda", with_f64_mlp=False):
        import torch
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt,
                                          device=device)
        mw = np.asarray(cloud.mlp_weights)
        return cls(t(cloud.positions, torch.float64),
                   t(cloud.log_scales, torch.float64),
                   t(cloud.rotations, torch.float64),
                   t(cloud.raw_opacities, torch.float64),
                   t(mw, torch.float32), cloud.mlp_dims,
                   t(mw, torch.float64) if with_f64_mlp else None)

    def to_host(self):
        return GaussianCloud(
            self.positions.double().cpu().numpy(),
            self.log_scales.double().cpu().numpy(),
            self.rotations.double().cpu().numpy(),
            self.raw_opacities.double().cpu().numpy(),
            (self.mlp_weights64 if self.mlp_weights64 is not None
             else self.mlp_weights).double().cpu().numpy(),
            self.mlp_dims)

    def cstruct(self):
        from ._lib import CCloud
        i, h, o = self.mlp_dims
        c = CCloud()
        c.n = self.n
        c.mlp_in, c.mlp_hidden, c.mlp_out = i, h, o
        c.positions = self.positions.data_ptr()
        c.log_scales = self.log_scales.data_ptr()
        c.rotations = self.rotations.data_ptr()
        c.raw_opacities = self.raw_opacities.data_ptr()
        c.mlp_weights = self.mlp_weights.data_ptr()
        c.mlp_weights64 = (self.mlp_weights64.data_ptr()
                           if self.mlp_weights64 is not None else None)
        return c
