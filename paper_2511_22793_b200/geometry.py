"""Receiver pose and projection constants (geometry.py:17-47 of the
reference).  The projection math itself runs on the device (K2/K6)."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

COV2D_REG = 0.3
FOOTPRINT_SIGMA = float(np.sqrt(2.0 * np.log(255.0)))
NEAR_PLANE = 0.05
FAR_PLANE = 1000.0
POLE_CLAMP_DEG = 89.0


@dataclass
class ViewPose:
    """Receiver position and world-to-receiver rotation W (geometry.py:34-47):
    ValueError unless W is orthonormal with det +1."""

    rx_position: np.ndarray
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))

    def __post_init__(self):
        self.rx_position = np.asarray(self.rx_position, np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, np.float64).reshape(3, 3)
        if not np.allclose(self.rotation.T @ self.rotation, np.eye(3),
                           atol=1e-9):
            raise ValueError("ViewPose.rotation must be orthonormal")
        if np.linalg.det(self.rotation) < 0:
            raise ValueError("ViewPose.rotation must be a proper rotation "
                             "(det +1)")

    def cstruct(self, w, h):
        from .engine import view_cstruct
        return view_cstruct(self, w, h)


def pixel_to_direction(u, v, w, h):
    """Unit direction of pixel (u, v)'s centre (geometry.py:83-95); used to
    place known-answer Gaussians."""
    u = np.asarray(u, np.float64)
    v = np.asarray(v, np.float64)
    if np.any(u < 0) or np.any(u >= w) or np.any(v < 0) or np.any(v >= h):
        raise ValueError("pixel index out of range")
    az = ((u + 0.5) * 2.0 / w - 1.0) * np.pi
    el = (v + 0.5) * (np.pi / 2.0) / h
    ce = np.cos(el)
    return np.stack([ce * np.sin(az), np.sin(el), ce * np.cos(az)], axis=-1)
