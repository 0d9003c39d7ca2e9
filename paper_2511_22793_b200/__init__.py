"""B200-native GSpaRC render/train hot path (arxiv 2511.22793).

Drop-in for the reference `rfsplat` renderer API on sm_100a CUDA kernels
behind the C ABI in include/gsparc_b200.h (libgsparc_b200.so, built in-tree
by `python -m paper_2511_22793_b200.build`).  No CPU fallback: entry points
raise when the library or a CUDA device is missing.
"""

from .geometry import ViewPose, pixel_to_direction
from .image import SpectrumImage
from .scene import (DeviceCloud, GaussianCloud, SceneBounds, init_uniform,
                    load_checkpoint, mlp_param_count, save_checkpoint)

__version__ = "0.1.0"

__all__ = ["ViewPose", "pixel_to_direction", "SpectrumImage", "DeviceCloud",
           "GaussianCloud", "SceneBounds", "init_uniform", "load_checkpoint",
           "mlp_param_count", "save_checkpoint"]
