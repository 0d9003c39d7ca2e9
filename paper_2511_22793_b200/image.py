"""Spectrum image container (image.py:20-43 of the reference).

`data` is an (h, w, c) array; row 0 is the horizon.  Images produced by the
CUDA path are device tensors, converted to NumPy lazily on first access of
`.data` so the drop-in API returns the reference's type without forcing a
device->host copy when the caller stays on the device (`.tensor`).
"""

from __future__ import annotations

import numpy as np


class SpectrumImage:
    def __init__(self, data):
        self._tensor = None
        self._data = None
        if hasattr(data, "is_cuda"):
            if data.dim() != 3 or min(data.shape) < 1:
                raise ValueError("spectrum data must be (h, w, c) with all "
                                 "dims >= 1")
            self._tensor = data
        else:
            d = np.asarray(data)
            if d.ndim == 2:
                d = d[:, :, None]
            if d.ndim != 3 or min(d.shape) < 1:
                raise ValueError("spectrum data must be (h, w, c) with all "
                                 "dims >= 1")
            self._data = d

    @property
    def data(self):
        if self._data is None:
            self._data = self._tensor.cpu().numpy()
        return self._data

    @data.setter
    def data(self, value):
        self._data = np.asarray(value)
        self._tensor = None

    @property
    def tensor(self):
        """Device tensor (h, w, c) when produced on the GPU, else None."""
        return self._tensor

    @property
    def height(self):
        return self.data.shape[0] if self._tensor is None else self._tensor.shape[0]

    @property
    def width(self):
        return self.data.shape[1] if self._tensor is None else self._tensor.shape[1]

    @property
    def channels(self):
        return self.data.shape[2] if self._tensor is None else self._tensor.shape[2]
