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


# ----------------------------------------------------------- wire formats
# RFSI (image.py:1-7, 64-86 of the reference): magic `RFSI`, u32 version=1,
# u32 width, u32 height, u32 channels, then h*w*c little-endian f32,
# row-major (row 0 = horizon).  Byte-compatible in both directions.
import struct  # noqa: E402

RFSI_MAGIC = b"RFSI"
RFSI_VERSION = 1
_RFSI_HDR = 20


def magnitude(image: SpectrumImage) -> SpectrumImage:
    """Per-pixel hypot(re, im) of a 2-channel image in f64 (image.py:46-51);
    stays on the device for device images."""
    if image.channels != 2:
        raise ValueError(f"magnitude needs 2 channels, got {image.channels}")
    t = image.tensor
    if t is not None:
        import torch
        d = t.double()
        return SpectrumImage(torch.hypot(d[..., 0], d[..., 1])[..., None])
    d = image.data.astype(np.float64)
    return SpectrumImage(np.hypot(d[:, :, 0], d[:, :, 1])[:, :, None])


def magnitude_backward(image: SpectrumImage, grad_mag):
    """dL/d|z| -> (re, im), zero at |z| = 0 (image.py:54-61)."""
    d = image.data.astype(np.float64)
    m = np.hypot(d[:, :, 0], d[:, :, 1])
    safe = np.where(m > 0.0, m, 1.0)
    g = np.asarray(grad_mag, dtype=np.float64).reshape(m.shape)
    scale = np.where(m > 0.0, g / safe, 0.0)
    return np.stack([d[:, :, 0] * scale, d[:, :, 1] * scale], axis=-1)


def _rfsi_header(w, h, c):
    return RFSI_MAGIC + struct.pack("<4I", RFSI_VERSION, w, h, c)


def save_rfsi(path, image: SpectrumImage):
    """image.py:64-69.  Device images are copied to the host once."""
    with open(path, "wb") as f:
        f.write(_rfsi_header(image.width, image.height, image.channels))
        f.write(np.ascontiguousarray(image.data, dtype="<f4").tobytes())


def _parse_rfsi(path, buf):
    if bytes(buf[:4]) != RFSI_MAGIC:
        raise ValueError(f"{path}: bad magic {bytes(buf[:4])!r}, expected RFSI")
    if len(buf) < _RFSI_HDR:
        raise ValueError(f"{path}: truncated RFSI header")
    version, w, h, c = struct.unpack("<4I", bytes(buf[4:_RFSI_HDR]))
    if version != RFSI_VERSION:
        raise ValueError(f"{path}: unsupported RFSI version {version}")
    count = w * h * c
    if len(buf) - _RFSI_HDR < 4 * count:
        raise ValueError(f"{path}: truncated RFSI payload "
                         f"({len(buf) - _RFSI_HDR} of {4 * count} bytes)")
    return w, h, c


def load_rfsi(path) -> SpectrumImage:
    """image.py:72-86 (same error messages)."""
    with open(path, "rb") as f:
        buf = f.read()
    w, h, c = _parse_rfsi(path, buf)
    data = np.frombuffer(buf, dtype="<f4", count=w * h * c,
                         offset=_RFSI_HDR).reshape(h, w, c)
    return SpectrumImage(data.copy())


def save_pgm(path, image: SpectrumImage):
    """8-bit P5 export of channel 0, clipped to [0, 1], zenith at the top
    (image.py:89-96)."""
    d = image.data[:, :, 0]
    pix = np.clip(d, 0.0, 1.0)
    pix = (pix * 255.0 + 0.5).astype(np.uint8)[::-1]
    with open(path, "wb") as f:
        f.write(f"P5\n{image.width} {image.height}\n255\n".encode())
        f.write(pix.tobytes())


def load_rfsi_batch(paths, device="cuda"):
    """Read RFSI files into one pinned host buffer (memory-mapped reads, no
    per-file allocation) and copy it to the device with one asynchronous
    H2D on the current stream.  Returns a f32 tensor [B, h, w, c]; all files
    must share (h, w, c)."""
    import torch
    paths = list(paths)
    if not paths:
        raise ValueError("load_rfsi_batch: no files")
    dims = None
    host = None
    for i, p in enumerate(paths):
        mm = np.memmap(p, dtype=np.uint8, mode="r")
        w, h, c = _parse_rfsi(p, mm)
        if dims is None:
            dims = (h, w, c)
            host = torch.empty((len(paths), h, w, c), dtype=torch.float32,
                               pin_memory=torch.cuda.is_available())
        elif dims != (h, w, c):
            raise ValueError(f"{p}: inconsistent image dims {(h, w, c)} vs {dims}")
        host[i].numpy().reshape(-1)[:] = np.frombuffer(
            mm, dtype="<f4", count=h * w * c, offset=_RFSI_HDR)
        del mm
    return host.to(device, non_blocking=True)


def save_rfsi_batch(paths, images):
    """Write a [B, h, w, c] (device or host) tensor as RFSI files: one D2H
    into pinned memory, then plain file writes."""
    import torch
    t = images if isinstance(images, torch.Tensor) else torch.as_tensor(images)
    if t.dim() != 4 or t.shape[0] != len(paths):
        raise ValueError("save_rfsi_batch: need [B, h, w, c] and B paths")
    host = torch.empty(t.shape, dtype=torch.float32,
                       pin_memory=t.is_cuda)
    host.copy_(t, non_blocking=t.is_cuda)
    if t.is_cuda:
        torch.cuda.current_stream().synchronize()
    B, h, w, c = t.shape
    hdr = _rfsi_header(w, h, c)
    arr = host.numpy()
    for i, p in enumerate(paths):
        with open(p, "wb") as f:
            f.write(hdr)
            f.write(np.ascontiguousarray(arr[i], dtype="<f4").tobytes())
