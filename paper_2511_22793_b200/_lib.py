"""ctypes binding of libgsparc_b200.so (include/gsparc_b200.h).

The CUDA library is the only compute path.  If it is missing, or no CUDA
device is visible, every product entry point raises -- there is no CPU
fallback.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgsparc_b200.so")
ABI_VERSION = 5
LOSS_STATS = 6  # GSPARC_LOSS_STATS

OK, ERR_ARG, ERR_CUDA, ERR_UNSUPPORTED = 0, 1, 2, 3
F32, F64 = 0, 1
LAZY_MLP, FORCE_FUSED = 1, 2
CNT_KEPT, CNT_PAIRS, CNT_OVERFLOW, CNT_LIVE, CNT_NONFINITE, CNT_BIGTILE, CNT_SORTED, CNT_CLAIMED, CNT_PXA_DONE = range(9)
NUM_COUNTERS = 16

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, \
    ctypes.c_void_p


class CCloud(ctypes.Structure):
    _fields_ = [("n", c_i64), ("mlp_in", c_i32), ("mlp_hidden", c_i32),
                ("mlp_out", c_i32), ("reserved", c_i32),
                ("positions", c_vp), ("log_scales", c_vp), ("rotations", c_vp),
                ("raw_opacities", c_vp), ("mlp_weights", c_vp),
                ("mlp_weights64", c_vp)]


class CView(ctypes.Structure):
    _fields_ = [("rx", c_dbl * 3), ("rotation", c_dbl * 9),
                ("width", c_i32), ("height", c_i32)]


_LAYOUT_OFFSETS = ("key", "rec32", "rec64", "rect", "counters", "tile_count",
                   "tile_cursor", "tile_start", "tile_stop", "pairs", "T",
                   "count", "last", "live", "live_list", "coef", "gcoef",
                   "ggeo", "pair_rec", "wstop", "rrec", "ch_idx", "ch_T",
                   "ch_n", "ch_rec")


class CLayout(ctypes.Structure):
    _fields_ = ([("total_bytes", c_i64), ("n", c_i64), ("pair_capacity", c_i64),
                 ("channels", c_i64)] +
                [(k, c_i32) for k in ("width", "height", "ntx", "nty", "ntiles",
                                      "dtype", "with_backward", "reserved")] +
                [("off_" + k, c_i64) for k in _LAYOUT_OFFSETS] +
                [("ch_slots", c_i64), ("off_ch_used", c_i64),
                 ("off_det_gcoef", c_i64), ("off_det_ggeo", c_i64),
                 ("off_stage", c_i64), ("off_seg", c_i64), ("seg_stride", c_i64),
                 ("off_pxw", c_i64), ("pxw_chunks", c_i64), ("off_ch_wm", c_i64),
                 ("off_det_inv", c_i64), ("off_sort_tmp", c_i64),
                 ("off_ch_pos", c_i64)])


class CEmitter(ctypes.Structure):
    _fields_ = [("position", c_dbl * 3), ("gain_re", c_dbl), ("gain_im", c_dbl),
                ("angular_spread", c_dbl)]


class CAdamConfig(ctypes.Structure):
    _fields_ = [(k, c_dbl) for k in (
        "position_lr_init", "position_lr_final", "position_lr_delay_mult",
        "position_lr_max_steps", "opacity_lr", "scaling_lr", "rotation_lr",
        "mlp_lr", "beta1", "beta2", "eps")]


_lib = None


def lib():
    """Load (once) and return the library; raise loudly if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with "
            "`python -m paper_2511_22793_b200.build` (no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    sig = {
        "gsparc_abi_version": (c_i32, []),
        "gsparc_last_error": (ctypes.c_char_p, []),
        "gsparc_plan_frame": (c_i32, [c_i64, c_i32, c_i32, c_i64, c_i64, c_i32,
                                      c_i32, P(CLayout)]),
        "gsparc_prepare": (c_i32, [P(CCloud), P(CView), c_vp, P(CLayout), c_vp]),
        "gsparc_bin_tiles": (c_i32, [c_vp, P(CLayout), c_vp]),
        "gsparc_mlp_coef": (c_i32, [P(CCloud), c_vp, c_i32, c_i32, c_vp,
                                    P(CLayout), c_vp]),
        "gsparc_raster_forward": (c_i32, [c_vp, P(CLayout), c_i32, c_i32, c_dbl,
                                          c_i32, c_vp, c_vp]),
        "gsparc_render_forward": (c_i32, [P(CCloud), P(CView), c_vp, c_i32,
                                          c_dbl, c_i32, c_vp, P(CLayout), c_vp,
                                          c_vp]),
        "gsparc_render_backward": (c_i32, [P(CCloud), P(CView), c_vp, c_i32,
                                           c_vp, c_i32, c_vp, P(CLayout), c_vp,
                                           c_i32, c_vp]),
        "gsparc_loss_scratch_bytes": (c_i64, [c_i32, c_i32, c_i32, c_i32]),
        "gsparc_loss_fwd_bwd": (c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32,
                                        c_i32, c_i32, c_dbl, c_vp, c_vp, c_vp,
                                        c_i64, c_vp]),
        "gsparc_adam_step": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32,
                                     c_vp, c_vp, c_vp, c_vp, c_vp,
                                     P(CAdamConfig), c_vp]),
        "gsparc_gt_spectrum": (c_i32, [c_vp, c_i32, P(c_dbl), c_dbl, c_vp, c_i32,
                                       c_i32, c_i32, c_dbl, c_i32, c_vp, c_vp]),
        "gsparc_rssi_energy": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_i32, c_i32,
                                       c_vp, c_i64, c_vp, c_vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    got = L.gsparc_abi_version()
    if got != ABI_VERSION:
        raise ImportError(f"libgsparc_b200 ABI {got}, expected {ABI_VERSION}")
    _lib = L
    return L


def exported_symbols():
    """Names declared in include/gsparc_b200.h (for the ABI test)."""
    return ["gsparc_abi_version", "gsparc_last_error", "gsparc_plan_frame",
            "gsparc_prepare", "gsparc_bin_tiles", "gsparc_mlp_coef",
            "gsparc_raster_forward", "gsparc_render_forward",
            "gsparc_render_backward", "gsparc_loss_scratch_bytes",
            "gsparc_loss_fwd_bwd", "gsparc_adam_step", "gsparc_gt_spectrum",
            "gsparc_rssi_energy"]


class GsparcError(RuntimeError):
    pass


def check(rc):
    if rc != OK:
        msg = lib().gsparc_last_error().decode(errors="replace")
        raise GsparcError(f"libgsparc_b200 error {rc}: {msg}")


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2511_22793_b200 needs a CUDA device "
                           "(B200, sm_100a); there is no CPU fallback")
    lib()
