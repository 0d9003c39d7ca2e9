"""CPU-side checks of the C ABI: the in-tree library loads, exports every
function declared in include/gsparc_b200.h, and the host-only entry points
(frame planning, error reporting) behave.  No kernels run here."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "gsparc_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+"
                                 r"(gsparc_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2511_22793_b200 import build
    build.build(verbose=False)
    from paper_2511_22793_b200 import _lib
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    from paper_2511_22793_b200 import _lib
    names = _declared()
    assert len(names) >= 12
    assert sorted(_lib.exported_symbols()) == names
    for n in names:
        assert hasattr(L, n), n


def test_abi_version(L):
    assert L.gsparc_abi_version() == 5


def test_plan_frame_layout(L):
    from paper_2511_22793_b200 import _lib
    lay = _lib.CLayout()
    rc = L.gsparc_plan_frame(4096, 360, 90, 128, 200000, _lib.F32, 1,
                             ctypes.byref(lay))
    assert rc == 0
    assert (lay.ntx, lay.nty, lay.ntiles) == (23, 6, 138)
    offs = [getattr(lay, "off_" + k) for k in _lib._LAYOUT_OFFSETS
            if k not in ("rec64", "pair_rec")]
    assert all(o % 256 == 0 for o in offs)
    assert len(set(offs)) == len(offs)
    assert lay.total_bytes >= lay.off_ggeo + 4096 * 8 * 4
    assert lay.off_pairs + 8 * 200000 <= lay.total_bytes
    # chunk slots bound the CTA chunk lists of any pair layout
    assert lay.ch_slots >= 2 * (200000 + 31 * 138) // 32
    assert lay.off_ch_T + 4 * 128 * lay.ch_slots <= lay.total_bytes
    # staged segments: one slot per (preprocess CTA of 128 Gaussians, tile)
    assert lay.seg_stride == 4096 // 128
    assert lay.off_stage % 256 == 0 and lay.off_seg % 256 == 0
    assert lay.off_stage + 8 * 200000 <= lay.off_seg
    assert lay.off_seg + 8 * 138 * lay.seg_stride <= lay.total_bytes
    # counters, tile_count, tile_cursor are contiguous (one clearing kernel)
    assert lay.off_counters < lay.off_tile_count < lay.off_tile_cursor < lay.off_key


def test_plan_frame_rejects_bad_args(L):
    from paper_2511_22793_b200 import _lib
    lay = _lib.CLayout()
    assert L.gsparc_plan_frame(16, 0, 90, 2, 100, _lib.F32, 0,
                               ctypes.byref(lay)) == _lib.ERR_ARG
    assert b"plan_frame" in L.gsparc_last_error()
    assert L.gsparc_plan_frame(16, 36, 9, 2, 100, 7, 0,
                               ctypes.byref(lay)) == _lib.ERR_ARG


def test_loss_scratch_bytes(L):
    assert L.gsparc_loss_scratch_bytes(2, 45, 90, 2) >= 8 * 11 * 2 * 2 * 45 * 90


def test_product_refuses_without_cuda(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2511_22793_b200 import _lib
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.require_cuda()


def test_library_is_sm100a(L):
    from paper_2511_22793_b200 import _lib
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
