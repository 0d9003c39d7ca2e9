"""pytest plugin: run the REFERENCE's own test files against the drop-in.

Loaded with `-p refsuite_plugin` by tests/test_gpu_reference_suite.py in a
subprocess whose rootdir is the reference's test directory
(baseline/_ref/rfsplat_tests, installed by scripts/install_reference.sh).

It imports the unmodified `rfsplat` package, then replaces the module
`rfsplat.rasterizer` (and the names `rfsplat/__init__.py` re-exports) by the
B200 drop-in `paper_2511_22793_b200.rasterizer` before any test module or
`rfsplat.optimize` / `rfsplat.rfsim` / `rfsplat.cli` binds them -- the one
line a maintainer would change to switch backends.  The
reference's own types (`rfsplat.scene.GaussianCloud`,
`rfsplat.geometry.ViewPose`) are passed to the drop-in unchanged.

`rasterize_reference` stays the reference's CPU brute-force oracle
(rasterizer.py:237-259), so the oracle-agreement tests compare the GPU path
against the reference's own CPU code.  Set REFSUITE_GPU_ORACLE=1 to use the
drop-in's device f64 oracle instead.
"""

import os
import sys
import types

import rfsplat  # noqa: F401  (the unmodified reference)
import rfsplat.rasterizer as _cpu

from paper_2511_22793_b200 import rasterizer as _gpu

_shim = types.ModuleType("rfsplat.rasterizer")
_shim.__doc__ = "B200 drop-in for rfsplat.rasterizer (tests/refsuite/refsuite_plugin.py)"
for _name in dir(_cpu):
    if not _name.startswith("__"):
        setattr(_shim, _name, getattr(_cpu, _name))
for _name in ("rasterize_forward", "rasterize_backward", "ParamGradients",
              "RenderAux", "ALPHA_MAX", "ALPHA_MIN", "T_EPS", "TILE"):
    setattr(_shim, _name, getattr(_gpu, _name))
if os.environ.get("REFSUITE_GPU_ORACLE"):
    _shim.rasterize_reference = _gpu.rasterize_reference
_shim.BACKEND = "paper_2511_22793_b200"
sys.modules["rfsplat.rasterizer"] = _shim
rfsplat.rasterizer = _shim
for _name in ("ParamGradients", "RenderAux", "rasterize_backward",
              "rasterize_forward", "rasterize_reference"):
    setattr(rfsplat, _name, getattr(_shim, _name))
for _mod in ("rfsplat.optimize", "rfsplat.rfsim", "rfsplat.cli"):
    assert _mod not in sys.modules, f"{_mod} bound the CPU rasterizer early"


def _banner():
    return (f"rfsplat.rasterizer -> {_shim.BACKEND} (B200 drop-in); "
            f"rasterize_reference -> "
            f"{'GPU f64' if os.environ.get('REFSUITE_GPU_ORACLE') else 'reference CPU'}")


def pytest_report_header(config):
    return [_banner()]


def pytest_terminal_summary(terminalreporter):
    # also under -q, where the report header is suppressed
    terminalreporter.write_line(_banner())
