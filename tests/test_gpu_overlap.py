"""The overlapped launch chain (programmatic dependent launches: frame clear
-> K2 -> K3 -> K4a -> streaming K1 -> K4b, with the sorted-tile queue and
the live list consumed while pass A runs) must produce exactly what the
ordinary stream-ordered chain produces: the overlap changes when kernels
run, never what they compute.  The ordinary chain runs in a subprocess with
GSPARC_NO_PDL=1 (the switch is read once per process)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_RENDER = r"""
import sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose
from paper_2511_22793_b200.engine import Renderer
dc = DeviceCloud.from_host(bench.bench_cloud({n}, {f}))
R = Renderer()
out = []
for seed in (11, 12):
    tx = torch.as_tensor(bench.sample_tx(seed, 1), device="cuda")
    for _ in range(2):  # the second render reuses the frame (counters re-cleared)
        img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=True)
    c = frame.counters().cpu().numpy()
    out.append(img.cpu().numpy())
    out.append(frame.view("tile_start", torch.int32, (frame.layout.ntiles + 1,)).cpu().numpy())
    out.append(c[:4].copy())
np.savez({path!r}, *out)
"""


def _render(tmp_path, env_extra, tag, n=20000, f=52):
    path = str(tmp_path / f"{tag}.npz")
    env = dict(os.environ)
    env.update(env_extra)
    code = _RENDER.format(root=ROOT, n=n, f=f, path=path)
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    z = np.load(path)
    return [z[k] for k in sorted(z.files, key=lambda s: int(s.split("_")[1]))]


def test_overlapped_chain_matches_stream_order(tmp_path):
    a = _render(tmp_path, {}, "pdl")
    b = _render(tmp_path, {"GSPARC_NO_PDL": "1"}, "ordered")
    assert len(a) == len(b) == 6
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert np.array_equal(x, y), "overlapped and stream-ordered renders differ"
    # the renders have contributions and a live list
    assert np.abs(a[0]).max() > 0
    assert a[2][3] > 0
