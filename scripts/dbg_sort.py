"""Tile-sort per-phase clocks (experiments): GSPARC_SORT_DBG=1, one config-3 render."""
import ctypes, os, sys
os.environ["GSPARC_SORT_DBG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose, _lib
from paper_2511_22793_b200.engine import Renderer
cloud = bench.bench_cloud(50000, 52)
dc = DeviceCloud.from_host(cloud)
R = Renderer()
tx = torch.as_tensor(bench.sample_tx(1000, 1), device="cuda")
for _ in range(3):
    img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=True)
torch.cuda.synchronize()
L = _lib.lib()
n = 138
host = (ctypes.c_longlong * (12288 * 16))()
assert L.gsparc_debug_copy(host, ctypes.c_int64(12288 * 16)) == 0
d = np.ctypeslib.as_array(host).reshape(12288, 16)[0 * 4096:0 * 4096 + n][:, :11]
ts = frame.view("tile_start", torch.int32, (n + 1,)).cpu().numpy()
ln = np.diff(ts)
# cycle stamps since kernel start: 0 pdl_wait done, 1 prologue (descriptor
# and count loads, segment scan), 9 segment copies, 2 min/max, 3 histogram,
# 4 bucket scatter, 5 bucket rank, 7 ties
cols = [0, 1, 9, 2, 3, 4, 5, 7]
names = ["wait", "prolog", "copy", "minmax", "hist", "scatter", "rank", "ties"]
def row(v):
    st = v[cols].astype(int)
    return " ".join("%s=%d" % (nm, st[k] - (st[k - 1] if k else 0)) for k, nm in enumerate(names)) + " total_after_wait=%d" % (st[-1] - st[0])
print("per-phase cycles (differences of consecutive stamps)")
print("avg       ", row(d.mean(0)))
small = ln < 2000
print("avg n<2000", row(d[small].mean(0)), "tiles", small.sum())
print("avg n>=2000", row(d[~small].mean(0)))
for r in np.argsort(-d[:, 7])[:4]:
    print("tile", r, "n", ln[r], row(d[r]))
for r in np.where(small)[0][:4]:
    print("tile", r, "n", ln[r], row(d[r]))
