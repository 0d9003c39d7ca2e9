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
d = np.ctypeslib.as_array(host).reshape(12288, 16)[0 * 4096:0 * 4096 + n][:, :10]
ts = frame.view("tile_start", torch.int32, (n + 1,)).cpu().numpy()
ln = np.diff(ts)
print("phase ends: prologue gather hist scan+scatter rank - ties+write | seg-scan search+load-issue")
print("avg", d.mean(0).astype(int))
for r in np.argsort(-d[:, 7])[:6]:
    print("tile", r, "n", ln[r], d[r].astype(int))
