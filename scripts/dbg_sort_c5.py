"""Tile-sort per-phase clocks for config 5's long lists (experiments):
GSPARC_SORT_DBG=1, one 4-TX render of the 500k-Gaussian scene at 720x180."""
import ctypes, os, sys
os.environ["GSPARC_SORT_DBG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_22793_b200 import ViewPose, _lib
from paper_2511_22793_b200.engine import Renderer
dc = bench.device_bench_cloud(500000, 256)
R = Renderer()
tx = torch.as_tensor(bench.sample_tx(1000, 4), device="cuda")
for _ in range(3):
    img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 720, 180, lazy=True)
torch.cuda.synchronize()
L = _lib.lib()
n = 540
host = (ctypes.c_longlong * (12288 * 16))()
assert L.gsparc_debug_copy(host, ctypes.c_int64(12288 * 16)) == 0
d = np.ctypeslib.as_array(host).reshape(12288, 16)[:n]
ts = frame.view("tile_start", torch.int32, (n + 1,)).cpu().numpy()
ln = np.diff(ts)
# 0 pdl wait, 1 prologue, 9 gather (windows to L2), 2 min/max, 3 histogram,
# 4 bucket scatter to scratch, 5 windows ranked in shared memory, 15-14 ns
cols = [0, 1, 9, 2, 3, 4, 5]
names = ["wait", "prolog", "gather", "minmax", "hist", "scatter", "windows"]
def row(v):
    st = v[cols].astype(int)
    return " ".join("%s=%d" % (nm, st[k] - (st[k - 1] if k else 0)) for k, nm in enumerate(names)) + \
        " total=%d  wall %.1f us" % (st[-1], (v[15] - v[14]) / 1e3)
print("per-phase cycles; lists mean %.0f max %d" % (ln.mean(), ln.max()))
print("avg", row(d.mean(0)))
for r in np.argsort(-ln)[:5]:
    print("tile", r, "n", ln[r], row(d[r]))
t0 = d[:, 14].min()
print("CTA start..end (us): first end %.1f, last end %.1f" % ((d[:, 15].min() - t0) / 1e3, (d[:, 15].max() - t0) / 1e3))
