"""Pass-B per-role timing for config 5 (experiments): GSPARC_PXB_DBG=1, one
4-TX render of the 500k-Gaussian scene at 720x180 (2048 columns in 16
channel-chunk CTAs per half tile; the rows hold the last-written chunk)."""
import ctypes, os, sys
os.environ["GSPARC_PXB_DBG"] = "1"
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
n = 1080
host = (ctypes.c_longlong * (12288 * 16))()
assert L.gsparc_debug_copy(host, ctypes.c_int64(12288 * 16)) == 0
d = np.ctypeslib.as_array(host).reshape(12288, 16)[2 * 4096:2 * 4096 + n].astype(np.float64)
nch = d[:, 11]
tot = d[:, 10]
print("CTAs %d, chunks per CTA mean %.1f max %d" % (n, nch.mean(), nch.max()))
print("cycles per CTA: total mean %.0f max %.0f; prologue %.0f; epilogue start %.0f (epilogue %.0f)" % (
    tot.mean(), tot.max(), d[:, 13].mean(), d[:, 14].mean(), (tot - d[:, 14]).mean()))
m = nch > 0
print("per chunk (group's own chunks = nch/2): wait-empty %.0f, compute %.0f, total/nch %.0f" % (
    ((d[m, 6] + d[m, 7]) / nch[m]).mean(), ((d[m, 8] + d[m, 9]) / nch[m]).mean(),
    ((d[m, 14] - d[m, 13]) / nch[m]).mean()))
wall = (d[:, 15] - d[:, 12]) / 1e3
print("wall per CTA us: mean %.1f max %.1f" % (wall.mean(), wall.max()))
