"""K2 per-phase clocks (experiments): GSPARC_PREP_DBG=1, one config-3 render."""
import ctypes, os, sys
os.environ["GSPARC_PREP_DBG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose, _lib
from paper_2511_22793_b200.engine import Renderer
cloud = bench.bench_cloud(50000, 52)
dc = DeviceCloud.from_host(cloud)
R = Renderer()
tx = torch.as_tensor(bench.sample_tx(1000, 1), device="cuda")
for _ in range(4):
    img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=True)
torch.cuda.synchronize()
L = _lib.lib()
host = (ctypes.c_longlong * (16384 * 16))()
assert L.gsparc_debug_copy(host, ctypes.c_int64(16384 * 16)) == 0
n = 391
d = np.ctypeslib.as_array(host).reshape(16384, 16)[3 * 4096:3 * 4096 + n]
print("clock64 phase ends per CTA (cycles): warps 0-7 chain end | sync1 | rect+hist | scan | seg | scatter")
print("avg", d[:, :13].mean(0).astype(int))
print("max", d[:, :13].max(0).astype(int))
t = d[:, 14:16]
print("span us %.1f; start spread %.1f; per-CTA dur max %.1f mean %.1f" % (
    (t[:, 1].max() - t[:, 0].min()) / 1e3, (t[:, 0].max() - t[:, 0].min()) / 1e3,
    (t[:, 1] - t[:, 0]).max() / 1e3, (t[:, 1] - t[:, 0]).mean() / 1e3))
for r in np.argsort(-d[:, 12])[:5]:
    print("cta", r, d[r, :13].astype(int))
