"""Pass-A per-role timing (experiments): run one config-3 render with
GSPARC_PXA_DBG=1 and summarise the clock64 counters per CTA."""
import ctypes, os, sys
os.environ["GSPARC_PXA_DBG"] = "1"
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
n = 276
host = (ctypes.c_longlong * (12288 * 16))()
assert L.gsparc_debug_copy(host, ctypes.c_int64(12288 * 16)) == 0
d = np.ctypeslib.as_array(host).reshape(12288, 16)[1 * 4096:1 * 4096 + n]
names = ["prod_wait_empty", "prod_total", "prod_chunks", "w0_wait_full", "w1_wait_full",
         "w2_wait_full", "w3_wait_full", "w0_comp", "w1_comp", "w2_comp", "w3_comp",
         "total", "nch"]
order = np.argsort(-d[:, 10])
print("avg:", {k: int(d[:, i].mean()) for i, k in enumerate(names)})
for r in order[:6]:
    print("cta", r, {k: int(d[r, i]) for i, k in enumerate(names)})
