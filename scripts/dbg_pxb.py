"""Pass-B per-role timing (experiments): run one config-3 render with
GSPARC_PXB_DBG=1 and summarise the clock64 counters per CTA."""
import ctypes, os, sys
os.environ["GSPARC_PXB_DBG"] = "1"
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
d = np.ctypeslib.as_array(host).reshape(12288, 16)[2 * 4096:2 * 4096 + n]
names = ["mma_wait", "", "", "", "", "", "w0_waitE", "w1_waitE", "w0_comp", "w1_comp",
         "total", "nch", "", "t_prologue_end", "t_epilogue_start"]
order = np.argsort(-d[:, 10])
print("avg:", {k: int(d[:, i].mean()) for i, k in enumerate(names)})
for r in order[:6]:
    print("cta", r, {k: int(d[r, i]) for i, k in enumerate(names)})
