"""Pass-B per-chunk phase split (experiments, config 3).  Reads the
GSPARC_PXB_DBG rows; the per-phase clock64 stamps it prints (slots 0-5, 8-9,
12-13) were a temporary patch of k_pxb's chunk loop (see
profiles/r02/SUMMARY.md), not kept in the kernel."""
import ctypes, os, sys
os.environ["GSPARC_PXB_DBG"] = "1"
sys.path.insert(0, "/root/repo")
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
host = (ctypes.c_longlong * (12288 * 16))()
assert L.gsparc_debug_copy(host, ctypes.c_int64(12288 * 16)) == 0
d = np.ctypeslib.as_array(host).reshape(12288, 16)[2 * 4096:2 * 4096 + 276].astype(float)
nch = d[:, 11]
m = nch > 0
def per(col): return (d[m, col] / np.maximum(1, nch[m] / 2)).mean()
print("per chunk per group (cycles): weights->TMEM g0 %.0f g1 %.0f | coef->smem g0 %.0f g1 %.0f | wait-empty g0 %.0f g1 %.0f | token g0 %.0f g1 %.0f | leader full-wait g0 %.0f" % (
    per(0), per(1), per(2), per(3), per(6), per(7), per(8), per(9), per(4)))
print("issue (chunk start -> loads issued) g0 %.0f g1 %.0f; gap chunk end -> next chunk start g0 %.0f" % (per(12), per(13), per(5)))
print("chunk start -> list index stored (waits for the prefetched index) g1 %.0f" % per(9))
print("CTA total %.0f, prologue %.0f, epilogue %.0f, main/nch %.0f" % (d[m,10].mean(), d[m,13].mean(), (d[m,10]-d[m,14]).mean(), ((d[m,14]-d[m,13])/nch[m]).mean()))
top = np.argsort(-d[:, 10])[:3]
for r in top:
    print("cta", r, "nch", nch[r], "total", d[r,10], "ta", d[r,0], d[r,1], "tb", d[r,2], d[r,3], "tw", d[r,6], d[r,7], "tok", d[r,8], d[r,9], "full", d[r,4])
