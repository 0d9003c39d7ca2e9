"""K5 work distribution (config 2): per half-tile CTA batches of 32 entries
(max wstop over its 4 warps), and the makespan of greedy list scheduling on
148 SMs (one CTA per SM) in launch order vs longest-first."""
import os, sys, heapq
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose
from paper_2511_22793_b200.engine import Renderer
cloud = bench.bench_cloud(16384, 1)
dc = DeviceCloud.from_host(cloud)
R = Renderer()
tx = torch.as_tensor(bench.sample_tx(7, 32), device="cuda")
img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, with_backward=True)
torch.cuda.synchronize()
nt = 138
ws = frame.view("wstop", torch.int32, (nt * 8,)).cpu().numpy().reshape(nt, 2, 4)
nb = (ws.max(axis=2) + 31) // 32          # [tile, half]
work = nb.reshape(-1).astype(float)        # blockIdx order = 2 tile + half
ov = 2.0                                   # per-CTA fixed cost in batch units (guess)
def makespan(order):
    h = [0.0] * 148
    for i in order:
        t = heapq.heappop(h)
        heapq.heappush(h, t + work[i] + ov)
    return max(h)
print("CTAs", len(work), "batches total", work.sum(), "max", work.max(), "mean %.1f" % work.mean())
print("per-SM lower bound %.1f" % ((work.sum() + ov * len(work)) / 148))
print("launch order makespan %.1f" % makespan(range(len(work))))
print("longest-first makespan %.1f" % makespan(np.argsort(-work, kind="stable")))
print("batches by tile row:", [int(nb.reshape(6, 23, 2)[r].sum()) for r in range(6)])
