"""Print the frame counters of one config-3 render (kept, pairs, live ...)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose, _lib
from paper_2511_22793_b200.engine import Renderer
cloud = bench.bench_cloud(50000, 52)
dc = DeviceCloud.from_host(cloud)
R = Renderer()
tx = torch.as_tensor(bench.sample_tx(1000, 1), device="cuda")
img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=True)
torch.cuda.synchronize()
c = frame.counters().cpu().numpy()
print("kept", c[_lib.CNT_KEPT], "pairs", c[_lib.CNT_PAIRS], "live", c[_lib.CNT_LIVE],
      "bigtile", c[_lib.CNT_BIGTILE])
ts = frame.view("tile_start", torch.int32, (frame.layout.ntiles + 1,)).cpu().numpy()
print("max tile list", int(np.diff(ts).max()))
chn = frame.view("ch_n", torch.int32, (2 * frame.layout.ntiles,)).cpu().numpy()
print("chunks with contributions per CTA: mean", chn.mean(), "max", chn.max())
for lazy in (True, False):
    for _ in range(3):
        R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=lazy)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=lazy)
    e1.record(); torch.cuda.synchronize()
    print("lazy", lazy, "ms/render (eager launches)", e0.elapsed_time(e1) / 20)
# used-entry statistics of the pass-B chunks (popcount of ch_used)
img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=True)
torch.cuda.synchronize()
Ly = frame.layout
ts = frame.view("tile_start", torch.int32, (Ly.ntiles + 1,)).cpu().numpy().astype(np.int64)
chn = frame.view("ch_n", torch.int32, (2 * Ly.ntiles,)).cpu().numpy()
used = frame.view("ch_used", torch.int32, (int(Ly.ch_slots),)).cpu().numpy().view(np.uint32)
pops, ksteps = [], []
for cta in range(2 * Ly.ntiles):
    t, h = cta >> 1, cta & 1
    s, ln = ts[t], ts[t + 1] - ts[t]
    slot0 = 2 * ((s + 31 * t) >> 5) + h * ((ln + 31) >> 5)
    for c in range(chn[cta]):
        u = int(used[slot0 + c])
        pops.append(bin(u).count("1"))
        ksteps.append(sum(1 for k in range(4) if (u >> (8 * k)) & 0xFF))
pops, ksteps = np.array(pops), np.array(ksteps)
print("chunks", len(pops), "used entries/chunk mean", pops.mean(), "K-steps mean", ksteps.mean(),
      "compacted K-steps mean", np.ceil(pops / 8).mean())
