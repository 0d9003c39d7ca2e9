"""Per-warp included entries per chunk (ch_wm) of config 3's pass A: how many
of a chunk's 32 entries actually contribute to each consumer warp's 16x2
pixels -- the bound on per-warp entry skipping."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose
from paper_2511_22793_b200.engine import Renderer
dc = DeviceCloud.from_host(bench.bench_cloud(50000, 52))
R = Renderer()
tx = torch.as_tensor(bench.sample_tx(1000, 1), device="cuda")
img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=True)
torch.cuda.synchronize()
Ly = frame.layout
ts = frame.view("tile_start", torch.int32, (Ly.ntiles + 1,)).cpu().numpy().astype(np.int64)
chn = frame.view("ch_n", torch.int32, (2 * Ly.ntiles,)).cpu().numpy()
wm = frame.view("ch_wm", torch.int32, (int(Ly.ch_slots) * 4,)).cpu().numpy().view(np.uint32)
used = frame.view("ch_used", torch.int32, (int(Ly.ch_slots),)).cpu().numpy().view(np.uint32)
pc = lambda x: bin(int(x)).count("1")
rows = []
for cta in range(2 * Ly.ntiles):
    t, h = cta >> 1, cta & 1
    s, ln = ts[t], ts[t + 1] - ts[t]
    slot0 = 2 * ((s + 31 * t) >> 5) + h * ((ln + 31) >> 5)
    n = min(int(chn[cta]), int(Ly.pxw_chunks))
    if n == 0:
        continue
    per_w = [np.mean([pc(wm[(slot0 + c) * 4 + w]) for c in range(n)]) for w in range(4)]
    cta_used = np.mean([pc(used[slot0 + c]) for c in range(n)])
    rows.append((n, cta, cta_used, per_w))
rows.sort(key=lambda r: -r[0])
print("CTA-used entries per chunk (mean over CTAs): %.1f" % np.mean([r[2] for r in rows]))
print("per-warp included entries per chunk (mean): %s" % np.round(np.mean([r[3] for r in rows], 0), 1))
print("heaviest CTAs: chunks, cta, CTA-used/chunk, per-warp included/chunk")
for r in rows[:10]:
    print(r[0], r[1], round(r[2], 1), np.round(r[3], 1))
