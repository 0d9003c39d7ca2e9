"""Config-2 scene: list entries K5 visits per half tile (max wstop) against
the entries pass A marked used (ch_used bits), i.e. how much of the
backward's batch work is on entries with no contribution in the CTA."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose
from paper_2511_22793_b200.engine import Renderer
for n, F in ((16384, 1), (50000, 52)):
    cloud = bench.bench_cloud(n, F)
    dc = DeviceCloud.from_host(cloud)
    R = Renderer()
    tx = torch.as_tensor(bench.sample_tx(1000, 1), device="cuda")
    img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=False)
    torch.cuda.synchronize()
    L = frame.layout
    nt = int(L.ntiles)
    ts = frame.view("tile_start", torch.int32, (nt + 1,)).cpu().numpy().astype(np.int64)
    ws = frame.view("wstop", torch.int32, (nt * 8,)).cpu().numpy()
    chn = frame.view("ch_n", torch.int32, (2 * nt,)).cpu().numpy()
    used = frame.view("ch_used", torch.int32, (int(L.ch_slots),)).cpu().numpy().view(np.uint32)
    tot_visit = tot_used = tot_chunks = 0
    for t in range(nt):
        s, ln = ts[t], ts[t + 1] - ts[t]
        for hf in range(2):
            nv = ws[t * 8 + hf * 4: t * 8 + hf * 4 + 4].max()
            slot0 = 2 * ((s + 31 * t) >> 5) + hf * ((ln + 31) >> 5)
            u = used[slot0: slot0 + chn[2 * t + hf]]
            tot_visit += nv
            tot_used += int(sum(bin(int(x)).count("1") for x in u))
            tot_chunks += len(u)
    print(f"n={n} F={F}: pairs {ts[-1]}, K5 visited entries {tot_visit}, used entries {tot_used} "
          f"({100 * tot_used / max(tot_visit, 1):.1f}%), chunks with contributions {tot_chunks}")
