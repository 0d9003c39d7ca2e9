"""Where does the config-3 end-to-end time go?  Times the bench's e2e loop
(rasterize_forward_batch, which host-syncs on the overflow counter every
call) against variants: no per-call sync (overflow read back with the image),
one stream, and the D2H alone.  Diagnostic only."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_22793_b200 import DeviceCloud, ViewPose  # noqa: E402
from paper_2511_22793_b200.engine import Renderer  # noqa: E402
from paper_2511_22793_b200.rasterizer import rasterize_forward_batch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n, w, h, F, B = bench.CONFIGS[cfg]
C = 2 * F
dc = DeviceCloud.from_host(bench.bench_cloud(n, F))
pose = ViewPose(np.zeros(3))
txs = bench.sample_tx(5, 400 * B)
R = Renderer()
lazy = C >= 16
img, frame = R.forward(dc, pose, torch.as_tensor(txs[:B], device="cuda"), w, h,
                       lazy=lazy)
stream = torch.cuda.current_stream()
cs = torch.cuda.Stream()
pin_tx = [torch.empty((B, 3), dtype=torch.float64).pin_memory() for _ in range(2)]
pin_img = [torch.empty((B, h, w, C), dtype=torch.float32).pin_memory() for _ in range(2)]
pin_cnt = [torch.empty(16, dtype=torch.int32).pin_memory() for _ in range(2)]
dev_img = [img, torch.empty_like(img)]
rendered = [torch.cuda.Event() for _ in range(2)]
copied = [torch.cuda.Event() for _ in range(2)]


def loop(nsteps, mode):
    for i in range(nsteps):
        k = i & 1
        pin_tx[k].copy_(torch.as_tensor(txs[i * B:(i + 1) * B]))
        stream.wait_event(copied[k])
        tx_dev = pin_tx[k].to("cuda", non_blocking=True)
        if mode == "sync":
            out, _ = rasterize_forward_batch(dc, pose, tx_dev, w, h, lazy=lazy,
                                             frame=frame, image=dev_img[k])
        else:
            out, _ = R.forward(dc, pose, tx_dev, w, h, frame=frame,
                               image=dev_img[k], lazy=lazy, sync_check=False)
        if mode == "onestream":
            pin_img[k].copy_(out, non_blocking=True)
            pin_cnt[k].copy_(frame.counters(), non_blocking=True)
            copied[k].record(stream)
            continue
        rendered[k].record(stream)
        cs.wait_event(rendered[k])
        with torch.cuda.stream(cs):
            pin_img[k].copy_(out, non_blocking=True)
            if mode != "sync":
                pin_cnt[k].copy_(frame.counters(), non_blocking=True)
            copied[k].record(cs)


def timeit(mode, nsteps=100):
    loop(4, mode)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    loop(nsteps, mode)
    stream.wait_stream(cs)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / nsteps


for mode in ("sync", "async", "onestream", "sync", "async"):
    ms = timeit(mode)
    print(f"{mode:10s} {ms * 1e3:8.1f} us/step  {B / ms * 1e3:9.1f} renders/s")
# D2H alone
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(50):
    pin_img[i & 1].copy_(dev_img[i & 1], non_blocking=True)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 50
print(f"d2h alone  {ms * 1e3:8.1f} us/step  {img.numel() * 4 / ms / 1e6:.1f} GB/s")
# render alone (graph-free, no sync)
a.record()
for i in range(50):
    R.forward(dc, pose, torch.as_tensor(txs[:B], device="cuda"), w, h, frame=frame,
              image=dev_img[0], lazy=lazy, sync_check=False)
b.record()
torch.cuda.synchronize()
print(f"render     {a.elapsed_time(b) / 50 * 1e3:8.1f} us/step (eager, no sync)")
