"""Per-CTA timeline of one config-3 render (experiments): globaltimer
start/end stamps of K2, K3 (per tile), K4a, K1 and K4b from the same render
(replayed from a CUDA graph with the L2 flushed, as bench.py; --eager for
host-enqueued launches), list lengths and pass A's chunks with contributions."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for e in ("GSPARC_SORT_DBG", "GSPARC_PXA_DBG", "GSPARC_PXB_DBG", "GSPARC_MLP_DBG", "GSPARC_PREP_DBG"):
    os.environ[e] = "1"
import numpy as np, torch
import bench
from paper_2511_22793_b200 import DeviceCloud, ViewPose, _lib
from paper_2511_22793_b200.engine import Renderer
cloud = bench.bench_cloud(50000, 52)
dc = DeviceCloud.from_host(cloud)
R = Renderer()
tx = torch.as_tensor(bench.sample_tx(1000, 1), device="cuda")
L = _lib.lib()
img, frame = R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, lazy=True)
torch.cuda.synchronize()
eager = "--eager" in sys.argv
def step():
    R.forward(dc, ViewPose(np.zeros(3)), tx, 360, 90, frame=frame, image=img, lazy=True,
              sync_check=False)
if eager:  # host-enqueued launches: later kernels may wait for the host
    for _ in range(5):
        step()
else:  # as bench.py: one CUDA graph per render, L2 flushed before it
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        flush.fill_(1)
        g.replay()
torch.cuda.synchronize()
host = (ctypes.c_longlong * (16384 * 16))()
assert L.gsparc_debug_copy(host, ctypes.c_int64(16384 * 16)) == 0
D = np.ctypeslib.as_array(host).reshape(4, 4096, 16)
nt = 138
ds, da, db = D[0, :nt], D[1, :2 * nt], D[2, :2 * nt]
ts = frame.view("tile_start", torch.int32, (nt + 1,)).cpu().numpy()
ln = np.diff(ts)
dk = D[3, :391]
t0 = dk[:, 14].min() if dk[:, 14].max() > 0 else ds[:, 14].min()
us = lambda v: (v - t0) / 1e3
s0, s1 = us(ds[:, 14]), us(ds[:, 15])
a0, a1 = us(da[:, 14]), us(da[:, 15])
b0, b1 = us(db[:, 12]), us(db[:, 15])
print("times in us from the first K2 CTA start (%s)" % ("eager" if eager else "graph, L2 flushed"))
print("K2  start %.1f..%.1f end max %.1f" % (us(dk[:, 14]).min(), us(dk[:, 14]).max(), us(dk[:, 15]).max()))
print("K3  start %.1f..%.1f end max %.1f mean %.1f" % (s0.min(), s0.max(), s1.max(), s1.mean()))
print("K4a start %.1f..%.1f end max %.1f; dur max %.1f mean %.1f" % (a0.min(), a0.max(), a1.max(), (a1 - a0).max(), (a1 - a0).mean()))
dm = D[3, 2048:2048 + 148]
m0, m1, mw = us(dm[:, 14]), us(dm[:, 15]), us(dm[:, 13])
print("K1  start %.1f..%.1f last Gaussian done %.1f end max %.1f" % (m0.min(), m0.max(), mw[dm[:, 13] > 0].max(), m1.max()))
bw = us(db[:, 5])
print("K4b work start (after the grid-dependency wait) %.1f..%.1f; work dur max %.1f mean %.1f" % (bw.min(), bw.max(), (b1 - bw).max(), (b1 - bw).mean()))
for c in np.argsort(-(b1 - bw))[:6]:
    print("  K4b cta", c, "nch", db[c, 11], "placed %.1f work %.1f..%.1f" % (b0[c], bw[c], b1[c]))
print("K4b start %.1f..%.1f end max %.1f; dur max %.1f mean %.1f" % (b0.min(), b0.max(), b1.max(), (b1 - b0).max(), (b1 - b0).mean()))
wait = a0 - np.repeat(s1, 2)
print("pass A start - own sort end: min %.1f max %.1f mean %.1f" % (wait.min(), wait.max(), wait.mean()))
print("tile len  sort[s,e]  passA[s,e]x2  nch  passB dur")
for t in np.argsort(-np.maximum(a1[0::2], a1[1::2]))[:12]:
    print(t, ln[t], "[%.1f %.1f]" % (s0[t], s1[t]),
          "[%.1f %.1f] [%.1f %.1f]" % (a0[2 * t], a1[2 * t], a0[2 * t + 1], a1[2 * t + 1]),
          da[2 * t:2 * t + 2, 12], ((db[2 * t:2 * t + 2, 15] - db[2 * t:2 * t + 2, 12]) / 1e3).round(1))
# pass A: consumers finished (stamp 11, cycles after the CTA start) -> CTA end
# (live-list append, completion count, final grid wait)
cons = a0 + (da[:, 11] - da[:, 13]) / 1965.0
tail = a1 - cons
print("pass A consumers done -> CTA end (live-list append): max %.1f mean %.1f us; latest consumer end %.1f, latest CTA end %.1f"
      % (tail.max(), tail.mean(), cons.max(), a1.max()))
# pass A roles of the last-finishing CTAs (cycles): producer waiting for a
# free ring slot, consumers waiting for a filled one / walking
print("pass A roles (cycles): cta tile.half nchunks prod_wait_empty prod_end | cons wait_full x4 | cons walk x4")
for c in np.argsort(-a1)[:10]:
    print(" ", c, "%d.%d" % (c >> 1, c & 1), da[c, 2], da[c, 0], da[c, 1], "|", da[c, 3:7], "|", da[c, 7:11])
