#!/usr/bin/env python
"""Benchmark of the GSpaRC render hot path on B200 (BASELINE.json metric:
"p50 per-TX render latency (ms); renders/s at 1/2/4/8 B200 vs CPU ref").

Default workload = BASELINE config 3 (the north_star latency target):
50k Gaussians (reference bench scene recipe, cli.py:239-246, GSPC-rounded),
90x360 equirect hemisphere x 52 OFDM subcarriers (C = 104 channels), one TX
per step, full pipeline K2 -> K3 -> K4a -> K1(live) -> K4b with the cloud
resident in HBM.  A step renders one transmitter position; `value` is
renders/s over all ranks (each rank renders its own TX shard, no
collective: weak scaling); ms_per_step / p50 / p99 are per-TX latency.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("p50 per-TX render latency (ms); renders/s at 1/2/4/8 B200 vs CPU "
          "ref")
CONFIGS = {
    # name: (N, W, H, F, tx per step)
    "c3": (50_000, 360, 90, 52, 1),
    "c1": (4_096, 360, 90, 1, 64),
    "c2": (16_384, 360, 90, 1, 32),   # training step (fwd+loss+bwd+Adam)
    # stress: 500k Gaussians, 180x720 x 256 subcarriers; 4096 TX over 8 GPUs
    # = 512 per GPU, rendered here 4 per step (geometry shared in a step)
    "c5": (500_000, 720, 180, 256, 4),
    # full training on a synthetic 5k-TX dataset (gen_dataset(seed=7, 5000,
    # random_scene(11, 6)), magnitude supervision), data-parallel: the
    # global batch of 32 TX is split across the ranks
    "c4": (16_384, 360, 90, 1, 32),
}
TRAIN_METRIC = "train iterations/s (global batch 32 TX)"


def device_bench_cloud(n, F, seed=0):
    """The bench-scene recipe (cli.py:239-246: uniform positions in
    [-5,-0.2,-5]x[5,3.2,5], log-scale ln(0.02 |diag|), identity rotations,
    logit -2, N(0,1) MLP weights x 0.3) drawn on the device with torch's
    generator -- the 17.6 GB of c5 weights never touch the host."""
    import torch
    from paper_2511_22793_b200 import DeviceCloud
    g = torch.Generator(device="cuda").manual_seed(seed)
    lo = torch.tensor([-5.0, -0.2, -5.0], dtype=torch.float64, device="cuda")
    hi = torch.tensor([5.0, 3.2, 5.0], dtype=torch.float64, device="cuda")
    pos = lo + (hi - lo) * torch.rand((n, 3), generator=g, dtype=torch.float64, device="cuda")
    diag = float(torch.linalg.norm(hi - lo))
    ls = torch.full((n, 3), float(np.log(0.02 * diag)), dtype=torch.float64, device="cuda")
    rot = torch.zeros((n, 4), dtype=torch.float64, device="cuda")
    rot[:, 0] = 1.0
    op = torch.full((n, 1), -2.0, dtype=torch.float64, device="cuda")
    dims = (5, 16, 2 * F)
    P = 5 * 16 + 16 + 16 * 2 * F + 2 * F
    mw = torch.randn((n, P), generator=g, dtype=torch.float32, device="cuda") * 0.3
    return DeviceCloud(pos.contiguous(), ls, rot, op, mw, dims)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-buffers", type=int, default=3,
                    help="render e2e: device/pinned image buffers in flight")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--deterministic", action="store_true",
                    help="c2: fixed-order (bit-reproducible) backward")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def dist_setup():
    """One process per GPU: cuda:LOCAL_RANK, NCCL.  With more ranks than
    visible GPUs (only for exercising the N>1 path on a 1-GPU box) ranks
    share devices and the collectives run over gloo; the line says so."""
    import torch
    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    oversub = world > ndev
    dev = local % max(ndev, 1)
    torch.cuda.set_device(dev)
    dist = None
    backend = None
    if world > 1:
        import torch.distributed as dist
        backend = "gloo" if oversub else "nccl"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    return rank, world, dev, dist, {"backend": backend,
                                    "oversubscribed": bool(oversub),
                                    "visible_gpus": ndev}


def self_launch(args):
    """`bench.py --gpus N` without torchrun: launch N ranks on this node
    (127.0.0.1 rendezvous) and pass rank 0's JSON line through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def sample_tx(seed, n, lo=(-4.0, 0.0, -4.0), hi=(4.0, 2.0, 4.0), keepout=1.0):
    """TX positions: rejection sampling of rfsim._sample_tx_positions
    (rfsim.py:120-128) around a receiver at the origin."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    while len(out) < n:
        p = rng.uniform(lo, hi)
        if np.linalg.norm(p) >= keepout:
            out.append(p)
    return np.asarray(out)


def bench_cloud(n, F):
    """Reference bench scene (cli.py:239-246) with mlp_out = 2F, rounded
    through GSPC so CPU and GPU see identical f32-representable values."""
    from paper_2511_22793_b200.scene import (SceneBounds, init_uniform,
                                             load_checkpoint, save_checkpoint)
    c = init_uniform(SceneBounds([-5, -0.2, -5], [5, 3.2, 5]), n, seed=0,
                     mlp_dims=(5, 16, 2 * F))
    c.mlp_weights *= 0.3
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "scene.gspc")
        save_checkpoint(p, c)
        return load_checkpoint(p)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,"
              "clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index),
                     f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------- CPU side
def host_info():
    """os.cpu_count() and the lscpu model name."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True,
                             timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_count": os.cpu_count() or 1, "model": model}


def oracle_cloud(cloud):
    import oracle as O
    return O.Cloud(*(np.asarray(getattr(cloud, g)) for g in O.GROUPS),
                   mlp_dims=cloud.mlp_dims)


def cpu_render(oc, tx, w, h, threads):
    """One full render with the NumPy oracle; returns (seconds, img, aux)."""
    import oracle as O
    t0 = time.perf_counter()
    img, aux = O.forward(oc, np.zeros(3), np.eye(3), tx, w, h, threads=threads)
    return time.perf_counter() - t0, img, aux


def _pool_render(a):
    oc, tx, w, h = a
    import oracle as O
    O.forward(oc, np.zeros(3), np.eye(3), tx, w, h, threads=1)


def cpu_pool_rate(oc, txs, w, h, procs):
    """renders/s of multiprocessing.Pool(procs) mapping distinct TX at
    threads=1."""
    import multiprocessing as mp
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_pool_render, [(oc, txs[0], w, h)] * procs)     # warm-up
        t0 = time.perf_counter()
        pool.map(_pool_render, [(oc, t, w, h) for t in txs])
        dt = time.perf_counter() - t0
    return len(txs) / dt


def stock_reference_pair_s(cloud, tx, w, h):
    """The UNMODIFIED reference (baseline/_ref/rfsplat, when installed) on one
    subcarrier pair of the C-wide cloud (a 5->16->2 head = rows of W2/b2;
    exact by linearity), threads=1; None if absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "rfsplat")):
        return None
    if ref not in sys.path:
        sys.path.append(ref)
    try:
        from rfsplat.geometry import ViewPose as RPose
        from rfsplat.rasterizer import rasterize_forward as rfwd
        from rfsplat.scene import GaussianCloud as RCloud
    except Exception:
        return None
    i, hd, o = cloud.mlp_dims
    mw = np.asarray(cloud.mlp_weights)
    head = i * hd + hd
    pair = np.concatenate([mw[:, :head], mw[:, head:head + 2 * hd],
                           mw[:, head + o * hd:head + o * hd + 2]], axis=1)
    rc = RCloud(np.asarray(cloud.positions), np.asarray(cloud.log_scales),
                np.asarray(cloud.rotations), np.asarray(cloud.raw_opacities),
                pair, mlp_dims=(i, hd, 2))
    t0 = time.perf_counter()
    rfwd(rc, RPose(np.zeros(3)), tx, w, h)
    return time.perf_counter() - t0


def cpu_baseline_render(cloud, txs, w, h, B, name, reps_n=5, budget_s=60.0):
    """CPU baseline of a render config on this host (rank 0, N=1 only):
    oracle latency at threads=N (>=5 reps) and threads=1, Pool renders/s
    (config 1), the stock reference per subcarrier pair (config 3).  Returns
    (cpu_baseline dict, oracle image + aux of txs[0] for the parity check)."""
    import oracle as O
    oc = oracle_cloud(cloud)
    hi = host_info()
    threads = hi["cpu_count"]
    t_first, img0, aux0 = cpu_render(oc, txs[0], w, h, threads)   # warm-up
    reps = max(1, min(reps_n, int(budget_s / 2 / max(t_first, 1e-3))))
    lat_n = [cpu_render(oc, txs[1 + k], w, h, threads)[0] for k in range(reps)]
    t1 = cpu_render(oc, txs[1], w, h, 1)[0]
    lat_1 = [t1]
    while sum(lat_1) < budget_s / 4 and len(lat_1) < reps_n:
        lat_1.append(cpu_render(oc, txs[1 + len(lat_1)], w, h, 1)[0])
    p = lambda v, q: 1e3 * float(np.percentile(v, q))
    out = {"value": B / (float(np.median(lat_n)) * B), "unit": "renders/s",
           "cores": threads, "kind": "port",
           "host": hi,
           "latency_ms": {"threads_N": {"threads": threads, "reps": len(lat_n),
                                        "p50": p(lat_n, 50), "p99": p(lat_n, 99)},
                          "threads_1": {"reps": len(lat_1), "p50": p(lat_1, 50),
                                        "p99": p(lat_1, 99)}},
           "sample": (f"NumPy oracle port (pinned to the reference by "
                      f"tests/test_oracle_golden.py) on the same GSPC-rounded "
                      f"scene: 1 warm-up + {len(lat_n)} full renders at "
                      f"threads={threads} (value = 1/p50) and {len(lat_1)} at "
                      f"threads=1, distinct TX")}
    if name == "c1":
        pool_tx = txs[:max(threads, 16)]
        rate = cpu_pool_rate(oc, pool_tx, w, h, threads)
        out["pool"] = {"renders_per_s": rate, "procs": threads,
                       "renders": len(pool_tx)}
        out["value"] = rate
        out["sample"] += (f"; value = multiprocessing.Pool({threads}) over "
                          f"{len(pool_tx)} distinct TX at threads=1")
    if name == "c3":
        pair = stock_reference_pair_s(cloud, txs[0], w, h)
        if pair is not None:
            F = cloud.mlp_dims[2] // 2
            out["stock_reference"] = {
                "pair_s_threads1": pair, "subcarriers": F,
                "extrapolated_render_s": pair * F,
                "renders_per_s": 1.0 / (pair * F),
                "note": "unmodified rfsplat.rasterize_forward on ONE "
                        "subcarrier pair (its rasterizer is 2-channel), "
                        "x F extrapolated: the reference's own way to "
                        "render CSI"}
    return out, (img0, aux0)


def image_parity(img, frame, ref_img, aux_ref, tol=1e-4):
    """SURVEY 8(d) parity metrics of one GPU render vs the oracle's:
    per-tile source sequences bit-exact, image normwise error on pixels
    whose contributor count agrees, threshold-flip count."""
    from paper_2511_22793_b200.rasterizer import RenderAux
    aux = RenderAux(frame, None, None, None, 0, np.float32, 0, None)
    got = aux.tile_sources()
    want = {k: aux_ref.prep.idx[v] for k, v in aux_ref.tiles.items()}
    tiles_ok = sorted(got) == sorted(want) and all(
        np.array_equal(got[k], want[k]) for k in want)
    cnt = frame.contrib_count().cpu().numpy()
    flip = cnt != aux_ref.contrib_count
    ok = ~flip
    err = np.abs(np.asarray(img, np.float64) - ref_img)
    scale = max(float(np.abs(ref_img).max()), 1e-30)
    e = float(err[ok].max(initial=0.0) / scale)
    return {"tiles_bit_exact": bool(tiles_ok),
            "pairs": int(sum(len(v) for v in want.values())),
            "image_normwise": e, "tolerance": tol, "flips": int(flip.sum()),
            "pixels": int(flip.size), "pass": bool(tiles_ok and e <= tol),
            "oracle": "oracle.forward f32 (NumPy restatement of "
                      "rasterizer.py:187-234)"}


def run_reference(args):
    """--impl reference: the reference algorithm (NumPy oracle port; the
    reference is pure Python and cannot be compiled) on host cores, rank 0
    only.  Render configs: full renders at threads=N.  Train configs: the
    per-TX train step (forward, magnitude, L1+SSIM, backward) scaled to the
    32-TX batch, plus one Adam update."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    n, w, h, F, B = CONFIGS[args.config]
    train = args.config in ("c2", "c4")
    cloud = bench_cloud(n, F) if args.config != "c5" else None
    if cloud is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "config 5 (17.6 GB scene) is not CPU-runnable; "
                          "see profiles/ for the reduced-size CPU sample"}))
        return 0
    oc = oracle_cloud(cloud)
    txs = sample_tx(1000, max(args.steps + args.warmup, 2) * (1 if train else B) + 1)
    threads = os.cpu_count() or 1
    budget_s = 150.0
    gt = np.random.default_rng(7).random((h, w, 1)) * 0.5

    def one(tx):
        t0 = time.perf_counter()
        img, aux = O.forward(oc, np.zeros(3), np.eye(3), tx, w, h,
                             threads=threads)
        if train:
            pred = O.magnitude(img)
            _, gp = O.loss_and_grad(pred, gt, 0.2)
            O.backward(O.magnitude_grad(img, gp[:, :, 0]), oc, tx, aux)
        return time.perf_counter() - t0

    t_one = one(txs[0])                                          # warm-up
    per_step_units = 1 if train else B
    k = max(1, min(args.steps, int(budget_s / max(t_one * per_step_units, 1e-9))))
    times = []
    for i in range(k):
        times.append(sum(one(txs[1 + i * per_step_units + b])
                         for b in range(per_step_units)))
    if train:
        g = {kk: np.zeros_like(v) for kk, v in oc.groups().items()}
        m = {kk: np.zeros_like(v) for kk, v in oc.groups().items()}
        v = {kk: np.zeros_like(a) for kk, a in oc.groups().items()}
        t0 = time.perf_counter()
        O.adam_update(oc.copy(), g, m, v, 0, O.AdamCfg())
        t_adam = time.perf_counter() - t0
        ms = 1e3 * (float(np.mean(times)) * B + t_adam)
        val, unit = 1e3 / ms, "it/s"
        sample = (f"{k} single-TX train steps (oracle forward + magnitude + "
                  f"L1/SSIM + backward, {n} Gaussians, {w}x{h}, threads="
                  f"{threads} for the forward tile pool) + one Adam update; "
                  f"a {B}-TX step = {B} x mean + Adam (extrapolated)")
        metric = TRAIN_METRIC
    else:
        ms = 1e3 * float(np.mean(times))
        val, unit = B * 1e3 / ms, "renders/s"
        sample = (f"{k} of {args.steps} requested steps timed (budget "
                  f"{budget_s:.0f} s), each a full {args.config} step: {B} "
                  f"render(s) of {n} Gaussians at {w}x{h}x{2 * F} channels "
                  f"with the NumPy oracle (tile thread pool, {threads} threads)")
        metric = METRIC
    line = {"impl": "reference", "metric": metric, "value": val,
            "unit": unit, "n_gpus": world, "steps": k,
            "warmup": 1, "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if train else "weak", "vs_baseline": None,
            "dtype": "f32" if not train else "f32 forward / f64 backward",
            "data": "synthetic (reference bench scene, seeded)",
            "config": workload_config(args.config),
            "cpu_baseline": {"value": val, "unit": unit,
                             "cores": threads, "kind": "port",
                             "host": host_info(), "sample": sample},
            "e2e": {"value": val, "unit": unit,
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not train:
        line["p50_ms"] = 1e3 * float(np.median(times)) / B
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name):
    n, w, h, F, B = CONFIGS[name]
    desc = {"c3": "config 3: CSI multi-frequency per-TX render latency",
            "c1": "config 1: batched forward of 64 TX positions",
            "c2": "config 2: training step (render + L1/SSIM + backward + "
                  "Adam) on a batch of 32 TX",
            "c5": "config 5 (stress): batched render, 4096 TX sharded over "
                  "the GPUs, 4 TX per step per GPU",
            "c4": "config 4: full training on a synthetic 5k-TX dataset, "
                  "data-parallel, global batch 32 TX split across the GPUs"}[name]
    return {"workload": f"{desc}; {n} Gaussians, {h}x{w} hemisphere x {F} "
                        f"subcarrier(s) ({2 * F} channels), {B} TX per step",
            "n_gaussians": n, "height": h, "width": w, "subcarriers": F,
            "channels": 2 * F, "tx_per_step": B,
            "scene": ("bench scene recipe (cli.py:239-246) drawn on the device"
                      if name == "c5" else
                      "reference bench scene (cli.py:239-246), GSPC-rounded"),
            "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": "tx-sharded (independent renders per GPU)"}


# ---------------------------------------------------------------- GPU side
def run_ours(args):
    import torch
    rank, world, local, dist, dinfo = dist_setup()
    from paper_2511_22793_b200 import DeviceCloud, ViewPose
    from paper_2511_22793_b200 import _lib
    from paper_2511_22793_b200.engine import Renderer
    from paper_2511_22793_b200.rasterizer import rasterize_forward_batch

    n, w, h, F, B = CONFIGS[args.config]
    C = 2 * F
    if args.config == "c5":  # 17.6 GB of weights: generated on the device
        cloud = None
        dc = device_bench_cloud(n, F)
        args.no_cpu_baseline = True
    else:
        cloud = bench_cloud(n, F)
        dc = DeviceCloud.from_host(cloud)
    pose = ViewPose(np.zeros(3))
    total_steps = args.steps + args.warmup
    # each rank renders its own TX shard (distinct seeds)
    txs_np = sample_tx(1000 + 7919 * rank, total_steps * B)
    tx_table = torch.as_tensor(txs_np, device="cuda").view(total_steps, B, 3)
    R = Renderer()
    lazy = C >= 16
    tx_buf = tx_table[0].clone()
    img, frame = R.forward(dc, pose, tx_buf, w, h, lazy=lazy)   # sizes frame
    cnt = R.check_frame(frame)
    pairs, kept = int(cnt[_lib.CNT_PAIRS]), int(cnt[_lib.CNT_KEPT])
    live = int(cnt[_lib.CNT_LIVE]) if lazy else None

    def step_eager():
        R.forward(dc, pose, tx_buf, w, h, frame=frame, image=img, lazy=lazy,
                  sync_check=False)

    graph = None
    if not args.no_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step_eager()
        torch.cuda.current_stream().wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step_eager()
    run = graph.replay if graph is not None else step_eager
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    for i in range(args.warmup):
        tx_buf.copy_(tx_table[i])
        run()
    torch.cuda.synchronize()

    def timed(nsteps, table_off):
        st = [torch.cuda.Event(enable_timing=True) for _ in range(nsteps)]
        en = [torch.cuda.Event(enable_timing=True) for _ in range(nsteps)]
        # hold the stream ~20 ms (untimed) so the host queues the steps
        # ahead of the device: a host hiccup (GIL, the clock sampler's
        # nvidia-smi) must not open a gap between a step's start event and
        # its launches
        torch.cuda._sleep(40_000_000)
        for i in range(nsteps):
            flush.fill_(i & 0xFF)                       # evict L2 (untimed)
            # the step's input (its TX) is placed in HBM before the timed
            # region, like the resident cloud
            tx_buf.copy_(tx_table[(table_off + i) % total_steps])
            st[i].record(stream)
            run()
            en[i].record(stream)
        torch.cuda.synchronize()
        return np.array([a.elapsed_time(b) for a, b in zip(st, en)])

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        times = timed(args.steps, args.warmup)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    R.check_frame(frame)
    total_ms = float(times.sum())
    if dist:
        total_ms = dist_max(dist, total_ms)
    renders = world * args.steps * B
    value = renders / (total_ms / 1e3)

    # ---- latency distribution: a separate >=1000-rep pass
    lat_reps = max(1000, args.steps)
    lat = timed(lat_reps, 0)
    R.check_frame(frame)
    per_step_launches = count_our_kernels(step_eager) or kernels_per_step(lazy)

    # ---- end-to-end through the public API (host TX in, host image out).
    # Renders run on the compute stream, each image's D2H on a copy stream
    # (double-buffered device images), so the copy of render i overlaps
    # render i+1 -- what a serving loop would do.  Every render's TX is
    # copied in from pinned memory and every image lands in pinned memory
    # inside the timed region.
    # NB image buffers in flight (render i reuses buffer i mod NB once its
    # copy from render i - NB has finished)
    NB = args.e2e_buffers
    pin_tx = [torch.empty((B, 3), dtype=torch.float64).pin_memory() for _ in range(NB)]
    pin_img = [torch.empty((B, h, w, C), dtype=torch.float32).pin_memory() for _ in range(NB)]
    dev_img = [img] + [torch.empty_like(img) for _ in range(NB - 1)]
    copy_stream = torch.cuda.Stream()
    rendered = [torch.cuda.Event() for _ in range(NB)]
    copied = [torch.cuda.Event() for _ in range(NB)]
    e2e_steps = min(args.steps, 100)
    checks = [None] * NB

    def e2e_run(n):
        for i in range(n):
            k = i % NB
            t = i % total_steps
            pin_tx[k].copy_(torch.as_tensor(txs_np[t * B:(t + 1) * B]))
            stream.wait_event(copied[k])          # image buffer k is free again
            tx_dev = pin_tx[k].to("cuda", non_blocking=True)
            # deferred overflow check: verified NB renders later, when
            # buffer k is reused (re-rendered on the rare overflow)
            if checks[k] is not None and not checks[k].ok():
                raise RuntimeError("pair buffer overflow in the e2e loop")
            out, _, checks[k] = rasterize_forward_batch(
                dc, pose, tx_dev, w, h, lazy=lazy, frame=frame,
                image=dev_img[k], sync=False)
            rendered[k].record(stream)
            copy_stream.wait_event(rendered[k])
            with torch.cuda.stream(copy_stream):
                pin_img[k].copy_(out, non_blocking=True)
                copied[k].record(copy_stream)

    e2e_run(4)
    torch.cuda.synchronize()
    e_s = torch.cuda.Event(enable_timing=True)
    e_e = torch.cuda.Event(enable_timing=True)
    e_s.record(stream)
    e2e_run(e2e_steps)
    stream.wait_stream(copy_stream)
    e_e.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e_s.elapsed_time(e_e) / e2e_steps
    if dist:
        e2e_ms = dist_max(dist, e2e_ms)
    e2e_val = world * B / (e2e_ms / 1e3)
    # the PCIe ceiling of that D2H: the same bytes, pinned, copy alone
    d2h_gbs = d2h_ceiling(dev_img[0], pin_img[0])

    # ---- per-stage timing (separate pass, CUDA events on the launch stream)
    stages = stage_times(R, dc, pose, tx_buf, w, h, frame, img, lazy, flush)
    dom = max(stages, key=lambda k: stages[k])
    # pass A and pass B take about the same time on config 3; the roofline
    # line reports pass B (the tensor-core stage, which moves most bytes)
    # unless another stage is clearly longer
    if "raster_accumulate" in stages and stages["raster_accumulate"] >= 0.95 * stages[dom]:
        dom = "raster_accumulate"

    # ---- parity of the benchmarked configuration (rank 0, N=1): the GPU
    # render of the cpu_baseline TX against the oracle's render of it
    cpu_line = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu_line, (ref_img, aux_ref) = cpu_baseline_render(
            cloud, txs_np, w, h, B, args.config)
        t0 = torch.as_tensor(txs_np[:1], device="cuda")
        pimg, pfr = R.forward(dc, pose, t0, w, h, lazy=lazy)
        parity = image_parity(pimg[0, ..., :C].cpu().numpy(), pfr, ref_img,
                              aux_ref)

    line = None
    if rank == 0:
        hbm, src = peaks()
        P = dc.P
        S = 4 * n * (11 + P)
        img_bytes = 4 * h * w * C * B
        bytes_fwd = S + B * (12 + 4 * h * w * C)
        ms = total_ms / args.steps
        nl = live if live is not None else n
        bytes_live = 44 * n + 4 * nl * P + B * (12 + 4 * h * w * C)
        roof = roofline_entry(dom, stages, n, P, C, B, h, w, live, pairs, hbm,
                              args.config)
        line = {
            "metric": METRIC, "value": value, "unit": "renders/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms,
            "p50_ms": float(np.percentile(lat, 50)),
            "p99_ms": float(np.percentile(lat, 99)),
            "latency_reps": int(lat_reps),
            "timed_p50_ms": float(np.percentile(times, 50)),
            "timed_p99_ms": float(np.percentile(times, 99)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": ("synthetic (bench scene recipe drawn on the device "
                                     "with torch's generator; random-init MLP weights)"
                                     if args.config == "c5" else
                                     "synthetic (reference bench scene recipe, "
                                     "seeded PCG64; random-init MLP weights)"),
            "config": dict(workload_config(args.config), **dinfo),
            "clocks": clocks.summary(),
            "e2e": {"value": e2e_val, "unit": "renders/s",
                    "h2d_bytes_per_step": 24 * B,
                    "d2h_bytes_per_step": img_bytes,
                    "ms_per_step": e2e_ms,
                    "d2h_ceiling_gbs": d2h_gbs,
                    "d2h_ceiling_renders_per_s": world * d2h_gbs * 1e9 / img_bytes * B
                    if d2h_gbs else None,
                    "path": "rasterize_forward_batch(pinned host TX -> device, "
                            "sync=False: each render's overflow flag read back "
                            "with it and checked before its buffer is reused) "
                            "+ D2H of every image into pinned memory on a copy "
                            "stream overlapping the next render",
                    "image_buffers": NB},
            "gpu_launches": int(args.steps * per_step_launches),
            "roofline": roof,
            "pipeline_hbm": {"algorithmic_bytes": bytes_fwd,
                             "achieved_gbs": bytes_fwd / (ms / 1e3) / 1e9,
                             "peak_gbs": hbm, "peak_source": src,
                             "frac": bytes_fwd / (ms / 1e3) / 1e9 / hbm,
                             "note": "SURVEY 8(d) bytes_fwd = S + B(12 + 4HWC)"
                                     " counts every Gaussian's MLP weights; "
                                     "the lazy MLP reads only live ones"},
            "pipeline_hbm_live": {"algorithmic_bytes": bytes_live,
                                  "achieved_gbs": bytes_live / (ms / 1e3) / 1e9,
                                  "frac": bytes_live / (ms / 1e3) / 1e9 / hbm,
                                  "note": "SURVEY 8(d) live-normalised: "
                                          "44N + 4 N_live P + B(12 + 4HWC)"},
            "live_fraction": (live / kept) if (live is not None and kept) else None,
            "pairs": pairs, "stages_us": stages,
            "stage_traffic": stage_traffic(stages, n, P, C, B, h, w, live, pairs,
                                           args.config),
        }
        if cpu_line is not None:
            line["cpu_baseline"] = cpu_line
            line["parity"] = parity
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def dist_max(dist, v):
    import torch
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def d2h_ceiling(src, dst, reps=20):
    """GB/s of a lone device->pinned-host copy of the image bytes."""
    import torch
    try:
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e.record()
        torch.cuda.synchronize()
        return src.numel() * src.element_size() * reps / (s.elapsed_time(e) / 1e3) / 1e9
    except Exception:
        return None


def kernels_per_step(lazy):
    # static fallback: frame clear, preprocess, tile_sort, raster pass(es), mlp
    return 6 if lazy else 5


def count_our_kernels(fn):
    """Kernels of libgsparc_b200 (names gs::k_*) launched by one call of fn,
    counted with the CUDA profiler (CUPTI); None if it is unavailable."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        n = sum(1 for e in prof.events()
                if e.device_type.name == "CUDA" and "gs::k_" in e.name)
        return n if n > 0 else None
    except Exception:
        return None


def stage_times(R, dc, pose, tx, w, h, frame, img, lazy, flush, reps=20):
    """Per-stage device time (us, median of reps, L2 flushed before each)."""
    import ctypes
    import torch
    from paper_2511_22793_b200._lib import check, lib
    L = frame.layout
    cc = dc.cstruct()
    view = pose.cstruct(w, h)
    C = dc.mlp_dims[2]
    B = int(tx.shape[0])
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    by = ctypes.byref
    calls = [("preprocess", lambda: check(lib().gsparc_prepare(
        by(cc), by(view), frame.ptr, by(L), st()))),
        ("bin_sort", lambda: check(lib().gsparc_bin_tiles(frame.ptr, by(L),
                                                          st())))]
    if lazy:
        calls += [("raster_weights", lambda: check(lib().gsparc_raster_forward(
            frame.ptr, by(L), B, C, 1e-4, 1, ctypes.c_void_p(img.data_ptr()),
            st()))),
            ("mlp_live", lambda: check(lib().gsparc_mlp_coef(
                by(cc), ctypes.c_void_p(tx.data_ptr()), B, 1, frame.ptr, by(L),
                st()))),
            ("raster_accumulate", lambda: check(lib().gsparc_raster_forward(
                frame.ptr, by(L), B, C, 1e-4, 2,
                ctypes.c_void_p(img.data_ptr()), st())))]
    else:
        calls += [("mlp", lambda: check(lib().gsparc_mlp_coef(
            by(cc), ctypes.c_void_p(tx.data_ptr()), B, 0, frame.ptr, by(L),
            st()))),
            ("raster_fused", lambda: check(lib().gsparc_raster_forward(
                frame.ptr, by(L), B, C, 1e-4, 0,
                ctypes.c_void_p(img.data_ptr()), st())))]
    res = {k: [] for k, _ in calls}
    stream = torch.cuda.current_stream()
    for _ in range(reps):
        flush.fill_(1)
        for name, fn in calls:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            res[name].append((a, b))
    torch.cuda.synchronize()
    return {k: float(np.median([a.elapsed_time(b) for a, b in v])) * 1e3
            for k, v in res.items()}


def ncu_kernel_stats(config, stage):
    """Per-launch DRAM traffic and issue/occupancy figures of a stage's
    kernel from the committed ncu --set full summary (profiles/ncu_kernels.json,
    written by scripts/ncu_summary.py from this round's capture); None if
    that config/stage was not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_kernels.json")) as f:
            return json.load(f)["configs"][config][stage]
    except (OSError, ValueError, KeyError):
        return None


def stage_bytes(n, P, C, B, h, w, live, pairs):
    """Algorithmic HBM bytes per launch of each render stage (DESIGN.md
    section 3's per-unit figures times the units of one launch)."""
    nl = live if live is not None else n
    return {
        # geometry read (f64 pos/scale/quat/logit = 88 B) + records written
        # (key 8 + rec32 32 + rect 16)
        "preprocess": n * (88 + 56),
        # rect + key read, pairs written and re-read/written by the sort
        "bin_sort": n * 24 + pairs * 8 * 3,
        # records gathered per visited pair are L2 hits; HBM-side: pairs +
        # aux planes written
        "raster_weights": pairs * 8 + h * w * 12 + n * 4,
        "mlp_live": nl * 4 * (P + B * C) + n * 4,
        "mlp": n * 4 * (P + B * C),
        "raster_accumulate": pairs * 8 + nl * 4 * B * C + 4 * h * w * B * C,
        "raster_fused": pairs * 8 + n * 4 * B * C + 4 * h * w * B * C + h * w * 12,
    }


def pipe_traffic(config):
    """In-pipeline DRAM bytes per stage (profiles/ncu_pipe_traffic.json,
    scripts/gpu_traffic_pipe.sh: ncu --cache-control none, so each kernel
    sees the L2 its predecessor left, as in the graph); {} if not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_pipe_traffic.json")) as f:
            return json.load(f)["configs"][config]
    except (OSError, ValueError, KeyError):
        return {}


def stage_traffic(stages, n, P, C, B, h, w, live, pairs, config):
    """Per stage: algorithmic bytes, measured in-pipeline DRAM bytes and
    their ratio (traffic well above the algorithmic bytes = wasted re-reads)."""
    per = stage_bytes(n, P, C, B, h, w, live, pairs)
    pt = pipe_traffic(config)
    out = {}
    for st in stages:
        if st not in per:
            continue
        d = pt.get(st, {}).get("dram_bytes")
        out[st] = {"algorithmic_bytes": per[st], "dram_bytes_in_pipeline": d,
                   "ratio": d / per[st] if d else None}
    return out


def roofline_entry(dom, stages, n, P, C, B, h, w, live, pairs, hbm, config):
    """Algorithmic bytes of the dominant stage / its measured duration."""
    us = stages[dom]
    per = stage_bytes(n, P, C, B, h, w, live, pairs)[dom]
    achieved = per / (us * 1e-6) / 1e9
    nc = ncu_kernel_stats(config, dom)
    out = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
           "unit": "GB/s", "frac": achieved / hbm,
           "traffic": nc.get("dram_bytes") if nc else None,
           "traffic_in_pipeline": pipe_traffic(config).get(dom, {}).get("dram_bytes"),
           "algorithmic_bytes": per, "launch_us": us,
           "note": "raster stages are issue/latency-bound (alpha compositing "
                   "on CUDA cores, sequential transmittance), so their HBM "
                   "fraction is low by nature; `latency` carries the ncu "
                   "issue-slot and occupancy figures of the same kernel"}
    if nc:
        out["latency"] = {k: v for k, v in nc.items() if k != "dram_bytes"}
    return out


def train_data(config, S, h, w):
    """(tx [S,3] f64 numpy, gt [S,h,w,1] f32 device).  c4: the reference's
    gen_dataset(seed=7, S, random_scene(11, 6), w, h) spectra (rfsim.py:
    131-172: PCG64 TX sampling, magnitude normalised by the dataset max),
    computed on the device with K9 instead of written as RFSI files.  c2:
    uniform random magnitude targets (round-1 workload)."""
    import torch
    if config == "c4":
        from paper_2511_22793_b200.rfsim import (_sample_tx_positions,
                                                 ground_truth_batch,
                                                 random_scene)
        scene = random_scene(11, 6)
        rng = np.random.Generator(np.random.PCG64(7))
        txs = _sample_tx_positions(rng, S, (-4.0, 0.0, -4.0), (4.0, 2.0, 4.0),
                                   scene.rx_position, 1.0)
        raw = torch.cat([ground_truth_batch(scene, txs[i:i + 512], w, h)
                         for i in range(0, S, 512)])
        gt = (raw / raw.max()).to(torch.float32)[..., None].contiguous()
        return txs, gt
    txs = sample_tx(7, S)
    gt = np.random.default_rng(7).random((S, h, w, 1), dtype=np.float32) * 0.5
    return txs, torch.as_tensor(gt, device="cuda")


def cpu_baseline_train(cloud, tx, gt, w, h, B, budget_s=40.0):
    """The oracle's per-TX train step (forward, magnitude, L1+SSIM,
    backward; optimize.py:273-296 without the Adam) on this host, x B +
    one Adam update = a B-TX step (the reference trains one TX per step)."""
    import oracle as O
    oc = oracle_cloud(cloud)
    threads = os.cpu_count() or 1
    ts = []
    while not ts or (sum(ts) < budget_s and len(ts) < 3):
        t0 = time.perf_counter()
        img, aux = O.forward(oc, np.zeros(3), np.eye(3), tx[len(ts)], w, h,
                             threads=threads)
        _, gp = O.loss_and_grad(O.magnitude(img), gt[len(ts)], 0.2)
        O.backward(O.magnitude_grad(img, gp[:, :, 0]), oc, tx[len(ts)], aux)
        ts.append(time.perf_counter() - t0)
    g = {k: np.zeros_like(v) for k, v in oc.groups().items()}
    t0 = time.perf_counter()
    O.adam_update(oc.copy(), g, {k: v.copy() for k, v in g.items()},
                  {k: v.copy() for k, v in g.items()}, 0, O.AdamCfg())
    t_adam = time.perf_counter() - t0
    step_s = float(np.median(ts)) * B + t_adam
    return {"value": 1.0 / step_s, "unit": "it/s", "cores": threads,
            "kind": "port", "host": host_info(),
            "per_tx_step_s": ts, "adam_s": t_adam,
            "sample": f"{len(ts)} single-TX oracle train steps (forward with a "
                      f"{threads}-thread tile pool, f64 backward) on the same "
                      f"scene and data; a {B}-TX step = {B} x median + one "
                      f"Adam update (extrapolated)"}


def train_stage_times(tr, flush, reps=10):
    """Per-stage device time (us) of the train step, L2 flushed first."""
    import torch
    calls = [("gather", tr._gather),
             ("render", lambda: tr.R.forward(tr.dev, tr.pose, tr.tx, tr.w, tr.h,
                                             frame=tr.frame, image=tr.img,
                                             lazy=False, sync_check=False)),
             ("loss", lambda: tr.loss.run(tr.img, tr.gt, tr.sup,
                                          tr.cfg.lambda_dssim)),
             ("backward", lambda: tr.R.backward(
                 tr.dev, tr.pose, tr.tx, tr.loss.dimg, tr.frame,
                 grad=tr.grad, deterministic=tr.cfg.deterministic)),
             ("adam", tr._update)]
    res = {k: [] for k, _ in calls}
    stream = torch.cuda.current_stream()
    for _ in range(reps):
        flush.fill_(1)
        for name, fn in calls:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            res[name].append((a, b))
    torch.cuda.synchronize()
    return {k: float(np.median([a.elapsed_time(b) for a, b in v])) * 1e3
            for k, v in res.items()}


def run_train(args):
    """--config c2 / c4: device train step (K2..K8) on a global batch of 32
    TX, data-parallel over ranks (contiguous shard per rank, one all-reduce
    of the flat gradient, identical Adam on every rank)."""
    import torch
    rank, world, local, dist, dinfo = dist_setup()
    from paper_2511_22793_b200 import ViewPose
    from paper_2511_22793_b200 import _lib
    from paper_2511_22793_b200.optimize import (TrainConfig, Trainer,
                                                sample_stream)
    n, w, h, F, B = CONFIGS[args.config]
    cloud = bench_cloud(n, F)
    S = 5000
    txs, gt = train_data(args.config, S, h, w)
    cfg = TrainConfig(width=w, height=h, batch_tx=B,
                      deterministic=args.deterministic)
    tr = Trainer(cloud, ViewPose(np.zeros(3)), cfg, txs, gt)
    if not args.no_graph:
        tr.capture()
    batches = list(sample_stream(S, cfg, 0, args.warmup + args.steps, B))
    for i in range(args.warmup):
        tr.step(batches[i])
    torch.cuda.synchronize()
    ok = tr.check()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for i in range(args.steps):
            stats = tr.step(batches[args.warmup + i])
        e1.record(stream)
        torch.cuda.synchronize()
    total_ms = e0.elapsed_time(e1)
    loss = float(stats[:, 0].mean().item())
    ok = tr.check() and ok
    if dist:
        total_ms = dist_max(dist, total_ms)
    ms = total_ms / args.steps
    per_step = count_our_kernels(lambda: tr.step(batches[0]))

    # ---- end to end: every step's TX and ground truth copied from pinned
    # host memory (the rank's shard of the batch), the step's loss stats
    # copied back to pinned memory
    Bl = tr.Bl
    gt_host = gt.cpu().pin_memory()
    tx_host = torch.as_tensor(np.asarray(txs, np.float64)).pin_memory()
    stage_gt = [torch.empty((Bl, h, w, 1), dtype=torch.float32).pin_memory()
                for _ in range(2)]
    stage_tx = [torch.empty((Bl, 3), dtype=torch.float64).pin_memory()
                for _ in range(2)]
    stats_host = [torch.empty((Bl, _lib.LOSS_STATS), dtype=torch.float64).pin_memory()
                  for _ in range(2)]
    # two device slots in the dataset buffers (samples [0, Bl) and [Bl, 2Bl)
    # are overwritten by the streamed batches): the H2D of step i+1 runs on
    # a copy stream while step i computes
    slot_idx = [torch.arange(k * Bl, (k + 1) * Bl, device="cuda") for k in range(2)]
    copy_stream = torch.cuda.Stream()
    copied = [torch.cuda.Event() for _ in range(2)]   # slot k filled (copy stream)
    used = [torch.cuda.Event() for _ in range(2)]     # slot k consumed (compute stream)
    for k in range(2):
        used[k].record(stream)
        copied[k].record(copy_stream)
    from paper_2511_22793_b200 import dp

    def e2e_run(nsteps):
        for i in range(nsteps):
            k = i & 1
            local_ids = dp.shard(np.asarray(batches[i % len(batches)]), tr.rank,
                                 tr.world)
            copied[k].synchronize()               # pinned stage k free again
            ids = torch.as_tensor(local_ids)
            torch.index_select(gt_host, 0, ids, out=stage_gt[k])
            torch.index_select(tx_host, 0, ids, out=stage_tx[k])
            copy_stream.wait_event(used[k])       # the step reading slot k is done
            with torch.cuda.stream(copy_stream):
                tr.gt_all[k * Bl:(k + 1) * Bl].copy_(stage_gt[k], non_blocking=True)
                tr.tx_all[k * Bl:(k + 1) * Bl].copy_(stage_tx[k], non_blocking=True)
                copied[k].record(copy_stream)
            stream.wait_event(copied[k])
            tr.idx.copy_(slot_idx[k])
            st = tr.step(None)
            used[k].record(stream)
            stats_host[k].copy_(st.to(torch.float64), non_blocking=True)

    e2e_steps = min(args.steps, 50)
    e2e_run(3)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_run(e2e_steps)
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / e2e_steps
    ok = tr.check() and ok
    if dist:
        e2e_ms = dist_max(dist, e2e_ms)

    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    stages = train_stage_times(tr, flush)
    line = None
    if rank == 0:
        hbm, src = peaks()
        P = tr.dev.P
        C = 2 * F
        Ssz = 4 * n * (11 + P)
        bytes_train = 10 * Ssz + B * 4 * h * w * (4 * C + 1)
        dom = max((k for k in stages if k != "gather"), key=lambda k: stages[k])
        roof = {"bound": "hbm", "kernel": f"train_step ({dom} dominates: "
                f"{stages[dom]:.0f} of {ms * 1e3:.0f} us)",
                "achieved": bytes_train / (ms / 1e3) / 1e9, "peak": hbm,
                "unit": "GB/s",
                "frac": bytes_train / (ms / 1e3) / 1e9 / hbm,
                "traffic": None, "algorithmic_bytes": bytes_train,
                "peak_source": src,
                "note": "SURVEY 8(d) bytes_train(B) = 10 S + B 4HW(4C + C_gt) "
                        "over the whole step (per-rank batch at N>1); the "
                        "step is latency-bound (per-TX raster chains)"}
        nc = ncu_kernel_stats(args.config, "backward")
        if nc:
            roof["latency"] = {"kernel": "backward", **nc}
        line = {"metric": TRAIN_METRIC,
                "value": 1e3 / ms, "unit": "it/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32",
                "data": ("synthetic 5k-TX dataset: gen_dataset(seed=7, 5000, "
                         "random_scene(11, 6)) spectra computed on the device "
                         "(K9), magnitude supervision"
                         if args.config == "c4" else
                         "synthetic (bench scene, random magnitude targets)"),
                "config": dict(workload_config(args.config),
                               parallelism=f"dp{world}",
                               per_rank_batch=Bl,
                               deterministic_backward=bool(args.deterministic),
                               l2="inputs (gt 648 MB + cloud) exceed L2; no flush",
                               **dinfo),
                "clocks": clocks.summary(), "renders_per_s": B * 1e3 / ms,
                "last_loss": loss, "healthy": bool(ok),
                "gpu_launches": int(per_step * args.steps) if per_step else None,
                "roofline": roof, "stages_us": stages,
                "e2e": {"value": 1e3 / e2e_ms, "unit": "it/s",
                        "ms_per_step": e2e_ms,
                        "h2d_bytes_per_step": Bl * (4 * h * w + 24),
                        "d2h_bytes_per_step": Bl * 8 * _lib.LOSS_STATS,
                        "path": "per step: the rank's batch of TX + ground "
                                "truth gathered on the host into pinned "
                                "memory, copied H2D on a copy stream into one "
                                "of two device slots (overlapping the previous "
                                "step), Trainer.step (graph + all-reduce + "
                                "Adam), loss stats copied D2H"}}
        if world == 1 and not args.no_cpu_baseline:
            gtn = gt[:3].double().cpu().numpy()
            line["cpu_baseline"] = cpu_baseline_train(cloud, txs[:3], gtn, w,
                                                      h, B)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.config in ("c2", "c4"):
        return run_train(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
