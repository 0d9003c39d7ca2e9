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
}


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
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--deterministic", action="store_true",
                    help="c2: fixed-order (bit-reproducible) backward")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


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
def cpu_render_time(cloud, tx, w, h, threads):
    """Time one full render of the same scene with the NumPy oracle."""
    import oracle as O
    oc = O.Cloud(*(np.asarray(getattr(cloud, g)) for g in O.GROUPS),
                 mlp_dims=cloud.mlp_dims)
    t0 = time.perf_counter()
    O.forward(oc, np.zeros(3), np.eye(3), tx, w, h, threads=threads)
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the reference algorithm (NumPy oracle port; the
    reference is pure Python and cannot be compiled) on host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    n, w, h, F, B = CONFIGS[args.config]
    cloud = bench_cloud(n, F)
    txs = sample_tx(1000, max(args.steps + args.warmup, 1))
    threads = os.cpu_count() or 1
    budget_s = 150.0
    t_one = cpu_render_time(cloud, txs[0], w, h, threads)      # warm-up
    k = max(1, min(args.steps, int(budget_s / max(t_one * B, 1e-9))))
    times = []
    for i in range(k):
        t = 0.0
        for b in range(B):
            t += cpu_render_time(cloud, txs[(1 + i * B + b) % len(txs)], w, h,
                                 threads)
        times.append(t)
    ms = 1e3 * float(np.mean(times))
    val = B * 1e3 / ms
    sample = (f"{k} of {args.steps} requested steps timed (budget {budget_s:.0f}"
              f" s), each a full {args.config} step: {B} render(s) of {n} "
              f"Gaussians at {w}x{h}x{2 * F} channels with the NumPy oracle "
              f"(tile thread pool, {threads} threads)")
    line = {"impl": "reference", "metric": METRIC, "value": val,
            "unit": "renders/s", "n_gpus": world, "steps": k,
            "warmup": 1, "ms_per_step": ms, "p50_ms": 1e3 * float(np.median(times)) / B,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (reference bench scene, seeded)",
            "config": workload_config(args.config),
            "cpu_baseline": {"value": val, "unit": "renders/s",
                             "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": val, "unit": "renders/s",
                    "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name):
    n, w, h, F, B = CONFIGS[name]
    desc = {"c3": "config 3: CSI multi-frequency per-TX render latency",
            "c1": "config 1: batched forward of 64 TX positions",
            "c2": "config 2: training step (render + L1/SSIM + backward + "
                  "Adam) on a batch of 32 TX",
            "c5": "config 5 (stress): batched render, 4096 TX sharded over "
                  "the GPUs, 4 TX per step per GPU"}[name]
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
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)                       # evict L2 (untimed)
            starts[i].record(stream)
            tx_buf.copy_(tx_table[args.warmup + i])
            run()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    R.check_frame(frame)
    per_step_launches = count_our_kernels(step_eager) or kernels_per_step(lazy)
    times = np.array([s.elapsed_time(e) for s, e in zip(starts, ends)])
    total_ms = float(times.sum())
    if dist:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    renders = world * args.steps * B
    value = renders / (total_ms / 1e3)

    # ---- end-to-end through the public API (host TX in, host image out).
    # Renders run on the compute stream, each image's D2H on a copy stream
    # (double-buffered device images), so the copy of render i overlaps
    # render i+1 -- what a serving loop would do.  Every render's TX is
    # copied in from pinned memory and every image lands in pinned memory
    # inside the timed region.
    pin_tx = [torch.empty((B, 3), dtype=torch.float64).pin_memory() for _ in range(2)]
    pin_img = [torch.empty((B, h, w, C), dtype=torch.float32).pin_memory() for _ in range(2)]
    dev_img = [img, torch.empty_like(img)]
    copy_stream = torch.cuda.Stream()
    rendered = [torch.cuda.Event() for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    e2e_steps = min(args.steps, 100)

    def e2e_run(n):
        for i in range(n):
            k = i & 1
            t = i % total_steps
            pin_tx[k].copy_(torch.as_tensor(txs_np[t * B:(t + 1) * B]))
            stream.wait_event(copied[k])          # image buffer k is free again
            tx_dev = pin_tx[k].to("cuda", non_blocking=True)
            out, _ = rasterize_forward_batch(dc, pose, tx_dev, w, h, lazy=lazy,
                                             frame=frame, image=dev_img[k])
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
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = world * B / (e2e_ms / 1e3)

    # ---- per-stage timing (separate pass, CUDA events on the launch stream)
    stages = stage_times(R, dc, pose, tx_buf, w, h, frame, img, lazy, flush)
    dom = max(stages, key=lambda k: stages[k])
    # pass A and pass B take about the same time on config 3; the roofline
    # line reports pass B (the tensor-core stage, which moves most bytes)
    # unless another stage is clearly longer
    if "raster_accumulate" in stages and stages["raster_accumulate"] >= 0.95 * stages[dom]:
        dom = "raster_accumulate"

    line = None
    if rank == 0:
        hbm, src = peaks()
        P = dc.P
        S = 4 * n * (11 + P)
        img_bytes = 4 * h * w * C * B
        bytes_fwd = S + B * (12 + 4 * h * w * C)
        ms = total_ms / args.steps
        roof = roofline_entry(dom, stages, n, P, C, B, h, w, live, pairs, hbm)
        line = {
            "metric": METRIC, "value": value, "unit": "renders/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "p50_ms": float(np.percentile(times, 50)),
            "p99_ms": float(np.percentile(times, 99)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": ("synthetic (bench scene recipe drawn on the device "
                                     "with torch's generator; random-init MLP weights)"
                                     if args.config == "c5" else
                                     "synthetic (reference bench scene recipe, "
                                     "seeded PCG64; random-init MLP weights)"),
            "config": workload_config(args.config),
            "clocks": clocks.summary(),
            "e2e": {"value": e2e_val, "unit": "renders/s",
                    "h2d_bytes_per_step": 24 * B,
                    "d2h_bytes_per_step": img_bytes,
                    "ms_per_step": e2e_ms,
                    "path": "rasterize_forward_batch(pinned host TX -> device) "
                            "+ D2H of every image into pinned memory on a copy "
                            "stream overlapping the next render"},
            "gpu_launches": int(args.steps * per_step_launches),
            "roofline": roof,
            "pipeline_hbm": {"algorithmic_bytes": bytes_fwd,
                             "achieved_gbs": bytes_fwd / (ms / 1e3) / 1e9,
                             "peak_gbs": hbm, "peak_source": src,
                             "frac": bytes_fwd / (ms / 1e3) / 1e9 / hbm,
                             "note": "SURVEY 8(d) bytes_fwd = S + B(12 + 4HWC)"
                                     " counts every Gaussian's MLP weights; "
                                     "the lazy MLP reads only live ones"},
            "live_fraction": (live / kept) if (live is not None and kept) else None,
            "pairs": pairs, "stages_us": stages,
        }
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            t = cpu_render_time(cloud, txs_np[0], w, h, threads)
            line["cpu_baseline"] = {
                "value": 1.0 / t, "unit": "renders/s", "cores": threads,
                "kind": "port",
                "sample": f"1 full render (same scene, TX {[round(float(v), 3) for v in txs_np[0]]}) "
                          "with the NumPy oracle, tile thread pool"}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


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


def roofline_entry(dom, stages, n, P, C, B, h, w, live, pairs, hbm):
    """Algorithmic bytes of the dominant stage / its measured duration."""
    us = stages[dom]
    nl = live if live is not None else n
    per = {
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
    }[dom]
    achieved = per / (us * 1e-6) / 1e9
    # DRAM bytes (read + write) of the same kernel per launch, from the
    # committed ncu --set full capture of this config (null if none)
    traffic = None
    try:
        tf = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                         "profiles", "r01", "ncu_traffic_c3.json")))
        if n == 50000 and C == 104:
            traffic = tf["per_launch_bytes"].get(dom)
    except (OSError, ValueError, KeyError):
        pass
    return {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm,
            "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
            "algorithmic_bytes": per, "launch_us": us,
            "note": "raster stages are issue/latency-bound (alpha compositing "
                    "on CUDA cores), so their HBM fraction is low by nature; "
                    "see profiles/ for issue-slot utilisation"}


def run_train(args):
    """--config c2: device train step (K2..K8), batch of 32 TX per step,
    data-parallel over ranks (global batch split, NCCL all-reduce)."""
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2511_22793_b200 import ViewPose
    from paper_2511_22793_b200.optimize import TrainConfig, Trainer
    n, w, h, F, B = CONFIGS[args.config]
    cloud = bench_cloud(n, F)
    S = 5000                                  # config-4 sized sample table
    txs = sample_tx(7, S)
    gt = np.random.default_rng(7).random((S, h, w, 1), dtype=np.float32) * 0.5
    cfg = TrainConfig(width=w, height=h, batch_tx=B, deterministic=args.deterministic)
    tr = Trainer(cloud, ViewPose(np.zeros(3)), cfg, txs, gt)
    if not args.no_graph:
        tr.capture()
    rng = np.random.Generator(np.random.PCG64(0))
    batches = [rng.integers(S, size=B) for _ in range(args.warmup + args.steps)]
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
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    per_step = count_our_kernels(lambda: tr.step(batches[0]))
    line = None
    if rank == 0:
        line = {"metric": "train iterations/s (global batch 32 TX)",
                "value": 1e3 / ms, "unit": "it/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (bench scene, random magnitude targets)",
                "config": dict(workload_config(args.config),
                               parallelism=f"dp{world}",
                               deterministic_backward=bool(args.deterministic)),
                "clocks": clocks.summary(), "renders_per_s": B * 1e3 / ms,
                "last_loss": loss, "healthy": bool(ok),
                "gpu_launches": int(per_step * args.steps) if per_step else None}
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c2":
        return run_train(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
