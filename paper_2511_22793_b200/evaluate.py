"""Batched evaluation of a trained cloud against a dataset (reference
cli.cmd_eval, cli.py:190-231, with optimize.ssim/mse/psnr,
optimize.py:134-202).

The reference renders one TX at a time and computes the metrics on the host.
Here a batch of transmitters is rendered at once (shared geometry), and K7
(the loss kernel, f64 arithmetic) produces per-image SSIM and MSE of the
magnitude prediction against the ground truth on the device, so only four
doubles per sample come back.  Output files and their formatting match the
reference (eval_per_sample.csv, eval_summary.csv).
"""

from __future__ import annotations

import csv
import math
import statistics
from pathlib import Path

import numpy as np
import torch

from .engine import LossWorkspace
from .rasterizer import rasterize_forward_batch
from .scene import DeviceCloud


def _psnr(m):
    """optimize.py:196-202: 10 log10(1/mse), +inf for identical images."""
    return math.inf if m == 0.0 else 10.0 * math.log10(1.0 / m)


def evaluate_arrays(cloud, pose, ids, txs, gt, w, h, supervision="magnitude",
                    batch=64):
    """Per-sample {"id", "ssim", "mse", "psnr"} rows.

    txs: [S,3] (numpy or tensor); gt: [S, h, w, c] device or host spectra
    (channel 0 is compared, as cmd_eval does with gt[:, :, :1])."""
    if supervision != "magnitude":
        raise ValueError("batched evaluation supports magnitude supervision "
                         "(the cmd_eval default)")
    dev = cloud if isinstance(cloud, DeviceCloud) else DeviceCloud.from_host(cloud)
    txs = torch.as_tensor(np.asarray(txs, np.float64)) \
        if not isinstance(txs, torch.Tensor) else txs
    gt = gt if isinstance(gt, torch.Tensor) else torch.as_tensor(np.asarray(gt))
    S = int(txs.shape[0])
    rows = []
    ws = None
    for s0 in range(0, S, batch):
        tb = txs[s0:s0 + batch]
        B = int(tb.shape[0])
        img, _ = rasterize_forward_batch(dev, pose, tb, w, h)
        C = int(img.shape[-1])
        if C != 2:
            raise ValueError(f"magnitude supervision needs 2 channels, got {C}")
        g = gt[s0:s0 + B, :, :, :1].to("cuda", torch.float32).contiguous()
        if ws is None or ws.shape[0] != B:
            ws = LossWorkspace(B, h, w, C, "cuda", dtype=torch.float32)
        _, stats = ws.run(img.contiguous(), g, 0, 0.0)
        st = stats.cpu().numpy()
        for b in range(B):
            m = float(st[b, 3])
            rows.append({"id": ids[s0 + b], "ssim": float(st[b, 2]),
                         "mse": m, "psnr": _psnr(m)})
    return rows


def evaluate_dataset(cloud, pose, index_path, w=None, h=None, batch=64):
    """cmd_eval's metric loop over a dataset directory (index.csv + RFSI
    files), loaded through one pinned buffer onto the device."""
    from .rfsim import load_dataset_device
    ids, tx, spectra = load_dataset_device(index_path)
    h = h or int(spectra.shape[1])
    w = w or int(spectra.shape[2])
    return evaluate_arrays(cloud, pose, ids, tx, spectra, w, h, batch=batch)


def summarize(rows):
    """Mean and median per metric (cli.py:213-217)."""
    out = []
    for key in ("ssim", "mse", "psnr"):
        vals = [r[key] for r in rows]
        out.append({"metric": key, "mean": statistics.fmean(vals),
                    "median": statistics.median(vals)})
    return out


def write_eval_csv(rows, out_dir):
    """eval_per_sample.csv and eval_summary.csv exactly as cli.py:205-224."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    with open(out / "eval_per_sample.csv", "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=["id", "ssim", "mse", "psnr"])
        wr.writeheader()
        for r in rows:
            wr.writerow({k: (f"{v:.6g}" if isinstance(v, float) else v)
                         for k, v in r.items()})
    summary = summarize(rows)
    with open(out / "eval_summary.csv", "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=["metric", "mean", "median"])
        wr.writeheader()
        for r in summary:
            wr.writerow({"metric": r["metric"], "mean": f"{r['mean']:.6g}",
                         "median": f"{r['median']:.6g}"})
    return summary
