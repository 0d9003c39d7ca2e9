"""Fold ncu --set full captures into profiles/ncu_kernels.json, the per-stage
kernel figures bench.py attaches to its roofline object (DRAM traffic per
launch, issue-slot utilisation, occupancy, warps per scheduler).

    python scripts/ncu_kernels_json.py CONFIG REP.ncu-rep [CONFIG REP ...]

Each capture's launches are grouped by kernel -> bench stage name; the
median over launches is recorded.  Run here on reports fetched from the
GPU box (gpurun_out/), commit the JSON."""
import csv
import io
import json
import os
import re
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_kernels.json")

STAGE = [  # (kernel-name regex, stage per config kind)
    (r"k_preprocess", "preprocess"),
    (r"k_tile_sort", "bin_sort"),
    (r"k_pxa<0>", "raster_weights"),
    (r"k_pxa<[1-9]", "raster_fused"),
    (r"k_pxb", "raster_accumulate"),
    (r"k_mlp_wide", "mlp"),
    (r"k_raster_bwd", "backward"),
    (r"k_gauss_bwd", "gauss_backward"),
    (r"k_adam", "adam"),
    (r"k_loss_band_fwd", "loss_fwd"),
    (r"k_loss_band_adj", "loss_adj"),
]
DETAILS = {"Duration": "duration_us", "Issue Slots Busy": "issue_slots_busy_pct",
           "Achieved Occupancy": "achieved_occupancy_pct",
           "Theoretical Occupancy": "theoretical_occupancy_pct",
           "Eligible Warps Per Scheduler": "eligible_warps_per_scheduler",
           "Active Warps Per Scheduler": "active_warps_per_scheduler",
           "Executed Ipc Active": "ipc_active",
           "DRAM Throughput": "dram_throughput_pct",
           "Compute (SM) Throughput": "sm_throughput_pct"}


def stage_of(name, config):
    for pat, st in STAGE:
        if re.search(pat, name):
            if st == "mlp" and config in ("c3", "c5"):
                return "mlp_live"
            return st
    return None


def load(rep, config):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ii, ki, mi, vi, ui = (h.index(k) for k in ("ID", "Kernel Name", "Metric Name",
                                               "Metric Value", "Metric Unit"))
    per = {}
    for r in rows[1:]:
        if r[mi] not in DETAILS:
            continue
        st = stage_of(r[ki], config)
        if st is None:
            continue
        v = float(r[vi].replace(",", ""))
        if r[mi] == "Duration":
            v = v / 1e3 if r[ui] in ("ns", "nsecond") else v
            v = v * 1e3 if r[ui] in ("ms", "msecond") else v
        per.setdefault(st, {}).setdefault(r[ii], {})[DETAILS[r[mi]]] = v
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, body = rows[0], rows[2:]
    for r in body:
        d = dict(zip(h, r))
        st = stage_of(d.get("Kernel Name", ""), config)
        if st is None:
            continue
        # the raw page's second row holds each metric's unit
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        try:
            b = sum(float(d[m].replace(",", "")) *
                    scale.get(rows[1][h.index(m)], 1)
                    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        except (KeyError, ValueError):
            continue
        per.setdefault(st, {}).setdefault(d["ID"], {})["dram_bytes"] = b
    out = {}
    for st, launches in per.items():
        keys = set().union(*launches.values())
        out[st] = {k: statistics.median(v[k] for v in launches.values() if k in v)
                   for k in keys}
        out[st]["launches"] = len(launches)
        out[st]["source"] = os.path.relpath(rep, ROOT)
    return out


def main(argv):
    data = {"note": "ncu --set full --clock-control none per-launch medians; "
                    "written by scripts/ncu_kernels_json.py", "configs": {}}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    for cfg, rep in zip(argv[0::2], argv[1::2]):
        data["configs"].setdefault(cfg, {}).update(load(rep, cfg))
    with open(OUT, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps(data, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1:])
