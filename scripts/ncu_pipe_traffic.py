"""Summarise scripts/gpu_traffic_pipe.sh's ncu CSVs: per kernel, the median
in-pipeline DRAM bytes (read + write) and duration over its launches.

    python scripts/ncu_pipe_traffic.py [--json] CONFIG CSV [CONFIG CSV ...]

--json merges the figures into profiles/ncu_pipe_traffic.json (per config,
per bench stage), which bench.py attaches to its roofline object as
`traffic_pipeline`."""
import csv, io, json, os, re, statistics, sys, collections

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_pipe_traffic.json")
STAGE = [(r"k_preprocess", "preprocess"), (r"k_tile_sort", "bin_sort"),
         (r"k_pxa<0>", "raster_weights"), (r"k_pxa<[1-9]", "raster_fused"),
         (r"k_pxb", "raster_accumulate"), (r"k_mlp", "mlp")]

def load(path):
    txt = open(path).read()
    i = txt.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    per = collections.defaultdict(lambda: collections.defaultdict(dict))
    for r in rows:
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1,
              "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}.get(u, 1)
        per[name][r["ID"]][r["Metric Name"]] = v
    out = {}
    for k, launches in per.items():
        L = list(launches.values())
        med = lambda m: statistics.median(x[m] for x in L if m in x)
        out[k] = {"launches": len(L), "dram_read_MB": med("dram__bytes_read.sum") / 1e6,
                  "dram_write_MB": med("dram__bytes_write.sum") / 1e6,
                  "duration_us": med("gpu__time_duration.sum")}
    return out

if __name__ == "__main__":
    args = sys.argv[1:]
    js = "--json" in args
    args = [a for a in args if a != "--json"]
    data = json.load(open(OUT)) if js and os.path.exists(OUT) else {
        "note": "ncu --cache-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                "gpu__time_duration.sum over a bench.py --no-graph run (scripts/gpu_traffic_pipe.sh): "
                "each kernel sees the L2 its predecessor left, as inside the timed graph; "
                "medians over launches", "configs": {}}
    for cfg, p in zip(args[0::2], args[1::2]):
        print(cfg, p)
        for k, v in sorted(load(p).items(), key=lambda kv: -kv[1]["duration_us"]):
            print("  %-40s n=%4d read %8.2f MB write %8.2f MB  %8.1f us" % (
                k[:40], v["launches"], v["dram_read_MB"], v["dram_write_MB"], v["duration_us"]))
            st = next((st for pat, st in STAGE if re.search(pat, k)), None)
            if st:
                if st == "mlp" and cfg in ("c3", "c5"):
                    st = "mlp_live"
                data["configs"].setdefault(cfg, {})[st] = {
                    "kernel": k, "dram_bytes": (v["dram_read_MB"] + v["dram_write_MB"]) * 1e6,
                    "dram_read_bytes": v["dram_read_MB"] * 1e6,
                    "dram_write_bytes": v["dram_write_MB"] * 1e6,
                    "duration_us_serialised": v["duration_us"],
                    "source": os.path.relpath(p, ROOT)}
    if js:
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
