"""Per-kernel DRAM bytes (read, write; MB) and duration (us) from an ncu
--set full report.  usage: ncu_dram.py rep [json_out]"""
import csv, io, json, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
res = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    name = d["Kernel Name"]
    def val(m, scale):
        v = float(d[m].replace(",", ""))
        un = u[m]
        f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3,
             "usecond": 1, "msecond": 1e3}.get(un, 1)
        return v * f / scale
    rd = val("dram__bytes_read.sum", 1e6)
    wr = val("dram__bytes_write.sum", 1e6)
    du = val("gpu__time_duration.sum", 1)
    print(f"{name[:40]} dram_read {rd:.6f} dram_write {wr:.6f} dur {du:.6f}")
    res.setdefault(name, {"dram_read_mb": rd, "dram_write_mb": wr, "dur_us": du,
                          "traffic_bytes": (rd + wr) * 1e6})
if len(sys.argv) > 2:
    json.dump(res, open(sys.argv[2], "w"), indent=1)
