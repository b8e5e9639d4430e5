"""Summarise ncu --set full reports into a JSON dict (dev tool; output goes to profiles/).
python tools/ncu_summary.py out.json name=path.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active": "fmaheavy_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "inst_executed",
}
SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")][:160]}
        for m, name in METRICS.items():
            if m not in head:
                continue
            v, u = r[head.index(m)], units[head.index(m)]
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if name == "duration":
                d["duration_us"] = round(x * SCALE.get(u, 1e-3), 3)
            elif name in ("dram_read", "dram_write"):
                d[name + "_bytes"] = int(x * SCALE.get(u, 1))
            elif name == "sm_clock":
                d["sm_clock_ghz"] = round(x / 1e9 if x > 1e6 else x, 3)
            else:
                d[name] = x
        res.append(d)
    return res


def main():
    out = {}
    for arg in sys.argv[2:]:
        name, path = arg.split("=", 1)
        out[name] = summarise(path)
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
