"""Summarise ncu reports into one JSON object per kernel launch (committed
under profiles/): duration, DRAM bytes and throughput, tensor-pipe and SM
utilisation, L2 hit rate, registers.

    python scripts/ncu_summary.py gpurun_out/r2a_*.ncu-rep > profiles/r2a_ncu_summary.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "launch__registers_per_thread": "regs",
    "smsp__inst_executed.sum": "warp_insts",
}
UNIT_SCALE = {"us": 1.0, "ns": 1e-3, "ms": 1e3, "msecond": 1e3, "usecond": 1.0, "nsecond": 1e-3,
              "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"report": path.split("/")[-1], "kernel": r[head.index("Kernel Name")][:80]}
        for k, name in KEYS.items():
            if k not in head:
                continue
            i = head.index(k)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if name == "duration_us":
                v *= UNIT_SCALE.get(u, 1.0)
            elif name.startswith("dram_") and name != "dram_pct":
                v = v * UNIT_SCALE.get(u, 1.0) / 1e6  # MB
                name += "_mb"
            elif name == "sm_clock":
                v = v * (1e9 if u.lower().startswith("g") else 1e6 if u.lower().startswith("m") else 1.0) / 1e6
                name = "sm_clock_mhz"
            rec[name] = round(v, 3)
        if "duration_us" in rec and "dram_read_mb" in rec:
            rec["dram_gbs"] = round((rec["dram_read_mb"] + rec.get("dram_write_mb", 0.0)) / rec["duration_us"] * 1e3, 1)
        out.append(rec)
    return out


if __name__ == "__main__":
    res = []
    for p in sys.argv[1:]:
        res.extend(summarise(p))
    print(json.dumps(res, indent=1))
