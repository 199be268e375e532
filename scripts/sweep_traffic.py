"""DRAM traffic of the megakernel over the whole bench sweep (ncu target and summariser).

    ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --csv --log-file gpurun_out/sweep_launches.csv python scripts/sweep_traffic.py run
    python scripts/sweep_traffic.py summarize gpurun_out/sweep_launches.csv > profiles/sweep_traffic.json

`run` makes one layer call per bench sweep point (27, on-device dispatch,
the bench's table and routings) after one warm-up call each; ncu replays
every launch with its caches flushed, so the weights are read cold as in the
bench.  `summarize` sums the DRAM bytes of the timed megakernel launches and
compares them with the algorithmic bytes of the same points:
the ratio is bench.py's roofline `traffic` evidence (> 1 = wasted re-reads).
"""
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def run():
    import torch

    import bench
    from paper_2604_26039_b200 import moe
    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs
    from paper_2604_26039_b200.sweep import make_inputs, make_weights

    geom = BASELINE_MODELS[bench.MODEL]
    pool = enumerate_b200_configs(geom, HardwareModel.b200())
    table, _ = bench.load_table(geom, pool, HardwareModel.b200())
    dtab = table.device_table()
    w1, w2 = make_weights(geom)
    for pt in bench.sweep_points(geom):
        x, ids, w = make_inputs(geom, pt["hist"], pt["seed"])
        ws = moe.Workspace(pt["S"], geom.K, geom.N // 2, geom.E, geom.top_k)
        for _ in range(2):  # warm-up, timed
            moe.fused_moe(x, w1, w2, w, ids, dtab, -1, workspace=ws)
        torch.cuda.synchronize()
        print("point", pt["S"], pt["beta"], "active", pt["hist"].active_experts, "cfg",
              dtab.pool_id(int(ws.sel[0].item())), "bytes", bench.layer_bytes(geom, pt["hist"], pt["S"]), flush=True)


def summarize(path):
    import bench
    from paper_2604_26039_b200.catalog import BASELINE_MODELS

    text = Path(path).read_text()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = {}
    for r in rows:
        if "fused_moe" not in r["Kernel Name"]:
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1.0, "nsecond": 1e-3,
                 "msecond": 1e3}.get(unit, 1.0)
        per.setdefault(int(r["ID"]), {})[r["Metric Name"]] = v * scale
    launches = [per[i] for i in sorted(per)]
    geom = BASELINE_MODELS[bench.MODEL]
    pts = bench.sweep_points(geom)
    if len(launches) != 2 * len(pts):
        raise SystemExit(f"expected {2 * len(pts)} megakernel launches, found {len(launches)}")
    timed = launches[1::2]  # the second call of each point
    dram = [m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in timed]
    alg = [bench.layer_bytes(geom, pt["hist"], pt["S"]) for pt in pts]
    out = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     "--clock-control none (caches flushed per launch), scripts/sweep_traffic.py run: "
                     "one megakernel launch per bench sweep point",
           "launches": len(timed), "dram_bytes_per_launch": sum(dram) / len(dram),
           "algorithmic_bytes_per_launch": sum(alg) / len(alg), "dram_over_algorithmic": sum(dram) / sum(alg),
           "per_point": [{"S": pt["S"], "beta": pt["beta"], "dram_mb": round(d / 1e6, 2),
                          "algorithmic_mb": round(a / 1e6, 2), "ratio": round(d / a, 4),
                          "us_cold": round(m["gpu__time_duration.sum"], 2)}
                         for pt, d, a, m in zip(pts, dram, alg, timed)]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        summarize(sys.argv[2])
