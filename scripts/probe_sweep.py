"""Exhaustive timing of every B200 config at chosen bench sweep points.

    python scripts/probe_sweep.py --points 1:0.2,8:0.5,512:0.2
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.moe import DeviceTable  # noqa: E402
from paper_2604_26039_b200.sweep import MeasuredTimer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--points", default="1:0.2,1:0.5,8:0.5,64:0.5,512:0.2,16:1.0")
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
geom = BASELINE_MODELS[bench.MODEL]
hw = HardwareModel.b200()
pool = enumerate_b200_configs(geom, hw)
cols = pool.columns()
n = len(pool)
flat = DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                   group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols.get("kps"), h3=cols.get("h3"), a=np.ones(n), b=np.zeros(n),
                   c=np.zeros(n), d=np.zeros(n), N=geom.N, kappa_ok=True, sm_count=148, ntile=cols["ntile"],
                   omega_max=float("inf"))
timer = MeasuredTimer(geom, flat, iters=a.iters)
allpts = bench.sweep_points(geom)
for spec in a.points.split(","):
    S, beta = spec.split(":")
    pt = [p for p in allpts if p["S"] == int(S) and p["beta"] == float(beta)][0]
    t = timer.pool_times(pool, pt["hist"], pt["seed"])
    order = np.argsort(t)
    print(f"S={S} beta={beta} active={pt['hist'].active_experts} bytes={bench.layer_bytes(geom, pt['hist'], int(S))/1e6:.1f}MB")
    for i in order[:6]:
        c = pool.by_id(int(i))
        print(f"   {t[i]:7.1f}us bm={c.bm} ttn={c.ttn} stg={c.stg} gm={int(c.group_m)} mode={c.mode} sk={c.split_k}")
    for sk in (2, 4):
        j = [i for i in order if pool.by_id(int(i)).split_k == sk][0]
        c = pool.by_id(int(j))
        print(f"   best sk={sk}: {t[j]:7.1f}us bm={c.bm} ttn={c.ttn} stg={c.stg}")
