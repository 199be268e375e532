"""A/B timing of forced configs with MeasuredTimer (development tool).

    RAMP_B200_LIB=<lib.so> python scripts/ab_time.py --points 16:0.5,1024:0.2 --cfgs "8,128,8,0,1,1,1;128,256,4,0,1,1,1"

Config spec: bm,ttn,stg,group_m,mode,split_k,kps[,h3].  Prints one line per
(point, config): median us over the timer's L2-flushed graph replays.
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, derive_seed  # noqa: E402
from paper_2604_26039_b200.moe import DeviceTable  # noqa: E402
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.sweep import MeasuredTimer, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--points", default="1:0.2,16:0.5,128:0.5,1024:0.2")
ap.add_argument("--cfgs", default="8,128,8,0,1,1,1;16,256,6,0,1,1,1;64,256,4,0,1,1,1;128,256,4,0,1,1,1")
ap.add_argument("--iters", type=int, default=9)
ap.add_argument("--model", default="OLMoE-1B-7B")
ap.add_argument("--dtype", default="bf16", choices=("bf16", "fp8"))
a = ap.parse_args()
geom = BASELINE_MODELS[a.model]
fp8 = a.dtype == "fp8"
pool = enumerate_b200_configs(geom, HardwareModel.b200(), dtype=a.dtype, phase3_chunks=not fp8, wide_tiles=not fp8,
                              fp8_wide_kps=fp8)
cols = pool.columns()
n = len(pool)
flat = DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                   group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols["kps"], h3=cols["h3"],
                   a=np.ones(n), b=np.zeros(n), c=np.zeros(n), d=np.zeros(n), N=geom.N, kappa_ok=True, sm_count=148)
want = [tuple(int(v) for v in c.split(",")) for c in a.cfgs.split(";")]
want = [w if len(w) == 8 else w + (1,) for w in want]  # h3 defaults to 1
ids = []
for w in want:
    m = [c.id for c in pool if (c.bm, c.ttn, c.stg, int(c.group_m), c.mode, c.split_k, c.kps, c.h3) == w]
    if not m:
        raise SystemExit(f"config {w} not in the pool")
    ids.append(m[0])
if fp8:
    from paper_2604_26039_b200.sweep import make_fp8_weights

    timer = MeasuredTimer(geom, flat, iters=a.iters, fp8_weights=make_fp8_weights(geom))
else:
    timer = MeasuredTimer(geom, flat, iters=a.iters)
for spec in a.points.split(","):
    S, beta = int(spec.split(":")[0]), float(spec.split(":")[1])
    hs = derive_seed(42, EVAL_HIST_DOMAIN, S, round(beta * 1000), 0)
    hist = sample_histogram(geom.E, S, geom.top_k, beta, hs).histogram
    x, tid, w = make_inputs(geom, hist, hs, "cuda")
    t = timer.time_configs(x, tid, w, ids)
    for cid, wspec, us in zip(ids, want, t):
        print(f"S={S} beta={beta} cfg {wspec}: {us:.2f} us")
