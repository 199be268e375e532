"""FP8 split-K feasibility probe (development tool): forced FP8 configs with
split_k in {1, 2, 4} on Qwen3-30B-A3B decode/prefill points -- output vs the
split_k = 1 output of the same tile shape, and MeasuredTimer latency."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_26039_b200 import moe  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, derive_seed  # noqa: E402
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.sweep import MeasuredTimer, make_fp8_weights, make_inputs  # noqa: E402

geom = BASELINE_MODELS["Qwen3-30B-A3B"]
# (bm, ttn, stg, split_k)
cfgs = [(16, 256, 4, 1), (16, 256, 4, 2), (16, 256, 4, 4), (32, 256, 4, 1), (32, 256, 4, 2), (32, 256, 4, 4),
        (16, 512, 3, 1), (16, 512, 3, 2)]
n = len(cfgs)
col = lambda i: np.array([c[i] for c in cfgs])  # noqa: E731
tab = moe.DeviceTable(bm=col(0), ttn=col(1), stg=col(2), split_k=col(3), group_m=np.zeros(n, np.int64),
                      mode=np.ones(n, np.int64), a=np.ones(n), b=np.zeros(n), c=np.zeros(n), d=np.zeros(n),
                      N=geom.N, kappa_ok=True, sm_count=148)
tab._fp8_ok = True  # probe: bypass the split_k == 1 guard
wq = make_fp8_weights(geom, seed=1)
timer = MeasuredTimer(geom, tab, iters=7, fp8_weights=wq)
for S, beta in ((8, 0.5), (32, 0.5), (128, 0.5)):
    hs = derive_seed(42, EVAL_HIST_DOMAIN, S, round(beta * 1000), 0)
    hist = sample_histogram(geom.E, S, geom.top_k, beta, hs).histogram
    x, ids, w = make_inputs(geom, hist, hs, "cuda")
    ws = moe.Workspace(S, geom.K, geom.N // 2, geom.E, geom.top_k)
    outs = []
    for i in range(n):
        o = moe.fused_moe_fp8(x, wq, w, ids, tab, i, workspace=ws).float()
        outs.append(o)
    torch.cuda.synchronize()
    t = timer.time_configs(x, ids, w, list(range(n)))
    for i, c in enumerate(cfgs):
        base = [j for j, d in enumerate(cfgs) if d[:3] == c[:3] and d[3] == 1][0]
        err = float((outs[i] - outs[base]).norm() / outs[base].norm())
        print(f"S={S} beta={beta} cfg bm{c[0]} ttn{c[1]} stg{c[2]} sk{c[3]}: {t[i]:.2f} us  rel vs sk1 {err:.2e}",
              flush=True)
