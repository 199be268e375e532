"""Inter-call overhead under CUDA-graph replay (development tool).

For a few sweep points, captures graphs of 8 back-to-back calls of: the full
layer (route + megakernel), the route kernel only, the megakernel only, and a
trivial torch kernel, and prints the per-call time of each.  The difference
full - (route stamps + megakernel stamps) is launch / teardown overhead.
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import MODEL, load_table  # noqa: E402
from paper_2604_26039_b200 import moe  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, derive_seed  # noqa: E402
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.sweep import make_inputs, make_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--points", default="1:0.2,16:1.0,512:0.2")
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--fp8", action="store_true", help="Qwen3-30B-A3B MXFP8 path with its fitted table")
a = ap.parse_args()
geom = BASELINE_MODELS["Qwen3-30B-A3B" if a.fp8 else MODEL]
dev = torch.device("cuda")
pool = enumerate_b200_configs(geom, HardwareModel.b200(), dtype="fp8" if a.fp8 else "bf16")
if a.fp8:
    from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store
    from paper_2604_26039_b200.dispatch import DispatchTable
    from paper_2604_26039_b200.sweep import make_fp8_weights
    store = read_coeff_store(ROOT / "paper_2604_26039_b200" / "data" / "coeffs_Qwen3-30B-A3B_b200_fp8.json")
    _, sm, co = parse_coeff_store(store)
    dtab = DispatchTable(model=geom.name, pool=pool, coefficients=co, sm_count=sm,
                         active=active_ids_of(store)).device_table(device=dev)
    wq = make_fp8_weights(geom, seed=1, device=dev)
else:
    table, _ = load_table(geom, pool, HardwareModel.b200())
    dtab = table.device_table(device=dev)
    w1, w2 = make_weights(geom, seed=1, device=dev)
H, I = geom.K, geom.N // 2
side = torch.cuda.Stream()


def graph(fn):
    with torch.cuda.stream(side):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(a.n):
                fn()
    torch.cuda.synchronize()
    return g


def timeit(g, reps=15):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / a.n)
    return float(np.median(ts[3:]))


t = torch.zeros(1, device=dev)
print(f"trivial kernel per call: {timeit(graph(lambda: t.add_(1))):.2f} us")
for spec in a.points.split(","):
    S, beta = int(spec.split(":")[0]), float(spec.split(":")[1])
    hs = derive_seed(42, EVAL_HIST_DOMAIN, S, round(beta * 1000), 0)
    hist = sample_histogram(geom.E, S, geom.top_k, beta, hs).histogram
    x, ids, w = make_inputs(geom, hist, hs, dev)
    ws = moe.Workspace(S, H, I, geom.E, geom.top_k, device=dev)
    out = torch.empty(S, H, dtype=torch.bfloat16, device=dev)

    def run(phases=3):
        if a.fp8:
            moe.fused_moe_fp8(x, wq, w, ids, dtab, -1, out=out, workspace=ws, phases=phases)
        else:
            moe.fused_moe(x, w1, w2, w, ids, dtab, -1, out=out, workspace=ws, phases=phases)

    res = {k: timeit(graph(lambda p=p: run(p))) for k, p in (("full", 3), ("route", 1), ("mega", 2))}
    print(f"S={S} beta={beta}: per call full {res['full']:.2f}  route-only {res['route']:.2f}  "
          f"mega-only {res['mega']:.2f}  (route+mega {res['route'] + res['mega']:.2f})", flush=True)
