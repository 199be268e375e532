"""One MXFP8 layer call through the public API, a few times (ncu target).

    python scripts/ncu_point_fp8.py --model Qwen3-30B-A3B --S 2048 --beta 0.5 [--reps 3]
    python scripts/ncu_point_fp8.py --model DeepSeek-V3 --S 256 --beta 0.5     # the bench EP leg at N=1

The config is the on-device dispatcher's pick from the shipped FP8 table
(`--cfg ID` forces one).  DeepSeek-V3 runs the EP leg's world-1 geometry
(all 256 experts local) with the DeepSeek-V3-EP8 table, as bench.py does.
"""
import argparse
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2604_26039_b200 import moe  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store  # noqa: E402
from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, DispatchTable, derive_seed  # noqa: E402
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.sweep import make_fp8_weights, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="Qwen3-30B-A3B")
ap.add_argument("--S", type=int, default=2048)
ap.add_argument("--beta", type=float, default=0.5)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--cfg", type=int, default=-1)
a = ap.parse_args()
geom = BASELINE_MODELS[a.model]
table_model = a.model
if not (ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{table_model}_b200_fp8.json").exists():
    table_model = "DeepSeek-V3-EP8" if a.model == "DeepSeek-V3" else a.model
pool = enumerate_b200_configs(geom, HardwareModel.b200(), dtype="fp8")
store = read_coeff_store(ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{table_model}_b200_fp8.json")
_, sm, co = parse_coeff_store(store)
dtab = DispatchTable(model=geom.name, pool=pool, coefficients=co, sm_count=sm,
                     active=active_ids_of(store)).device_table()
hs = derive_seed(42, EVAL_HIST_DOMAIN, a.S, round(a.beta * 1000), 0)
hist = sample_histogram(geom.E, a.S, geom.top_k, a.beta, hs).histogram
weights = make_fp8_weights(geom)
x, ids, w = make_inputs(geom, hist, hs)
H, I = geom.K, geom.N // 2
ws = moe.Workspace(a.S, H, I, geom.E, geom.top_k)
for _ in range(a.reps):
    out = moe.fused_moe_fp8(x, weights, w, ids, dtab, a.cfg, workspace=ws)
torch.cuda.synchronize()
sel = dtab.pool_id(int(ws.sel[0].item()))
nbytes = hist.active_experts * 3 * H * I * (1 + 1 / 32) + a.S * H * 4 + 8 * a.S * geom.top_k
print("point", a.model, a.S, a.beta, "active", hist.active_experts, "cfg", sel, pool.by_id(sel).to_dict(),
      "bytes", int(nbytes), "flop", 6 * a.S * geom.top_k * H * I)
