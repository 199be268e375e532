"""Route-kernel step clocks (development tool; needs a -DRAMP_ROUTE_CLOCKS
build, e.g. RAMP_B200_LIB=scripts/_ab/lib_rclk.so): one layer call at a bench
point, thread 0's clock64() at every RCLK(k) of csrc/route.cu[h], printed as
cycles since RCLK(0).

    RAMP_B200_LIB=... python scripts/route_clocks.py --S 2048 --beta 0.5 --model Qwen3-30B-A3B --fp8
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2604_26039_b200 import _lib, moe  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store  # noqa: E402
from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, DispatchTable, derive_seed  # noqa: E402
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.sweep import make_fp8_weights, make_inputs, make_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="OLMoE-1B-7B")
ap.add_argument("--S", type=int, default=512)
ap.add_argument("--beta", type=float, default=0.5)
ap.add_argument("--fp8", action="store_true")
a = ap.parse_args()
geom = BASELINE_MODELS[a.model]
dt = "fp8" if a.fp8 else "bf16"
pool = enumerate_b200_configs(geom, HardwareModel.b200(), dtype=dt)
tag = f"{a.model}_b200" + ("_fp8" if a.fp8 else "")
store = read_coeff_store(ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{tag}.json")
_, sm, co = parse_coeff_store(store)
dtab = DispatchTable(model=a.model, pool=pool, coefficients=co, sm_count=sm, active=active_ids_of(store)).device_table()
hs = derive_seed(42, EVAL_HIST_DOMAIN, a.S, round(a.beta * 1000), 0)
hist = sample_histogram(geom.E, a.S, geom.top_k, a.beta, hs).histogram
x, ids, w = make_inputs(geom, hist, hs)
ws = moe.Workspace(a.S, geom.K, geom.N // 2, geom.E, geom.top_k)
if a.fp8:
    wq = make_fp8_weights(geom)
    run = lambda: moe.fused_moe_fp8(x, wq, w, ids, dtab, -1, workspace=ws)  # noqa: E731
else:
    w1, w2 = make_weights(geom)
    run = lambda: moe.fused_moe(x, w1, w2, w, ids, dtab, -1, workspace=ws)  # noqa: E731
for _ in range(3):
    run()
torch.cuda.synchronize()
buf = torch.zeros(149 * 32 + 148 * 16 * 4, dtype=torch.int64, device="cuda")
_lib.load().ramp_set_profile_buffer(buf.data_ptr())
run()
torch.cuda.synchronize()
_lib.load().ramp_set_profile_buffer(None)
r = buf[148 * 32: 149 * 32].cpu().numpy()
clk = buf[148 * 32 + 16: 148 * 32 + 16 + 25].cpu().numpy().astype(np.int64)
base = clk[0] if clk[0] else 0
print(f"{a.model} S={a.S} beta={a.beta} n={a.S * geom.top_k} active={hist.active_experts}")
print("globaltimer (ns from start): hist %d dispatch %d scan+pad %d align %d done %d" %
      tuple(r[i] - r[0] for i in (1, 2, 5, 3, 4)))
print("RCLK cycles since RCLK(0):", {k: int(clk[k] - base) for k in range(25) if clk[k]})
