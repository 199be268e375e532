"""One bench sweep point through the public API, a few times (ncu target).

    python scripts/ncu_point.py --S 16 --beta 1.0 [--reps 3]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2604_26039_b200 import moe  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.sweep import make_inputs, make_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--S", type=int, default=16)
ap.add_argument("--beta", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
geom = BASELINE_MODELS[bench.MODEL]
pool = enumerate_b200_configs(geom, HardwareModel.b200())
table, _ = bench.load_table(geom, pool, HardwareModel.b200())
pt = [p for p in bench.sweep_points(geom) if p["S"] == a.S and p["beta"] == a.beta][0]
w1, w2 = make_weights(geom)
x, ids, w = make_inputs(geom, pt["hist"], pt["seed"])
ws = moe.Workspace(a.S, geom.K, geom.N // 2, geom.E, geom.top_k)
for _ in range(a.reps):
    out = moe.fused_moe(x, w1, w2, w, ids, table.device_table(), -1, workspace=ws)
torch.cuda.synchronize()
cfg = int(ws.sel[0].item())
print("point", a.S, a.beta, "active", pt["hist"].active_experts, "cfg", cfg, pool.by_id(cfg).to_dict(),
      "bytes", bench.layer_bytes(geom, pt["hist"], a.S))
