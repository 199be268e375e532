"""One small fused-MoE layer call (BF16 or MXFP8) for compute-sanitizer runs.

    compute-sanitizer --tool memcheck --error-exitcode 99 python scripts/sanitize_case.py --dtype bf16

Device dispatch over the full B200 pool of a small geometry (a uniform
table), then two forced configs covering split-K / fused mode, each checked
against the fp32 oracle, so a sanitizer run also proves the result.
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.moe_ref import fused_moe_ref, fused_moe_ref_fp8  # noqa: E402
from paper_2604_26039_b200 import moe  # noqa: E402
from paper_2604_26039_b200.catalog import MoeGeometry  # noqa: E402
from paper_2604_26039_b200.config_space import enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.quant import prepare_mxfp8_weights  # noqa: E402
from tests._util import random_moe  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", choices=("bf16", "fp8"), default="bf16")
a = ap.parse_args()
E, H, I, k, S = 8, 256, 256, 2, 24
pool = enumerate_b200_configs(MoeGeometry(name="san", E=E, N=2 * I, K=H, top_k=k), dtype=a.dtype)
cols = pool.columns()
n = len(pool)
one = np.ones(n)
table = moe.DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                        group_m=cols["group_m"].astype(np.int64), mode=cols.get("mode"), kps=cols.get("kps"),
                        h3=cols.get("h3"), a=one + 1e-3 * cols["bm"], b=0 * one, c=0 * one, d=0 * one, N=2 * I,
                        kappa_ok=False, sm_count=148)
x, w1, w2, w, ids = random_moe(S, H, I, E, k, seed=4)
xt = torch.from_numpy(x).to("cuda", torch.bfloat16)
wt, it = torch.from_numpy(w).cuda(), torch.from_numpy(ids).cuda()
ws = moe.Workspace(S, H, I, E, k)
picks = [-1]
picks += [c.id for c in pool if c.split_k > 1][:1]
picks += [c.id for c in pool if c.mode == 0][:1]
picks += [c.id for c in pool if getattr(c, "kps", 1) > 1][:1]
if a.dtype == "fp8":
    wq = prepare_mxfp8_weights(torch.from_numpy(w1).cuda(), torch.from_numpy(w2).cuda())
    d1, d2 = (t.cpu().numpy() for t in wq.dequantize())
    ref = fused_moe_ref_fp8(x, d1, d2, w, ids)
else:
    w1t, w2t = torch.from_numpy(w1).to("cuda", torch.bfloat16), torch.from_numpy(w2).to("cuda", torch.bfloat16)
    ref = fused_moe_ref(x, w1, w2, w, ids)
for cid in picks:
    if a.dtype == "fp8":
        o = moe.fused_moe_fp8(xt, wq, wt, it, table, cid, workspace=ws)
    else:
        o = moe.fused_moe(xt, w1t, w2t, wt, it, table, cid, workspace=ws)
    o = o.float().cpu().numpy()
    err = float(np.linalg.norm(o - ref) / np.linalg.norm(ref))
    print(f"{a.dtype} cfg {cid} -> {int(ws.sel[0].item())}: rel err {err:.2e}", flush=True)
    if not err < 1e-2:
        sys.exit(3)
print("sanitize_case ok")
