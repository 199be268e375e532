"""Every config of the MXFP8 pools (Qwen3-30B-A3B, DeepSeek-V3) at the shipped
tables' test routings (tests/test_gpu_shipped.py, reduced E, real d_model /
d_ff) against the oracle, one call at a time with a synchronize after each --
a hang names its config (development tool; run under `timeout`).

    timeout 400 python scripts/fp8_config_sweep.py [Qwen3|DeepSeek]
"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import tests.test_gpu_shipped as T
from paper_2604_26039_b200 import moe
from paper_2604_26039_b200.catalog import BASELINE_MODELS
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs
from paper_2604_26039_b200.quant import prepare_mxfp8_weights
from oracle.moe_ref import bf16_round
from tests._util import random_moe
only = sys.argv[1] if len(sys.argv) > 1 else None
for fname, model, dtype, E in T.SHIPPED:
    if dtype != "fp8" or (only and only not in model):
        continue
    g = BASELINE_MODELS[model]; H, I, k = g.K, g.N // 2, g.top_k
    pool = enumerate_b200_configs(g, HardwareModel.b200(), dtype=dtype)
    table = T._uniform_table(pool)
    gen = torch.Generator(device="cuda").manual_seed(7)
    w1 = (torch.randn(E, 2 * I, H, device="cuda", generator=gen) * H ** -0.5).to(torch.bfloat16)
    w2 = (torch.randn(E, H, I, device="cuda", generator=gen) * I ** -0.5).to(torch.bfloat16)
    wq = prepare_mxfp8_weights(w1, w2); d1, d2 = wq.dequantize()
    for S, skew in T.ROUTINGS[model]:
        x, _, _, w, ids = random_moe(S, 128, 128, E, k, seed=S, skew=skew)
        x = bf16_round(np.random.default_rng(S).standard_normal((S, H)).astype(np.float32))
        rows = np.random.default_rng(1).choice(S, size=min(S, T.N_ROWS), replace=False)
        ref = T._rows_ref(x, d1, d2, w, ids, rows, True)
        xt = torch.from_numpy(x).to("cuda", torch.bfloat16); wt, it = torch.from_numpy(w).cuda(), torch.from_numpy(ids).cuda()
        ws = moe.Workspace(S, H, I, E, k)
        for c in pool:
            print(f"{model} S={S} cfg {c.id} {c.to_dict()}", end=" ", flush=True)
            o = moe.fused_moe_fp8(xt, wq, wt, it, table, c.id, workspace=ws)
            torch.cuda.synchronize()
            err = T._rel(o.float()[torch.as_tensor(rows, device="cuda")].cpu().numpy(), ref)
            print(f"err {err:.2e}{'  BAD' if not err < 1e-2 else ''}", flush=True)
print("hunt done", flush=True)
