"""Run one (S, skew, config) point a few times -- the target for ncu captures."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_26039_b200 import moe as M  # noqa: E402
from paper_2604_26039_b200.catalog import MoeGeometry  # noqa: E402
from paper_2604_26039_b200.config_space import enumerate_b200_configs  # noqa: E402
from scripts.probe import topk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--S", type=int, default=512)
ap.add_argument("--skew", type=float, default=0.0)
ap.add_argument("--bm", type=int, default=64)
ap.add_argument("--ttn", type=int, default=512)
ap.add_argument("--stg", type=int, default=2)
ap.add_argument("--gm", type=int, default=0)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--sk", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--E", type=int, default=64)
ap.add_argument("--H", type=int, default=2048)
ap.add_argument("--I", type=int, default=1024)
ap.add_argument("--k", type=int, default=8)
ap.add_argument("--prof", action="store_true")
ap.add_argument("--fp8", action="store_true", help="the MXFP8 megakernel (FP8 pool)")
ap.add_argument("--kps", type=int, default=1)
ap.add_argument("--beta", type=float, default=None,
                help="route with the reference sampler's histogram at this beta (instead of --skew)")
a = ap.parse_args()
E, H, I, k, S = a.E, a.H, a.I, a.k, a.S
gen = torch.Generator(device="cuda").manual_seed(0)
w1 = (torch.randn(E, 2 * I, H, device="cuda", generator=gen) / H ** 0.5).to(torch.bfloat16)
w2 = (torch.randn(E, H, I, device="cuda", generator=gen) / I ** 0.5).to(torch.bfloat16)
pool = enumerate_b200_configs(MoeGeometry(name="p", E=E, N=2 * I, K=H, top_k=k), dtype="fp8" if a.fp8 else "bf16")
cols = pool.columns()
n = len(pool)
table = M.DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                      group_m=cols["group_m"].astype(np.int64), mode=cols.get("mode"), kps=cols.get("kps"), h3=cols.get("h3"), a=np.ones(n), b=np.zeros(n), c=np.zeros(n),
                      d=np.zeros(n), N=2 * I, kappa_ok=False, sm_count=148)
cfg = [c.id for c in pool if (c.bm, c.ttn, c.stg, int(c.group_m), c.mode, c.split_k, c.kps) ==
       (a.bm, a.ttn, a.stg, a.gm, a.mode, a.sk, a.kps)][0]
if a.fp8:
    from paper_2604_26039_b200.quant import prepare_mxfp8_weights
    wq = prepare_mxfp8_weights(w1, w2)
    run = lambda: M.fused_moe_fp8(x, wq, w, ids, table, cfg, workspace=ws)  # noqa: E731
else:
    run = lambda: M.fused_moe(x, w1, w2, w, ids, table, cfg, workspace=ws)  # noqa: E731
x = torch.randn(S, H, device="cuda", generator=gen).to(torch.bfloat16)
if a.beta is None:
    ids, w = topk(S, k, E, a.skew, gen)
else:
    from paper_2604_26039_b200.routing import sample_histogram
    from paper_2604_26039_b200.sweep import make_inputs

    g_ = MoeGeometry(name="p", E=E, N=2 * I, K=H, top_k=k)
    hist = sample_histogram(E, S, k, a.beta, 4242).histogram
    x, ids, w = make_inputs(g_, hist, 4242)
    print("active experts", hist.active_experts)
ws = M.Workspace(S, H, I, E, k)
for _ in range(a.reps):
    out = run()
torch.cuda.synchronize()
if a.prof:
    from paper_2604_26039_b200 import _lib
    buf = torch.zeros(149 * 32, dtype=torch.int64, device="cuda")
    _lib.load().ramp_set_profile_buffer(buf.data_ptr())
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    out = run()
    e1.record()
    torch.cuda.synchronize()
    _lib.load().ramp_set_profile_buffer(None)
    allb = buf.view(149, 32).cpu().numpy().astype(np.float64)
    pr = allb[:148]
    rt = allb[148]
    t0 = rt[0]
    tl = ["entry", "start", "gathered", "producer_done", "epilogue_done", "end_arrive", "end_pass", "final"]
    print("timeline (us from route start): " + "  ".join(
        f"{n} {np.min(pr[:, 16 + i] - t0) / 1e3:.1f}/{np.median(pr[:, 16 + i] - t0) / 1e3:.1f}/{np.max(pr[:, 16 + i] - t0) / 1e3:.1f}"
        for i, n in enumerate(tl) if np.all(pr[:, 16 + i] > 0)))
    print('route stamps (ns from start): hist %.0f dispatch %.0f scan+pad %.0f align %.0f done %.0f' % tuple(rt[i] - rt[0] for i in (1, 2, 5, 3, 4)))
    names = ["pr_wait_empty", "pr_issue", "mma_wait_full", "mma_wait_acc", "mma_wait_act", "epi_wait_acc",
             "epi_swiglu", "epi_wait_chunk", "epi_scatter", "total", "items", "epi_meta", "pr_wait_dep",
             "lat_tma", "lat_release", "n_stages"]
    act = pr[:, 10] > 0
    print(f"S={S} cfg bm={a.bm} ttn={a.ttn} stg={a.stg}: {e0.elapsed_time(e1)*1000:.1f} us (with profiling)")
    for i, nme in enumerate(names):
        col = pr[act, i]
        print(f"  {nme:14s} mean {col.mean():12.0f}  max {col.max():12.0f}")
print("ok", cfg, out.float().abs().mean().item())
