"""Where does a layer call's time go under CUDA-graph replay?  (development tool)

For sweep points of the bench, captures graphs of the full layer (route +
megakernel), route only and megakernel only, times their replays with CUDA
events, and replays once more with the globaltimer profile buffer to print
the per-phase timeline (ns from the route kernel's start).
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from bench import MODEL, load_table  # noqa: E402
from paper_2604_26039_b200 import _lib, moe  # noqa: E402
from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, derive_seed  # noqa: E402
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.sweep import make_inputs, make_weights  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--points", default="1:0.2,16:1.0,512:0.2")
ap.add_argument("--cfg", default="-1", help="comma list of forced config ids (-1: dispatcher)")
ap.add_argument("--flat", action="store_true", help="flat cost table over the current pool (forced configs only)")
ap.add_argument("--fp8", action="store_true", help="Qwen3-30B-A3B MXFP8 path with its fitted table")
a = ap.parse_args()
geom = BASELINE_MODELS["Qwen3-30B-A3B" if a.fp8 else MODEL]
dev = torch.device("cuda")
pool = enumerate_b200_configs(geom, HardwareModel.b200(), dtype="fp8" if a.fp8 else "bf16")
if a.flat:
    cols = pool.columns()
    n = len(pool)
    dtab = moe.DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                           group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols.get("kps"), h3=cols.get("h3"), a=np.ones(n), b=np.zeros(n),
                           c=np.zeros(n), d=np.zeros(n), N=geom.N, kappa_ok=True, sm_count=148, device=dev)
elif a.fp8:
    from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store
    from paper_2604_26039_b200.dispatch import DispatchTable
    from paper_2604_26039_b200.sweep import make_fp8_weights
    store = read_coeff_store(ROOT / "paper_2604_26039_b200" / "data" / "coeffs_Qwen3-30B-A3B_b200_fp8.json")
    _, sm, co = parse_coeff_store(store)
    dtab = DispatchTable(model=geom.name, pool=pool, coefficients=co, sm_count=sm,
                         active=active_ids_of(store)).device_table(device=dev)
else:
    table, _ = load_table(geom, pool, HardwareModel.b200())
    dtab = table.device_table(device=dev)
if a.fp8:
    wq = make_fp8_weights(geom, seed=1, device=dev)
else:
    w1, w2 = make_weights(geom, seed=1, device=dev)
H, I = geom.K, geom.N // 2
lib = _lib.load()
side = torch.cuda.Stream()


def graph(fn):
    with torch.cuda.stream(side):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            fn()
    torch.cuda.synchronize()
    return g


def timeit(g, n=20):
    ts = []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts[3:]))


empty = torch.zeros(1, device=dev)
g_empty = graph(lambda: empty.add_(1))
print(f"trivial graph (1 torch kernel): {timeit(g_empty):.2f} us")
for spec, forced in [(p, int(f)) for p in a.points.split(",") for f in a.cfg.split(",")]:
    S, beta = int(spec.split(":")[0]), float(spec.split(":")[1])
    hs = derive_seed(42, EVAL_HIST_DOMAIN, S, round(beta * 1000), 0)
    hist = sample_histogram(geom.E, S, geom.top_k, beta, hs).histogram
    x, ids, w = make_inputs(geom, hist, hs, dev)
    ws = moe.Workspace(S, H, I, geom.E, geom.top_k, device=dev)
    out = torch.empty(S, H, dtype=torch.bfloat16, device=dev)

    def run(phases=3):
        if a.fp8:
            moe.fused_moe_fp8(x, wq, w, ids, dtab, forced, out=out, workspace=ws, phases=phases)
        else:
            moe.fused_moe(x, w1, w2, w, ids, dtab, forced, out=out, workspace=ws, phases=phases)

    full, route, mega = graph(run), graph(lambda: run(1)), graph(lambda: run(2))
    t_full, t_route, t_mega = timeit(full), timeit(route), timeit(mega)
    cfg = dtab.pool_id(int(ws.sel[0].item()))
    c = pool.by_id(cfg)
    buf = torch.zeros(149 * 32 + 148 * 16 * 4, dtype=torch.int64, device=dev)
    lib.ramp_set_profile_buffer(buf.data_ptr())
    gp = graph(run)
    lib.ramp_set_profile_buffer(None)
    for _ in range(2):
        gp.replay()
    torch.cuda.synchronize()
    buf.zero_()  # job-log rows of earlier replays would otherwise linger
    gp.replay()
    torch.cuda.synchronize()
    hb = buf.cpu().numpy().astype(np.float64)
    allb = hb[:149 * 32].reshape(149, 32)
    jl = hb[149 * 32:].reshape(148, 16, 4)
    pr, rt = allb[:148], allb[148]
    t0 = rt[0]
    tl = ["entry", "start", "gathered", "producer_done", "epilogue_done", "end_arrive", "end_pass", "final",
          "cfg", "first_expert", "first_issue", "unused", "first_acc", "role", "claimed"]
    def q3(v):
        v = (v[v > 0] - t0) / 1e3
        return f"{np.min(v):.1f}/{np.median(v):.1f}/{np.max(v):.1f}" + ("" if len(v) == len(pr) else f"({len(v)})")
    line = "  ".join(f"{n} {q3(pr[:, 16 + i])}" for i, n in enumerate(tl) if np.any(pr[:, 16 + i] > 0))
    print(f"S={S} beta={beta} active={hist.active_experts} cfg {cfg} (bm {c.bm} ttn {c.ttn} stg {c.stg} gm "
          f"{int(c.group_m)} mode {c.mode} sk {c.split_k}): full {t_full:.2f} us  route {t_route:.2f}  "
          f"mega {t_mega:.2f}")
    print(f"   route stamps (us): hist {(rt[1]-t0)/1e3:.2f} dispatch {(rt[2]-t0)/1e3:.2f} "
          f"align {(rt[3]-t0)/1e3:.2f} done {(rt[4]-t0)/1e3:.2f}  [dispatch: mt {(rt[12]-t0)/1e3:.2f} "
          f"eval {(rt[13]-t0)/1e3:.2f} reduced {(rt[14]-t0)/1e3:.2f}; align scan+pad {(rt[5]-t0)/1e3:.2f}]  cycles entry->dispatched {rt[7]-rt[6]:.0f}"
          + (f"  [first pass started {(rt[15]-t0)/1e3:.2f}]" if rt[15] > 0 else ""))
    rc = hb[148 * 32 + 16:148 * 32 + 16 + 25]  # -DRAMP_ROUTE_CLOCKS build (spills into the job-log area)
    if rc[0] > 0:  # clock64 points of the route block, cycles from entry
        print("   route clocks: " + " ".join(f"{k}:{int(rc[k] - rc[0])}" for k in range(25) if rc[k] > 0))
    print(f"   timeline (us from route start, min/median/max over CTAs): {line}")
    # per-job log: phase-1 (kind 0) jobs are ids < nJobA
    npp = int(ws.sel[1].item())
    mt = npp // c.bm
    stripes = I // (c.ttn // 2)
    sk = c.split_k if c.mode == 1 else 1
    nja = mt * stripes * sk
    rows = [r for r in jl.reshape(-1, 4) if r[1] > 0]
    for kind, name in ((0, "phase-1"), (1, "phase-3")):
        rr = np.array([r for r in rows if (r[0] < nja) == (kind == 0)])
        if len(rr) == 0:
            continue
        cl, iss, dn = (rr[:, 1] - t0) / 1e3, (rr[:, 2] - t0) / 1e3, (rr[:, 3] - t0) / 1e3
        q = lambda v: f"{v.min():.1f}/{np.median(v):.1f}/{v.max():.1f}"  # noqa: E731
        print(f"   {name} jobs {len(rr)} (of {nja if kind == 0 else 'n/a'}): claimed {q(cl)}  loads-issued {q(iss)}  "
              f"done {q(dn)}  claim->done {q(dn - cl)}")
