"""One-time B200 profiling sweep -> reference-format trace -> fit -> coeffs.

    python scripts/profile_b200.py --model OLMoE-1B-7B [--plan-reps 3] [--iters 3]

This is the RaMP offline step run on the real megakernel:
for every (S, beta) point of ramp's profiling plan (5 batch sizes x 5 skews,
ramp/cost_model.py:212-231) and every routing seed, every config of the B200
pool is launched and timed (sweep.MeasuredTimer), the samples are written in
ramp's trace CSV schema (loadable by ramp.load_trace), and each config's four
coefficients are fitted with the reference's OLS (cost_model.fit).  The model
variant (P2 / P3 / P4, the reference's ablation ladder) is chosen by held-out
dispatch regret on the sweep itself (choose_variant), together with the B200
variant B4 (cost_model.py: waves on the job grid, traffic terms on the
HBM-equivalent grid with a fitted per-config L2-reuse factor).
`--refit` skips the GPU sweep and refits from an existing trace.
Outputs (under paper_2604_26039_b200/data/ unless --out is given):
    trace_<model>_b200.csv, coeffs_<model>_b200.json, fit_<model>_b200.json
Then it evaluates the fitted table against an exhaustive on-GPU sweep over the
reference's held-out test points: regret_<model>_b200.csv / speedup_... .csv
and a JSON summary.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs  # noqa: E402
from paper_2604_26039_b200.cost_model import (B200_BATCH_SIZES, b4_features, coeff_store_dict, fit, fit_b4, profiling_plan,  # noqa: E402
                                              useful_configs, write_coeff_store)
from paper_2604_26039_b200.routing import sample_histogram  # noqa: E402
from paper_2604_26039_b200.dispatch import DispatchTable, evaluate_regret, speedup_ra_vs_static  # noqa: E402
from paper_2604_26039_b200.moe import DeviceTable  # noqa: E402
from paper_2604_26039_b200.sweep import MeasuredTimer, make_fp8_weights  # noqa: E402
from paper_2604_26039_b200.trace import load_trace, profile  # noqa: E402


def _fit_all(pool, by_cfg, hw, variant, geom):
    cols = pool.columns()
    out = {}
    for cid, ss in by_cfg.items():
        if variant in ("B4", "B4r"):
            jpm = int(cols["ntile"][cid] * cols["split_k"][cid])
            out[cid] = fit_b4(ss, b4_features(ss, geom, int(cols["bm"][cid]), jpm), hw, relative=variant == "B4r")
        else:
            out[cid] = fit(ss, hw, variant)
    return out


def choose_variant(pool, trace, hw, geom):
    """Pick the cost-model variant (the reference's P2 / P3 / P4,
    ramp/cost_model.py:163-196, or the B200 "B4") with the lowest held-out
    dispatch regret: for every routing seed of every plan point, fit on the
    other seeds, select on it with the table's own host predictor, compare
    with the measured best there; mean over all folds."""
    points: dict = {}
    for s in trace.samples:
        points.setdefault((s.S, s.beta_target), {}).setdefault(s.seed, {})[s.config_id] = s
    n_seeds = min(len(v) for v in points.values())
    ids = [c.id for c in pool]
    out = {}
    for variant in ("P2", "P3", "P4", "B4", "B4r"):
        regs = []
        for hold in range(n_seeds):
            train: dict[int, list] = {c: [] for c in ids}
            test = []
            for _, by_seed in sorted(points.items()):
                seeds = sorted(by_seed)
                for j, sd in enumerate(seeds):
                    if j == hold:
                        test.append(by_seed[sd])
                    else:
                        for c in ids:
                            train[c].append(by_seed[sd][c])
            reports = _fit_all(pool, train, hw, variant, geom)
            table = DispatchTable(model="cv", pool=pool, coefficients={c: r.coefficients for c, r in reports.items()},
                                  sm_count=hw.sm_count)
            for pt in test:
                s0 = pt[ids[0]]
                hist = sample_histogram(geom.E, s0.S, geom.top_k, s0.beta_target, s0.seed).histogram
                t = np.array([pt[c].time_us for c in ids])
                regs.append(t[table.host_select(hist)] / t.min() - 1.0)
        out[variant] = float(np.mean(regs))
    return min(out, key=out.get), out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="OLMoE-1B-7B", choices=sorted(BASELINE_MODELS))
    ap.add_argument("--plan-reps", type=int, default=3)
    ap.add_argument("--eval-reps", type=int, default=2)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--out", default=str(ROOT / "paper_2604_26039_b200" / "data"))
    ap.add_argument("--skip-eval", action="store_true")
    ap.add_argument("--eval-iters", type=int, default=7)
    ap.add_argument("--dtype", default="bf16", choices=("bf16", "fp8"))
    ap.add_argument("--refit", action="store_true", help="reuse the existing trace (no profiling sweep)")
    ap.add_argument("--prune-tol", type=float, default=0.05,
                    help="keep as dispatch candidates only configs within this fraction of the best at some "
                         "profiled point (0: keep all)")
    a = ap.parse_args()
    out = Path(a.out)
    out.mkdir(parents=True, exist_ok=True)
    geom = BASELINE_MODELS[a.model]
    hw = HardwareModel.b200()
    pool = enumerate_b200_configs(geom, hw, dtype=a.dtype)
    cols = pool.columns()
    n = len(pool)
    plan = profiling_plan(geom, batch_sizes=B200_BATCH_SIZES)
    tag = f"{a.model}_b200" + ("_fp8" if a.dtype == "fp8" else "")
    trace_path = out / f"trace_{tag}.csv"
    t0 = time.time()
    def make_timer():
        flat = DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                           group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols.get("kps"), h3=cols.get("h3"), a=np.ones(n),
                           b=np.zeros(n), c=np.zeros(n), d=np.zeros(n), N=geom.N, kappa_ok=False,
                           sm_count=hw.sm_count)
        if a.dtype == "fp8":
            return MeasuredTimer(geom, flat, iters=a.iters, fp8_weights=make_fp8_weights(geom))
        return MeasuredTimer(geom, flat, iters=a.iters)

    timer = None
    if a.refit:
        trace = load_trace(trace_path, pool)
    else:
        timer = make_timer()
        if trace_path.exists():
            trace_path.unlink()
        trace = profile(pool, geom, plan, timer, seeds_per_point=a.plan_reps, trace_path=trace_path)
    t_prof = time.time() - t0
    by_cfg: dict[int, list] = {}
    for s in trace.samples:
        by_cfg.setdefault(s.config_id, []).append(s)
    variant, validation = choose_variant(pool, trace, hw, geom)
    reports = _fit_all(pool, by_cfg, hw, variant, geom)
    store = coeff_store_dict(a.model, hw.sm_count, reports)
    active = useful_configs(trace.samples, a.prune_tol) if a.prune_tol > 0 else None
    if active is not None:
        store["active_ids"] = list(active)
    write_coeff_store(out / f"coeffs_{tag}.json", store)
    r2 = np.array([r.r_squared for r in reports.values()])
    summary = {"model": a.model, "pool": n, "plan_points": len(plan), "samples": len(trace.samples),
               "profile_s": round(t_prof, 1), "r2_median": float(np.median(r2)), "r2_min": float(r2.min()),
               "variant": variant, "heldout_regret_by_variant": validation,
               "active_configs": None if active is None else len(active), "prune_tol": a.prune_tol}
    print(json.dumps(summary), flush=True)
    if not a.skip_eval:
        table = DispatchTable(model=a.model, pool=pool,
                              coefficients={c: r.coefficients for c, r in reports.items()},
                              sm_count=hw.sm_count, active=active)
        t0 = time.time()
        timer = timer or make_timer()
        timer.iters = a.eval_iters
        reg = evaluate_regret(table, pool, geom, timer, seeds_per_point=a.eval_reps)
        spd = speedup_ra_vs_static(table, pool, geom, timer, seeds_per_point=a.eval_reps)
        (out / f"regret_{tag}.csv").write_text(reg.to_csv())
        (out / f"speedup_{tag}.csv").write_text(spd.to_csv())
        summary.update({"eval_s": round(time.time() - t0, 1), "regret": reg.aggregate(),
                        "speedup": spd.aggregate()})
        print(json.dumps({"regret": reg.aggregate(), "speedup": spd.aggregate()}), flush=True)
    (out / f"fit_{tag}.json").write_text(json.dumps(summary, indent=2) + "\n")


if __name__ == "__main__":
    main()
