"""Generate the golden fixtures that pin `oracle/` and the host mirror to the reference.

Run HERE (the build container), never on the GPU box:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

It imports the reference `ramp` package read-only from /root/reference and
writes small JSON fixtures next to this script.  The fixtures are committed;
the tests only read them, so nothing at test time touches /root/reference.

What each fixture pins (reference file:line of the producing function):
  seeds.json       derive_seed               ramp/oracle.py:69-71
  histograms.json  sample_histogram          ramp/routing.py:148-188
                   balancedness              ramp/routing.py:77-87
  pools.json       enumerate_configs         ramp/config_space.py:195-252
                   classify_regime           ramp/catalog.py:128-137
  grids.json       pool_grids / grid_size    ramp/routing.py:191-216
  fits.json        fit / r_squared           ramp/cost_model.py:163-209
  tables.json      profile + fit + select_config + predict_batch
                                             ramp/oracle.py:257-297, ramp/dispatch.py:89-122,
                                             ramp/cost_model.py:104-114
  eval.json        evaluate_regret / speedup_ra_vs_static / static_best
                                             ramp/dispatch.py:131-339
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

import ramp  # noqa: E402
from ramp import (  # noqa: E402
    DispatchTable,
    ExpertHistogram,
    HardwareModel,
    MoeGeometry,
    OracleParams,
    StepCache,
    balancedness,
    classify_regime,
    enumerate_configs,
    evaluate_regret,
    find_model,
    fit,
    profile,
    region_variables,
    round_robin,
    sample_histogram,
    select_config,
    speedup_ra_vs_static,
    static_best,
)
from ramp.cost_model import ProfilingSample, predict_batch, profiling_plan  # noqa: E402
from ramp.dispatch import default_test_points  # noqa: E402
from ramp.oracle import derive_seed, simulate_pool_times  # noqa: E402
from ramp.routing import BetaUnreachableError, pool_grids  # noqa: E402

OUT = Path(__file__).resolve().parent
MASTER = 42

# BASELINE.json model shapes (N = 2 * d_ff, K = d_model) plus the reference's
# own catalog rows and test geometries.
BASELINE_GEOMS = {
    "OLMoE-1B-7B": dict(E=64, N=2 * 1024, K=2048, top_k=8),
    "Qwen3-30B-A3B": dict(E=128, N=2 * 768, K=2048, top_k=8),
    "Mixtral-8x7B": dict(E=8, N=2 * 14336, K=4096, top_k=2),
    "DeepSeek-V3": dict(E=256, N=2 * 2048, K=7168, top_k=8),
}
TEST_GEOMS = {
    "tiny": dict(E=4, N=256, K=1024, top_k=2),
    "deep": dict(E=32, N=1024, K=16384, top_k=8),
}
B200_HW = dict(sm_count=148, elem_size=2)


def geom(name: str) -> MoeGeometry:
    if name in BASELINE_GEOMS:
        return MoeGeometry(name=name, **BASELINE_GEOMS[name])
    if name in TEST_GEOMS:
        return MoeGeometry(name=name, **TEST_GEOMS[name])
    return find_model(name)


def pool_for(name: str, hw_over: dict | None):
    g = geom(name)
    hw = HardwareModel.from_overrides(hw_over or {})
    return enumerate_configs(g, hw, classify_regime(region_variables(g)))


def pool_columns(pool) -> dict:
    return {
        k: [int(getattr(c, k)) for c in pool]
        for k in ("bm", "bn", "wn", "stg", "ttn", "group_m", "split_k")
    }


def digest(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()


def dump(name: str, obj) -> None:
    path = OUT / name
    path.write_text(json.dumps(obj, sort_keys=True, separators=(",", ":")) + "\n")
    print(f"wrote {path} ({path.stat().st_size} bytes)")


def gen_seeds():
    rows = []
    for keys in ([42, 1, 8, 300, 0], [42, 3, 16, 500, 2], [42, 4, 1024, 1000, 1], [7], [0, 0],
                 [42, 6, 64, 200, 0], [42, 7, 512, 500, 2], [42, 8, 0, 0, 0], [2**40, 5]):
        rows.append({"keys": keys, "seed": str(derive_seed(*keys))})
    dump("seeds.json", rows)


def gen_histograms():
    rows = []
    models = {**BASELINE_GEOMS, "tiny": TEST_GEOMS["tiny"]}
    for name, g in models.items():
        for S in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024):
            for beta in (0.2, 0.3, 0.5, 0.8, 1.0):
                for rep in range(2):
                    seed = derive_seed(MASTER, 3, S, round(beta * 1000), rep)
                    entry = {"model": name, "E": g["E"], "S": S, "top_k": g["top_k"],
                             "beta": beta, "seed": str(seed)}
                    try:
                        smp = sample_histogram(g["E"], S, g["top_k"], beta, seed)
                    except BetaUnreachableError as exc:
                        entry["unreachable"] = str(exc)
                    else:
                        entry["counts"] = list(smp.histogram.counts)
                        entry["beta_achieved"] = smp.beta_achieved
                    rows.append(entry)
    # balancedness on hand-built histograms
    extra = []
    for counts in ([5, 0, 0, 0], [1, 1, 1, 1], [3, 1, 0, 7], [100] + [0] * 63, [2] * 64, [9]):
        extra.append({"counts": counts, "beta": balancedness(ExpertHistogram(tuple(counts)))})
    dump("histograms.json", {"samples": rows, "balancedness": extra})


def gen_pools():
    out = []
    names = ["tiny", "deep", "OLMoE", "Qwen3", "DSv3-EP8", "Mixtral", "DSv3-TP8", "DBRX",
             *BASELINE_GEOMS]
    for name in names:
        for hw_tag, hw_over in (("h200", None), ("b200", B200_HW)):
            pool = pool_for(name, hw_over)
            cols = pool_columns(pool)
            rep = pool.regime
            entry = {
                "geom": name, "hw": hw_tag, "size": len(pool), "digest": digest(cols),
                "regime": rep.regime, "group_m_required": rep.group_m_required,
                "split_k_eligible": rep.split_k_eligible,
            }
            if name in ("tiny", "deep", "OLMoE") or (name == "OLMoE-1B-7B" and hw_tag == "b200"):
                entry["columns"] = cols
            out.append(entry)
    dump("pools.json", out)


def gen_grids():
    out = []
    for name, hw_over in (("OLMoE", None), ("deep", None), ("OLMoE-1B-7B", B200_HW),
                          ("Mixtral-8x7B", B200_HW)):
        pool = pool_for(name, hw_over)
        g = pool.geom
        for S, beta, rep in ((1, 0.2, 0), (16, 0.5, 0), (64, 1.0, 0), (512, 0.2, 1), (8, 0.5, 1)):
            seed = derive_seed(MASTER, 3, S, round(beta * 1000), rep)
            try:
                hist = sample_histogram(g.E, S, g.top_k, beta, seed).histogram
            except BetaUnreachableError:
                continue
            grids = pool_grids(pool, hist)
            out.append({"geom": name, "hw": "b200" if hw_over else "h200",
                        "counts": list(hist.counts), "grids": [int(x) for x in grids]})
    dump("grids.json", out)


def gen_fits():
    rng = np.random.default_rng(1234)
    out = []
    hw = HardwareModel()
    cases = []
    # well-posed staircase data, sub-wave data (log term active), rank-deficient data
    g1 = np.array([10, 40, 90, 130, 200, 300, 420, 700], dtype=np.int64)
    cases.append(("staircase", g1, 20 + 5 * np.ceil(g1 / 132) + 0.03 * g1 + rng.normal(0, 0.2, g1.size)))
    g2 = np.array([1, 3, 8, 16, 30, 60, 90, 120], dtype=np.int64)
    cases.append(("subwave", g2, 15 + 2.5 * np.log(g2 + 1.0) + 0.01 * g2 + rng.normal(0, 0.05, g2.size)))
    g3 = np.array([5, 5, 10, 10, 20, 20], dtype=np.int64)
    cases.append(("onewave", g3, 30 + 0.5 * g3))
    g4 = np.array([132, 264, 396, 528, 132, 264], dtype=np.int64)
    cases.append(("collinear", g4, 10 + 0.1 * g4))
    for tag, g, t in cases:
        samples = [ProfilingSample(config_id=0, S=8, beta_target=0.5, seed=i, g=int(gv),
                                   time_us=float(round(tv, 6)))
                   for i, (gv, tv) in enumerate(zip(g, t))]
        for variant in ("P2", "P3", "P4"):
            rep = fit(samples, hw, variant)
            co = rep.coefficients
            out.append({"case": tag, "variant": variant, "g": [int(x) for x in g],
                        "t": [s.time_us for s in samples],
                        "a": co.a, "b": co.b, "c": co.c, "d": co.d, "uses_log": co.uses_log,
                        "r_squared": rep.r_squared, "median_grid": rep.median_grid,
                        "condition_flag": rep.condition_flag})
    dump("fits.json", out)


def fitted_table(pool, params, plan_kwargs=None, seeds=3):
    g = pool.geom
    plan = profiling_plan(g, **(plan_kwargs or {}))
    trace = profile(pool, g, plan, params, seeds_per_point=seeds, master_seed=MASTER)
    by_cfg: dict[int, list] = {}
    for s in trace.samples:
        by_cfg.setdefault(s.config_id, []).append(s)
    coeffs = {cid: fit(ss, pool.hw, "P4").coefficients for cid, ss in by_cfg.items()}
    return DispatchTable(model=g.name, pool=pool, coefficients=coeffs, sm_count=pool.hw.sm_count)


def gen_tables():
    out = []
    setups = [
        ("OLMoE", None, OracleParams(), None),
        ("deep", None, OracleParams(), dict(batch_sizes=(8, 32, 128), betas=(0.3, 0.5, 1.0))),
        ("OLMoE-1B-7B", B200_HW, OracleParams(sm_count=148, elem_size=2), None),
    ]
    for name, hw_over, params, plan_kwargs in setups:
        pool = pool_for(name, hw_over)
        table = fitted_table(pool, params, plan_kwargs, seeds=2 if name == "deep" else 3)
        g = pool.geom
        coeffs = [[table.coefficients[i].a, table.coefficients[i].b, table.coefficients[i].c,
                   table.coefficients[i].d, table.coefficients[i].uses_log] for i in range(len(pool))]
        picks = []
        for S in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024):
            for beta in (0.2, 0.5, 0.8, 1.0):
                for rep in range(3):
                    seed = derive_seed(MASTER, 3, S, round(beta * 1000), rep)
                    try:
                        hist = sample_histogram(g.E, S, g.top_k, beta, seed).histogram
                    except BetaUnreachableError:
                        continue
                    before = table.evaluations
                    sel = select_config(table, hist, None, 0)
                    picks.append({"counts": list(hist.counts), "selected": sel,
                                  "evaluations": table.evaluations - before})
        # hand-built extremes: one hot expert, everything on one expert, empty
        for counts in ([g.top_k] + [0] * (g.E - 1), [0] * (g.E - 1) + [g.top_k * 4096],
                       [0] * g.E, list(round_robin(g.E, g.E * 104).counts)):
            before = table.evaluations
            sel = select_config(table, ExpertHistogram(tuple(counts)), None, 0)
            picks.append({"counts": counts, "selected": sel,
                          "evaluations": table.evaluations - before})
        # one full prediction vector, to pin predict_batch's fp64 arithmetic
        hist = sample_histogram(g.E, 64, g.top_k, 0.5, derive_seed(MASTER, 3, 64, 500, 0)).histogram
        grids = pool_grids(pool, hist)
        pred = predict_batch(table._a, table._b, table._c, table._d, grids, table.sm_count)
        out.append({"geom": name, "hw": "b200" if hw_over else "h200", "sm_count": table.sm_count,
                    "coeffs": coeffs, "picks": picks,
                    "predict": {"counts": list(hist.counts), "grids": [int(x) for x in grids],
                                "pred": [float(x).hex() for x in pred]}})
    dump("tables.json", out)


def gen_eval():
    pool = pool_for("OLMoE", None)
    g = pool.geom
    params = OracleParams()
    table = fitted_table(pool, params)
    points = [(8, 0.2), (16, 0.5), (64, 0.5), (128, 1.0), (1024, 0.8)]
    reg = evaluate_regret(table, pool, g, params, test_points=points, seeds_per_point=2,
                          master_seed=MASTER)
    spd = speedup_ra_vs_static(table, pool, g, params, points=points, seeds_per_point=2,
                               master_seed=MASTER)
    quiet = OracleParams(noise_cv=0.0)
    rr = round_robin(g.E, 64 * g.top_k)
    sim = simulate_pool_times(pool, rr, quiet, point_seed=0)
    noisy = simulate_pool_times(pool, rr, params, point_seed=derive_seed(MASTER, 2, 64, 1000, 0))
    dump("eval.json", {
        "points": points,
        "regret_csv": reg.to_csv(), "regret": reg.aggregate(),
        "speedup_csv": spd.to_csv(), "speedup": spd.aggregate(),
        "static_best_8_64": static_best(pool, g, params, [8, 64]),
        "default_test_points": [list(p) for p in default_test_points(g)],
        "sim_quiet_rr64": [float(x).hex() for x in sim],
        "sim_noisy_rr64": [float(x).hex() for x in noisy],
    })


if __name__ == "__main__":
    print(f"reference ramp {ramp.__version__} from {ramp.__file__}")
    gen_seeds()
    gen_histograms()
    gen_pools()
    gen_grids()
    gen_fits()
    gen_tables()
    gen_eval()
