"""Kernel-agnostic dispatch: the RaMP pipeline driven by a
third-party kernel's measured timings instead of the B200 megakernel's.

    python scripts/profile_thirdparty.py --model OLMoE-1B-7B

vLLM's Triton fused_moe (`fused_experts`) is timed on B200 under every config
of a triton-family pool (BLOCK_SIZE_M/N/K x GROUP_SIZE_M), over the profiling
plan, into a trace CSV in the reference schema; the per-config four-term fit,
the dispatcher (the same on-device fp64 kernel) and the regret / speedup
harness are the ones the megakernel uses -- only the timing source changes.
This mirrors the paper's Alpha-MoE experiment and the
reference's criterion 12 (tests/test_acceptance.py:423-457).
Outputs under paper_2604_26039_b200/data/: trace_/coeffs_/regret_/speedup_/fit_<model>_vllm-triton.*
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2604_26039_b200.catalog import BASELINE_MODELS  # noqa: E402
from paper_2604_26039_b200.config_space import HardwareModel, enumerate_triton_configs  # noqa: E402
from paper_2604_26039_b200.cost_model import coeff_store_dict, profiling_plan, write_coeff_store  # noqa: E402
from paper_2604_26039_b200.dispatch import DispatchTable, evaluate_regret, speedup_ra_vs_static  # noqa: E402
from paper_2604_26039_b200.thirdparty import VllmTritonTimer  # noqa: E402
from paper_2604_26039_b200.trace import profile  # noqa: E402
from scripts.profile_b200 import _fit_all, choose_variant  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="OLMoE-1B-7B", choices=sorted(BASELINE_MODELS))
    ap.add_argument("--plan-reps", type=int, default=2)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--eval-reps", type=int, default=1)
    ap.add_argument("--out", default=str(ROOT / "paper_2604_26039_b200" / "data"))
    a = ap.parse_args()
    out = Path(a.out)
    geom = BASELINE_MODELS[a.model]
    hw = HardwareModel.b200()
    pool = enumerate_triton_configs(geom, hw)
    plan = profiling_plan(geom, batch_sizes=(8, 32, 128, 512))
    tag = f"{a.model}_vllm-triton"
    t0 = time.time()
    timer = VllmTritonTimer(geom, iters=a.iters)
    trace_path = out / f"trace_{tag}.csv"
    if trace_path.exists():
        trace_path.unlink()
    trace = profile(pool, geom, plan, timer, seeds_per_point=a.plan_reps, trace_path=trace_path)
    t_prof = time.time() - t0
    by_cfg: dict[int, list] = {}
    for s in trace.samples:
        by_cfg.setdefault(s.config_id, []).append(s)
    variant, validation = choose_variant(pool, trace, hw, geom)
    reports = _fit_all(pool, by_cfg, hw, variant, geom)
    write_coeff_store(out / f"coeffs_{tag}.json", coeff_store_dict(a.model, hw.sm_count, reports))
    table = DispatchTable(model=a.model, pool=pool, coefficients={c: r.coefficients for c, r in reports.items()},
                          sm_count=hw.sm_count)
    t1 = time.time()
    reg = evaluate_regret(table, pool, geom, timer, seeds_per_point=a.eval_reps)
    spd = speedup_ra_vs_static(table, pool, geom, timer, seeds_per_point=a.eval_reps)
    (out / f"regret_{tag}.csv").write_text(reg.to_csv())
    (out / f"speedup_{tag}.csv").write_text(spd.to_csv())
    summary = {"kernel": "vLLM Triton fused_moe (fused_experts) under override_config", "model": a.model,
               "pool": len(pool), "plan_points": len(plan), "samples": len(trace.samples),
               "profile_s": round(t_prof, 1), "variant": variant, "heldout_regret_by_variant": validation,
               "eval_s": round(time.time() - t1, 1), "regret": reg.aggregate(), "speedup": spd.aggregate()}
    (out / f"fit_{tag}.json").write_text(json.dumps(summary, indent=2) + "\n")
    print(json.dumps(summary), flush=True)


if __name__ == "__main__":
    main()
