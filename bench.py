"""Benchmark: the OLMoE-1B-7B fused-MoE layer sweep on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload ("step"): one pass over the beta x batch sweep of BASELINE.json
configs[1] -- OLMoE-1B-7B (E=64, top-8, d=2048, d_ff=1024), BF16,
S in {1,2,4,...,512} x beta in {0.2,0.5,1.0} (beta=1 is unreachable for
S*k < E and dropped, as ramp.profiling_plan drops it) -- 27 layer calls, each
routed by the on-device dispatcher (routing-aware, forced_cfg = -1).  The
histograms are the reference's own evaluation draws
(sample_histogram(E, S, 8, beta, derive_seed(42, 3, S, 1000*beta, 0))),
expanded into concrete top-k ids; tokens, routing weights and expert weights
are synthetic / random-init.  Every layer call uses the next of 8 resident
copies of the expert weights (8 x 805 MB >> 126 MB L2), so weights are cold as
in a real multi-layer model; no flush is needed inside the timed region.

metric / value: whole-job TFLOP/s over the sweep (6*S*k*H*I per layer, all
ranks' layers / max-over-ranks time); the per-point microseconds, the
routing-aware-vs-static speedup and the dispatch regret against an
exhaustive on-GPU sweep are reported beside it.  N > 1 runs independent
replicas (the OLMoE layer is not expert-sharded).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MODEL = "OLMoE-1B-7B"
BATCHES = (1, 2, 4, 8, 16, 32, 64, 128, 256, 512)
BETAS = (0.2, 0.5, 1.0)
N_COPIES = 8
METRIC = "fused-MoE layer TFLOP/s over the OLMoE-1B-7B beta x batch sweep (routing-aware dispatch)"


def sweep_points(geom):
    from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, derive_seed
    from paper_2604_26039_b200.routing import BetaUnreachableError, sample_histogram

    pts = []
    for S in BATCHES:
        for beta in BETAS:
            seed = derive_seed(42, EVAL_HIST_DOMAIN, S, round(beta * 1000), 0)
            try:
                hist = sample_histogram(geom.E, S, geom.top_k, beta, seed).histogram
            except BetaUnreachableError:
                continue
            pts.append(dict(S=S, beta=beta, seed=seed, hist=hist))
    return pts


def layer_flops(geom, S):
    return 6 * S * geom.top_k * geom.K * (geom.N // 2)


def layer_bytes(geom, hist, S):
    """Algorithmic HBM bytes of one layer call: active experts'
    weights once, tokens in and out once, ids + weights."""
    H, I = geom.K, geom.N // 2
    return hist.active_experts * 3 * H * I * 2 + S * H * 4 + 8 * S * geom.top_k


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML
    polling thread (2 ms period; the timed region can be only tens of ms,
    shorter than nvidia-smi's start-up), nvidia-smi as the fallback."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        self.gpu = int(ids[gpu]) if gpu < len(ids) and ids[gpu].isdigit() else gpu
        self.rows, self.max_mhz, self.stop, self.thread, self.err = [], None, threading.Event(), None, None

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            bits = (N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap)

            def poll():
                while True:
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append((float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                                      tuple(n for n, b in zip(self.NAMES, bits) if r & b)))
                    if self.stop.wait(0.002):
                        break

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
        except Exception as e:  # no NVML: fall back to one nvidia-smi read after the region
            self.err = repr(e)
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread is not None:
            self.thread.join(timeout=2)
        elif not self.rows:
            self._smi()

    def _smi(self):
        q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
            "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20).stdout
            f = [x.strip() for x in out.strip().split(",")]
            self.max_mhz = float(f[1])
            self.rows.append((float(f[0]), tuple(n for n, v in zip(self.NAMES, f[2:]) if v == "Active")))
        except Exception as e:
            self.err = (self.err or "") + " / nvidia-smi: " + repr(e)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [f"no clock samples ({self.err})"]}
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])), "sm_max_mhz": self.max_mhz,
                "reasons": sorted({n for r in self.rows for n in r[1]}), "samples": len(self.rows),
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


# ------------------------------------------------------------------ CPU oracle
def cpu_weights(geom, seed=42):
    """fp32 host copy of random-init weights for the CPU (oracle) arm."""
    rng = np.random.default_rng(seed)
    E, H, I = geom.E, geom.K, geom.N // 2
    w1 = (rng.standard_normal((E, 2 * I, H), dtype=np.float32) * np.float32(H ** -0.5))
    w2 = (rng.standard_normal((E, H, I), dtype=np.float32) * np.float32(I ** -0.5))
    return w1, w2


def cpu_inputs(geom, pt):
    from paper_2604_26039_b200.dispatch import derive_seed
    from paper_2604_26039_b200.routing import topk_from_histogram

    S, k = pt["S"], geom.top_k
    ids = topk_from_histogram(pt["hist"].counts, S, k, derive_seed(pt["seed"], 6) % (2 ** 63))
    rng = np.random.default_rng(derive_seed(pt["seed"], 8))
    lg = rng.standard_normal((S, k)).astype(np.float32)
    w = np.exp(lg - lg.max(1, keepdims=True))
    w /= w.sum(1, keepdims=True)
    x = rng.standard_normal((S, geom.K)).astype(np.float32)
    return x, ids, w.astype(np.float32)


def run_cpu_sweep(geom, pts, w1, w2, budget_s=None):
    """One pass of the fp32 oracle over the sweep points (bounded by budget_s)."""
    from oracle.moe_ref import fused_moe_ref

    flops, t_total, n = 0, 0.0, 0
    for pt in pts:
        x, ids, w = cpu_inputs(geom, pt)
        t0 = time.perf_counter()
        fused_moe_ref(x, w1, w2, w, ids)
        t_total += time.perf_counter() - t0
        flops += layer_flops(geom, pt["S"])
        n += 1
        if budget_s is not None and t_total > budget_s:
            break
    return flops, t_total, n


def reference_arm(args, geom):
    """--impl reference: the reference path has no fused-MoE kernel, so its CPU
    implementation of the layer is the oracle port (oracle/moe_ref.py, the
    paper's three phases in fp32 numpy with all host threads)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pts = sweep_points(geom)
    w1, w2 = cpu_weights(geom)
    for _ in range(args.warmup):
        run_cpu_sweep(geom, pts[:3], w1, w2)
    flops, secs = 0, 0.0
    for _ in range(args.steps):
        f, t, _ = run_cpu_sweep(geom, pts, w1, w2)
        flops += f
        secs += t
    value = flops / secs / 1e12
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (random-init weights, reference evaluation histograms)",
            "config": {"workload": f"{MODEL} MoE layer beta x batch sweep, fp32 CPU oracle port",
                       "points": len(pts)},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                             "sample": f"full {len(pts)}-point sweep per step, numpy fp32 (oracle/moe_ref.py)"},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ FP8 leg
def fp8_row_errors(geom, wq, x, ids, w, out, n_rows=16, seed=0):
    """Norm-wise relative error of the MXFP8 layer on a sample of output rows
    against (a) plain fp32 math on the dequantised expert weights (tokens and
    activations unquantised: north_star's "vs the reference's fp32 output")
    and (b) the same math with the tokens and SwiGLU activations quantised per
    32 exactly as the kernel does (what is left: accumulation order, bf16 out)."""
    import torch

    from paper_2604_26039_b200.quant import GROUP, mx_dequantize, quantize_tokens_ref, untile_scales

    H, I, k = geom.K, geom.N // 2, geom.top_k
    S = x.shape[0]
    rows = np.random.default_rng(seed).choice(S, size=min(n_rows, S), replace=False)
    r1, r2 = 2 * I // 128, H // 128
    cache = {}

    def expert(e):
        if e not in cache:
            s1 = untile_scales(wq.w1_sf[e * r1:(e + 1) * r1]).reshape(2 * I, H // GROUP)
            s2 = untile_scales(wq.w2_sf[e * r2:(e + 1) * r2]).reshape(H, I // GROUP)
            cache[e] = (mx_dequantize(wq.w1_q[e], s1), mx_dequantize(wq.w2_q[e], s2))
        return cache[e]

    ref32 = torch.zeros(len(rows), H, device=x.device)
    refq = torch.zeros_like(ref32)
    xf = x.float()
    for r, t in enumerate(rows):
        xq = quantize_tokens_ref(xf[t][None])[0]
        for j in range(k):
            d1, d2 = expert(int(ids[t, j]))
            h = d1 @ xf[t]
            ref32[r] += float(w[t, j]) * (d2 @ (torch.nn.functional.silu(h[:I]) * h[I:]))
            hq = d1 @ xq
            aq = quantize_tokens_ref((torch.nn.functional.silu(hq[:I]) * hq[I:])[None])[0]
            refq[r] += float(w[t, j]) * (d2 @ aq)
    o = out.float()[rows]
    return {"rows": len(rows), "vs_fp32": float((o - ref32).norm() / ref32.norm()),
            "vs_mx_emulation": float((o - refq).norm() / refq.norm())}



FP8_MODEL = "Qwen3-30B-A3B"
FP8_BATCHES = (1, 8, 32, 128, 512, 2048)
FP8_BETAS = (0.5, 0.55)  # 12 / 15 of 128 experts active: BASELINE configs[2]'s 8-14% skew
FP8_COPIES = 4


def fp8_leg(dev):
    """BASELINE configs[2]: Qwen3-30B-A3B MoE layer, MXFP8 block-scaled, skewed
    routing, on-device dispatch over the FP8 pool with its own fitted table.
    Untimed by the step contract; reported as a side object of the line."""
    import torch

    from paper_2604_26039_b200 import moe
    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs
    from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store
    from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, DispatchTable, derive_seed
    from paper_2604_26039_b200.routing import BetaUnreachableError, sample_histogram
    from paper_2604_26039_b200.sweep import make_fp8_weights, make_inputs

    geom = BASELINE_MODELS[FP8_MODEL]
    path = ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{FP8_MODEL}_b200_fp8.json"
    if not path.exists():
        return {"skipped": f"{path.name} missing (scripts/profile_b200.py --model {FP8_MODEL} --dtype fp8)"}
    pool = enumerate_b200_configs(geom, HardwareModel.b200(), dtype="fp8")
    store = read_coeff_store(path)
    _, sm, co = parse_coeff_store(store)
    dtab = DispatchTable(model=FP8_MODEL, pool=pool, coefficients=co, sm_count=sm,
                         active=active_ids_of(store)).device_table(device=dev)
    copies = [make_fp8_weights(geom, seed=100 + c, device=dev) for c in range(FP8_COPIES)]
    H, I, E, k = geom.K, geom.N // 2, geom.E, geom.top_k
    side = torch.cuda.Stream(device=dev)
    rows = []
    for S in FP8_BATCHES:
        for beta in FP8_BETAS:
            hs = derive_seed(42, EVAL_HIST_DOMAIN, S, round(beta * 1000), 0)
            try:
                hist = sample_histogram(E, S, k, beta, hs).histogram
            except BetaUnreachableError:
                continue  # dropped, as ramp.profiling_plan drops unreachable points
            x, ids, w = make_inputs(geom, hist, hs, dev)
            ws = moe.Workspace(S, H, I, E, k, device=dev)
            out = torch.empty(S, H, dtype=torch.bfloat16, device=dev)
            # one graph of 2 x FP8_COPIES back-to-back layer calls over the
            # rotating copies (graph-launch latency amortised as in the BF16
            # per-point latency); per-call time = replay time / calls
            n_calls = 2 * FP8_COPIES
            with torch.cuda.stream(side):
                for c in range(FP8_COPIES):
                    moe.fused_moe_fp8(x, copies[c], w, ids, dtab, -1, out=out, workspace=ws)
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    for c in range(n_calls):
                        moe.fused_moe_fp8(x, copies[c % FP8_COPIES], w, ids, dtab, -1, out=out, workspace=ws)
            torch.cuda.synchronize()
            ts = []
            for r in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3 / n_calls)
            us = float(np.median(ts[2:]))
            a = hist.active_experts
            nbytes = a * 3 * H * I * (1 + 1 / 32) + S * H * 4 + 8 * S * k
            c = pool.by_id(dtab.pool_id(int(ws.sel[0].item())))
            rows.append({"S": S, "beta": beta, "active": a, "us": round(us, 2),
                         "tflops": round(6 * S * k * H * I / us / 1e6, 2), "gbs": round(nbytes / us / 1e3, 1),
                         "cfg": {"id": c.id, "bm": c.bm, "ttn": c.ttn, "stg": c.stg, "group_m": int(c.group_m)}})
    # accuracy on the last point's routing (full geometry, sampled rows)
    acc = fp8_row_errors(geom, copies[0], x, ids, w,
                         moe.fused_moe_fp8(x, copies[0], w, ids, dtab, -1, workspace=ws))
    acc["point"] = {"S": rows[-1]["S"], "beta": rows[-1]["beta"]}
    del copies
    torch.cuda.empty_cache()
    return {"accuracy": acc, "workload": f"{FP8_MODEL} MoE layer (E=128, top-8, d=2048, d_ff=768) MXFP8 W8A8, skewed routing "
                        f"beta in {FP8_BETAS} (12/15 of 128 experts active), on-device dispatch over the FP8 pool",
            "dtype": "e4m3 x e4m3 (UE8M0 per 32) -> fp32", "l2": f"{FP8_COPIES} rotating weight copies",
            "timing": f"graph of {2 * FP8_COPIES} back-to-back layer calls, median replay time / calls",
            "us_geomean": float(np.exp(np.mean([np.log(r["us"]) for r in rows]))), "points": rows,
            "coeffs": path.name}


# ------------------------------------------------------------------ Mixtral leg
MIX_MODEL = "Mixtral-8x7B"
MIX_POINTS = ((64, 1.0), (512, 1.0), (512, 0.5))


def mixtral_leg(dev):
    """BASELINE configs[3]: Mixtral-8x7B MoE layer (E=8, top-2, d=4096,
    d_ff=14336), BF16, the large-K regime.  No fitted table ships for this
    geometry (a full profiling sweep of 614 configs at ~0.5 ms per call is a
    separate offline job), so this leg is a bounded exhaustive search over the
    large-tile split-mode candidates (bm 16..128, ttn 256/512, split-K 1/4)
    and reports the best config per point with and without split-K.  Untimed
    by the step contract; reported as a side object of the line."""
    import torch

    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs
    from paper_2604_26039_b200.dispatch import EVAL_HIST_DOMAIN, derive_seed
    from paper_2604_26039_b200.moe import DeviceTable
    from paper_2604_26039_b200.routing import sample_histogram
    from paper_2604_26039_b200.sweep import MeasuredTimer, make_inputs

    geom = BASELINE_MODELS[MIX_MODEL]
    pool = enumerate_b200_configs(geom, HardwareModel.b200())
    cols = pool.columns()
    n = len(pool)
    best_stg: dict = {}
    for c in pool:
        if c.mode == 1 and not c.group_m and c.kps == 1 and c.bm >= 16 and c.ttn >= 256:
            key = (c.bm, c.ttn, c.split_k)
            if key not in best_stg or c.stg > pool.by_id(best_stg[key]).stg:
                best_stg[key] = c.id
    cand = sorted(best_stg.values())
    flat = DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                       group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols["kps"], h3=cols["h3"], a=np.ones(n),
                       b=np.zeros(n), c=np.zeros(n), d=np.zeros(n), N=geom.N, kappa_ok=True, sm_count=148,
                       device=dev)
    timer = MeasuredTimer(geom, flat, iters=3, device=dev)
    H, I = geom.K, geom.N // 2
    # the fitted table (scripts/profile_b200.py --model Mixtral-8x7B), when shipped: the
    # on-device dispatcher's pick over the whole pool, timed the same way
    dtab = None
    path = ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{MIX_MODEL}_b200.json"
    if path.exists():
        from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store
        from paper_2604_26039_b200.dispatch import DispatchTable
        from paper_2604_26039_b200.moe import Workspace, fused_moe

        store = read_coeff_store(path)
        _, sm, co = parse_coeff_store(store)
        dtab = DispatchTable(model=MIX_MODEL, pool=pool, coefficients=co, sm_count=sm,
                             active=active_ids_of(store)).device_table(device=dev)
    rows = []
    for S, beta in MIX_POINTS:
        hs = derive_seed(42, EVAL_HIST_DOMAIN, S, round(beta * 1000), 0)
        hist = sample_histogram(geom.E, S, geom.top_k, beta, hs).histogram
        x, ids, w = make_inputs(geom, hist, hs, dev)
        t = timer.time_configs(x, ids, w, cand)
        i = int(np.argmin(t))
        c = pool.by_id(cand[i])
        no_sk = min(tt for tt, cid in zip(t, cand) if pool.by_id(cid).split_k == 1)
        nbytes = hist.active_experts * 3 * H * I * 2 + S * H * 4
        rows.append({"S": S, "beta": beta, "active": hist.active_experts, "us": round(float(t[i]), 2),
                     "tflops": round(6 * S * geom.top_k * H * I / t[i] / 1e6, 2), "gbs": round(nbytes / t[i] / 1e3, 1),
                     "best_without_split_k_us": round(float(no_sk), 2),
                     "cfg": {"id": c.id, "bm": c.bm, "ttn": c.ttn, "stg": c.stg, "split_k": c.split_k}})
        if dtab is not None:
            ws = Workspace(S, H, I, geom.E, geom.top_k, device=dev)
            fused_moe(x, timer.w1, timer.w2, w, ids, dtab, -1, workspace=ws)
            sel = dtab.pool_id(int(ws.sel[0].item()))
            t_sel = float(timer.time_configs(x, ids, w, [sel])[0])
            cs = pool.by_id(sel)
            rows[-1]["dispatched"] = {"us": round(t_sel, 2), "vs_best_candidate": round(t_sel / float(t[i]), 4),
                                      "cfg": {"id": cs.id, "bm": cs.bm, "ttn": cs.ttn, "stg": cs.stg,
                                              "split_k": cs.split_k, "mode": cs.mode}}
    del timer
    torch.cuda.empty_cache()
    return {"workload": f"{MIX_MODEL} MoE layer (E=8, top-2, d=4096, d_ff=14336) BF16, large-K regime",
            "method": f"exhaustive search over {len(cand)} large-tile split-mode candidates per point "
                      "(L2 flushed before each timed replay)"
                      + ("; 'dispatched' = the on-device dispatcher's pick over the full pool with the fitted "
                         f"table {path.name}, timed the same way" if dtab is not None else ""),
            "points": rows}


# ------------------------------------------------------------------ EP leg
EP_MODEL = "DeepSeek-V3"
EP_LOCAL = "DeepSeek-V3-EP8"
EP_TOKENS = 256     # tokens per rank per layer call
EP_BETA = 0.5


def ep_leg(dev, world, rank, iters=10, warmup=3):
    """BASELINE configs[4]: DeepSeek-V3 MoE layer (E=256, top-8, d=7168,
    d_ff=2048), MXFP8, expert-parallel over the `world` ranks of this run:
    the library's own NCCL communicator (ramp_ep_dispatch: pack kernel + one
    grouped all-to-all of fixed-capacity MXFP8 blocks), the FP8 megakernel on
    each rank's E/world experts straight off the wire (on-device dispatch over
    the FP8 pool with the EP8 local table), ramp_ep_combine (all-to-all back +
    reduce kernel).  No host synchronisation anywhere, so the layer is
    captured and replayed as a CUDA graph.  At world 1 the same exchange runs
    over a one-rank communicator, next to the identity shortcut (no exchange).
    Every rank runs it; the layer time is the max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2604_26039_b200 import ep
    from paper_2604_26039_b200.catalog import BASELINE_MODELS, MoeGeometry
    from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs
    from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store
    from paper_2604_26039_b200.dispatch import DispatchTable, derive_seed
    from paper_2604_26039_b200.routing import sample_histogram
    from paper_2604_26039_b200.sweep import make_fp8_weights, make_inputs

    if not dist.is_initialized():
        return {"skipped": "needs a torch.distributed process group"}
    geom = BASELINE_MODELS[EP_MODEL]
    if geom.E % world:
        return {"skipped": f"E={geom.E} does not split over {world} ranks"}
    per = geom.E // world
    # the table fitted for this rank's local expert count when one ships
    # (world 1: all 256 experts, "DeepSeek-V3"; world 8: 32, "DeepSeek-V3-EP8"),
    # else the EP8 one (the kernel geometry N, K is the same; the B4 traffic
    # terms were fitted on 32-expert histograms)
    local_name = {1: EP_MODEL, 8: EP_LOCAL}.get(world, EP_LOCAL)
    path = ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{local_name}_b200_fp8.json"
    if not path.exists():
        path = ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{EP_LOCAL}_b200_fp8.json"
    if not path.exists():
        return {"skipped": f"{path.name} missing (scripts/profile_b200.py --model {EP_LOCAL} --dtype fp8)"}
    table_matches = path.name == f"coeffs_{local_name}_b200_fp8.json" and world in (1, 8)
    lgeom = MoeGeometry(name=f"{EP_MODEL}-EP{world}", E=per, N=geom.N, K=geom.K, top_k=geom.top_k)
    pool = enumerate_b200_configs(lgeom, HardwareModel.b200(), dtype="fp8")
    store = read_coeff_store(path)
    _, sm, co = parse_coeff_store(store)
    dtab = DispatchTable(model=lgeom.name, pool=pool, coefficients=co, sm_count=sm,
                         active=active_ids_of(store)).device_table(device=dev)
    weights = make_fp8_weights(lgeom, seed=1000 + rank, device=dev)
    hs = derive_seed(42, 9, EP_TOKENS, round(EP_BETA * 1000), rank)
    hist = sample_histogram(geom.E, EP_TOKENS, geom.top_k, EP_BETA, hs).histogram
    x, ids, w = make_inputs(geom, hist, hs, dev)
    local_fn = ep.make_local_megakernel(weights, dtab)
    comm = ep.EPComm()
    side = torch.cuda.Stream(device=dev)

    def timed(fn):
        """Graph of 4 back-to-back layer calls; median per-call time, max over ranks."""
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                fn()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(4):
                    fn()
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 4)
        t = torch.tensor([float(np.median(ts))], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    us = timed(lambda: ep.ep_moe_layer(x, ids, w, geom.E, local_fn, wire="fp8", comm=comm))
    plan, rx, rids, rw = ep.dispatch(x, ids, w, geom.E, wire="fp8", comm=comm)
    local_us = timed(lambda: local_fn(rx, rids, rw))
    ident_us = timed(lambda: ep.ep_moe_layer(x, ids, w, geom.E, local_fn, wire="fp8")) if world == 1 else None
    acc = None
    if world == 1:  # every expert is local: sample rows of the exchanged layer against fp32
        acc = fp8_row_errors(geom, weights, x, ids, w,
                             ep.ep_moe_layer(x, ids, w, geom.E, local_fn, wire="fp8", comm=comm))
    torch.cuda.synchronize()
    overflow = int(plan.overflow.item())
    rows = torch.tensor([float(plan.counts.sum().item())], device=dev)
    dist.all_reduce(rows, op=dist.ReduceOp.MAX)
    comm.close()
    flops = world * 6 * EP_TOKENS * geom.top_k * geom.K * (geom.N // 2)
    del weights
    torch.cuda.empty_cache()
    out = {"workload": f"{EP_MODEL} MoE layer (E=256, top-8, d=7168, d_ff=2048) MXFP8, expert-parallel over "
                       f"{world} GPU(s): {per} experts/rank, {EP_TOKENS} tokens/rank, beta={EP_BETA}",
           "exchange": "ramp_ep_dispatch / ramp_ep_combine: pack kernel + one grouped NCCL all-to-all of "
                       "fixed-capacity blocks (MXFP8 rows + local ids/weights; no host read), the FP8 megakernel "
                       "on the MXFP8 rows as they arrived, NCCL all-to-all back + reduce kernel",
           "world": world, "us_per_layer": us, "local_megakernel_us": local_us,
           "exchange_overhead": us / local_us, "rows_sent_max": int(rows.item()), "overflow": overflow,
           "dispatch_wire_bytes": plan.wire_bytes, "tflops": flops / us / 1e6,
           "timing": "CUDA graph of 4 layer calls, median of iters, max over ranks", "coeffs": path.name}
    if acc is not None:
        out["accuracy"] = acc
    if world == 1:
        out["identity_us_per_layer"] = ident_us
        out["note"] = ("world 1: the exchange runs over a one-rank NCCL communicator (self send/recv); "
                       "identity_us_per_layer = the no-exchange shortcut")
    out["table_fitted_for_local_experts"] = table_matches
    return out


# ------------------------------------------------------------------ report helpers
def load_peaks():
    """MEASURED_PEAKS.json (driver-written) or the profiling guide's fallbacks."""
    pk_path = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(pk_path.read_text()) if pk_path.exists() else {}
    src = "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    return float(peaks.get("hbm_gbs", 6650.0)), float(peaks.get("bf16_tflops", 2250.0)), src


def roofline_summary(geom, pts, per_point, step_us, k3_bytes, k3_time):
    """The layer roofline over the sweep.  Per point, the roofline time is
    max(algorithmic bytes / HBM peak, FLOP / dense BF16 peak);
    frac = sum of roofline times / the CUDA-event time of the whole step
    (route kernel, prologue and megakernel of all 27 layer calls), and
    achieved = frac x peak, the HBM-equivalent bandwidth of the step.  The
    megakernel-only window (globaltimer, route kernel excluded) is kept
    separately."""
    hbm, tf, src = load_peaks()
    t_roof, t_bytes, fr = 0.0, 0.0, []
    for pt, r in zip(pts, per_point):
        b = layer_bytes(geom, pt["hist"], pt["S"])
        f = layer_flops(geom, pt["S"])
        tr = max(b / hbm / 1e3, f / tf / 1e6)  # us
        t_roof += tr
        t_bytes += b / hbm / 1e3
        fr.append(tr / r["us"])
    frac = t_roof / step_us
    n_hbm = sum(1 for pt in pts if layer_bytes(geom, pt["hist"], pt["S"]) / hbm / 1e3 >=
                layer_flops(geom, pt["S"]) / tf / 1e6)
    out = {"bound": "hbm", "achieved": frac * hbm, "peak": hbm, "unit": "GB/s", "frac": frac,
           "traffic": None, "kernel": "route_kernel + fused_moe_kernel<0> (whole layer)",
           "peak_source": src, "tensor_peak_tflops": tf,
           "points_hbm_bound": n_hbm, "points_tensor_bound": len(pts) - n_hbm,
           "bytes_only_frac": t_bytes / step_us, "per_point_geomean_frac": float(np.exp(np.mean(np.log(fr)))),
           "megakernel_window_frac": (k3_bytes / k3_time / 1e3) / hbm,
           "note": "frac = sum over the 27 points of max(bytes/hbm_peak, flop/bf16_peak) / CUDA-event step time; "
                   "achieved = frac * peak (HBM-equivalent GB/s); megakernel_window_frac = algorithmic bytes / "
                   "megakernel globaltimer window (route kernel excluded)"}
    tr_path = ROOT / "profiles" / "sweep_traffic.json"
    if tr_path.exists():
        t = json.loads(tr_path.read_text())
        out["traffic"] = t.get("dram_bytes_per_launch")
        out["traffic_vs_algorithmic"] = t.get("dram_over_algorithmic")
        out["traffic_source"] = t.get("source")
    return out


def compact_leg(leg, keys):
    """A side leg for the JSON line: its summary fields plus one short row per
    point (the full records go to the per-point file)."""
    if not isinstance(leg, dict) or "points" not in leg:
        return leg
    out = {k: v for k, v in leg.items() if k not in ("points", "workload", "method", "timing", "dtype", "l2")}
    out["workload"] = leg.get("workload", "")[:120]
    out["points_" + "_".join(keys)] = [[r.get(k) for k in keys] + ([r["dispatched"]["us"]] if "dispatched" in r else [])
                                       for r in leg["points"]]
    return out


# Descriptive strings that live in the per-point file only (the driver keeps
# a bounded tail of stdout: the JSON line stays under ~4 KB).
_FILE_ONLY_KEYS = ("note", "traffic_source", "method", "impl", "how", "exchange", "timing")


def compact_line(line):
    """The printed line: every nested float to 4 significant digits and the
    long descriptions dropped (the full line is in the per-point file)."""

    def walk(o, top=False):
        if isinstance(o, float) and not top:
            return float(f"{o:.4g}")
        if isinstance(o, dict):
            return {k: walk(v) for k, v in o.items() if not (k in _FILE_ONLY_KEYS and isinstance(v, str))}
        if isinstance(o, list):
            return [walk(v) for v in o]
        return o

    out = {k: walk(v, top=True) for k, v in line.items() if k != "per_point_us"}
    if isinstance(line.get("e2e"), dict):
        out["e2e"]["value"] = line["e2e"]["value"]
    return out


def write_per_point(per_point):
    """The per-point detail goes to a file (the JSON line stays short)."""
    d = ROOT / "gpurun_out" if (ROOT / "gpurun_out").is_dir() else ROOT
    path = d / "bench_per_point.json"
    try:
        path.write_text(json.dumps(per_point, indent=1) + "\n")
    except OSError:
        return None
    return str(path.relative_to(ROOT))


def cpu_baseline(geom, pts, table):
    """The CPU reference arms, timed on this box's host cores (bounded):
    the fp32 oracle of the layer with every thread and with one thread, and
    the reference's numpy dispatch path (ramp.select_config restated in
    oracle/ramp_ref.select_np) on the same table and histograms as the device
    dispatcher."""
    from oracle.ramp_ref import select_np
    from threadpoolctl import threadpool_limits

    w1c, w2c = cpu_weights(geom)
    run_cpu_sweep(geom, pts[:2], w1c, w2c)
    f, t, n = run_cpu_sweep(geom, pts, w1c, w2c, budget_s=20.0)
    out = {"value": f / t / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
           "sample": f"first {n} of {len(pts)} sweep points (fp32 numpy oracle, oracle/moe_ref.py)"}
    with threadpool_limits(limits=1):
        f1, t1, n1 = run_cpu_sweep(geom, pts, w1c, w2c, budget_s=8.0)
    out["single_thread"] = {"value": f1 / t1 / 1e12, "unit": "TFLOP/s", "cores": 1,
                            "sample": f"first {n1} sweep points, BLAS limited to 1 thread (threadpoolctl)"}
    cols = table.pool.columns()
    act = table._active
    args = dict(bm=cols["bm"][act], ttn=cols["ttn"][act], split_k=cols["split_k"][act], a=table._a[act],
                b=table._b[act], c=table._c[act], d=table._d[act], N=geom.N, sm=table.sm_count,
                kappa_ok=bool(table._kappa_ok), ntile=cols["ntile"][act], omega_max=table._omega_max,
                lam=None if table._lam is None else table._lam[act])
    ts = []
    for pt in pts:
        counts = np.asarray(pt["hist"].counts)
        select_np(counts=counts, **args)
        t0 = time.perf_counter()
        for _ in range(20):
            select_np(counts=counts, **args)
        ts.append((time.perf_counter() - t0) / 20 * 1e6)
    out["dispatch"] = {"us_per_call_median": float(np.median(ts)), "us_per_call_max": float(np.max(ts)),
                       "candidates": int(act.sum()), "cores": 1,
                       "impl": "ramp.select_config's numpy path (pool_grids -> gate -> predict_batch -> argmin), "
                               "oracle/ramp_ref.select_np, on the bench table and the 27 sweep histograms; "
                               "the device dispatcher runs inside the route kernel (no host round trip)"}
    return out


# ------------------------------------------------------------------ GPU arm
def load_table(geom, pool, hw):
    from paper_2604_26039_b200.cost_model import active_ids_of, parse_coeff_store, read_coeff_store
    from paper_2604_26039_b200.dispatch import DispatchTable

    path = ROOT / "paper_2604_26039_b200" / "data" / f"coeffs_{MODEL}_b200.json"
    if not path.exists():
        raise SystemExit(f"{path} missing: run scripts/profile_b200.py on a B200 first")
    store = read_coeff_store(path)
    _, sm, coeffs = parse_coeff_store(store)
    return DispatchTable(model=MODEL, pool=pool, coefficients=coeffs, sm_count=sm,
                         active=active_ids_of(store)), path


def _ensure_single_pg() -> bool:
    """A one-rank NCCL process group (127.0.0.1), so the EP leg's collectives
    run unchanged at N=1."""
    import torch
    import torch.distributed as dist

    if dist.is_initialized():
        return True
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    return True


def ours(args, geom):
    import torch
    import torch.distributed as dist

    from paper_2604_26039_b200 import _lib, moe
    from paper_2604_26039_b200.config_space import HardwareModel, enumerate_b200_configs
    from paper_2604_26039_b200.dispatch import DispatchTable, evaluate_regret, speedup_ra_vs_static
    from paper_2604_26039_b200.sweep import MeasuredTimer, make_inputs, make_weights

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.require_device()
    dev = torch.device("cuda", local)
    hw = HardwareModel.b200()
    pool = enumerate_b200_configs(geom, hw)
    table, coeff_path = load_table(geom, pool, hw)
    dtab = table.device_table(device=dev)
    pts = sweep_points(geom)
    copies = [make_weights(geom, seed=42 + c, device=dev) for c in range(N_COPIES)]
    inputs = [make_inputs(geom, pt["hist"], pt["seed"], dev) for pt in pts]
    H, I = geom.K, geom.N // 2
    wss = [moe.Workspace(pt["S"], H, I, geom.E, geom.top_k, device=dev) for pt in pts]
    outs = [torch.empty(pt["S"], H, dtype=torch.bfloat16, device=dev) for pt in pts]
    step_flops = sum(layer_flops(geom, pt["S"]) for pt in pts)
    stream = torch.cuda.current_stream()

    def layer(p, c, phases=3):
        x, ids, w = inputs[p]
        w1, w2 = copies[c % N_COPIES]
        moe.fused_moe(x, w1, w2, w, ids, dtab, -1, out=outs[p], workspace=wss[p], phases=phases)

    # The serving path replays CUDA graphs (no per-layer host work): one graph
    # per weight-rotation offset, each holding the whole 27-layer sweep.
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    graphs = {}
    with torch.cuda.stream(side):
        for p in range(len(pts)):
            layer(p, p)  # warm-up outside capture (encodes the cached tensor maps)
        for off in sorted({(i * len(pts)) % N_COPIES for i in range(N_COPIES)}):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for p in range(len(pts)):
                    layer(p, off + p)
            graphs[off] = g
    stream.wait_stream(side)
    torch.cuda.synchronize()

    def step(i):
        graphs[(i * len(pts)) % N_COPIES].replay()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(i)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for i in range(args.steps):
            step(args.warmup + i)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = step_flops * args.steps * world / (ms / 1e3) / 1e12

    # ---------------- expert-parallel DeepSeek-V3 leg (every rank: collectives)
    ep_res = None
    if not args.no_ep:
        try:
            ep_res = ep_leg(dev, world, rank) if (world > 1 or _ensure_single_pg()) else None
        except Exception as exc:  # noqa: BLE001 - reported in the line, never fatal for the main metric
            ep_res = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    # ---------------- diagnostics (untimed): per-point latency, megakernel roofline
    per_point = []
    k3_bytes, k3_time = 0.0, 0.0
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def graph_of(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                fn()
        torch.cuda.synchronize()
        return g

    # per-point layer time: a graph of 8 back-to-back calls (rotating weight
    # copies), so graph-launch latency is amortised as in the step graph;
    # megakernel time: first CTA past the route hand-off -> last CTA exit, from the kernel's own
    # globaltimer stamps (the kernel duration, as ncu counts it)
    prof_buf = torch.zeros(149 * 32 + 148 * 16 * 4, dtype=torch.int64, device=dev)
    lib = _lib.load()
    for p, pt in enumerate(pts):
        g8 = graph_of(lambda: [layer(p, c) for c in range(N_COPIES)])
        lat = []
        for r in range(5):
            a0, a1 = ev(), ev()
            a0.record()
            g8.replay()
            a1.record()
            torch.cuda.synchronize()
            lat.append(a0.elapsed_time(a1) * 1e3 / N_COPIES)
        lib.ramp_set_profile_buffer(prof_buf.data_ptr())
        gp = graph_of(lambda: layer(p, 1))
        lib.ramp_set_profile_buffer(None)
        k3 = []
        for r in range(4):
            prof_buf.zero_()
            gp.replay()
            torch.cuda.synchronize()
            st = prof_buf[:148 * 32].view(148, 32).cpu().numpy()
            k3.append((st[:, 23].max() - st[:, 17].min()) / 1e3)  # kTsFinal - kTsStart (after the route), ns -> us
        cfg = dtab.pool_id(int(wss[p].sel[0].item()))
        us, k3us = float(np.median(lat)), float(np.median(k3[1:]))
        nbytes = layer_bytes(geom, pt["hist"], pt["S"])
        k3_bytes += nbytes
        k3_time += k3us
        c = pool.by_id(cfg)
        per_point.append({"S": pt["S"], "beta": pt["beta"], "active": pt["hist"].active_experts, "us": round(us, 2),
                          "megakernel_us": round(k3us, 2), "tflops": round(layer_flops(geom, pt["S"]) / us / 1e6, 2),
                          "gbs": round(nbytes / k3us / 1e3, 1),
                          "cfg": {"id": cfg, "bm": c.bm, "ttn": c.ttn, "stg": c.stg, "group_m": int(c.group_m),
                                  "mode": c.mode, "split_k": c.split_k}})
    geo_us = math.exp(np.mean([math.log(r["us"]) for r in per_point]))

    # ---------------- routing-aware vs static and regret against an exhaustive on-GPU sweep
    ra = None
    if not args.no_sweep:
        # the exhaustive sweep times every pool config, pruned or not
        full_tab = DispatchTable(model=MODEL, pool=pool, coefficients=table.coefficients,
                                 sm_count=table.sm_count).device_table(device=dev)
        timer = MeasuredTimer(geom, full_tab, w1=copies[0][0], w2=copies[0][1], iters=9, device=dev)
        points = [(pt["S"], pt["beta"]) for pt in pts]
        t_ra = time.time()
        ns = args.regret_seeds
        spd = speedup_ra_vs_static(table, pool, geom, timer, points=points, seeds_per_point=ns)
        reg = evaluate_regret(table, pool, geom, timer, test_points=points, seeds_per_point=ns)
        agg = reg.aggregate()
        ra = {"ra_vs_static_geomean": spd.geomean, "per_beta": spd.aggregate()["per_beta_geomean"],
              "regret_mean_pct": reg.mean * 100, "regret_max_pct": reg.max * 100,
              "regret_sweep_only_mean_pct": agg["sweep_only_mean"] * 100,
              "regret_sweep_only_max_pct": agg["sweep_only_max"] * 100,
              "points": len(points), "seeds_per_point": ns, "records": len(reg.records),
              "winners_curse_retimed": agg["retimed"],
              "method": "regret = selected / exhaustive best - 1 over every pool config, L2 flushed per replay; "
                        "when the pick is not the sweep's winner both are re-timed side by side with 4x the "
                        "replays and the faster is the best (deviation from ramp.evaluate_regret, which uses the "
                        "sweep minimum: reported as regret_sweep_only_*)",
              "worst": [{"S": r.S, "beta": r.beta, "regret_pct": round(r.regret * 100, 2), "sel": r.selected_id,
                         "best": r.best_id} for r in sorted(reg.records, key=lambda r: -r.regret)[:3]],
              "wall_s": round(time.time() - t_ra, 1)}

    # ---------------- e2e through the public API with host buffers
    # Each layer's request (tokens, top-k ids, top-k weights) sits in ONE
    # pinned host block and moves with one copy into one device block, the
    # three tensors being typed views of it (16-byte aligned: H % 8 == 0,
    # 4-byte ids / weights in rows of top_k).
    def _views(buf, x, ids, w):
        nx, ni = x.numel() * x.element_size(), ids.numel() * ids.element_size()
        nw = w.numel() * w.element_size()
        return (buf[:nx].view(x.dtype).view(x.shape), buf[nx:nx + ni].view(ids.dtype).view(ids.shape),
                buf[nx + ni:nx + ni + nw].view(w.dtype).view(w.shape))

    pinned, host_blocks, dev_blocks, dev_bufs = [], [], [], []
    for (x, ids, w), pt in zip(inputs, pts):
        nb = x.numel() * x.element_size() + ids.numel() * ids.element_size() + w.numel() * w.element_size()
        hb = torch.empty(nb, dtype=torch.uint8).pin_memory()
        for dst, src in zip(_views(hb, x, ids, w), (x, ids, w)):
            dst.copy_(src.cpu())
        db = torch.empty(nb, dtype=torch.uint8, device=dev)
        host_blocks.append(hb)
        dev_blocks.append(db)
        dev_bufs.append(_views(db, x, ids, w))
        pinned.append((*_views(hb, x, ids, w), torch.empty(pt["S"], H, dtype=torch.bfloat16).pin_memory()))
    h2d = sum(b.numel() for b in host_blocks)
    d2h = sum(o.numel() * o.element_size() for *_, o in pinned)

    # The serving loop as a CUDA graph: every replay copies each layer's
    # inputs (one block) from pinned host memory (copy-in stream, running ahead), runs the
    # layer once its inputs have landed, and copies its output back to the
    # host (copy-out stream) while the next layer computes.
    cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def e2e_body(off):
        ev_in = [torch.cuda.Event() for _ in pts]
        ev_done = [torch.cuda.Event() for _ in pts]
        cin.wait_stream(side)
        cout.wait_stream(side)
        with torch.cuda.stream(cin):
            for p, (hb, db) in enumerate(zip(host_blocks, dev_blocks)):
                db.copy_(hb, non_blocking=True)  # the layer's x, ids and weights in one transfer
                ev_in[p].record(cin)
        for p, (dx, di, dw) in enumerate(dev_bufs):
            side.wait_event(ev_in[p])
            w1, w2 = copies[(off + p) % N_COPIES]
            moe.fused_moe(dx, w1, w2, dw, di, dtab, -1, out=outs[p], workspace=wss[p])
            ev_done[p].record(side)
            with torch.cuda.stream(cout):
                cout.wait_event(ev_done[p])
                pinned[p][3].copy_(outs[p], non_blocking=True)
        side.wait_stream(cin)
        side.wait_stream(cout)

    e2e_graphs = {}
    with torch.cuda.stream(side):
        e2e_body(0)  # warm-up outside capture
        for off in sorted({(i * len(pts)) % N_COPIES for i in range(N_COPIES)}):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                e2e_body(off)
            e2e_graphs[off] = g
    torch.cuda.synchronize()

    def e2e_step(i):
        e2e_graphs[(i * len(pts)) % N_COPIES].replay()

    e2e_step(0)
    torch.cuda.synchronize()
    f0, f1 = ev(), ev()
    f0.record()
    for i in range(max(1, args.steps // 2)):
        e2e_step(i + 1)
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = f0.elapsed_time(f1) / max(1, args.steps // 2)
    # the outputs really came back: spot-check the last layer's host copy
    if not torch.equal(pinned[-1][3], outs[-1].cpu()):
        raise SystemExit("e2e: host output differs from the device result")
    if not all(torch.equal(a, b) for a, b in zip(dev_bufs[-1], inputs[-1])):
        raise SystemExit("e2e: the copied-in request differs from the layer's inputs")
    e2e_val = step_flops / (e2e_ms / 1e3) / 1e12

    # ---------------- CPU baseline (oracle port, bounded sample)
    cpu = None
    if not args.no_cpu:
        cpu = cpu_baseline(geom, pts, table)

    mix = None
    if not args.no_mixtral:
        try:
            mix = mixtral_leg(dev)
        except Exception as exc:  # noqa: BLE001 - reported in the line, never fatal for the main metric
            mix = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    fp8 = None
    if not args.no_fp8:
        try:
            fp8 = fp8_leg(dev)
        except Exception as exc:  # noqa: BLE001 - reported in the line, never fatal for the main metric
            fp8 = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    roof = roofline_summary(geom, pts, per_point, ms / args.steps * 1e3, k3_bytes, k3_time)
    pp_path = write_per_point({"olmoe": per_point, "fp8": fp8, "mixtral": mix})
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, reference evaluation histograms)",
        "config": {"workload": f"{MODEL} MoE layer (E=64, top-8, d=2048, d_ff=1024) BF16, S=1..512 x "
                               f"beta in {{0.2,0.5,1.0}} ({len(pts)} layer calls/step), routing-aware dispatch",
                   "l2": f"inputs larger than L2: {N_COPIES} rotating weight copies of 805 MB",
                   "parallelism": "replicas" if world > 1 else "single GPU", "coeffs": coeff_path.name},
        "gpu_launches": 2 * len(pts) * args.steps,
        "us_per_layer_geomean": geo_us,
        "roofline": roof,
        "clocks": clocks.summary(),
        "e2e": {"value": e2e_val, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "how": "public fused_moe() per layer from pinned host inputs (x, topk ids, topk weights) to a pinned "
                       "host output, replayed as one CUDA graph per step; copies on their own streams overlap the "
                       "neighbouring layers' compute"},
        "cpu_baseline": cpu,
        "dispatch": ra,
        "per_point_us": [[r["S"], r["beta"], r["us"]] for r in per_point],
        "per_point_file": pp_path,
        "fp8": compact_leg(fp8, ("S", "beta", "us", "tflops")),
        "mixtral": compact_leg(mix, ("S", "beta", "us")),
        "ep": ep_res,
    }
    if pp_path:  # the full line (with the descriptions) next to the per-point detail
        write_per_point({"olmoe": per_point, "fp8": fp8, "mixtral": mix, "line_full": line})
    print(json.dumps(compact_line(line)), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-sweep", action="store_true", help="skip the exhaustive RA/static/regret sweep")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline")
    ap.add_argument("--no-fp8", action="store_true", help="skip the Qwen3 FP8 side measurement")
    ap.add_argument("--no-ep", action="store_true", help="skip the DeepSeek-V3 expert-parallel side measurement")
    ap.add_argument("--no-mixtral", action="store_true", help="skip the Mixtral large-K side measurement")
    ap.add_argument("--regret-seeds", type=int, default=3,
                    help="routing seeds per sweep point in the regret / RA-vs-static evaluation (reference: 3)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    from paper_2604_26039_b200.catalog import BASELINE_MODELS

    geom = BASELINE_MODELS[MODEL]
    if args.impl == "reference":
        reference_arm(args, geom)
    else:
        ours(args, geom)


if __name__ == "__main__":
    main()
