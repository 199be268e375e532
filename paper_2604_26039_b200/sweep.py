"""Measured kernel times on the B200: the timer behind the profiling sweep,
the exhaustive on-GPU search and the regret / speedup reports.

`MeasuredTimer.pool_times(pool, hist, ...)` replaces the reference's
`simulate_pool_times` (ramp/oracle.py:197-254): for one routing histogram it
builds concrete top-k routing (routing.topk_from_histogram), then launches
the fused-MoE megakernel once per pool config (forced config id, same
inputs) and returns the per-config microseconds.  Each config is captured in
a CUDA graph and replayed `iters` times; before every replay the L2 is
flushed (a 256 MiB memset > 126 MB L2), because in a real model the next
layer's weights are cold; the reported time is the median of the CUDA-event
intervals around the replays.  All configs of one histogram are timed in
the same run, so selected-vs-best comparisons share conditions (the
measured counterpart of the simulator's shared noise draw).
"""

from __future__ import annotations

import numpy as np
import torch

from .catalog import MoeGeometry
from .config_space import ConfigPool
from .dispatch import derive_seed
from .moe import DeviceTable, Workspace, fused_moe, fused_moe_fp8
from .routing import ExpertHistogram, topk_from_histogram

TOPK_DOMAIN = 6      # seed domains for the concrete inputs of a histogram
WEIGHT_DOMAIN = 7
ACT_DOMAIN = 8


def make_weights(geom: MoeGeometry, seed: int = 42, device="cuda"):
    """Random-init expert weights of the geometry: w1 [E, 2I, H] ~ N(0, 1/H),
    w2 [E, H, I] ~ N(0, 1/I), bf16 (there is no checkpoint access)."""
    E, I, H = geom.E, geom.N // 2, geom.K
    g = torch.Generator(device=device).manual_seed(derive_seed(seed, WEIGHT_DOMAIN) % (2**63))
    w1 = torch.empty(E, 2 * I, H, dtype=torch.bfloat16, device=device)
    w2 = torch.empty(E, H, I, dtype=torch.bfloat16, device=device)
    for e in range(E):  # per expert keeps the fp32 temporaries small
        w1[e] = (torch.randn(2 * I, H, generator=g, device=device) * H ** -0.5).to(torch.bfloat16)
        w2[e] = (torch.randn(H, I, generator=g, device=device) * I ** -0.5).to(torch.bfloat16)
    return w1, w2


def make_fp8_weights(geom: MoeGeometry, seed: int = 42, device="cuda"):
    """make_weights, quantised to MXFP8 operands expert by expert."""
    from .quant import MxFp8Weights, prepare_mxfp8_weights

    w1, w2 = make_weights(geom, seed, device)
    parts = [prepare_mxfp8_weights(w1[e:e + 1], w2[e:e + 1]) for e in range(geom.E)]
    del w1, w2
    return MxFp8Weights(*(torch.cat([getattr(p, f) for p in parts]) for f in ("w1_q", "w1_sf", "w2_q", "w2_sf")))


def make_inputs(geom: MoeGeometry, hist: ExpertHistogram, seed: int, device="cuda"):
    """Tokens, top-k ids and weights realising `hist` exactly."""
    k = geom.top_k
    if hist.total % k:
        raise ValueError(f"histogram total {hist.total} is not a multiple of top_k={k}")
    S = hist.total // k
    ids = topk_from_histogram(hist.counts, S, k, derive_seed(seed, TOPK_DOMAIN) % (2**63))
    rng = np.random.default_rng(derive_seed(seed, ACT_DOMAIN))
    logits = rng.standard_normal((S, k)).astype(np.float32)
    w = np.exp(logits - logits.max(1, keepdims=True))
    w /= w.sum(1, keepdims=True)
    x = rng.standard_normal((S, geom.K)).astype(np.float32)
    return (torch.from_numpy(x).to(device, torch.bfloat16), torch.from_numpy(ids).to(device),
            torch.from_numpy(w.astype(np.float32)).to(device))


class MeasuredTimer:
    """Times every config of a pool on one histogram with the real megakernel."""

    def __init__(self, geom: MoeGeometry, table: DeviceTable, w1=None, w2=None, iters: int = 5,
                 flush_mb: int = 256, device="cuda", fp8_weights=None):
        """`fp8_weights` (quant.MxFp8Weights): time the FP8 megakernel instead."""
        self.geom = geom
        self.table = table
        self.iters = iters
        self.device = device
        self.fp8 = fp8_weights
        if w1 is None and fp8_weights is None:
            w1, w2 = make_weights(geom, device=device)
        self.w1, self.w2 = w1, w2
        self.flush = torch.empty(flush_mb << 20, dtype=torch.uint8, device=device)
        self._memo: dict = {}  # (counts, seed) -> times: regret and speedup share one sweep per point

    def quiet(self) -> "MeasuredTimer":
        return self

    def time_configs(self, x, ids, w, config_ids) -> np.ndarray:
        S, H = x.shape
        I = self.geom.N // 2
        ws = Workspace(S, H, I, self.geom.E, self.geom.top_k, device=self.device)
        out = torch.empty(S, H, dtype=torch.bfloat16, device=self.device)
        res = np.empty(len(config_ids))
        stream = torch.cuda.Stream()
        for n, cid in enumerate(config_ids):
            if self.fp8 is not None:
                call = lambda: fused_moe_fp8(x, self.fp8, w, ids, self.table, int(cid), out=out,  # noqa: E731
                                             workspace=ws)
            else:
                call = lambda: fused_moe(x, self.w1, self.w2, w, ids, self.table, int(cid), out=out,  # noqa: E731
                                         workspace=ws)
            with torch.cuda.stream(stream):
                call()  # warm-up (also encodes the cached tensor maps)
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=stream):
                    call()
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(self.iters)]
                for e0, e1 in ev:
                    self.flush.zero_()
                    e0.record(stream)
                    graph.replay()
                    e1.record(stream)
            stream.synchronize()
            # CUDA event timestamps are quantised (~0.5-1 us on this part):
            # average the middle replays instead of taking one median sample
            ts = np.sort([e0.elapsed_time(e1) * 1e3 for e0, e1 in ev])
            trim = len(ts) // 4
            res[n] = float(ts[trim:len(ts) - trim].mean())
        return res

    def confirm(self, pool: ConfigPool, hist: ExpertHistogram, point_seed: int, config_ids, factor: int = 4):
        """Re-time a few configs side by side with `factor` x the replays
        (the regret harness's winner's-curse correction)."""
        x, ids, w = make_inputs(self.geom, hist, point_seed, self.device)
        iters = self.iters
        self.iters = iters * factor
        try:
            return self.time_configs(x, ids, w, list(config_ids))
        finally:
            self.iters = iters

    def pool_times(self, pool: ConfigPool, hist: ExpertHistogram, point_seed: int, shared_noise: bool = False,
                   grids=None) -> np.ndarray:
        key = (hist.counts, point_seed, len(pool), self.iters)
        if key not in self._memo:
            x, ids, w = make_inputs(self.geom, hist, point_seed, self.device)
            self._memo[key] = self.time_configs(x, ids, w, [c.id for c in pool])
        return self._memo[key].copy()
