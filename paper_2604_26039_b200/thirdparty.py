"""Kernel-agnostic trace source (the reference's
"real kernel timings can be substituted", pkg/README.md:17-18, and its
acceptance criterion 12, tests/test_acceptance.py:423-457).

`VllmTritonTimer` times a third-party fused-MoE kernel -- vLLM's Triton
`fused_experts` -- under every config of a triton-family pool
(config_space.enumerate_triton_configs), with the same `pool_times`
interface as sweep.MeasuredTimer.  The profiling sweep, the trace CSV in the
reference schema, the OLS fit, the dispatcher and the regret / speedup
harness are then exactly the ones the B200 megakernel uses
(scripts/profile_thirdparty.py): only the timing source changes.

vLLM is a test-time dependency of this module alone (imported lazily); the
product path never calls it.
"""

from __future__ import annotations

import numpy as np
import torch

from .catalog import MoeGeometry
from .config_space import ConfigPool, triton_config_dict
from .routing import ExpertHistogram
from .sweep import make_inputs, make_weights


class VllmTritonTimer:
    """Times vLLM's Triton fused_moe (`fused_experts`) per triton-family config."""

    def __init__(self, geom: MoeGeometry, iters: int = 5, flush_mb: int = 256, device="cuda", seed: int = 42):
        self.geom = geom
        self.iters = iters
        self.device = device
        self.w1, self.w2 = make_weights(geom, seed=seed, device=device)
        self.flush = torch.empty(flush_mb << 20, dtype=torch.uint8, device=device)
        self._memo: dict = {}

    def quiet(self) -> "VllmTritonTimer":
        return self

    def time_configs(self, pool: ConfigPool, x, ids, w, config_ids) -> np.ndarray:
        from vllm.model_executor.layers.fused_moe import override_config
        from vllm.model_executor.layers.fused_moe.fused_moe import fused_experts

        res = np.empty(len(config_ids))
        for n, cid in enumerate(config_ids):
            with override_config(triton_config_dict(pool.by_id(int(cid)))):
                fused_experts(x, self.w1, self.w2, w, ids)  # compile + warm-up
                ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                      for _ in range(self.iters)]
                for e0, e1 in ev:
                    self.flush.zero_()  # cold weights, as for the megakernel's timer
                    e0.record()
                    fused_experts(x, self.w1, self.w2, w, ids)
                    e1.record()
                torch.cuda.synchronize()
            ts = np.sort([e0.elapsed_time(e1) * 1e3 for e0, e1 in ev])
            trim = len(ts) // 4
            res[n] = float(ts[trim:len(ts) - trim].mean())
        return res

    def pool_times(self, pool: ConfigPool, hist: ExpertHistogram, point_seed: int, shared_noise: bool = False,
                   grids=None) -> np.ndarray:
        key = (hist.counts, point_seed, len(pool), self.iters)
        if key not in self._memo:
            x, ids, w = make_inputs(self.geom, hist, point_seed, self.device)
            self._memo[key] = self.time_configs(pool, x, ids, w, [c.id for c in pool])
        return self._memo[key].copy()

    def confirm(self, pool: ConfigPool, hist: ExpertHistogram, point_seed: int, config_ids, factor: int = 4):
        x, ids, w = make_inputs(self.geom, hist, point_seed, self.device)
        iters = self.iters
        self.iters = iters * factor
        try:
            return self.time_configs(pool, x, ids, w, list(config_ids))
        finally:
            self.iters = iters
