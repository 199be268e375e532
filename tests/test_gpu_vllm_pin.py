"""Pins the fused-forward and alignment oracle (oracle/moe_ref.py, whose
semantics come from PAPER.md:155-169 and vLLM's conventions)
to an independent implementation: vLLM's `fused_experts` (Triton, BF16) and
`moe_align_block_size` (CUDA op), on identical inputs, on the GPU box.

vLLM is third-party library code used here only as the independent checker
(SURVEY.md 8c names its layout as the convention); the product never calls it.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.moe_ref import bf16_round, fused_moe_ref, moe_align_ref  # noqa: E402
from tests._util import random_moe  # noqa: E402

pytestmark = pytest.mark.gpu


def _vllm():
    try:
        from vllm.model_executor.layers.fused_moe.fused_moe import fused_experts
        from vllm.model_executor.layers.fused_moe.moe_align_block_size import moe_align_block_size
    except Exception as exc:  # noqa: BLE001
        pytest.fail(f"vLLM is part of this image but did not import: {exc!r}")
    return fused_experts, moe_align_block_size


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("S,E,k,H,I,skew", [(16, 64, 8, 2048, 1024, None), (200, 16, 4, 512, 768, 0.4),
                                           (3, 8, 2, 4096, 1792, None)])
def test_oracle_matches_vllm_fused_experts(S, E, k, H, I, skew):
    fused_experts, _ = _vllm()
    x, w1, w2, w, ids = random_moe(S, H, I, E, k, seed=S + E, skew=skew)
    ref = fused_moe_ref(x, w1, w2, w, ids, act_dtype=bf16_round)
    out = fused_experts(torch.from_numpy(x).to("cuda", torch.bfloat16), torch.from_numpy(w1).to("cuda", torch.bfloat16),
                        torch.from_numpy(w2).to("cuda", torch.bfloat16), torch.from_numpy(w).cuda(),
                        torch.from_numpy(ids).cuda())
    torch.cuda.synchronize()
    err = _rel(out.float().cpu().numpy(), ref)
    # both compute in bf16 operands / fp32 accumulation with a bf16 output
    assert err < 1e-2, err


@pytest.mark.parametrize("S,k,E,bm,skew", [(16, 8, 64, 16, None), (512, 8, 64, 64, 0.3), (7, 2, 8, 128, None),
                                           (1000, 8, 256, 32, 0.1)])
def test_oracle_alignment_matches_vllm(S, k, E, bm, skew):
    """Same padded length and per-block expert map, and for every expert the
    same multiset of assignment indices over its blocks (vLLM places an
    expert's assignments with atomics, so which of that expert's blocks an
    index lands in is unspecified; the oracle and the route kernel sort
    stably), and the same number of padding sentinels."""
    _, moe_align_block_size = _vllm()
    _, _, _, _, ids = random_moe(S, 8, 8, E, k, seed=S, skew=skew)
    h_ref, s_ref, t_ref, n_ref = moe_align_ref(ids, E, bm)
    sid, eid, npp = moe_align_block_size(torch.from_numpy(ids).cuda(), bm, E)
    torch.cuda.synchronize()
    n = int(npp.item())
    assert n == n_ref
    sid = sid.cpu().numpy()[:n]
    eid = eid.cpu().numpy()[:n // bm]
    np.testing.assert_array_equal(eid, t_ref)
    pad = ids.size
    for e in np.unique(t_ref):
        rows = np.concatenate([np.arange(b * bm, (b + 1) * bm) for b in np.flatnonzero(t_ref == e)])
        a, r = sid[rows], s_ref[rows]
        np.testing.assert_array_equal(np.sort(a[a < pad]), np.sort(r[r < pad]))
        assert (a >= pad).sum() == (r >= pad).sum()
