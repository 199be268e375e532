"""Shared helpers for the tests: golden fixtures, synthetic MoE inputs, tables."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"

GEOMS = {
    "tiny": dict(E=4, N=256, K=1024, top_k=2),
    "deep": dict(E=32, N=1024, K=16384, top_k=8),
    "OLMoE": dict(E=64, N=2048, K=2048, top_k=8),
    "OLMoE-1B-7B": dict(E=64, N=2048, K=2048, top_k=8),
}


@lru_cache(maxsize=None)
def golden(name: str):
    return json.loads((GOLDEN / name).read_text())


def pool_columns(geom: str, hw: str) -> dict:
    for entry in golden("pools.json"):
        if entry["geom"] == geom and entry["hw"] == hw and "columns" in entry:
            return {k: np.asarray(v, dtype=np.int64) for k, v in entry["columns"].items()}
    raise KeyError((geom, hw))


def kappa_ok(geom: str) -> bool:
    return GEOMS[geom]["K"] / 128 >= 48


def random_moe(S, H, I, E, k, seed=0, skew=None, dup=False):
    """bf16-representable fp32 inputs (numpy) for the fused MoE layer."""
    from oracle.moe_ref import bf16_round

    rng = np.random.default_rng(seed)
    x = bf16_round(rng.standard_normal((S, H)).astype(np.float32))
    w1 = bf16_round((rng.standard_normal((E, 2 * I, H)) / np.sqrt(H)).astype(np.float32))
    w2 = bf16_round((rng.standard_normal((E, H, I)) / np.sqrt(I)).astype(np.float32))
    logits = rng.standard_normal((S, k)).astype(np.float32)
    w = np.exp(logits) / np.exp(logits).sum(1, keepdims=True)
    if dup:
        ids = rng.integers(0, E, size=(S, k))
    elif skew is not None:
        p = np.exp(-skew * np.arange(E))
        p /= p.sum()
        ids = np.stack([rng.choice(E, size=k, replace=False, p=p) for _ in range(S)]) if S else np.zeros((0, k))
    else:
        ids = np.stack([rng.choice(E, size=k, replace=False) for _ in range(S)]) if S else np.zeros((0, k))
    return x, w1, w2, w.astype(np.float32), ids.astype(np.int32)
