"""The fp32 fused-MoE / alignment oracle: frozen vectors and independent
re-derivations (CPU only).  PARITY UNPINNED BY THE REFERENCE (it has no
implementation of either); see oracle/moe_ref.py."""

from pathlib import Path

import numpy as np
import pytest

from oracle.moe_ref import bf16_round, fused_moe_ref, moe_align_ref
from tests._util import random_moe

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "moe_small.npz")


@pytest.mark.parametrize("tag", ["a", "b"])
def test_frozen_vectors(tag):
    g = {k[2:]: GOLD[k] for k in GOLD.files if k.startswith(tag + "_")}
    y = fused_moe_ref(g["x"], g["w1"], g["w2"], g["w"], g["ids"])
    np.testing.assert_allclose(y, g["out"], rtol=1e-6, atol=1e-6)
    h, s, t, npp = moe_align_ref(g["ids"], g["w1"].shape[0], 4)
    np.testing.assert_array_equal(h, g["hist"])
    np.testing.assert_array_equal(s, g["sorted"])
    np.testing.assert_array_equal(t, g["tiles"])


def test_matches_per_token_loop():
    x, w1, w2, w, ids = random_moe(6, 64, 64, 5, 3, seed=3, dup=True)
    I = 64
    ref = np.zeros_like(x)
    for t in range(x.shape[0]):
        for j in range(ids.shape[1]):
            e = ids[t, j]
            h = w1[e] @ x[t]
            a = h[:I] / (1 + np.exp(-h[:I])) * h[I:]
            ref[t] += w[t, j] * (w2[e] @ a)
    np.testing.assert_allclose(fused_moe_ref(x, w1, w2, w, ids), ref, rtol=2e-5, atol=2e-5)


@pytest.mark.parametrize("E,bm", [(8, 4), (64, 16), (3, 128)])
def test_align_invariants(E, bm):
    rng = np.random.default_rng(E + bm)
    ids = rng.integers(0, E, size=(50, 4))
    h, s, t, npp = moe_align_ref(ids, E, bm)
    n = ids.size
    assert npp % bm == 0 and len(s) == npp and len(t) == npp // bm
    assert np.array_equal(h, np.bincount(ids.ravel(), minlength=E))
    real = s[s < n]
    assert sorted(real.tolist()) == list(range(n))            # a permutation plus padding
    for tile, e in enumerate(t):                               # every tile holds one expert
        rows = s[tile * bm:(tile + 1) * bm]
        rows = rows[rows < n]
        assert (ids.ravel()[rows] == e).all()
        assert (np.diff(rows) > 0).all()                       # stable within an expert
    assert npp == sum(-(-c // bm) * bm for c in h)             # == m_tile_counts * bm


def test_bf16_round():
    x = np.array([1.0, 1.00390625, -2.5, 3.1415926], dtype=np.float32)
    r = bf16_round(x)
    assert r[0] == 1.0 and r[2] == -2.5
    assert abs(r[3] - 3.140625) < 1e-7


def test_nonlocal_slots_are_skipped():
    """-1 (expert-parallel: owned by another rank) == the slot removed."""
    from oracle.moe_ref import fused_moe_ref, moe_align_ref

    rng = np.random.default_rng(0)
    S, H, I, E, k = 9, 16, 8, 4, 3
    x = rng.standard_normal((S, H)).astype(np.float32)
    w1 = rng.standard_normal((E, 2 * I, H)).astype(np.float32)
    w2 = rng.standard_normal((E, H, I)).astype(np.float32)
    ids = rng.integers(0, E, size=(S, k)).astype(np.int32)
    w = rng.random((S, k)).astype(np.float32)
    mask = rng.random((S, k)) < 0.4
    ids_m = np.where(mask, -1, ids)
    w_zero = np.where(mask, 0.0, w).astype(np.float32)
    np.testing.assert_allclose(fused_moe_ref(x, w1, w2, w, ids_m), fused_moe_ref(x, w1, w2, w_zero, ids),
                               rtol=1e-5, atol=1e-5)
    hist, sorted_ids, tiles, npp = moe_align_ref(ids_m, E, 2)
    assert hist.sum() == (~mask).sum()
    flat = ids_m.reshape(-1)
    assert all(flat[a] >= 0 for a in sorted_ids if a < flat.size)
