"""fp32 CPU oracle of the fused MoE layer and of moe_align_block_size.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  PARITY UNPINNED BY THE
REFERENCE: /root/reference has no fused-MoE forward and no alignment code
(SURVEY.md 0.2); the semantics follow the paper's three-phase description
(up-projection, SwiGLU, down-projection + scatter via
atomic add) with vLLM's weight layout (w1 = [E, 2I, H] with
the gate half first, w2 = [E, H, I]).
"""

from __future__ import annotations

import numpy as np


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def fused_moe_ref(x: np.ndarray, w1: np.ndarray, w2: np.ndarray, topk_w: np.ndarray,
                  topk_ids: np.ndarray, act_dtype=None) -> np.ndarray:
    """out[t] = sum_j w[t,j] * W2[e] (silu(W1g[e] x_t) * W1u[e] x_t), e = ids[t,j].

    All math in fp32.  `act_dtype` optionally rounds the SwiGLU activation
    (e.g. to bf16 via a callable) to model the kernel's on-chip precision;
    the default keeps it fp32 (the reference-precision oracle).
    """
    x = np.asarray(x, dtype=np.float32)
    S, H = x.shape
    E, two_i, _ = w1.shape
    I = two_i // 2
    k = topk_ids.shape[1]
    out = np.zeros((S, H), dtype=np.float32)
    flat_ids = np.asarray(topk_ids).reshape(-1)
    flat_w = np.asarray(topk_w, dtype=np.float32).reshape(-1)
    tok = np.repeat(np.arange(S), k)
    for e in np.unique(flat_ids):
        if e == -1:
            continue  # non-local slot (expert-parallel convention): no work
        sel = np.nonzero(flat_ids == e)[0]
        xe = x[tok[sel]]                                   # gather  [n, H]
        h = xe @ np.asarray(w1[e], dtype=np.float32).T     # phase 1 [n, 2I]
        a = silu(h[:, :I]) * h[:, I:]                      # phase 2 [n, I]
        if act_dtype is not None:
            a = act_dtype(a)
        y = a @ np.asarray(w2[e], dtype=np.float32).T      # phase 3 [n, H]
        np.add.at(out, tok[sel], y * flat_w[sel, None])    # weighted scatter-reduce
    return out


def topk_softmax_ref(logits: np.ndarray, k: int, renormalize: bool):
    """Router top-k (vLLM fused_topk semantics, the contract of
    ramp_fused_moe_gating_bf16): fp32 softmax over the experts, the k highest
    probabilities per token (ties to the lower expert id), weights = those
    probabilities, divided by their sum when `renormalize`.
    Returns (weights [S, k] fp32, ids [S, k] int32)."""
    z = np.asarray(logits, dtype=np.float32)
    p = np.exp(z - z.max(axis=1, keepdims=True))
    p = p / p.sum(axis=1, keepdims=True)
    ids = np.argsort(-z, axis=1, kind="stable")[:, :k]   # stable: ties keep the lower id first
    w = np.take_along_axis(p, ids, axis=1)
    if renormalize:
        w = w / w.sum(axis=1, keepdims=True)
    return w.astype(np.float32), ids.astype(np.int32)


def moe_align_ref(topk_ids: np.ndarray, E: int, bm: int):
    """Histogram + stable alignment (the contract of ramp_moe_align).

    Slots holding -1 (an expert owned by another rank) are skipped.
    Returns (hist[E], sorted_ids[n_post_pad], tile_expert[n_post_pad/bm], n_post_pad):
    flat assignment indices grouped by expert in ascending order, each
    expert's run padded with the sentinel n = topk_ids.size up to a multiple
    of bm; tile_expert[t] is the expert owning rows [t*bm, (t+1)*bm).
    The M-tile count n_post_pad/bm equals m_tile_counts (ramp/routing.py:197-203).
    """
    flat = np.asarray(topk_ids, dtype=np.int64).reshape(-1)
    n = flat.size
    valid = flat != -1  # -1 = non-local slot (expert-parallel convention): skipped
    if n and valid.any() and (flat[valid].min() < 0 or flat[valid].max() >= E):
        raise ValueError("expert id out of range")
    hist = np.bincount(flat[valid], minlength=E).astype(np.int64)
    padded = -(-hist // bm) * bm
    key = np.where(valid, flat, E)  # skipped slots sort after every expert
    order = np.argsort(key, kind="stable")
    sorted_ids = np.full(int(padded.sum()), n, dtype=np.int64)
    tile_expert = np.repeat(np.arange(E), padded // bm)
    starts = np.concatenate(([0], np.cumsum(padded)[:-1]))
    cstarts = np.concatenate(([0], np.cumsum(hist)[:-1]))
    for e in range(E):
        c = hist[e]
        if c:
            sorted_ids[starts[e]:starts[e] + c] = order[cstarts[e]:cstarts[e] + c]
    return hist, sorted_ids, tile_expert, int(padded.sum())


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 (ties to even), returned as fp32."""
    u = np.asarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def e4m3_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest OCP E4M3 value (ties to even, saturating at
    +-448, subnormal step 2^-9), returned as fp32 -- cvt.rn.satfinite.e4m3x2."""
    a = np.asarray(a, dtype=np.float32)
    m = np.minimum(np.abs(a), np.float32(448.0)).astype(np.float64)
    e = np.floor(np.log2(np.where(m > 0, m, 1.0)))
    step = np.exp2(np.maximum(e, -6.0) - 3.0)
    q = np.minimum(np.round(m / step) * step, 448.0)
    return (np.sign(a) * q).astype(np.float32)


def mx_fake_quant(v: np.ndarray, group: int = 32) -> np.ndarray:
    """MXFP8 quantise-dequantise along the last axis: one power-of-two scale
    2^ceil(log2(amax / 448)) per `group` elements (clamped to UE8M0's
    [-127, 127]), elements rounded to E4M3.  The megakernel applies exactly
    this to every gathered token row and every SwiGLU activation row."""
    v = np.asarray(v, dtype=np.float32)
    g = v.reshape(*v.shape[:-1], v.shape[-1] // group, group)
    amax = np.abs(g).max(axis=-1, keepdims=True)
    with np.errstate(divide="ignore"):
        ex = np.where(amax > 0, np.ceil(np.log2(amax.astype(np.float64) / 448.0)), -127.0)
    ex = np.clip(ex, -127, 127)
    return (e4m3_round(g * np.exp2(-ex)) * np.exp2(ex)).astype(np.float32).reshape(v.shape)


def fused_moe_ref_fp8(x, w1, w2, topk_w, topk_ids) -> np.ndarray:
    """W8A8 MXFP8 layer semantics on already-dequantised expert weights:
    tokens and activations go through mx_fake_quant, all math in fp32."""
    return fused_moe_ref(mx_fake_quant(x), w1, w2, topk_w, topk_ids, act_dtype=mx_fake_quant)
