"""CPU restatement of the expert-parallel pack / reduce kernels -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py).

Parity unpinned by the reference: /root/reference is single-GPU and has no
exchange code; this restates the contract of csrc/ep.cu
(owner rank r holds experts [r*E/P, (r+1)*E/P); one row per
unique (token, rank) pair, in token order; fixed `cap` rows per destination,
padding rows with ids -1; the MXFP8 wire is the megakernel's own operand
quantisation, oracle/moe_ref.mx_fake_quant's rule) with plain loops, and
`RefKernels` plugs it into paper_2604_26039_b200.ep on CPU tensors (the gloo
tests) -- the device kernels are compared with it bit for bit on the GPU.
"""

from __future__ import annotations

import numpy as np
import torch


def mx_quantize_bytes(x: np.ndarray):
    """MXFP8 of fp32 rows: (e4m3 bytes [R, H], UE8M0 [R, H/32]) with the
    exact scale rule of oracle/moe_ref.mx_fake_quant."""
    x = np.asarray(x, dtype=np.float32)
    R, H = x.shape
    g = x.reshape(R, H // 32, 32)
    amax = np.abs(g).max(axis=-1, keepdims=True)
    with np.errstate(divide="ignore"):
        ex = np.where(amax > 0, np.ceil(np.log2(amax.astype(np.float64) / 448.0)), -127.0)
    ex = np.clip(ex, -127, 127)
    scaled = (g * np.exp2(-ex)).astype(np.float32).reshape(R, H)
    q = torch.from_numpy(np.clip(scaled, -448.0, 448.0)).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    return q, (ex[..., 0] + 127).astype(np.uint8)


def mx_dequantize_bytes(q: np.ndarray, sf: np.ndarray) -> np.ndarray:
    v = torch.from_numpy(np.ascontiguousarray(q)).view(torch.float8_e4m3fn).float().numpy()
    R, H = v.shape
    return (v.reshape(R, H // 32, 32) * np.exp2(sf.astype(np.float64) - 127.0)[..., None]).reshape(R, H).astype(
        np.float32)


def ep_pack_ref(x, ids, w, E: int, world: int, cap: int, wire: str = "bf16"):
    """numpy: returns send_x ([world*cap, H] bf16-as-fp32 or e4m3 bytes),
    send_sf ([world*cap, H/32] or None), send_ids, send_w, pos [S, world],
    counts [world], overflow (0/1).  Unwritten payload rows are zero."""
    x = np.asarray(x, dtype=np.float32)
    ids = np.asarray(ids)
    w = np.asarray(w, dtype=np.float32)
    S, H = x.shape
    k = ids.shape[1]
    per = E // world
    send_x = np.zeros((world * cap, H), dtype=np.uint8 if wire == "fp8" else np.float32)
    send_sf = np.zeros((world * cap, H // 32), dtype=np.uint8) if wire == "fp8" else None
    send_ids = np.full((world * cap, k), -1, dtype=np.int32)
    send_w = np.zeros((world * cap, k), dtype=np.float32)
    pos = np.full((S, world), -1, dtype=np.int32)
    counts = np.zeros(world, dtype=np.int64)
    overflow = 0
    q, sf = mx_quantize_bytes(x) if wire == "fp8" and S else (None, None)
    for t in range(S):
        for d in range(world):
            own = [(j, int(e)) for j, e in enumerate(ids[t]) if 0 <= e < E and e // per == d]
            if not own:
                continue
            row = counts[d]
            counts[d] += 1
            if row >= cap:
                overflow = 1
                continue
            pos[t, d] = row
            r = d * cap + row
            if wire == "fp8":
                send_x[r], send_sf[r] = q[t], sf[t]
            else:
                send_x[r] = x[t]
            for j, e in own:
                send_ids[r, j] = e - d * per
                send_w[r, j] = w[t, j]
    return send_x, send_sf, send_ids, send_w, pos, np.minimum(counts, cap).astype(np.int32), overflow


def ep_reduce_ref(back, pos, world: int, cap: int) -> np.ndarray:
    """out[t] = sum over ranks d in order of back[d*cap + pos[t, d]] (fp32)."""
    back = np.asarray(back, dtype=np.float32)
    pos = np.asarray(pos)
    S = pos.shape[0]
    out = np.zeros((S, back.shape[1]), dtype=np.float32)
    for t in range(S):
        for d in range(world):
            if pos[t, d] >= 0:
                out[t] += back[d * cap + pos[t, d]]
    return out


class RefKernels:
    """paper_2604_26039_b200.ep's `kernels=` interface on CPU tensors."""

    def pack(self, x, topk_ids, topk_w, E, world, cap, wire):
        sx, ssf, sid, sw, pos, cnt, ovf = ep_pack_ref(x.float().numpy(), topk_ids.numpy(), topk_w.numpy(), E, world,
                                                     cap, wire)
        send_x = torch.from_numpy(sx) if wire == "fp8" else torch.from_numpy(sx).to(x.dtype)
        return (send_x, None if ssf is None else torch.from_numpy(ssf), torch.from_numpy(sid),
                torch.from_numpy(sw), torch.from_numpy(pos), torch.from_numpy(cnt),
                torch.tensor([ovf], dtype=torch.int32))

    def reduce(self, back, pos, world, cap):
        return torch.from_numpy(ep_reduce_ref(back.float().numpy(), pos.numpy(), world, cap)).to(back.dtype)
