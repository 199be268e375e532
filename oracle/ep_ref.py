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


def row_layout_ref(H: int, k: int, wire: str):
    """(off_sf, off_ids, off_w, row_bytes) of one wire row: the token at 0 (H
    bf16, or H e4m3 + H/32 UE8M0 at off_sf = H), k int32 ids at the next
    16-byte boundary, k fp32 weights right after, row padded to 16 bytes."""
    fp8 = wire == "fp8"
    tok = H + H // 32 if fp8 else 2 * H
    off_ids = -(-tok // 16) * 16
    off_w = off_ids + 4 * k
    return (H if fp8 else -1), off_ids, off_w, -(-(off_w + 4 * k) // 16) * 16


def _bf16_bytes(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16).view(torch.uint8).numpy()


def ep_pack_ref(x, ids, w, E: int, world: int, cap: int, wire: str = "bf16"):
    """numpy: returns send [world*cap, row_bytes] uint8 (the wire rows, see
    row_layout_ref; bytes the kernel does not define -- padding rows' tokens,
    alignment gaps -- are zero here), pos [S, world], counts [world],
    overflow (0/1)."""
    x = np.asarray(x, dtype=np.float32)
    ids = np.asarray(ids)
    w = np.asarray(w, dtype=np.float32)
    S, H = x.shape
    k = ids.shape[1]
    per = E // world
    off_sf, off_ids, off_w, rb = row_layout_ref(H, k, wire)
    send = np.zeros((world * cap, rb), dtype=np.uint8)
    fill_ids = np.full(k, -1, dtype=np.int32).view(np.uint8)
    for r in range(world * cap):  # padding rows: ids -1, weights 0
        send[r, off_ids:off_ids + 4 * k] = fill_ids
    pos = np.full((S, world), -1, dtype=np.int32)
    counts = np.zeros(world, dtype=np.int64)
    overflow = 0
    if wire == "fp8":
        q, sf = mx_quantize_bytes(x) if S else (None, None)
    else:
        xb = _bf16_bytes(x) if S else None
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
                send[r, :H] = q[t]
                send[r, off_sf:off_sf + H // 32] = sf[t]
            else:
                send[r, :2 * H] = xb[t]
            rid = np.full(k, -1, dtype=np.int32)
            rw = np.zeros(k, dtype=np.float32)
            for j, e in own:
                rid[j] = e - d * per
                rw[j] = w[t, j]
            send[r, off_ids:off_ids + 4 * k] = rid.view(np.uint8)
            send[r, off_w:off_w + 4 * k] = rw.view(np.uint8)
    return send, pos, np.minimum(counts, cap).astype(np.int32), overflow


def ep_rows_defined(send: np.ndarray, counts, cap: int, H: int, k: int, wire: str) -> np.ndarray:
    """Byte mask of the wire rows the pack kernel defines: the ids / weights
    of every row, the token (and scales) of the rows below each count."""
    off_sf, off_ids, off_w, rb = row_layout_ref(H, k, wire)
    m = np.zeros(send.shape, dtype=bool)
    m[:, off_ids:off_w + 4 * k] = True
    tok = [(0, H), (off_sf, off_sf + H // 32)] if wire == "fp8" else [(0, 2 * H)]
    for d, c in enumerate(counts):
        for a, b in tok:
            m[d * cap:d * cap + int(c), a:b] = True
    return m


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
        send, pos, cnt, ovf = ep_pack_ref(x.float().numpy(), topk_ids.numpy(), topk_w.numpy(), E, world, cap, wire)
        return (torch.from_numpy(send), torch.from_numpy(pos), torch.from_numpy(cnt),
                torch.tensor([ovf], dtype=torch.int32))

    def reduce(self, back, pos, world, cap):
        return torch.from_numpy(ep_reduce_ref(back.float().numpy(), pos.numpy(), world, cap)).to(back.dtype)
