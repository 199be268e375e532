"""Block-scaled FP8 (MXFP8) operand preparation for the FP8 megakernel path.

The Blackwell tensor core's block-scaled FP8 MMA
(`tcgen05.mma ... kind::mxf8f6f4.block_scale`) takes E4M3 operands with one
UE8M0 (power-of-two) scale per 32 consecutive K elements of every row.
DeepSeek-style checkpoints ship E4M3 weights with one fp32 scale per 128x128
block (hard part 3); `requantize_block128` turns them into MX form
once at load time (dequantise, then per-32 power-of-two scales), which the
hardware then applies inside the MMA -- no per-K-block promotion in registers.

Layouts produced here:
  q   [..., K] float8_e4m3fn  (row-major, K contiguous)
  sf  [..., K/32] uint8 UE8M0 (value 2^(sf - 127))
and `tile_scales` rearranges sf into the 512-byte blocks the kernel copies
smem -> TMEM verbatim: for every 128-row block and every 128-element K block,
byte (r % 32) * 16 + (r // 32) * 4 + kg holds the scale of row r, K group kg
(the canonical K-major scale-factor atom of the MX MMA).
"""

from __future__ import annotations

import torch

E4M3_MAX = 448.0
GROUP = 32


def mx_quantize(t: torch.Tensor, group: int = GROUP):
    """Per-`group` power-of-two scaled E4M3 quantisation along the last dim."""
    if t.shape[-1] % group:
        raise ValueError(f"last dim {t.shape[-1]} must be a multiple of {group}")
    x = t.float().reshape(*t.shape[:-1], t.shape[-1] // group, group)
    amax = x.abs().amax(dim=-1, keepdim=True).clamp_min(2.0 ** -120)
    exp = torch.ceil(torch.log2(amax / E4M3_MAX)).clamp(-127, 127)
    q = (x / torch.exp2(exp)).clamp(-E4M3_MAX, E4M3_MAX).to(torch.float8_e4m3fn)
    sf = (exp.squeeze(-1) + 127).to(torch.uint8)
    return q.reshape(t.shape), sf


def mx_dequantize(q: torch.Tensor, sf: torch.Tensor, group: int = GROUP) -> torch.Tensor:
    x = q.float().reshape(*q.shape[:-1], q.shape[-1] // group, group)
    return (x * torch.exp2(sf.float() - 127.0).unsqueeze(-1)).reshape(q.shape)


def block128_quantize(w: torch.Tensor):
    """DeepSeek-style E4M3 with one fp32 scale per 128x128 block (amax/448)."""
    *lead, R, K = w.shape
    if R % 128 or K % 128:
        raise ValueError("rows and K must be multiples of 128")
    x = w.float().reshape(*lead, R // 128, 128, K // 128, 128)
    s = x.abs().amax(dim=(-3, -1), keepdim=True).clamp_min(1e-12) / E4M3_MAX
    q = (x / s).to(torch.float8_e4m3fn).reshape(w.shape)
    return q, s.reshape(*lead, R // 128, K // 128)


def requantize_block128(q: torch.Tensor, scale: torch.Tensor):
    """128x128-block-scaled E4M3 -> MXFP8 (per-32 UE8M0)."""
    *lead, R, K = q.shape
    w = q.float().reshape(*lead, R // 128, 128, K // 128, 128) * scale.reshape(*lead, R // 128, 1, K // 128, 1)
    return mx_quantize(w.reshape(q.shape))


def tile_scales(sf: torch.Tensor) -> torch.Tensor:
    """[..., R, K/32] UE8M0 -> [..., R/128, K/128, 512] canonical SF atoms."""
    *lead, R, G = sf.shape
    if R % 128 or G % 4:
        raise ValueError("rows must be a multiple of 128 and K a multiple of 128")
    x = sf.reshape(*lead, R // 128, 4, 32, G // 4, 4)          # [.., rb, r1, r0, kb, kg]
    x = x.permute(*range(len(lead)), len(lead), len(lead) + 3, len(lead) + 2, len(lead) + 1, len(lead) + 4)
    return x.reshape(*lead, R // 128, G // 4, 512).contiguous()  # byte r0*16 + r1*4 + kg
