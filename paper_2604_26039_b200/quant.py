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

from dataclasses import dataclass

import torch

E4M3_MAX = 448.0
GROUP = 32


def mx_quantize(t: torch.Tensor, group: int = GROUP):
    """Per-`group` power-of-two scaled E4M3 quantisation along the last dim."""
    if t.shape[-1] % group:
        raise ValueError(f"last dim {t.shape[-1]} must be a multiple of {group}")
    x = t.float().reshape(*t.shape[:-1], t.shape[-1] // group, group)
    amax = x.abs().amax(dim=-1, keepdim=True)
    # exactly ceil(log2(amax / 448)) (the megakernel's rule, csrc/ptx.cuh
    # mx_exponent): amax = m * 2^e with m in [0.5, 1), 448 = 0.875 * 2^9
    m, e = torch.frexp(amax)
    exp = torch.where(amax > 0, e - 9 + (m > 0.875).to(e.dtype), torch.full_like(e, -127)).clamp(-127, 127).float()
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


def untile_scales(tiled: torch.Tensor) -> torch.Tensor:
    """Inverse of `tile_scales`: [..., R/128, K/128, 512] -> [..., R, K/32]."""
    *lead, RB, KB, _ = tiled.shape
    x = tiled.reshape(*lead, RB, KB, 32, 4, 4)                  # [.., rb, kb, r0, r1, kg]
    n = len(lead)
    x = x.permute(*range(n), n, n + 3, n + 2, n + 1, n + 4)     # [.., rb, r1, r0, kb, kg]
    return x.reshape(*lead, RB * 128, KB * 4).contiguous()


@dataclass
class MxFp8Weights:
    """Expert weights in the FP8 megakernel's operand format.

    w1_q [E, 2I, H] / w2_q [E, H, I] float8_e4m3fn, and their UE8M0 scales as
    canonical 512-byte atoms: w1_sf [E*2I/128, H/128, 512], w2_sf
    [E*H/128, I/128, 512] (rows of all experts flattened, so the kernel
    indexes a row block as (expert*rows + row) / 128)."""

    w1_q: torch.Tensor
    w1_sf: torch.Tensor
    w2_q: torch.Tensor
    w2_sf: torch.Tensor

    @property
    def shape(self):
        E, two_i, H = self.w1_q.shape
        return E, H, two_i // 2

    def to(self, device) -> "MxFp8Weights":
        return MxFp8Weights(*(t.to(device) for t in (self.w1_q, self.w1_sf, self.w2_q, self.w2_sf)))

    def dequantize(self):
        """fp32 (w1, w2) the FP8 MMAs multiply by -- the oracle's weights."""
        E, H, I = self.shape
        s1 = untile_scales(self.w1_sf).reshape(E, 2 * I, H // GROUP)
        s2 = untile_scales(self.w2_sf).reshape(E, H, I // GROUP)
        return mx_dequantize(self.w1_q, s1), mx_dequantize(self.w2_q, s2)


def _pack(w1_q, s1, w2_q, s2) -> MxFp8Weights:
    E, two_i, H = w1_q.shape
    I = two_i // 2
    return MxFp8Weights(w1_q.contiguous(), tile_scales(s1.reshape(E * two_i, H // GROUP)),
                        w2_q.contiguous(), tile_scales(s2.reshape(E * H, I // GROUP)))


def prepare_mxfp8_weights(w1: torch.Tensor, w2: torch.Tensor) -> MxFp8Weights:
    """bf16 / fp32 expert weights (vLLM layout) -> MXFP8 operands."""
    q1, s1 = mx_quantize(w1)
    q2, s2 = mx_quantize(w2)
    return _pack(q1, s1, q2, s2)


def prepare_block128_weights(w1_q, w1_scale, w2_q, w2_scale) -> MxFp8Weights:
    """A DeepSeek-style checkpoint (E4M3 + one fp32 scale per 128x128 block)
    -> MXFP8 operands, once at load time."""
    q1, s1 = requantize_block128(w1_q, w1_scale)
    q2, s2 = requantize_block128(w2_q, w2_scale)
    return _pack(q1, s1, q2, s2)


def quantize_tokens_ref(x: torch.Tensor) -> torch.Tensor:
    """What the megakernel's phase-0 gather does to every token row (per-token,
    per-32 UE8M0 + E4M3), returned dequantised; for tests."""
    q, s = mx_quantize(x)
    return mx_dequantize(q, s)
