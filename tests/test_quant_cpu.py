"""MXFP8 preparation (quant.py) on CPU: round trips, scale format, SF tiling."""

import numpy as np
import pytest
import torch

from paper_2604_26039_b200 import quant as Q


def test_mx_round_trip_error():
    torch.manual_seed(0)
    x = torch.randn(64, 256) * torch.logspace(-3, 3, 64)[:, None]
    q, sf = Q.mx_quantize(x)
    assert q.dtype == torch.float8_e4m3fn and sf.dtype == torch.uint8 and sf.shape == (64, 8)
    y = Q.mx_dequantize(q, sf)
    rel = (y - x).abs() / x.abs().clamp_min(1e-30)
    assert float(rel.median()) < 0.04
    assert float(((y - x).norm() / x.norm())) < 0.04
    # scales are powers of two with |x / scale| <= 448
    s = torch.exp2(sf.float() - 127)
    assert float((x.reshape(64, 8, 32).abs().amax(-1) / s).max()) <= 448.0


def test_block128_to_mx():
    torch.manual_seed(1)
    w = torch.randn(2, 256, 384) * 0.02
    q, s = Q.block128_quantize(w)
    assert s.shape == (2, 2, 3)
    q2, sf = Q.requantize_block128(q, s)
    y = Q.mx_dequantize(q2, sf)
    assert float((y - w).norm() / w.norm()) < 0.06


def test_tile_scales_layout():
    R, K = 256, 512
    sf = torch.arange(R * (K // 32), dtype=torch.int64).reshape(R, K // 32) % 251
    t = Q.tile_scales(sf.to(torch.uint8))
    assert t.shape == (2, 4, 512)
    for r in (0, 5, 31, 32, 77, 127, 128, 255):
        for g in (0, 3, 5, 15):
            rb, rr, kb, kg = r // 128, r % 128, g // 4, g % 4
            assert int(t[rb, kb, (rr % 32) * 16 + (rr // 32) * 4 + kg]) == int(sf[r, g]) % 256
