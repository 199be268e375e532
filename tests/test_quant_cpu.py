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


def test_oracle_mx_fake_quant_matches_quantiser():
    """The oracle's numpy MXFP8 restatement and the torch operand quantiser
    agree bit for bit (incl. zero groups, tiny and huge magnitudes)."""
    import numpy as np

    from oracle.moe_ref import mx_fake_quant
    from paper_2604_26039_b200.quant import mx_dequantize, mx_quantize

    rng = np.random.default_rng(0)
    for scale in (1e-30, 1e-3, 1.0, 1e3, 1e30):
        x = (rng.standard_normal((32, 256)) * scale * np.exp(rng.standard_normal((32, 256)))).astype(np.float32)
        x[3, :32] = 0
        q, s = mx_quantize(torch.from_numpy(x))
        assert np.array_equal(mx_fake_quant(x), mx_dequantize(q, s).numpy())


def test_mxfp8_weights_roundtrip_and_layout():
    from paper_2604_26039_b200.quant import (prepare_block128_weights, prepare_mxfp8_weights, tile_scales,
                                             untile_scales, block128_quantize)

    g = torch.Generator().manual_seed(0)
    w1 = torch.randn(4, 512, 256, generator=g)
    w2 = torch.randn(4, 256, 256, generator=g)
    m = prepare_mxfp8_weights(w1, w2)
    assert m.shape == (4, 256, 256)
    assert tuple(m.w1_sf.shape) == (4 * 512 // 128, 256 // 128, 512)
    assert tuple(m.w2_sf.shape) == (4 * 256 // 128, 256 // 128, 512)
    d1, d2 = m.dequantize()
    assert float((d1 - w1).norm() / w1.norm()) < 0.04
    assert float((d2 - w2).norm() / w2.norm()) < 0.04
    s = torch.randint(0, 255, (384, 64), dtype=torch.uint8, generator=g)
    assert torch.equal(untile_scales(tile_scales(s)), s)
    b = prepare_block128_weights(*block128_quantize(w1), *block128_quantize(w2))
    e1, _ = b.dequantize()
    assert float((e1 - w1).norm() / w1.norm()) < 0.06


def test_fp8_pool_and_table_gate():
    import numpy as np

    from paper_2604_26039_b200.catalog import BASELINE_MODELS
    from paper_2604_26039_b200.config_space import b200_smem_bytes_fp8, enumerate_b200_configs
    from paper_2604_26039_b200.moe import DeviceTable

    g = BASELINE_MODELS["Qwen3-30B-A3B"]
    for dtype, want in (("fp8", True), ("bf16", False)):
        pool = enumerate_b200_configs(g, dtype=dtype)
        cols = pool.columns()
        n = len(pool)
        t = DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                        group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols.get("kps"), h3=cols.get("h3"), a=np.ones(n), b=np.zeros(n),
                        c=np.zeros(n), d=np.zeros(n), N=g.N, kappa_ok=False, sm_count=148, device="cpu")
        assert t.fp8_compatible() is want
        if dtype == "fp8":
            # split mode, ttn >= 256; every bm of the BF16 space, kps 1/2 and
            # split-K for the small token blocks (the polymorphic FP8 space)
            assert all(c.mode == 1 and c.ttn >= 256 and c.kps in (1, 2) for c in pool)
            assert {c.bm for c in pool} == {4, 8, 16, 32, 64, 128}
            assert {c.kps for c in pool} == {1, 2} and {c.split_k for c in pool} == {1, 2}
            assert all(0 < b200_smem_bytes_fp8(c.bm, c.ttn, c.stg, c.kps) <= 232448 for c in pool)
            assert len(pool) >= 100
            lib_sizes = {(c.bm, c.ttn, c.stg, c.kps): b200_smem_bytes_fp8(c.bm, c.ttn, c.stg, c.kps) for c in pool}
            from paper_2604_26039_b200 import _lib
            try:
                lib = _lib.load()
            except Exception:  # noqa: BLE001 - the C ABI test covers loading
                lib = None
            if lib is not None:
                for (bm, ttn, stg, kps), b in lib_sizes.items():
                    assert lib.ramp_config_smem_bytes_fp8_kps(bm, ttn, stg, kps) == b
