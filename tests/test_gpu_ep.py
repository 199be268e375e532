"""Expert-parallel kernels and exchange on the GPU (north_star (4)).

* ramp_ep_pack / ramp_ep_reduce (csrc/ep.cu) bit for bit against the oracle
  restatement (oracle/ep_ref.py) for 1, 2, 4 and 8 destination ranks, bf16
  and MXFP8 wires, full capacity and an overflowing one;
* a P-rank expert-parallel layer simulated on one GPU with the real kernels
  (every rank's pack, the all-to-all as block slicing, every rank's
  megakernel on its local experts -- the FP8 one straight off the MXFP8 wire --
  and the reduce) against the dense fp32 oracle;
* the library's own NCCL communicator (ramp_ep_dispatch / ramp_ep_combine)
  at world 1, against the torch.distributed exchange and the identity path.
"""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle.ep_ref import (ep_pack_ref, ep_reduce_ref, ep_rows_defined, mx_dequantize_bytes,  # noqa: E402
                           mx_quantize_bytes)
from oracle.moe_ref import bf16_round, fused_moe_ref, fused_moe_ref_fp8  # noqa: E402
from tests._util import random_moe  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _require_gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_2604_26039_b200 import _lib

    _lib.require_device()


def _rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).norm() / b.norm())


def _ids(rng, S, E, k, mode):
    if mode == "distinct":
        return np.stack([rng.choice(E, size=k, replace=False) for _ in range(S)]).astype(np.int32)
    if mode == "skew":
        return rng.integers(0, 3, size=(S, k)).astype(np.int32)
    ids = rng.integers(0, E, size=(S, k)).astype(np.int32)
    ids[rng.random((S, k)) < 0.2] = -1
    return ids


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("wire", ["bf16", "fp8"])
@pytest.mark.parametrize("S,mode,cap", [(37, "distinct", None), (300, "dup", None), (64, "skew", 20), (0, "dup", 8)])
def test_pack_and_reduce_bit_exact(world, wire, S, mode, cap):
    from paper_2604_26039_b200.ep import DeviceKernels

    E, k, H = 32, 8, 384
    rng = np.random.default_rng(S + world)
    x = bf16_round(rng.standard_normal((S, H)).astype(np.float32) * 3)
    ids = _ids(rng, S, E, k, mode)
    w = rng.random((S, k)).astype(np.float32)
    cap = S if cap is None else cap
    K = DeviceKernels()
    got = K.pack(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(ids).cuda(),
                 torch.from_numpy(w).cuda(), E, world, cap, wire)
    torch.cuda.synchronize()
    send, pos, cnt, ovf = (t.cpu() for t in got)
    rsend, rpos, rcnt, rovf = ep_pack_ref(x, ids, w, E, world, cap, wire)
    np.testing.assert_array_equal(pos.numpy(), rpos)
    np.testing.assert_array_equal(cnt.numpy(), rcnt)
    assert int(ovf.item()) == rovf
    assert tuple(send.shape) == rsend.shape
    # every byte the kernel defines (ids / weights of every row, token and
    # scales of the rows below each count), bit for bit
    m = ep_rows_defined(rsend, rcnt, cap, H, k, wire)
    np.testing.assert_array_equal(send.numpy()[m], rsend[m])
    # reduce: rank-order fp32 sum of bf16 rows, rounded once
    back = bf16_round(rng.standard_normal((world * cap, H)).astype(np.float32))
    out = K.reduce(torch.from_numpy(back).cuda().to(torch.bfloat16), pos.cuda(), world, cap)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.float().cpu().numpy(), bf16_round(ep_reduce_ref(back, rpos, world, cap)))


def _fp8_table(E, H, I, k):
    import paper_2604_26039_b200.moe as M
    from paper_2604_26039_b200.catalog import MoeGeometry
    from paper_2604_26039_b200.config_space import enumerate_b200_configs

    pool = enumerate_b200_configs(MoeGeometry(name="ep", E=E, N=2 * I, K=H, top_k=k), dtype="fp8")
    cols = pool.columns()
    n = len(pool)
    a = 10.0 + cols["bm"] * 0.01
    return M.DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                         group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols["kps"], h3=cols["h3"],
                         a=a, b=np.zeros(n), c=np.zeros(n), d=np.zeros(n), N=2 * I, kappa_ok=True, sm_count=148)


def _bf16_table(E, H, I, k):
    import paper_2604_26039_b200.moe as M
    from paper_2604_26039_b200.catalog import MoeGeometry
    from paper_2604_26039_b200.config_space import enumerate_b200_configs

    pool = enumerate_b200_configs(MoeGeometry(name="ep", E=E, N=2 * I, K=H, top_k=k))
    cols = pool.columns()
    n = len(pool)
    a = 10.0 + cols["bm"] * 0.01 + (1 - cols["mode"]) * 0.5
    return M.DeviceTable(bm=cols["bm"], ttn=cols["ttn"], stg=cols["stg"], split_k=cols["split_k"],
                         group_m=cols["group_m"].astype(np.int64), mode=cols["mode"], kps=cols["kps"], h3=cols["h3"],
                         a=a, b=np.zeros(n), c=np.zeros(n), d=np.zeros(n), N=2 * I, kappa_ok=True, sm_count=148)


@pytest.mark.parametrize("world,wire", [(2, "bf16"), (4, "fp8"), (8, "fp8")])
def test_simulated_multi_rank_layer(world, wire):
    """P ranks on one GPU: pack on every rank, all-to-all as block slicing,
    the local megakernel per rank, the reverse exchange, the reduce."""
    from paper_2604_26039_b200.ep import DeviceKernels, make_local_megakernel, row_fields
    from paper_2604_26039_b200.quant import prepare_mxfp8_weights

    E, k, H, I, S = 32, 4, 512, 256, 48
    _, w1, w2, _, _ = random_moe(1, H, I, E, k, seed=7)
    per = E // world
    K = DeviceKernels()
    ranks = []
    for r in range(world):
        x, _, _, w, ids = random_moe(S, H, I, E, k, seed=100 + r, skew=0.15 if r % 2 else None)
        ranks.append((x, w, ids))
    cap = S
    packs = []
    for x, w, ids in ranks:
        packs.append(K.pack(torch.from_numpy(x).cuda().to(torch.bfloat16), torch.from_numpy(ids).cuda(),
                            torch.from_numpy(w).cuda(), E, world, cap, wire))
    partial = []
    for r in range(world):
        blk = slice(r * cap, (r + 1) * cap)  # block r of every sender
        rows = torch.cat([p[0][blk] for p in packs])
        rx, rids, rw = row_fields(rows, H, k, wire)  # row-strided views, read in place by the megakernel
        lw1 = torch.from_numpy(w1[r * per:(r + 1) * per]).cuda()
        lw2 = torch.from_numpy(w2[r * per:(r + 1) * per]).cuda()
        if wire == "fp8":
            fn = make_local_megakernel(prepare_mxfp8_weights(lw1, lw2), _fp8_table(per, H, I, k))
        else:
            fn = make_local_megakernel((lw1.to(torch.bfloat16), lw2.to(torch.bfloat16)), _bf16_table(per, H, I, k))
        partial.append(fn(rx, rids, rw))
    for s, (x, w, ids) in enumerate(ranks):
        back = torch.cat([partial[r][s * cap:(s + 1) * cap] for r in range(world)])
        out = K.reduce(back, packs[s][1], world, cap).float().cpu().numpy()
        if wire == "fp8":
            wq = prepare_mxfp8_weights(torch.from_numpy(w1).cuda(), torch.from_numpy(w2).cuda())
            d1, d2 = (t.cpu().numpy() for t in wq.dequantize())
            ref = fused_moe_ref_fp8(x, d1, d2, w, ids)
            tol = 2e-2  # per-rank partial sums are rounded to bf16 before the reduce
        else:
            ref = fused_moe_ref(x, w1, w2, w, ids)
            tol = 1e-2
        err = float(np.linalg.norm(out - ref) / np.linalg.norm(ref))
        assert err < tol, (world, wire, s, err)


def test_mxfp8_wire_matches_megakernel_quantisation():
    """The wire's MXFP8 rows, fed to the FP8 megakernel pre-quantised, give
    the same layer as letting the megakernel quantise the bf16 rows itself
    (one quantisation rule: oracle/moe_ref.mx_fake_quant's)."""
    import paper_2604_26039_b200.moe as M
    from paper_2604_26039_b200.quant import prepare_mxfp8_weights

    E, k, H, I, S = 16, 4, 512, 256, 40
    x, w1, w2, w, ids = random_moe(S, H, I, E, k, seed=11)
    q, sf = mx_quantize_bytes(x)
    wq = prepare_mxfp8_weights(torch.from_numpy(w1).cuda(), torch.from_numpy(w2).cuda())
    tab = _fp8_table(E, H, I, k)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    wt, it = torch.from_numpy(w).cuda(), torch.from_numpy(ids).cuda()
    a = M.fused_moe_fp8(xt, wq, wt, it, tab, 0)
    b = M.fused_moe_fp8((torch.from_numpy(q).cuda(), torch.from_numpy(sf).cuda()), wq, wt, it, tab, 0)
    torch.cuda.synchronize()
    # identical operands; only the order of the fp32 output reductions (atomics) may differ
    assert _rel(a, b) < 1e-3


def _nccl_world1(fn):
    import socket

    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        return fn()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("wire", ["bf16", "fp8"])
def test_nccl_exchange_world1(wire):
    """The C-ABI NCCL path (ramp_ep_dispatch / ramp_ep_combine), the
    torch.distributed exchange and the identity path agree at world 1, and
    the NCCL path replays inside a CUDA graph."""
    from paper_2604_26039_b200.ep import EPComm, ep_moe_layer, make_local_megakernel
    from paper_2604_26039_b200.quant import prepare_mxfp8_weights

    E, k, H, I, S = 16, 4, 512, 256, 64
    x, w1, w2, w, ids = random_moe(S, H, I, E, k, seed=21)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    wt, it = torch.from_numpy(w).cuda(), torch.from_numpy(ids).cuda()
    if wire == "fp8":
        fn = make_local_megakernel(prepare_mxfp8_weights(torch.from_numpy(w1).cuda(), torch.from_numpy(w2).cuda()),
                                   _fp8_table(E, H, I, k))
    else:
        fn = make_local_megakernel((torch.from_numpy(w1).cuda().to(torch.bfloat16),
                                    torch.from_numpy(w2).cuda().to(torch.bfloat16)), _bf16_table(E, H, I, k))

    def body():
        comm = EPComm()
        try:
            ident = ep_moe_layer(xt, it, wt, E, fn, wire=wire)
            tdist = ep_moe_layer(xt, it, wt, E, fn, wire=wire, exchange="always")
            nccl = ep_moe_layer(xt, it, wt, E, fn, wire=wire, comm=comm)
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    cap_out = ep_moe_layer(xt, it, wt, E, fn, wire=wire, comm=comm)
            g.replay()
            torch.cuda.synchronize()
            res = ident, tdist, nccl, cap_out.clone()
            del g  # a captured graph holds the communicator's operations: free it before the communicator
            torch.cuda.synchronize()
            return res
        finally:
            comm.close()

    ident, tdist, nccl, graphed = _nccl_world1(body)
    # same operands on every path (only the order of the fp32 output atomics
    # differs); one bf16 round of the partial sums separates the exchange
    # paths from the identity one
    assert _rel(tdist, nccl) < 1e-3 and _rel(nccl, graphed) < 1e-3 and _rel(ident, nccl) < 1e-2
    if wire == "fp8":  # against the W8A8 MXFP8 semantics on the dequantised weights
        wq = prepare_mxfp8_weights(torch.from_numpy(w1).cuda(), torch.from_numpy(w2).cuda())
        d1, d2 = (t.cpu().numpy() for t in wq.dequantize())
        ref, tol = fused_moe_ref_fp8(x, d1, d2, w, ids), 2e-2
    else:
        ref, tol = fused_moe_ref(x, w1, w2, w, ids), 1e-2
    for o in (ident, nccl):
        err = float(np.linalg.norm(o.float().cpu().numpy() - ref) / np.linalg.norm(ref))
        assert err < tol, err


def _rows_of(x_fields, ids, w, H, k, wire):
    """A [S, row_bytes] wire-row buffer holding these tokens / ids / weights."""
    from paper_2604_26039_b200.ep import row_fields, row_layout

    S = ids.shape[0]
    rows = torch.full((S, row_layout(H, k, wire).row_bytes), 0x5A, dtype=torch.uint8, device="cuda")
    rx, rids, rw = row_fields(rows, H, k, wire)
    if wire == "fp8":
        rx[0].copy_(x_fields[0])
        rx[1].copy_(x_fields[1])
    else:
        rx.copy_(x_fields)
    rids.copy_(ids)
    rw.copy_(w)
    return rows, (rx, rids, rw)


@pytest.mark.parametrize("S,bm", [(6, 16), (300, 64), (2100, 128)])
@pytest.mark.parametrize("dtype", ["bf16", "fp8", "fp8_prequant"])
def test_row_strided_inputs_match_dense(S, bm, dtype):
    """ramp_fused_moe_strided (tokens, scales, ids and weights read in place
    from the wire's rows) equals the dense entry on the same operands -- the
    decode gather4 path (bm 16), the phase-0 gather, and S*k > kIdCache
    (the route kernel's uncached id reads)."""
    import paper_2604_26039_b200.moe as M
    from paper_2604_26039_b200.catalog import MoeGeometry
    from paper_2604_26039_b200.config_space import enumerate_b200_configs
    from paper_2604_26039_b200.quant import prepare_mxfp8_weights

    E, k, H, I = 16, 8, 512, 256
    x, w1, w2, w, ids = random_moe(S, H, I, E, k, seed=S + bm)
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    wt, it = torch.from_numpy(w).cuda(), torch.from_numpy(ids).cuda()
    fp8 = dtype != "bf16"
    pool = enumerate_b200_configs(MoeGeometry(name="rows", E=E, N=2 * I, K=H, top_k=k), dtype="fp8" if fp8 else "bf16")
    cfg = next(c.id for c in pool if c.bm == bm and c.mode == 1 and c.split_k == 1)
    if fp8:
        tab = _fp8_table(E, H, I, k)
        wq = prepare_mxfp8_weights(torch.from_numpy(w1).cuda(), torch.from_numpy(w2).cuda())
        if dtype == "fp8_prequant":
            q, sf = (torch.from_numpy(a).cuda() for a in mx_quantize_bytes(x))
            dense = M.fused_moe_fp8((q, sf), wq, wt, it, tab, cfg)
            _, (rx, rids, rw) = _rows_of((q, sf), it, wt, H, k, "fp8")
            assert not rx[0].is_contiguous() and not rids.is_contiguous()
            got = M.fused_moe_fp8(rx, wq, rw, rids, tab, cfg)
        else:
            dense = M.fused_moe_fp8(xt, wq, wt, it, tab, cfg)
            _, (rx, rids, rw) = _rows_of(xt, it, wt, H, k, "bf16")
            got = M.fused_moe_fp8(rx, wq, rw, rids, tab, cfg)
    else:
        tab = _bf16_table(E, H, I, k)
        w1b, w2b = (torch.from_numpy(a).cuda().to(torch.bfloat16) for a in (w1, w2))
        dense = M.fused_moe(xt, w1b, w2b, wt, it, tab, cfg)
        _, (rx, rids, rw) = _rows_of(xt, it, wt, H, k, "bf16")
        got = M.fused_moe(rx, w1b, w2b, rw, rids, tab, cfg)
    torch.cuda.synchronize()
    assert _rel(got, dense) < 1e-3  # same operands: only the fp32 output atomics' order may differ
