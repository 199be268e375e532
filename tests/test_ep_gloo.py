"""Expert-parallel dispatch / combine on gloo (CPU), world sizes 1, 2, 4 and 8:
the sharded layer must equal the dense oracle on the same inputs.

The exchange protocol of paper_2604_26039_b200.ep runs unchanged (fixed
`cap`-row blocks per destination through torch.distributed.all_to_all_single,
padding rows with ids -1, combine in rank order); the pack / reduce kernels
are the oracle's CPU restatement (oracle/ep_ref.RefKernels) -- the device
kernels are held to that restatement bit for bit in tests/test_gpu_ep.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _routing(rng, S, E, k, mode):
    if S == 0:
        return np.zeros((0, k), dtype=np.int32)
    if mode == "distinct":
        return np.stack([rng.choice(E, size=k, replace=False) for _ in range(S)]).astype(np.int32)
    if mode == "skew":  # every slot on the first two experts: most ranks receive nothing
        return rng.integers(0, 2, size=(S, k)).astype(np.int32)
    if mode == "dup":  # duplicated experts per token and invalid (-1) slots
        ids = rng.integers(0, E, size=(S, k)).astype(np.int32)
        ids[rng.random((S, k)) < 0.2] = -1
        return ids
    raise ValueError(mode)


def _worker(rank, world, port, E, S, k, H, I, q, wire, mode, cap, empty_rank=-1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.ep_ref import RefKernels, mx_dequantize_bytes, mx_quantize_bytes
        from oracle.moe_ref import bf16_round, fused_moe_ref
        from paper_2604_26039_b200.ep import ep_moe_layer

        rng = np.random.default_rng(123)  # same weights on every rank
        w1 = (rng.standard_normal((E, 2 * I, H)) / np.sqrt(H)).astype(np.float32)
        w2 = (rng.standard_normal((E, H, I)) / np.sqrt(I)).astype(np.float32)
        r2 = np.random.default_rng(1000 + rank)  # each rank has its own tokens
        if rank == empty_rank:
            S = 0
        x = r2.standard_normal((S, H)).astype(np.float32)
        ids = _routing(r2, S, E, k, mode).reshape(S, k)
        lg = r2.standard_normal((S, k)).astype(np.float32)
        w = (np.exp(lg) / np.exp(lg).sum(1, keepdims=True)).astype(np.float32)
        per = E // world
        lo = rank * per

        def local_fn(rx, rids, rw):
            xr = mx_dequantize_bytes(rx[0].numpy(), rx[1].numpy()) if isinstance(rx, tuple) else rx.float().numpy()
            return torch.from_numpy(fused_moe_ref(xr, w1[lo:lo + per], w2[lo:lo + per], rw.numpy(), rids.numpy()))

        out = ep_moe_layer(torch.from_numpy(x), torch.from_numpy(ids), torch.from_numpy(w), E, local_fn, wire=wire,
                           cap=cap, kernels=RefKernels(), exchange="always")
        if wire == "fp8":  # the wire carries MXFP8 token rows: the reference sees the same rounding
            x = mx_dequantize_bytes(*mx_quantize_bytes(x))
        else:  # bf16 token rows
            x = bf16_round(x)
        ref = fused_moe_ref(x, w1, w2, w, ids)
        assert tuple(out.shape) == (S, H)
        q.put((rank, float(np.abs(out.numpy() - ref).max(initial=0.0)), float(np.abs(ref).max(initial=0.0))))
    finally:
        dist.destroy_process_group()


def _run(world, E, S, k, wire, mode, cap=None, H=128, I=32, empty_rank=-1):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, E, S, k, H, I, q, wire, mode, cap, empty_rank))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, scale in res:
        assert err <= 1e-4 * max(1.0, scale), (world, rank, err)
    return res


@pytest.mark.parametrize("world,E,S,k,wire,mode", [
    (2, 8, 13, 2, "bf16", "distinct"),
    (2, 16, 9, 4, "fp8", "dup"),
    (4, 16, 11, 4, "fp8", "skew"),
    (8, 64, 5, 8, "bf16", "skew"),
])
def test_ep_matches_dense(world, E, S, k, wire, mode):
    _run(world, E, S, k, wire, mode)


def test_ep_world1_exchange_path():
    """world_size 1 with the exchange forced (pack -> self all-to-all -> reduce)."""
    _run(1, 8, 11, 2, "bf16", "dup")


def test_ep_empty_rank_batch():
    """A rank with no tokens still takes part in the exchanges (cap is the
    common per-rank capacity, here the other ranks' batch)."""
    _run(3, 9, 7, 2, "bf16", "distinct", cap=7, empty_rank=1)


@pytest.mark.parametrize("wire", ["bf16", "fp8"])
def test_ep_world1_identity_path(wire):
    """world_size 1, exchange='auto': the layer runs on the inputs directly."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    p = ctx.Process(target=_identity_worker, args=(port, q, wire))
    p.start()
    err, scale = q.get(timeout=120)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert err <= 1e-4 * max(1.0, scale)


def _identity_worker(port, q, wire):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        from oracle.moe_ref import fused_moe_ref
        from paper_2604_26039_b200.ep import dispatch, ep_moe_layer

        rng = np.random.default_rng(5)
        E, S, k, H, I = 8, 9, 2, 128, 32
        w1 = (rng.standard_normal((E, 2 * I, H)) / np.sqrt(H)).astype(np.float32)
        w2 = (rng.standard_normal((E, H, I)) / np.sqrt(I)).astype(np.float32)
        x = rng.standard_normal((S, H)).astype(np.float32)
        ids = _routing(rng, S, E, k, "distinct")
        w = np.full((S, k), 0.5, dtype=np.float32)
        plan, rx, _, _ = dispatch(torch.from_numpy(x), torch.from_numpy(ids), torch.from_numpy(w), E, wire=wire)
        assert plan.identity and plan.pos is None
        out = ep_moe_layer(torch.from_numpy(x), torch.from_numpy(ids), torch.from_numpy(w), E,
                           lambda rx, ri, rw: torch.from_numpy(fused_moe_ref(rx.numpy(), w1, w2, rw.numpy(),
                                                                             ri.numpy())), wire=wire)
        ref = fused_moe_ref(x, w1, w2, w, ids)
        q.put((float(np.abs(out.numpy() - ref).max()), float(np.abs(ref).max())))
    finally:
        dist.destroy_process_group()


def test_pack_ref_contract():
    """The oracle pack itself: one row per unique (token, rank), token order,
    local ids, padding rows -1, overflow flagged when cap is too small."""
    from oracle.ep_ref import ep_pack_ref, ep_reduce_ref, row_layout_ref

    x = np.random.default_rng(0).standard_normal((4, 128)).astype(np.float32)
    ids = np.array([[0, 5], [5, 6], [1, 1], [7, -1]], dtype=np.int32)
    w = np.array([[0.1, 0.2], [0.3, 0.4], [0.5, 0.6], [0.7, 0.8]], dtype=np.float32)
    send, pos, cnt, ovf = ep_pack_ref(x, ids, w, 8, 2, 4)
    _, off_ids, off_w, rb = row_layout_ref(128, 2, "bf16")
    assert send.shape == (8, rb) and rb % 16 == 0 and off_ids == 256
    sid = np.ascontiguousarray(send[:, off_ids:off_ids + 8]).view(np.int32)
    sw = np.ascontiguousarray(send[:, off_w:off_w + 8]).view(np.float32)
    sx = torch.from_numpy(np.ascontiguousarray(send[:, :256])).view(torch.bfloat16).float().numpy()
    assert cnt.tolist() == [2, 3] and ovf == 0
    assert pos.tolist() == [[0, 0], [-1, 1], [1, -1], [-1, 2]]
    assert sid[0].tolist() == [0, -1] and sid[4].tolist() == [-1, 1] and sid[5].tolist() == [1, 2]
    assert sid[6].tolist() == [3, -1] and sid[3].tolist() == [-1, -1] and sid[7].tolist() == [-1, -1]
    assert sw[5].tolist() == pytest.approx([0.3, 0.4]) and sw[4].tolist() == pytest.approx([0.0, 0.2])
    np.testing.assert_array_equal(sx[5], torch.from_numpy(x[1]).to(torch.bfloat16).float().numpy())
    back = np.arange(8 * 128, dtype=np.float32).reshape(8, 128)
    red = ep_reduce_ref(back, pos, 2, 4)
    np.testing.assert_array_equal(red[0], back[0] + back[4])
    *_, ovf2 = ep_pack_ref(x, ids, w, 8, 2, 2)
    assert ovf2 == 1
