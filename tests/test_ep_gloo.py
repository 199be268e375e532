"""Expert-parallel dispatch / combine on world_size 2 (gloo, CPU): the
sharded layer must equal the dense oracle on the same inputs."""

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


def _worker(rank, world, port, E, S, k, H, I, q, wire="bf16"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.moe_ref import fused_moe_ref
        from paper_2604_26039_b200.ep import ep_moe_layer

        rng = np.random.default_rng(123)  # same weights on every rank
        w1 = (rng.standard_normal((E, 2 * I, H)) / np.sqrt(H)).astype(np.float32)
        w2 = (rng.standard_normal((E, H, I)) / np.sqrt(I)).astype(np.float32)
        r2 = np.random.default_rng(1000 + rank)  # each rank has its own tokens
        x = r2.standard_normal((S, H)).astype(np.float32)
        ids = np.stack([r2.choice(E, size=k, replace=False) for _ in range(S)]).astype(np.int32)
        lg = r2.standard_normal((S, k)).astype(np.float32)
        w = (np.exp(lg) / np.exp(lg).sum(1, keepdims=True)).astype(np.float32)
        per = E // world
        lo = rank * per

        def local_fn(rx, rids, rw):
            return torch.from_numpy(fused_moe_ref(rx.numpy(), w1[lo:lo + per], w2[lo:lo + per], rw.numpy(),
                                                  rids.numpy()))

        out = ep_moe_layer(torch.from_numpy(x), torch.from_numpy(ids), torch.from_numpy(w), E, local_fn, wire=wire)
        if wire == "fp8":  # the wire carries MXFP8 token rows: the reference sees the same rounding
            from paper_2604_26039_b200.quant import mx_dequantize, mx_quantize

            x = mx_dequantize(*mx_quantize(torch.from_numpy(x))).numpy()
        ref = fused_moe_ref(x, w1, w2, w, ids)
        q.put((rank, float(np.abs(out.numpy() - ref).max()), float(np.abs(ref).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("E,S,k,wire", [(8, 13, 2, "bf16"), (16, 5, 4, "bf16"), (16, 9, 4, "fp8")])
def test_ep_world2_matches_dense(E, S, k, wire):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, E, S, k, 32, 16, q, wire)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, scale in res:
        assert err <= 1e-4 * max(1.0, scale), (rank, err)


@pytest.mark.parametrize("wire", ["bf16", "fp8"])
def test_ep_world1_identity_path(wire):
    """world_size 1: the exchange-free path equals the dense oracle."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    p = ctx.Process(target=_worker, args=(0, 1, port, 8, 11, 2, 32, 16, q, wire))
    p.start()
    rank, err, scale = q.get(timeout=120)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert err <= 1e-4 * max(1.0, scale), (rank, err)

