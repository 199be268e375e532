"""Expert parallelism for the expert-sharded configs (north_star (4)).

Rank r of a P-rank group owns experts [r*E/P, (r+1)*E/P).  One MoE layer:

  1. dispatch: every (token, expert) assignment goes to the owner rank of its
     expert.  Assignments of one token bound for the same rank are merged
     into one row (the token is sent once per destination rank, with its k
     slots as rank-local expert ids, -1 for the other ranks' slots), so the
     wire carries unique (token, rank) pairs -- the "pre-reduce per
     (token, rank)" of SURVEY §8e.
  2. the owner runs the fused-MoE megakernel on its local experts: the
     received rows are its tokens (slots with expert -1 are skipped by the
     route kernel, so they cost no work);
  3. combine: the per-(token, rank) partial outputs travel back and are
     summed, in rank order, into the origin tokens.

Every buffer on the wire has a FIXED capacity -- `cap` rows per destination
(cap = S by default, which never drops a pair; rows past a destination's
count carry ids -1) -- so no split size is ever read on the host: the whole
layer is asynchronous and CUDA-graph capturable.  The pack (step 1's
row/slot construction, bf16 or MXFP8 rows) and the reduce (step 3's sum)
are device kernels of libramp_b200 (`ramp_ep_pack` / `ramp_ep_reduce`,
csrc/ep.cu).  A wire row is one self-contained message -- the token, its
scales, its k local ids and weights at fixed offsets (`row_layout`) -- so a
dispatch is ONE send / receive per peer, and the receiving megakernel reads
the fields in place (row-strided inputs, `ramp_fused_moe_strided`).  The
exchanges run either through this library's own NCCL communicator
(`EPComm`: `ramp_ep_dispatch` / `ramp_ep_combine`, one grouped NCCL
send/recv per direction, the C ABI a reference-side integration binds) or
through `torch.distributed.all_to_all_single` on the packed rows (any
backend; what the gloo CPU tests drive, with the oracle's restatement of the
two kernels injected as `kernels=`).

With the MXFP8 wire the received rows stay MXFP8 (e4m3 + one UE8M0 scale per
32 features, 0.52x the bf16 bytes) and feed the FP8 megakernel directly
(`moe.fused_moe_fp8` with a pre-quantised pair): the wire's quantisation IS
the megakernel's operand quantisation, nothing is expanded back to bf16.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib

WIRES = {"bf16": 0, "fp8": 1}  # RAMP_EP_WIRE_BF16 / RAMP_EP_WIRE_MXFP8


@dataclass
class EPPlan:
    """Send-side bookkeeping of one dispatch (kept for the combine)."""

    world: int
    cap: int
    wire: str
    pos: torch.Tensor | None       # [S, world] int32: row of (token, rank) in the send blocks, -1 = not sent
    counts: torch.Tensor | None    # [world] int32 (device): rows sent to each rank
    overflow: torch.Tensor | None  # [1] int32 (device): 1 if some rank needed more than cap rows
    wire_bytes: int = 0            # bytes this rank puts on the wire per dispatch (fixed blocks)
    identity: bool = False         # world 1, no exchange: the layer ran on the inputs directly


def expert_owner(ids: torch.Tensor, E: int, world: int) -> torch.Tensor:
    per = E // world
    return torch.div(ids, per, rounding_mode="floor")


@dataclass(frozen=True)
class RowLayout:
    """Byte offsets of one wire row (csrc/ep.cu ep_row_layout,
    ramp_ep_row_layout): token at 0 (H bf16, or H e4m3 then H/32 UE8M0 at
    off_sf), k int32 local ids at off_ids, k fp32 weights at off_w."""

    off_sf: int
    off_ids: int
    off_w: int
    row_bytes: int


def row_layout(H: int, k: int, wire: str) -> RowLayout:
    fp8 = wire == "fp8"
    tok = H + H // 32 if fp8 else 2 * H
    off_ids = (tok + 15) // 16 * 16
    off_w = off_ids + 4 * k
    return RowLayout(H if fp8 else -1, off_ids, off_w, (off_w + 4 * k + 15) // 16 * 16)


def row_fields(rows: torch.Tensor, H: int, k: int, wire: str):
    """(x, ids, w) views of a [n, row_bytes] uint8 row buffer: x is [n, H]
    bf16, or the pair (e4m3 bytes [n, H], UE8M0 [n, H/32]); ids [n, k] int32;
    w [n, k] fp32 -- row-strided views, no copy."""
    L = row_layout(H, k, wire)
    ids = rows[:, L.off_ids:L.off_ids + 4 * k].view(torch.int32)
    w = rows[:, L.off_w:L.off_w + 4 * k].view(torch.float32)
    if wire == "fp8":
        x = (rows[:, :H], rows[:, L.off_sf:L.off_sf + H // 32])
    else:
        x = rows[:, :2 * H].view(torch.bfloat16)
    return x, ids, w


class DeviceKernels:
    """The pack / reduce kernels of libramp_b200 (csrc/ep.cu).  CUDA tensors
    only; there is no CPU path."""

    def pack(self, x, topk_ids, topk_w, E: int, world: int, cap: int, wire: str):
        lib = _lib.load()
        S, H = x.shape
        k = topk_ids.shape[1]
        dev = x.device
        for name, t, dt in (("x", x, torch.bfloat16), ("topk_ids", topk_ids, torch.int32),
                            ("topk_w", topk_w, torch.float32)):
            if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous {dt} CUDA tensor (there is no CPU path)")
        send = torch.empty(world * cap, row_layout(H, k, wire).row_bytes, dtype=torch.uint8, device=dev)
        pos = torch.empty(S, world, dtype=torch.int32, device=dev)
        counts = torch.empty(world, dtype=torch.int32, device=dev)
        overflow = torch.empty(1, dtype=torch.int32, device=dev)  # written by the pack kernel
        _lib.check(lib.ramp_ep_pack(x.data_ptr(), topk_ids.data_ptr(), topk_w.data_ptr(), S, H, E, k, world, cap,
                                    WIRES[wire], send.data_ptr(), pos.data_ptr(), counts.data_ptr(),
                                    overflow.data_ptr(), _stream()))
        return send, pos, counts, overflow

    def reduce(self, back, pos, world: int, cap: int):
        lib = _lib.load()
        S = pos.shape[0]
        H = back.shape[1]
        if back.dtype != torch.bfloat16 or not back.is_cuda or not back.is_contiguous():
            raise ValueError("partial outputs must be a contiguous bf16 CUDA tensor")
        out = torch.empty(S, H, dtype=torch.bfloat16, device=back.device)
        _lib.check(lib.ramp_ep_reduce(back.data_ptr(), pos.data_ptr(), S, H, world, cap, out.data_ptr(), _stream()))
        return out


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class EPComm:
    """libramp_b200's own NCCL communicator over a torch.distributed group
    (rank 0 creates the NCCL unique id, the group broadcasts it).  With it,
    dispatch / combine are single C-ABI calls (pack + one grouped NCCL
    all-to-all; all-to-all + reduce), capturable in a CUDA graph."""

    def __init__(self, group=None):
        lib = _lib.load()
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(lib.ramp_ep_get_unique_id(uid))
        obj = [uid.raw]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        self._comm = ctypes.c_void_p()
        _lib.check(lib.ramp_ep_comm_init(ctypes.byref(self._comm), obj[0], self.world, self.rank))

    @property
    def handle(self):
        return self._comm

    def close(self):
        """ncclCommDestroy.  CUDA graphs that captured this communicator's
        exchanges must be destroyed first (NCCL waits for their operations)."""
        if self._comm:
            _lib.load().ramp_ep_comm_destroy(self._comm)
            self._comm = ctypes.c_void_p()


def dispatch(x: torch.Tensor, topk_ids: torch.Tensor, topk_w: torch.Tensor, E: int, group=None,
             wire: str = "bf16", cap: int | None = None, comm: EPComm | None = None, kernels=None,
             exchange: str = "auto"):
    """Route token rows to expert owners.

    Returns (plan, recv_x, recv_ids [P*cap, k] rank-local expert ids, recv_w
    [P*cap, k]); recv_x is [P*cap, H] bf16, or the pair (e4m3 bytes
    [P*cap, H], UE8M0 scales [P*cap, H/32]) with wire="fp8" -- all four are
    row-strided views of the one received row buffer (`row_fields`), which
    the megakernel reads in place.  Block s of the received rows came from
    rank s; rows past its count have ids -1.

    exchange="auto" takes the identity shortcut at world 1 (every expert is
    local: the layer runs on the inputs, no pack, no collective);
    "always" packs and exchanges at every world size (the measured path)."""
    if wire not in WIRES:
        raise ValueError(f"wire must be bf16 or fp8, got {wire!r}")
    if exchange not in ("auto", "always"):
        raise ValueError(f"exchange must be 'auto' or 'always', got {exchange!r}")
    world = comm.world if comm is not None else dist.get_world_size(group)
    if E % world:
        raise ValueError(f"E={E} does not split over {world} ranks")
    S, H = x.shape
    k = topk_ids.shape[1]
    if world == 1 and exchange == "auto" and comm is None:
        plan = EPPlan(world=1, cap=S, wire=wire, pos=None, counts=None, overflow=None, identity=True)
        return plan, x, topk_ids, topk_w
    cap = S if cap is None else int(cap)
    if cap < 0:
        raise ValueError("cap must be >= 0")
    dev = x.device
    L = row_layout(H, k, wire)
    recv = torch.empty(world * cap, L.row_bytes, dtype=torch.uint8, device=dev)
    if comm is not None:
        lib = _lib.load()
        send = torch.empty_like(recv)
        pos = torch.empty(S, world, dtype=torch.int32, device=dev)
        counts = torch.empty(world, dtype=torch.int32, device=dev)
        overflow = torch.empty(1, dtype=torch.int32, device=dev)  # written by the pack kernel
        for name, t, dt in (("x", x, torch.bfloat16), ("topk_ids", topk_ids, torch.int32),
                            ("topk_w", topk_w, torch.float32)):
            if t.dtype != dt or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous {dt} CUDA tensor (there is no CPU path)")
        _lib.check(lib.ramp_ep_dispatch(
            comm.handle, x.data_ptr(), topk_ids.data_ptr(), topk_w.data_ptr(), S, H, E, k, cap, WIRES[wire],
            send.data_ptr(), pos.data_ptr(), counts.data_ptr(), overflow.data_ptr(), recv.data_ptr(), _stream()))
    else:
        kernels = kernels or DeviceKernels()
        send, pos, counts, overflow = kernels.pack(x, topk_ids, topk_w, E, world, cap, wire)
        # equal blocks of cap rows: no split sizes to exchange first
        dist.all_to_all_single(recv, send, group=group)
    plan = EPPlan(world=world, cap=cap, wire=wire, pos=pos, counts=counts, overflow=overflow,
                  wire_bytes=world * cap * L.row_bytes)
    rx, rids, rw = row_fields(recv, H, k, wire)
    return plan, rx, rids, rw


def combine(plan: EPPlan, partial: torch.Tensor, group=None, comm: EPComm | None = None, kernels=None) -> torch.Tensor:
    """Return the per-(token, rank) partial outputs [P*cap, H] to their origin
    ranks and sum them (rank order, fp32) into [S, H]."""
    if plan.identity:
        return partial  # one row per token, already in token order
    back = torch.empty_like(partial)
    if comm is not None:
        lib = _lib.load()
        S = plan.pos.shape[0]
        H = partial.shape[1]
        out = torch.empty(S, H, dtype=partial.dtype, device=partial.device)
        _lib.check(lib.ramp_ep_combine(comm.handle, partial.data_ptr(), back.data_ptr(), plan.pos.data_ptr(), S, H,
                                       plan.cap, out.data_ptr(), _stream()))
        return out
    dist.all_to_all_single(back, partial.contiguous(), group=group)
    return (kernels or DeviceKernels()).reduce(back, plan.pos, plan.world, plan.cap)


def ep_moe_layer(x, topk_ids, topk_w, E: int, local_fn, group=None, wire: str = "bf16", cap: int | None = None,
                 comm: EPComm | None = None, kernels=None, exchange: str = "auto"):
    """dispatch -> local_fn(recv_x, recv_ids, recv_w) -> combine."""
    plan, rx, rids, rw = dispatch(x, topk_ids, topk_w, E, group, wire=wire, cap=cap, comm=comm, kernels=kernels,
                                  exchange=exchange)
    partial = local_fn(rx, rids, rw)
    return combine(plan, partial, group, comm=comm, kernels=kernels)


def make_local_megakernel(weights, table, workspace_cache: dict | None = None):
    """local_fn running the B200 megakernel on this rank's experts.
    `weights` is (w1_local, w2_local) bf16 or a quant.MxFp8Weights of the
    local experts (then `table` must be an FP8 pool's).  The FP8 megakernel
    also takes the MXFP8 wire's (e4m3, scales) rows as they arrived."""
    from .moe import Workspace, fused_moe, fused_moe_fp8

    cache = workspace_cache if workspace_cache is not None else {}
    fp8 = not isinstance(weights, tuple)
    if fp8:
        E_l, H, I = weights.shape
    else:
        w1_local, w2_local = weights
        E_l, two_i, H = w1_local.shape
        I = two_i // 2

    def run(rx, rids, rw):
        rows = (rx[0] if isinstance(rx, tuple) else rx).shape[0]
        if rows == 0:
            return torch.zeros(0, H, dtype=torch.bfloat16, device=rids.device)
        key = (rows, rids.shape[1])
        ws = cache.get(key)
        if ws is None:
            ws = cache[key] = Workspace(rows, H, I, E_l, rids.shape[1], device=rids.device)
        if fp8:
            return fused_moe_fp8(rx, weights, rw, rids, table, workspace=ws)
        if isinstance(rx, tuple):
            raise ValueError("the BF16 megakernel takes bf16 rows: use wire='bf16' (or an FP8 table)")
        return fused_moe(rx, w1_local, w2_local, rw, rids, table, workspace=ws)

    return run
