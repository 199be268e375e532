"""Expert parallelism for the expert-sharded configs (north_star (4)).

Rank r of a P-rank group owns experts [r*E/P, (r+1)*E/P).  One MoE layer:

  1. dispatch: every (token, expert) assignment is routed to the owner rank
     of its expert.  Assignments of one token bound for the same rank are
     merged into one row (the token is sent once per destination rank, with up
     to k (local expert, weight) pairs), so the wire carries unique
     (token, rank) pairs -- the "pre-reduce per (token, rank)" of SURVEY §8e.
  2. the owner runs the fused-MoE megakernel on its local experts: the
     received rows are its tokens, their local expert ids / weights its top-k
     (slots of other ranks' experts carry expert -1 and weight 0; the route
     kernel skips them, so they cost no work);
  3. combine: the per-(token, rank) partial outputs travel back and are
     summed into the origin tokens.

The exchanges are NCCL all-to-alls (torch.distributed.all_to_all_single over
NVLink 5 / NVSwitch); the split sizes need one small host read of the
per-destination counts (exchanged with an all-to-all of int64 counts first;
the (token, rank) pairs come from a [world, S] mask whose nonzeros are read
with the already-known size, so that read is the only device sync).
The local computation is pluggable (`local_fn`), which lets the gloo CPU tests
check the routing, packing and combine arithmetic against a dense oracle.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass
class EPPlan:
    """Send-side bookkeeping of one dispatch (kept for the combine)."""

    send_counts: list[int]
    recv_counts: list[int]
    order: torch.Tensor        # unique (token, rank) pairs sorted by destination rank
    pair_token: torch.Tensor   # origin token of every sent row (sorted order)
    wire_bytes: int = 0        # token-row payload this rank sent (dispatch direction)


def expert_owner(ids: torch.Tensor, E: int, world: int) -> torch.Tensor:
    per = E // world
    return torch.div(ids, per, rounding_mode="floor")


def dispatch(x: torch.Tensor, topk_ids: torch.Tensor, topk_w: torch.Tensor, E: int, group=None,
             wire: str = "bf16"):
    """Route token rows to expert owners.  Returns (plan, recv_x [R, H],
    recv_ids [R, k] local expert ids, recv_w [R, k]).

    wire = "fp8" sends the token rows as MXFP8 -- E4M3 plus
    one UE8M0 scale per 32 features, the operand format of the FP8 megakernel,
    H + H/32 bytes per row instead of 2H -- and the receiver expands them back
    exactly (E4M3 x 2^k is representable in bf16); the FP8 megakernel then
    re-derives the same per-32 scales in its gather.  The combine stays bf16."""
    if wire not in ("bf16", "fp8"):
        raise ValueError(f"wire must be bf16 or fp8, got {wire!r}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = E // world
    S, k = topk_ids.shape
    dev = x.device
    if world == 1:
        # One rank owns every expert: each token is one row and the exchanges
        # are identities -- no collectives and no host read, so the layer
        # stays asynchronous (the MXFP8 wire rounding is still applied, so
        # the numerics match the multi-rank path).
        pair_token = torch.arange(S, device=dev)
        recv_x = x
        if wire == "fp8":
            from .quant import mx_dequantize, mx_quantize

            recv_x = mx_dequantize(*mx_quantize(x)).to(x.dtype)
        plan = EPPlan(send_counts=[S], recv_counts=[S], order=pair_token, pair_token=pair_token, wire_bytes=0)
        return plan, recv_x, topk_ids.to(torch.int32), topk_w
    owner = expert_owner(topk_ids.long(), E, world)                     # [S, k]
    # unique (token, rank) pairs as a [world, S] mask: its row-major nonzeros
    # are ordered by destination rank then token (no sort, no device sync)
    mask = torch.zeros(world, S, dtype=torch.bool, device=dev)
    mask[owner, torch.arange(S, device=dev)[:, None].expand(S, k)] = True
    send_counts = mask.sum(1)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    counts = torch.cat([send_counts, recv_counts]).tolist()              # the one host read
    sc, rc = counts[:world], counts[world:]
    pairs = torch.nonzero_static(mask.reshape(-1), size=sum(sc)).squeeze(1)
    pair_rank = torch.div(pairs, S, rounding_mode="floor")
    pair_token = pairs % S
    # per sent row: the token's assignments that live on that rank (others -> weight 0)
    row_owner = owner[pair_token]                                        # [P, k]
    hit = row_owner == pair_rank[:, None]
    # slots of other ranks' experts carry -1: the route kernel skips them
    row_ids = torch.where(hit, topk_ids[pair_token].long() - pair_rank[:, None] * per, -1)
    row_w = torch.where(hit, topk_w[pair_token], torch.zeros((), dtype=topk_w.dtype, device=dev))
    send_x = x[pair_token].contiguous()
    R = sum(rc)
    H = x.shape[1]
    if wire == "fp8":
        from .quant import GROUP, mx_dequantize, mx_quantize

        q, sf = mx_quantize(send_x)
        recv_q = torch.empty(R, H, dtype=torch.uint8, device=dev)
        recv_sf = torch.empty(R, H // GROUP, dtype=torch.uint8, device=dev)
        dist.all_to_all_single(recv_q, q.view(torch.uint8).contiguous(), rc, sc, group=group)
        dist.all_to_all_single(recv_sf, sf.contiguous(), rc, sc, group=group)
        recv_x = mx_dequantize(recv_q.view(torch.float8_e4m3fn), recv_sf).to(x.dtype)
        wire_bytes = int(send_x.shape[0]) * (H + H // GROUP)
    else:
        recv_x = torch.empty(R, H, dtype=x.dtype, device=dev)
        dist.all_to_all_single(recv_x, send_x, rc, sc, group=group)
        wire_bytes = int(send_x.numel() * send_x.element_size())
    if topk_w.dtype == torch.float32:
        # local ids (int32) and weights (fp32 bits) travel as one [P, k, 2] int32 exchange
        meta = torch.stack([row_ids.to(torch.int32), row_w.contiguous().view(torch.int32)], dim=-1).contiguous()
        recv_meta = torch.empty(R, k, 2, dtype=torch.int32, device=dev)
        dist.all_to_all_single(recv_meta, meta, rc, sc, group=group)
        recv_ids = recv_meta[..., 0].contiguous()
        recv_w = recv_meta[..., 1].contiguous().view(torch.float32)
    else:
        recv_ids = torch.empty(R, k, dtype=torch.int32, device=dev)
        recv_w = torch.empty(R, k, dtype=topk_w.dtype, device=dev)
        dist.all_to_all_single(recv_ids, row_ids.to(torch.int32).contiguous(), rc, sc, group=group)
        dist.all_to_all_single(recv_w, row_w.contiguous(), rc, sc, group=group)
    plan = EPPlan(send_counts=sc, recv_counts=rc, order=pairs, pair_token=pair_token, wire_bytes=wire_bytes)
    return plan, recv_x, recv_ids, recv_w


def combine(plan: EPPlan, partial: torch.Tensor, S: int, group=None) -> torch.Tensor:
    """Return per-(token, rank) partial outputs to their origin and sum them."""
    if dist.get_world_size(group) == 1:
        return partial  # one row per token, already in token order
    back = torch.empty(sum(plan.send_counts), partial.shape[1], dtype=partial.dtype, device=partial.device)
    dist.all_to_all_single(back, partial.contiguous(), plan.send_counts, plan.recv_counts, group=group)
    out = torch.zeros(S, partial.shape[1], dtype=torch.float32, device=partial.device)
    out.index_add_(0, plan.pair_token, back.float())
    return out.to(partial.dtype)


def ep_moe_layer(x, topk_ids, topk_w, E: int, local_fn, group=None, wire: str = "bf16"):
    """dispatch -> local_fn(recv_x, recv_ids, recv_w) -> combine."""
    plan, rx, rids, rw = dispatch(x, topk_ids, topk_w, E, group, wire=wire)
    partial = local_fn(rx, rids, rw)
    return combine(plan, partial, x.shape[0], group)


def make_local_megakernel(weights, table, workspace_cache: dict | None = None):
    """local_fn running the B200 megakernel on this rank's experts.
    `weights` is (w1_local, w2_local) bf16 or a quant.MxFp8Weights of the
    local experts (then `table` must be an FP8 pool's)."""
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
        if rx.shape[0] == 0:
            return torch.zeros(0, rx.shape[1], dtype=rx.dtype, device=rx.device)
        key = (rx.shape[0], rids.shape[1])
        ws = cache.get(key)
        if ws is None:
            ws = cache[key] = Workspace(rx.shape[0], H, I, E_l, rids.shape[1], device=rx.device)
        if fp8:
            return fused_moe_fp8(rx.contiguous(), weights, rw.float().contiguous(), rids.contiguous(), table,
                                 workspace=ws)
        return fused_moe(rx.contiguous(), w1_local, w2_local, rw.float().contiguous(), rids.contiguous(), table,
                         workspace=ws)

    return run
