"""PyTorch host API of the fused-MoE hot path.

`fused_moe` is the drop-in for the kernel the reference simulates
(`simulate_pool_times`, ramp/oracle.py:197-254) fused with the dispatch call
in front of it (`select_config`, ramp/dispatch.py:89-122).  Tensors are torch
CUDA tensors; the heavy lifting is one C-ABI call into libramp_b200.so, which
launches three kernels (route, megakernel, finalize) on the current stream
with no host synchronisation.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


@dataclass
class DeviceTable:
    """Device-resident dispatch table (`ramp_table_t`): per-config integer
    fields and the four fitted floats (ramp/dispatch.py:57-86).  Arrays are
    kept alive by this object; `struct` is what the C ABI receives."""

    bm: np.ndarray
    ttn: np.ndarray
    stg: np.ndarray
    split_k: np.ndarray
    group_m: np.ndarray
    mode: np.ndarray | None
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    d: np.ndarray
    N: int
    kappa_ok: bool
    sm_count: int
    device: torch.device | str = "cuda"
    ntile: np.ndarray | None = None   # work tiles per M-tile (default ceil(N/ttn))
    omega_max: float = 0.0            # split-K gate threshold (<= 0: the reference's 0.2)
    lam: np.ndarray | None = None     # B4 L2-reuse factor per config (None: the reference model)
    kps: np.ndarray | None = None     # k-blocks per pipeline stage per config (None: 1)
    h3: np.ndarray | None = None      # split phase-3 H chunks per job per config (None: 1)
    id_map: np.ndarray | None = None  # table index -> pool id (a pruned table); None: identity
    step_cache: "DeviceStepCache | None" = None  # device StepCache (None: every call dispatches)
    _tensors: dict = field(default_factory=dict, repr=False)
    struct: _lib.RampTable | None = field(default=None, repr=False)

    def __post_init__(self) -> None:
        n = len(self.bm)
        if n == 0:
            raise ValueError("dispatch table over an empty pool")
        if self.mode is None:
            self.mode = np.zeros(n, dtype=np.int64)
        for name in ("ttn", "stg", "split_k", "group_m", "mode", "a", "b", "c", "d"):
            if len(getattr(self, name)) != n:
                raise ValueError(f"column {name} has length {len(getattr(self, name))}, expected {n}")
        ubm, ubm_index = np.unique(np.asarray(self.bm, dtype=np.int64), return_inverse=True)
        if len(ubm) > 128:
            raise ValueError("at most 128 distinct bm values are supported")
        i32 = dict(dtype=torch.int32, device=self.device)
        f64 = dict(dtype=torch.float64, device=self.device)
        t = self._tensors
        for name in ("bm", "ttn", "stg", "split_k", "group_m", "mode"):
            t[name] = torch.as_tensor(np.asarray(getattr(self, name), dtype=np.int32), **i32)
        t["ubm"] = torch.as_tensor(ubm.astype(np.int32), **i32)
        t["ubm_index"] = torch.as_tensor(ubm_index.astype(np.int32), **i32)
        for name in ("a", "b", "c", "d"):
            t[name] = torch.as_tensor(np.asarray(getattr(self, name), dtype=np.float64), **f64)
        if self.ntile is not None:
            if len(self.ntile) != n:
                raise ValueError("ntile must have one entry per config")
            t["ntile"] = torch.as_tensor(np.asarray(self.ntile, dtype=np.int32), **i32)
        s = _lib.RampTable()
        s.n_cfg = n
        s.n_ubm = len(ubm)
        s.N = int(self.N)
        s.kappa_ok = int(bool(self.kappa_ok))
        s.sm_count = int(self.sm_count)
        for name in ("bm", "ttn", "stg", "split_k", "group_m", "mode", "ubm", "ubm_index", "a", "b", "c", "d"):
            setattr(s, name, t[name].data_ptr())
        s.ntile = t["ntile"].data_ptr() if "ntile" in t else None
        s.omega_max = float(self.omega_max)
        if self.lam is not None:
            if len(self.lam) != n:
                raise ValueError("lam must have one entry per config")
            t["lam"] = torch.as_tensor(np.asarray(self.lam, dtype=np.float64), **f64)
        s.lam = t["lam"].data_ptr() if "lam" in t else None
        if self.kps is not None:
            kps = np.asarray(self.kps, dtype=np.int64)
            if len(kps) != n:
                raise ValueError("kps must have one entry per config")
            if not np.isin(kps, (1, 2, 4)).all():
                raise ValueError("kps values must be 1, 2 or 4")
            t["kps"] = torch.as_tensor(kps.astype(np.int32), **i32)
        s.kps = t["kps"].data_ptr() if "kps" in t else None
        if self.h3 is not None:
            h3 = np.asarray(self.h3, dtype=np.int64)
            if len(h3) != n:
                raise ValueError("h3 must have one entry per config")
            if not np.isin(h3, (1, 2, 4)).all():
                raise ValueError("h3 values must be 1, 2 or 4")
            t["h3"] = torch.as_tensor(h3.astype(np.int32), **i32)
        s.h3 = t["h3"].data_ptr() if "h3" in t else None
        s.step_cache = self.step_cache.buf.data_ptr() if self.step_cache is not None else None
        s.step_cache_cap = self.step_cache.capacity if self.step_cache is not None else 0
        self.struct = s

    def __len__(self) -> int:
        return len(self.bm)

    def pool_id(self, index: int) -> int:
        """Pool id of table entry `index` (what the device reports in sel)."""
        return int(index) if self.id_map is None else int(self.id_map[int(index)])

    def table_index(self, pool_id: int) -> int:
        """Table entry of a pool id (forced configs); -1 stays -1."""
        if pool_id < 0 or self.id_map is None:
            return int(pool_id)
        hit = np.flatnonzero(np.asarray(self.id_map) == int(pool_id))
        if len(hit) == 0:
            raise ValueError(f"config {pool_id} is not a candidate of this (pruned) table")
        return int(hit[0])

    @property
    def ref(self):
        return ctypes.byref(self.struct)

    def fp8_compatible(self) -> bool:
        """Every config runnable by the FP8 megakernel (split mode, ttn >= 256,
        ramp_config_smem_bytes_fp8_kps > 0)."""
        ok = getattr(self, "_fp8_ok", None)
        if ok is not None:
            return ok
        lib = _lib.load()
        kps = self.kps if self.kps is not None else np.ones(len(self.bm), dtype=np.int64)
        self._fp8_ok = all(int(m) == 1 and lib.ramp_config_smem_bytes_fp8_kps(int(bm), int(t), int(st), int(kp)) > 0
                           for bm, t, st, m, kp in zip(self.bm, self.ttn, self.stg, self.mode, kps))
        return self._fp8_ok


class DeviceStepCache:
    """Device-resident StepCache (ramp/dispatch.py:40-54): per step, M = the
    histogram total -> selected config.  The route kernel consults it before
    dispatching and clears it when the step changes; `advance()` starts a new
    step with a device-side increment, so it can live inside a captured CUDA
    graph (one advance per replayed step)."""

    def __init__(self, capacity: int = 64, device="cuda"):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = int(capacity)
        # {current step, cached step, n, (M, cfg) x capacity}; cached step -1: empty
        self.buf = torch.zeros(3 + 2 * self.capacity, dtype=torch.int32, device=device)
        self.buf[1] = -1

    def advance(self) -> None:
        self.buf[0:1].add_(1)

    def entries(self) -> dict[int, int]:
        """Host copy {M: cfg} of the current step's entries (diagnostics)."""
        h = self.buf.cpu().tolist()
        if h[1] != h[0]:
            return {}
        return {h[3 + 2 * q]: h[4 + 2 * q] for q in range(h[2])}


def workspace_bytes(S: int, H: int, I: int, E: int, top_k: int) -> int:
    return int(_lib.load().ramp_fused_moe_workspace_size(S, H, I, E, top_k))


class Workspace:
    """Reusable device workspace for `fused_moe`: route outputs, the fp32
    accumulator, expert-sorted tokens and split-mode activations.  Zeroed
    once at allocation.  One workspace serves every call whose shape fits:
    the library lays its regions out for the largest token count the buffer
    holds (so a smaller S reuses the same offsets), and re-zeroes it itself
    when the geometry (H, I, E, top_k) changes between calls."""

    CTRL_BAD_IDS = 4  # int32 word of the control block: set by a call whose ids left [-1, E)

    def __init__(self, S: int, H: int, I: int, E: int, top_k: int, device="cuda"):
        self.key = (S, H, I, E, top_k)
        n = workspace_bytes(S, H, I, E, top_k)
        self.buf = torch.zeros(max(n, 256), dtype=torch.uint8, device=device)
        self.sel = torch.zeros(4, dtype=torch.int32, device=device)

    def fits(self, S: int, H: int, I: int, E: int, top_k: int) -> bool:
        return self.buf.numel() >= workspace_bytes(S, H, I, E, top_k)

    def invalid_ids(self) -> bool:
        """True if the last call on this workspace saw a top-k id outside
        [0, E) other than -1 (those slots were skipped).  Reads one device
        word (synchronises the current stream)."""
        w = self.buf[4 * self.CTRL_BAD_IDS:4 * self.CTRL_BAD_IDS + 4].view(torch.int32)
        return bool(int(w.item()) != 0)


def _row_stride(name: str, t: torch.Tensor) -> int:
    """0 for a contiguous tensor; the row stride (elements) of a row-strided
    2-D view with a unit inner stride (e.g. one field of the expert-parallel
    wire's rows, ep.dispatch); anything else is rejected."""
    if t.is_contiguous():
        return 0
    if t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]:
        return int(t.stride(0))
    raise ValueError(f"{name} must be contiguous or a row-strided [rows, n] view with unit inner stride")


def _strided_call(lib, x, x_sf, w1, w1_sf, w2, w2_sf, topk_w, topk_ids, strides, S, H, I, E, k, table, forced_cfg,
                  out, workspace, phases):
    _lib.check(lib.ramp_fused_moe_strided(
        x.data_ptr(), None if x_sf is None else x_sf.data_ptr(), w1.data_ptr(),
        None if w1_sf is None else w1_sf.data_ptr(), w2.data_ptr(), None if w2_sf is None else w2_sf.data_ptr(),
        topk_w.data_ptr(), topk_ids.data_ptr(), ctypes.byref(strides), S, H, I, E, k, table.ref,
        table.table_index(int(forced_cfg)), out.data_ptr(), workspace.sel.data_ptr(), workspace.buf.data_ptr(),
        workspace.buf.numel(), int(phases), _stream()))


def _token_strides(hidden_states, x_sf, topk_weights, topk_ids):
    """ramp_row_strides_t of the per-token inputs, or None when all are dense."""
    xs = _row_stride("hidden_states", hidden_states) * hidden_states.element_size()
    sfs = 0 if x_sf is None else _row_stride("x_sf", x_sf)
    ws = _row_stride("topk_weights", topk_weights)
    ids = _row_stride("topk_ids", topk_ids)
    if not (xs or sfs or ws or ids):
        return None
    return _lib.RowStrides(xs, sfs, ids, ws)


def _raise_if_invalid_ids(ws: Workspace, E: int) -> None:
    # the reference's ExpertHistogram rejects out-of-range experts with a
    # ValueError (ramp/routing.py:45-50); the device flags them and skips them
    if ws.invalid_ids():
        raise ValueError(f"topk_ids hold expert ids outside [0, {E}) (other than -1, a non-local EP slot)")


def fused_moe(
    hidden_states: torch.Tensor,
    w1: torch.Tensor,
    w2: torch.Tensor,
    topk_weights: torch.Tensor,
    topk_ids: torch.Tensor,
    table: DeviceTable,
    forced_cfg: int = -1,
    out: torch.Tensor | None = None,
    workspace: Workspace | None = None,
    phases: int = 3,
    validate: bool = False,
) -> torch.Tensor:
    """Fused MoE layer forward, BF16:

        out[t] = sum_j w[t, j] * W2[e] (silu(W1[e, :I] x_t) * W1[e, I:] x_t),  e = ids[t, j]

    hidden_states [S, H] bf16; w1 [E, 2I, H] bf16 (gate rows first, vLLM
    layout); w2 [E, H, I] bf16; topk_weights [S, k] fp32; topk_ids [S, k]
    int32 (the per-token inputs may also be row-strided views, e.g. fields of
    the expert-parallel wire's rows).  `forced_cfg < 0` lets the on-device dispatcher choose the tile
    config from the live histogram; a config id forces it (static dispatch or
    the exhaustive sweep).  The selection record {cfg, n_post_pad, n_mtiles,
    n_eval} is left in `workspace.sel` (device int32[4]).  `phases` = 1 / 2
    runs only the route kernel / only the megakernel (ramp_fused_moe_bf16_ex).
    Ids outside [0, E) other than -1 are skipped on the device and flagged;
    `validate=True` checks the flag after the call and raises ValueError, as
    the reference's ExpertHistogram does (costs one stream synchronisation).
    """
    lib = _lib.load()
    S, H = hidden_states.shape
    E, two_i, H1 = w1.shape
    I = two_i // 2
    k = topk_ids.shape[1]
    if H1 != H or tuple(w2.shape) != (E, H, I):
        raise ValueError(f"shape mismatch: x {tuple(hidden_states.shape)}, w1 {tuple(w1.shape)}, w2 {tuple(w2.shape)}")
    for name, t, dt in (("hidden_states", hidden_states, torch.bfloat16), ("w1", w1, torch.bfloat16),
                        ("w2", w2, torch.bfloat16), ("topk_weights", topk_weights, torch.float32),
                        ("topk_ids", topk_ids, torch.int32)):
        if t.dtype != dt:
            raise ValueError(f"{name} must be {dt}, got {t.dtype}")
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    for name, t in (("w1", w1), ("w2", w2)):
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    strides = _token_strides(hidden_states, None, topk_weights, topk_ids)
    if tuple(topk_weights.shape) != (S, k):
        raise ValueError("topk_weights must be [S, top_k]")
    if out is None:
        out = torch.empty(S, H, dtype=torch.bfloat16, device=hidden_states.device)
    if workspace is None or not workspace.fits(S, H, I, E, k):
        workspace = Workspace(S, H, I, E, k, device=hidden_states.device)
    if strides is not None:
        _strided_call(lib, hidden_states, None, w1, None, w2, None, topk_weights, topk_ids, strides, S, H, I, E, k,
                      table, forced_cfg, out, workspace, phases)
        if validate and phases & 1:
            _raise_if_invalid_ids(workspace, E)
        return out
    _lib.check(
        lib.ramp_fused_moe_bf16_ex(
            hidden_states.data_ptr(), w1.data_ptr(), w2.data_ptr(), topk_weights.data_ptr(),
            topk_ids.data_ptr(), S, H, I, E, k, table.ref, table.table_index(int(forced_cfg)), out.data_ptr(),
            workspace.sel.data_ptr(), workspace.buf.data_ptr(), workspace.buf.numel(), int(phases), _stream(),
        )
    )
    if validate and phases & 1:
        _raise_if_invalid_ids(workspace, E)
    return out


def fused_moe_gating(
    hidden_states: torch.Tensor,
    w1: torch.Tensor,
    w2: torch.Tensor,
    gating_output: torch.Tensor,
    topk: int,
    renormalize: bool,
    table: DeviceTable,
    forced_cfg: int = -1,
    out: torch.Tensor | None = None,
    workspace: Workspace | None = None,
    return_topk: bool = False,
):
    """The BF16 layer from the router's logits (router fusion),
    vLLM's `fused_moe(hidden_states, w1, w2, gating_output, topk, renormalize)`
    contract: per token the softmax top-k of `gating_output` [S, E] (fp32 or
    bf16) -- highest probabilities first, ties to the lower expert id; weights
    are the fp32 softmax probabilities, renormalised over the k picks when
    `renormalize` -- computed inside the route kernel, which then dispatches,
    aligns and launches the megakernel as `fused_moe` does.  With
    `return_topk` the (topk_weights, topk_ids) it chose are returned too."""
    lib = _lib.load()
    S, H = hidden_states.shape
    E, two_i, H1 = w1.shape
    I = two_i // 2
    k = int(topk)
    if H1 != H or tuple(w2.shape) != (E, H, I):
        raise ValueError(f"shape mismatch: x {tuple(hidden_states.shape)}, w1 {tuple(w1.shape)}, w2 {tuple(w2.shape)}")
    if tuple(gating_output.shape) != (S, E):
        raise ValueError(f"gating_output must be [S, E] = {(S, E)}, got {tuple(gating_output.shape)}")
    if gating_output.dtype not in (torch.float32, torch.bfloat16):
        raise ValueError(f"gating_output must be float32 or bfloat16, got {gating_output.dtype}")
    for name, t, dt in (("hidden_states", hidden_states, torch.bfloat16), ("w1", w1, torch.bfloat16),
                        ("w2", w2, torch.bfloat16), ("gating_output", gating_output, gating_output.dtype)):
        if t.dtype != dt:
            raise ValueError(f"{name} must be {dt}, got {t.dtype}")
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    dev = hidden_states.device
    topk_w = torch.empty(S, k, dtype=torch.float32, device=dev)
    topk_ids = torch.empty(S, k, dtype=torch.int32, device=dev)
    if out is None:
        out = torch.empty(S, H, dtype=torch.bfloat16, device=dev)
    if workspace is None or not workspace.fits(S, H, I, E, k):
        workspace = Workspace(S, H, I, E, k, device=dev)
    _lib.check(
        lib.ramp_fused_moe_gating_bf16(
            hidden_states.data_ptr(), w1.data_ptr(), w2.data_ptr(), gating_output.data_ptr(),
            int(gating_output.dtype == torch.bfloat16), int(bool(renormalize)), topk_w.data_ptr(),
            topk_ids.data_ptr(), S, H, I, E, k, table.ref, table.table_index(int(forced_cfg)), out.data_ptr(),
            workspace.sel.data_ptr(), workspace.buf.data_ptr(), workspace.buf.numel(), _stream(),
        )
    )
    return (out, topk_w, topk_ids) if return_topk else out


def fused_moe_fp8(
    hidden_states: torch.Tensor,
    weights,
    topk_weights: torch.Tensor,
    topk_ids: torch.Tensor,
    table: DeviceTable,
    forced_cfg: int = -1,
    out: torch.Tensor | None = None,
    workspace: Workspace | None = None,
    phases: int = 3,
    validate: bool = False,
) -> torch.Tensor:
    """Fused MoE layer forward, block-scaled FP8 (W8A8 MXFP8).

    `weights` is a quant.MxFp8Weights (E4M3 experts + UE8M0 scale atoms, from
    prepare_mxfp8_weights or prepare_block128_weights).  hidden_states stay
    bf16 [S, H]; the megakernel quantises each gathered token row (one scale
    per 32 features) -- or hidden_states is a pair (x_q [S, H] e4m3 / uint8,
    x_sf [S, H/32] uint8 UE8M0) of tokens already in that format (e.g. off the
    MXFP8 expert-parallel wire), which phase 0 then only moves -- and the
    SwiGLU activation the same way, multiplies with
    kind::mxf8f6f4.block_scale MMAs and accumulates in fp32; the output is
    bf16.  The table must be an FP8 pool (enumerate_b200_configs(...,
    dtype="fp8")); `forced_cfg` / `phases` / `validate` as in `fused_moe`.
    """
    lib = _lib.load()
    x_sf = None
    if isinstance(hidden_states, (tuple, list)):
        hidden_states, x_sf = hidden_states
        if hidden_states.dtype == torch.float8_e4m3fn:
            hidden_states = hidden_states.view(torch.uint8)
    S, H = hidden_states.shape
    E, H1, I = weights.shape
    k = topk_ids.shape[1]
    if H1 != H:
        raise ValueError(f"shape mismatch: x {tuple(hidden_states.shape)}, experts d_model {H1}")
    extra = ()
    if x_sf is not None:
        if tuple(x_sf.shape) != (S, H // 32):
            raise ValueError("x_sf must be [S, H/32] (one UE8M0 scale per 32 features)")
        extra = (("x_sf", x_sf, torch.uint8),)
    for name, t, dt in (("hidden_states", hidden_states, torch.uint8 if x_sf is not None else torch.bfloat16),
                        *extra,
                        ("w1_q", weights.w1_q, torch.float8_e4m3fn), ("w2_q", weights.w2_q, torch.float8_e4m3fn),
                        ("w1_sf", weights.w1_sf, torch.uint8), ("w2_sf", weights.w2_sf, torch.uint8),
                        ("topk_weights", topk_weights, torch.float32), ("topk_ids", topk_ids, torch.int32)):
        if t.dtype != dt:
            raise ValueError(f"{name} must be {dt}, got {t.dtype}")
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    for name, t in (("w1_q", weights.w1_q), ("w2_q", weights.w2_q), ("w1_sf", weights.w1_sf),
                    ("w2_sf", weights.w2_sf)):
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    strides = _token_strides(hidden_states, x_sf, topk_weights, topk_ids)
    if tuple(weights.w1_sf.shape) != (E * 2 * I // 128, H // 128, 512) or \
            tuple(weights.w2_sf.shape) != (E * H // 128, I // 128, 512):
        raise ValueError("scale atoms must be tiled [rows/128, K/128, 512] (quant.tile_scales)")
    if tuple(topk_weights.shape) != (S, k):
        raise ValueError("topk_weights must be [S, top_k]")
    if not table.fp8_compatible():
        raise ValueError("table holds configs the FP8 megakernel cannot run (use an FP8 pool)")
    if out is None:
        out = torch.empty(S, H, dtype=torch.bfloat16, device=hidden_states.device)
    if workspace is None or not workspace.fits(S, H, I, E, k):
        workspace = Workspace(S, H, I, E, k, device=hidden_states.device)
    tail = (weights.w1_q.data_ptr(), weights.w1_sf.data_ptr(), weights.w2_q.data_ptr(),
            weights.w2_sf.data_ptr(), topk_weights.data_ptr(), topk_ids.data_ptr(), S, H, I, E, k, table.ref,
            table.table_index(int(forced_cfg)), out.data_ptr(), workspace.sel.data_ptr(), workspace.buf.data_ptr(),
            workspace.buf.numel(), int(phases), _stream())
    if strides is not None:
        _strided_call(lib, hidden_states, x_sf, weights.w1_q, weights.w1_sf, weights.w2_q, weights.w2_sf,
                      topk_weights, topk_ids, strides, S, H, I, E, k, table, forced_cfg, out, workspace, phases)
    elif x_sf is None:
        _lib.check(lib.ramp_fused_moe_fp8(hidden_states.data_ptr(), *tail))
    else:
        _lib.check(lib.ramp_fused_moe_fp8_prequant(hidden_states.data_ptr(), x_sf.data_ptr(), *tail))
    if validate and phases & 1:
        _raise_if_invalid_ids(workspace, E)
    return out


def moe_align_block_size(topk_ids: torch.Tensor, num_experts: int, block_size: int):
    """Histogram + alignment on the GPU (north_star (1)).

    Returns (sorted_token_ids, expert_ids, num_tokens_post_padded, hist), the
    vLLM names: sorted ids are flat assignment indices (padding value =
    topk_ids.numel()), expert_ids the expert of every block_size-row tile.
    Buffers are sized to the worst case; only the first
    num_tokens_post_padded entries (resp. / block_size) are meaningful."""
    lib = _lib.load()
    if topk_ids.dtype != torch.int32 or not topk_ids.is_cuda:
        raise ValueError("topk_ids must be an int32 CUDA tensor")
    ids = topk_ids.contiguous().view(-1)
    n = ids.numel()
    cap = int(lib.ramp_align_capacity(n, num_experts, block_size))
    dev = ids.device
    sorted_ids = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    expert_ids = torch.empty(max(cap // block_size, 1), dtype=torch.int32, device=dev)
    npp = torch.empty(1, dtype=torch.int32, device=dev)
    hist = torch.empty(num_experts, dtype=torch.int32, device=dev)
    _lib.check(
        lib.ramp_moe_align(ids.data_ptr(), n, num_experts, block_size, hist.data_ptr(),
                           sorted_ids.data_ptr(), expert_ids.data_ptr(), npp.data_ptr(), _stream())
    )
    return sorted_ids, expert_ids, npp, hist


def dispatch_select(hist: torch.Tensor, table: DeviceTable, want_grids: bool = False,
                    want_pred: bool = False):
    """On-device dispatcher over a device histogram (north_star (3)).

    Returns device tensors (cfg[1], n_eval[1], grids or None, pred or None);
    nothing is copied to the host."""
    lib = _lib.load()
    if hist.dtype != torch.int32 or not hist.is_cuda:
        raise ValueError("hist must be an int32 CUDA tensor")
    dev = hist.device
    cfg = torch.empty(1, dtype=torch.int32, device=dev)
    n_eval = torch.empty(1, dtype=torch.int32, device=dev)
    grids = torch.empty(len(table), dtype=torch.int64, device=dev) if want_grids else None
    pred = torch.empty(len(table), dtype=torch.float64, device=dev) if want_pred else None
    _lib.check(
        lib.ramp_dispatch_select(hist.contiguous().data_ptr(), hist.numel(), table.ref, cfg.data_ptr(),
                                 n_eval.data_ptr(), _ptr(grids), _ptr(pred), _stream())
    )
    return cfg, n_eval, grids, pred


def flops(S: int, top_k: int, H: int, I: int) -> int:
    """Algorithmic FLOPs of one layer call: 6*S*k*H*I."""
    return 6 * S * top_k * H * I


def algorithmic_bytes(active_experts: int, S: int, top_k: int, H: int, I: int, w_bytes: int = 2,
                      x_bytes: int = 2, out_bytes: int = 2) -> int:
    """Bytes a perfect kernel must move: active experts' weights once, the
    activations in and out once, ids+weights."""
    return active_experts * 3 * H * I * w_bytes + S * H * (x_bytes + out_bytes) + 8 * S * top_k
