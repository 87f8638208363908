"""Tensor-level API over the C-ABI (the form the hot loop uses).

Every function takes CUDA tensors, allocates its outputs with torch on the
same device, and launches the sm_100a kernels on torch's current stream.
Per-token Python objects cost 10-80 us each in the reference,
so the reference-compatible object API (model.py, substitution.py, ...)
is a thin adapter over these functions.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _native as N
from .errors import InputError

KIND_KEPT, KIND_SUBSTITUTED, KIND_ONDEMAND, KIND_DROPPED = 0, 1, 2, 3
FALLBACK_PREFETCH, FALLBACK_DROP = 0, 1
METHOD_BUDDY, METHOD_ORIGINAL, METHOD_IDENTITY = 0, 1, 2
ACT_TANH, ACT_SWIGLU = 0, 1
ROW_ALIGN = 16


def _p(t):
    return None if t is None else t.data_ptr()


def _s():
    return torch.cuda.current_stream().cuda_stream


def _cuda(t, name, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InputError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise InputError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise InputError(f"{name} must be contiguous")
    return t


@dataclass
class RouteTensors:
    logits: torch.Tensor   # [B,E] f32 (or f64 on the logits-boundary path)
    topk: torch.Tensor     # [B,k] i32
    probs: torch.Tensor    # [B,k] f32
    tae: torch.Tensor      # [B]   f64
    margin: torch.Tensor   # [B]   f64
    allowed: torch.Tensor  # [B]   u8
    probs64: torch.Tensor | None = None


def gate_topk(x, wg, bias, k: int, temperature: float = 1.0, tau: float = -1.0, gamma: float | None = None):
    """K1: fused fp32 router (model.route_batch + gating.tae/margin/token_gate)."""
    _cuda(x, "x", torch.float32)
    _cuda(wg, "wg", torch.float32)
    B, d = x.shape
    E = wg.shape[0]
    if bias is not None:
        _cuda(bias, "bias", torch.float32)
    dev = x.device
    out = RouteTensors(
        logits=torch.empty(B, E, device=dev, dtype=torch.float32),
        topk=torch.empty(B, k, device=dev, dtype=torch.int32),
        probs=torch.empty(B, k, device=dev, dtype=torch.float32),
        tae=torch.empty(B, device=dev, dtype=torch.float64),
        margin=torch.empty(B, device=dev, dtype=torch.float64),
        allowed=torch.empty(B, device=dev, dtype=torch.uint8))
    N.call("bm_gate_topk", _p(x), _p(wg), _p(bias), B, E, d, k, float(temperature), float(tau),
           -1.0 if gamma is None else float(gamma), _p(out.logits), _p(out.topk), _p(out.probs), _p(out.tae),
           _p(out.margin), _p(out.allowed), _s())
    return out


def select_topk_f64(logits, k: int, temperature: float = 1.0, tau: float = -1.0, gamma: float | None = None):
    """Selection + gates from given float64 logits (the parity boundary)."""
    _cuda(logits, "logits", torch.float64)
    B, E = logits.shape
    dev = logits.device
    out = RouteTensors(
        logits=logits,
        topk=torch.empty(B, k, device=dev, dtype=torch.int32),
        probs=torch.empty(B, k, device=dev, dtype=torch.float32),
        tae=torch.empty(B, device=dev, dtype=torch.float64),
        margin=torch.empty(B, device=dev, dtype=torch.float64),
        allowed=torch.empty(B, device=dev, dtype=torch.uint8),
        probs64=torch.empty(B, k, device=dev, dtype=torch.float64))
    N.call("bm_select_topk_f64", _p(logits), B, E, k, float(temperature), float(tau),
           -1.0 if gamma is None else float(gamma), _p(out.topk), _p(out.probs), _p(out.probs64), _p(out.tae),
           _p(out.margin), _p(out.allowed), _s())
    return out


@dataclass
class DeviceTable:
    """Dense buddy table in HBM (buddies.BuddyTable as SoA)."""
    ids: torch.Tensor      # [E,K] i32, -1 padded
    weights: torch.Tensor  # [E,K] f64
    lens: torch.Tensor     # [E]   i32

    @property
    def num_experts(self):
        return self.ids.shape[0]

    @property
    def k_max(self):
        return self.ids.shape[1]


def bitmap_from_mask(mask, device=None) -> torch.Tensor:
    """Residency mask (bool[E]) -> packed u32 bitmap tensor (bit e of word e//32)."""
    import numpy as np
    m = np.asarray(mask, dtype=bool)
    E = m.size
    words = np.zeros((E + 31) // 32, dtype=np.uint32)
    for e in np.flatnonzero(m):
        words[e >> 5] |= np.uint32(1) << np.uint32(e & 31)
    t = torch.from_numpy(words.view(np.int32).copy())
    return t.to(device) if device is not None else t


@dataclass
class PlanTensors:
    executed: torch.Tensor  # [B,k] i32
    kind: torch.Tensor      # [B,k] u8
    used: torch.Tensor      # [B]   i32
    delta: torch.Tensor     # [1]   f64
    batch_allowed: torch.Tensor  # [1] u8


def buddy_remap(topk, token_allowed, bitmap, table: DeviceTable | None, *, H: int = 16, rho=None,
                fallback: int = FALLBACK_PREFETCH, method: int = METHOD_BUDDY, beta: float = 1.0,
                eta: float = 0.0, kappa: float = 0.0, use_local_logit: bool = True, partition_of=None,
                hop: float = 1.0, logits=None, num_experts: int | None = None) -> PlanTensors:
    """K2: warp-ballot buddy remap (substitution.substitute_batch / ondemand_plan / identity_plan)."""
    _cuda(topk, "topk", torch.int32)
    B, k = topk.shape
    E = table.num_experts if table is not None else int(num_experts)
    dev = topk.device
    out = PlanTensors(torch.empty(B, k, device=dev, dtype=torch.int32),
                      torch.empty(B, k, device=dev, dtype=torch.uint8),
                      torch.empty(B, device=dev, dtype=torch.int32),
                      torch.empty(1, device=dev, dtype=torch.float64),
                      torch.empty(1, device=dev, dtype=torch.uint8))
    lg, lg64 = None, 0
    if logits is not None:
        lg, lg64 = logits, int(logits.dtype == torch.float64)
    N.call("bm_buddy_remap", _p(topk), _p(token_allowed), _p(lg), lg64, B, k, E, _p(bitmap),
           _p(table.ids) if table is not None else None, _p(table.weights) if table is not None else None,
           _p(table.lens) if table is not None else None, table.k_max if table is not None else 1, int(H),
           -1 if rho is None else int(rho), int(fallback), int(method), float(beta), float(eta), float(kappa),
           int(bool(use_local_logit)), _p(partition_of), float(hop), _p(out.executed), _p(out.kind),
           _p(out.used), _p(out.delta), _p(out.batch_allowed), _s())
    return out


@dataclass
class Permutation:
    count: torch.Tensor     # [E]   i32 real rows per expert
    offset: torch.Tensor    # [E+1] i32 padded segment starts
    row_token: torch.Tensor  # [r_max] i32
    slot_row: torch.Tensor  # [B*k] i32
    r_max: int


def permute(executed, kind, num_experts: int, align: int = ROW_ALIGN) -> Permutation:
    """K3: stable warp-scan grouping of executed slots by expert."""
    B, k = executed.shape
    r_max = int(N.lib().bm_permute_rows_max(B, k, num_experts, align))
    r_max = (r_max + align - 1) // align * align
    dev = executed.device
    p = Permutation(torch.empty(num_experts, device=dev, dtype=torch.int32),
                    torch.empty(num_experts + 1, device=dev, dtype=torch.int32),
                    torch.full((max(r_max, 1),), -1, device=dev, dtype=torch.int32),
                    torch.empty(B * k, device=dev, dtype=torch.int32), r_max)
    ns = int(N.lib().bm_permute_scratch_elems(B, k, num_experts))
    scratch = torch.empty(max(ns, 1), device=dev, dtype=torch.int32)
    N.call("bm_permute_ws", _p(executed), _p(kind), B, k, num_experts, align, _p(p.count), _p(p.offset),
           _p(p.row_token), _p(p.slot_row), _p(scratch), ns, _s())
    return p


def append_shared(executed, kind, probs, num_experts: int, num_shared: int):
    """Plan [B,k] -> [B,k+S] with shared experts E..E+S-1 (kept, weight 1)."""
    B, k = executed.shape
    kt = k + num_shared
    dev = executed.device
    ex = torch.empty(B, kt, device=dev, dtype=torch.int32)
    kd = torch.empty(B, kt, device=dev, dtype=torch.uint8)
    pr = torch.empty(B, kt, device=dev, dtype=torch.float32)
    N.call("bm_append_shared", _p(executed), _p(kind), _p(probs), B, k, num_experts, num_shared, _p(ex), _p(kd),
           _p(pr), _s())
    return ex, kd, pr


def gather_rows(x, perm: Permutation, layout: int = 0):
    """Permuted activations: layout 0 row-major [r_max,d] in x's dtype (fp32, or
    f64 for the reference-precision path); layout 1 bf16 SW128 planes."""
    B, d = x.shape
    E = perm.count.shape[0]
    if layout == 0 and x.dtype == torch.float64:
        _cuda(x, "x", torch.float64)
        out = torch.empty(perm.r_max, d, device=x.device, dtype=torch.float64)
        N.call("bm_gather_rows_f64", _p(x), B, d, _p(perm.row_token), _p(perm.offset), E, perm.r_max, _p(out), _s())
        return out
    _cuda(x, "x", torch.float32)
    if layout == 0:
        out = torch.empty(perm.r_max, d, device=x.device, dtype=torch.float32)
    else:
        out = torch.zeros(d // 64, perm.r_max, 64, device=x.device, dtype=torch.bfloat16)
    N.call("bm_gather_rows", _p(x), B, d, _p(perm.row_token), _p(perm.offset), E, perm.r_max, layout, _p(out), _s())
    return out


def combine(y_perm, perm: Permutation, probs, kind, h_in=None, residual_scale: float = 0.5, out=None):
    """K5: gate-weighted combine (+ layer_update when h_in is given); fp32, or
    f64 when y_perm is float64 (then probs / h_in / out are float64 too)."""
    B, k = probs.shape
    d = y_perm.shape[-1]
    f64 = y_perm.dtype == torch.float64
    dt = torch.float64 if f64 else torch.float32
    for t, nm in ((y_perm, "y_perm"), (probs, "probs")) + (((h_in, "h_in"),) if h_in is not None else ()):
        _cuda(t, nm, dt)
    if out is None:
        out = torch.empty(B, d, device=y_perm.device, dtype=dt)
    N.call("bm_combine_f64" if f64 else "bm_combine", _p(y_perm), _p(perm.slot_row), _p(probs), _p(kind), B, k, d,
           _p(h_in), float(residual_scale), _p(out), _s())
    return out


def expert_ffn_f32(x_perm, perm: Permutation, w_arena, buf_of_expert, d: int, f: int, act: int):
    """SIMT grouped FFN over an arena of expert buffers: fp32 (parity mode), or
    f64 (the reference's precision) when x_perm and w_arena are float64."""
    E = perm.count.shape[0]
    dt = torch.float64 if x_perm.dtype == torch.float64 else torch.float32
    _cuda(x_perm, "x_perm", dt)
    _cuda(w_arena, "w_arena", dt)
    h = torch.empty(perm.r_max, f, device=x_perm.device, dtype=dt)
    y = torch.empty(perm.r_max, d, device=x_perm.device, dtype=dt)
    buf_elems = w_arena.shape[1] if w_arena.dim() == 2 else w_arena[0].numel()
    N.call("bm_expert_ffn_f64" if dt == torch.float64 else "bm_expert_ffn_f32", _p(x_perm), _p(perm.count),
           _p(perm.offset), E, d, f, act, _p(w_arena), buf_elems, _p(buf_of_expert), perm.r_max, _p(h), _p(y), _s())
    return y


def pack_expert_bf16(w1, w3, w2, act: int, out=None):
    """Row-major bf16 expert matrices -> one UMMA-tiled buffer (bmoe.h layout).
    SwiGLU: w1, w3 [f,d], w2 [d,f]. Tanh: w1 = Win^T [f,d], w2 = Wout^T [d,f], w3 None."""
    f, d = w1.shape
    n = (3 if act == ACT_SWIGLU else 2) * d * f
    if out is None:
        out = torch.empty(n, device=w1.device, dtype=torch.bfloat16)
    for t, nm in ((w1, "w1"), (w2, "w2")) + (((w3, "w3"),) if act == ACT_SWIGLU else ()):
        _cuda(t, nm, torch.bfloat16)
    N.call("bm_pack_expert_bf16", _p(w1), _p(w3), _p(w2), d, f, act, _p(out), _s())
    return out


def pack_arena_bf16(arena_rowmajor, d: int, f: int, act: int):
    """[n_bufs, buf_elems] row-major arena -> UMMA-tiled arena (same shape)."""
    out = torch.empty_like(arena_rowmajor)
    for b in range(arena_rowmajor.shape[0]):
        row = arena_rowmajor[b]
        if act == ACT_SWIGLU:
            pack_expert_bf16(row[: f * d].view(f, d), row[f * d: 2 * f * d].view(f, d), row[2 * f * d:].view(d, f),
                             act, out[b])
        else:
            pack_expert_bf16(row[: f * d].view(f, d), None, row[f * d:].view(d, f), act, out[b])
    return out


class FfnWorkspace:
    """Reusable workspace for the bf16 tcgen05 grouped FFN."""

    def __init__(self, E, d, f, r_max, n_tile=64, device="cuda"):
        self.E, self.d, self.f, self.r_max, self.n_tile = E, d, f, r_max, n_tile
        nbytes = int(N.lib().bm_expert_ffn_bf16_workspace(E, d, f, r_max, n_tile))
        self.buf = torch.zeros(nbytes, device=device, dtype=torch.uint8)  # counters start at zero
        self.nbytes = nbytes


def expert_ffn_bf16(x_perm_sw, perm: Permutation, w_arena, buf_of_expert, d: int, f: int, act: int,
                    ws: FfnWorkspace, y_perm=None):
    """bf16 tcgen05/TMEM/TMA grouped FFN (swap-AB, stream-K, fused SwiGLU/tanh)."""
    E = perm.count.shape[0]
    _cuda(x_perm_sw, "x_perm", torch.bfloat16)
    _cuda(w_arena, "w_arena", torch.bfloat16)
    if y_perm is None:
        y_perm = torch.empty(perm.r_max, d, device=x_perm_sw.device, dtype=torch.float32)
    n_bufs = w_arena.shape[0]
    N.call("bm_expert_ffn_bf16", _p(x_perm_sw), _p(perm.count), _p(perm.offset), E, d, f, act, _p(w_arena),
           n_bufs, _p(buf_of_expert), perm.r_max, ws.n_tile, _p(ws.buf), ws.nbytes, _p(y_perm), _s())
    return y_perm


def expert_ffn_bf16_combine(x_perm_sw, perm: Permutation, w_arena, buf_of_expert, d: int, f: int, act: int,
                            ws: FfnWorkspace, probs, kind, h, residual_scale: float = 0.5, y_perm=None):
    """K4 + K5: the bf16 grouped FFN, then the gate-weighted combine and
    layer_update in place on h [B][d] fp32 (model.py:334-347). At decode
    widths one launch does both (bit-identical to expert_ffn_bf16 + combine)."""
    E = perm.count.shape[0]
    B, k = probs.shape
    _cuda(x_perm_sw, "x_perm", torch.bfloat16)
    _cuda(w_arena, "w_arena", torch.bfloat16)
    _cuda(probs, "probs", torch.float32)
    _cuda(h, "h", torch.float32)
    if y_perm is None:
        y_perm = torch.empty(perm.r_max, d, device=x_perm_sw.device, dtype=torch.float32)
    N.call("bm_expert_ffn_bf16_combine", _p(x_perm_sw), _p(perm.count), _p(perm.offset), E, d, f, act, _p(w_arena),
           w_arena.shape[0], _p(buf_of_expert), perm.r_max, ws.n_tile, _p(ws.buf), ws.nbytes, _p(y_perm),
           _p(perm.slot_row), _p(probs), _p(kind), B, k, _p(h), float(residual_scale), _s())
    return h


def coact_count(topk, num_experts: int, counts=None, pairs=None, check: bool = True):
    """K6: accumulate binary co-activation counts (u64, stored in int64 tensors).

    Rows with an out-of-range or repeated id are not counted; with ``check``
    (one readback of a device counter) they raise InputError like observe()
    (profiler.py:76-80)."""
    _cuda(topk, "topk", torch.int32)
    Nn, k = topk.shape
    dev = topk.device
    if counts is None:
        counts = torch.zeros(num_experts, device=dev, dtype=torch.int64)
    if pairs is None:
        pairs = torch.zeros(num_experts, num_experts, device=dev, dtype=torch.int64)
    bad = torch.zeros(1, device=dev, dtype=torch.int32)
    N.call("bm_coact_count", _p(topk), Nn, k, num_experts, _p(counts), _p(pairs), _p(bad), _s())
    if check and Nn:
        nbad = int(bad.item())
        if nbad:
            raise InputError(f"{nbad} routing rows with duplicate or out-of-range expert ids were not counted")
    return counts, pairs


def coact_weighted(topk, probs, num_experts: int, w: float = 1.0, pw=None):
    Nn, k = topk.shape
    if pw is None:
        pw = torch.zeros(num_experts, num_experts, device=topk.device, dtype=torch.float64)
    N.call("bm_coact_weighted", _p(topk), _p(probs), Nn, k, num_experts, float(w), _p(pw), _s())
    return pw


def counts_to_f64(main, warm=None, w_warm: float = 0.0):
    out = torch.empty(main.shape, device=main.device, dtype=torch.float64)
    N.call("bm_counts_to_f64", _p(warm), _p(main), main.numel(), float(w_warm), _p(out), _s())
    return out


def buddy_rank(pair_matrix64, eps: float, alpha: float, k_max: int) -> DeviceTable:
    """K7: bit-exact buddy table from an f64 pair matrix."""
    _cuda(pair_matrix64, "pair_matrix", torch.float64)
    E = pair_matrix64.shape[0]
    dev = pair_matrix64.device
    t = DeviceTable(torch.empty(E, k_max, device=dev, dtype=torch.int32),
                    torch.empty(E, k_max, device=dev, dtype=torch.float64),
                    torch.empty(E, device=dev, dtype=torch.int32))
    N.call("bm_buddy_rank", _p(pair_matrix64), E, float(eps), float(alpha), int(k_max), _p(t.ids),
           _p(t.weights), _p(t.lens), _s())
    return t


def synth_bf16(lut, base: int, out) -> torch.Tensor:
    """Fill the bf16 tensor ``out`` with synthetic weights (bm_synth_bf16):
    lut = 65,536 bf16 quantiles (device, int16 or bfloat16 view), base = the
    matrix key of synth.matrix_key."""
    _cuda(lut, "lut")
    _cuda(out, "out", torch.bfloat16)
    if lut.numel() != 65536:
        raise InputError("synth lut must hold 65536 entries")
    N.call("bm_synth_bf16", _p(lut), int(base), out.numel(), _p(out), _s())
    return out


def sm_count() -> int:
    return int(N.lib().bm_device_sm_count())


# ------------------------------------------------------------------ fetch codec
XFER_CHUNK = 2048


def xfer_encode(src) -> torch.Tensor:
    """Lossless exponent coding of a bf16 tensor (numel a multiple of 2048)
    into a device blob (uint8), the expert-transfer format (bm_xfer_encode)."""
    _cuda(src, "src", torch.bfloat16)
    n = src.numel()
    bound = int(N.lib().bm_xfer_blob_bound(n))
    if bound < 0:
        raise InputError(f"xfer_encode: numel {n} must be a positive multiple of {XFER_CHUNK}")
    blob = torch.empty(bound + 256, dtype=torch.uint8, device=src.device)
    off = (-blob.data_ptr()) % 256
    out = blob[off:off + bound]
    nb = N.C.c_int64()
    N.call("bm_xfer_encode", src.data_ptr(), n, out.data_ptr(), bound, N.C.byref(nb), _s())
    return out[: nb.value]


def xfer_decode(blob, n_values: int, out=None) -> torch.Tensor:
    """Decode a blob made by xfer_encode back into n_values bf16 (bit-exact)."""
    _cuda(blob, "blob", torch.uint8)
    if blob.data_ptr() % 256:
        raise InputError("xfer_decode: blob must be 256-byte aligned")
    out = torch.empty(n_values, dtype=torch.bfloat16, device=blob.device) if out is None else out
    N.call("bm_xfer_decode", blob.data_ptr(), out.data_ptr(), n_values, _s())
    return out
