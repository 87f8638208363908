"""MoE substrate and layer forward — the reference ``model`` API
(model.py:1-382) with routing, forward and layer_update on the GPU.

``route_batch`` runs K1 (fused fp32 gate + top-k); ``forward_batch`` runs
K3 permute -> K4 grouped FFN (the reference's tanh expert) -> K5 combine;
``layer_update`` is K5's epilogue. Inputs/outputs stay numpy float64 like the
reference, and so does the arithmetic of this API's forward: the f64 SIMT
variants of K4/K5 (the engine's fp32 parity path and bf16 tensor-core path
are the throughput forms of the same kernels).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops, substrate
from .errors import InputError, InternalError
from .substrate import ModelSpec, readout_head, token_stream  # noqa: F401  (re-exported API)

_RESIDUAL_SCALE = 0.5


def _dev():
    if not torch.cuda.is_available():
        raise InternalError("the B200 path needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class Expert:
    """One expert FFN: y = tanh(x @ w_in) @ w_out (model.py:85-99)."""
    layer: int
    id: int
    w_in: np.ndarray
    w_out: np.ndarray

    @property
    def size_bytes(self) -> int:
        return self.w_in.nbytes + self.w_out.nbytes

    def __call__(self, x: np.ndarray) -> np.ndarray:
        # single-expert convenience: route through the grouped FFN with one slot
        one_d = np.asarray(x).ndim == 1
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        B = x.shape[0]
        E, d, f = 1, self.w_in.shape[0], self.w_in.shape[1]
        arena = np.concatenate([self.w_in.T.reshape(1, -1), self.w_out.T.reshape(1, -1)], axis=1)
        y = _grouped_forward(x, np.zeros((B, 1), np.int64), np.zeros((B, 1), np.uint8), np.ones((B, 1)),
                             torch.tensor(arena, dtype=torch.float64, device=_dev()), E, d, f)
        return y if one_d is False else y[0]


@dataclass(frozen=True)
class RouterDecision:
    """Routing outcome for one token at one layer (model.py:102-116)."""
    token: int
    layer: int
    logits: np.ndarray
    topk: np.ndarray
    probs_renorm: np.ndarray
    temperature: float = 1.0


class Model:
    """Same fields as the reference Model (model.py:119-198); the router and
    expert stacks are mirrored to HBM on first use."""

    def __init__(self, spec: ModelSpec):
        spec.validate()
        self.spec = spec
        E, C = spec.experts_per_layer, spec.num_clusters
        self.cluster_of = (np.arange(E) * C) // E
        self.cluster_dirs = substrate.cluster_dirs(spec)
        self.cluster_dirs.setflags(write=False)
        gw, gb = substrate.gate_weights(spec)
        gw.setflags(write=False)
        gb.setflags(write=False)
        self.gate_w, self.gate_b = gw, gb
        self._stacks: dict = {}
        self._dev_gate = None
        self._dev_arena: dict = {}

    @property
    def expert_bytes(self) -> int:
        s = self.spec
        return 2 * s.hidden_dim * s.ffn_dim * 8

    def layer_stack(self, layer: int):
        self._check_layer(layer)
        if layer not in self._stacks:
            w_in, w_out = substrate.layer_stack(self.spec, layer)
            w_in.setflags(write=False)
            w_out.setflags(write=False)
            self._stacks[layer] = (w_in, w_out)
            self._dev_arena.pop(layer, None)
        return self._stacks[layer]

    def expert(self, layer: int, expert_id: int) -> Expert:
        self._check_layer(layer)
        if not (0 <= expert_id < self.spec.experts_per_layer):
            raise InputError(f"expert id {expert_id} out of range")
        w_in, w_out = self.layer_stack(layer)
        return Expert(layer=layer, id=expert_id, w_in=w_in[expert_id], w_out=w_out[expert_id])

    def _check_layer(self, layer: int) -> None:
        substrate.check_layer(self.spec, layer)

    # device mirrors -------------------------------------------------------
    def device_gate(self, layer: int):
        if self._dev_gate is None:
            d = _dev()
            self._dev_gate = (torch.tensor(self.gate_w, dtype=torch.float32, device=d),
                              torch.tensor(self.gate_b, dtype=torch.float32, device=d))
        return self._dev_gate[0][layer], self._dev_gate[1][layer]

    def device_arena(self, layer: int):
        """f64 TANH arena [E, f*d + d*f]: [Win^T | Wout^T] per expert."""
        if layer not in self._dev_arena:
            w_in, w_out = self.layer_stack(layer)
            E = w_in.shape[0]
            arena = np.concatenate([np.transpose(w_in, (0, 2, 1)).reshape(E, -1),
                                    np.transpose(w_out, (0, 2, 1)).reshape(E, -1)], axis=1)
            self._dev_arena[layer] = torch.tensor(arena, dtype=torch.float64, device=_dev())
        return self._dev_arena[layer]


def build_model(spec: ModelSpec) -> Model:
    return Model(spec)


def route_batch(model: Model, x: np.ndarray, layer: int, temperature: float = 1.0, tokens=None) -> list:
    """K1 on the GPU (model.py:231-280). Selection is made on fp32 logits; the
    returned logits are those fp32 values as float64, and probs_renorm are
    computed in f64 from them (bm_select_topk_f64), so a decision's topk and
    probabilities are mutually consistent bit for bit."""
    model._check_layer(layer)
    if temperature <= 0:
        raise InputError("temperature must be > 0")
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    if x.shape[1] != model.spec.hidden_dim:
        raise InputError(f"embedding dim {x.shape[1]} != hidden_dim {model.spec.hidden_dim}")
    if not np.isfinite(x).all():
        raise InputError("non-finite embedding")
    k = model.spec.top_k
    wg, bg = model.device_gate(layer)
    xd = torch.tensor(x, dtype=torch.float32, device=wg.device)
    r = ops.gate_topk(xd, wg, bg, k, temperature)
    s = ops.select_topk_f64(r.logits.double(), k, temperature)
    z = s.logits.cpu().numpy()
    tk = s.topk.cpu().numpy().astype(np.int64)
    pr = s.probs64.cpu().numpy()
    if tokens is None:
        tokens = range(x.shape[0])
    out = []
    for row, tok in zip(range(x.shape[0]), tokens):
        zr = z[row].copy()
        zr.setflags(write=False)
        out.append(RouterDecision(token=int(tok), layer=layer, logits=zr, topk=tk[row].copy(),
                                  probs_renorm=pr[row].copy(), temperature=float(temperature)))
    return out


def route(model: Model, x: np.ndarray, layer: int, temperature: float = 1.0, token: int = 0) -> RouterDecision:
    return route_batch(model, np.asarray(x)[None, :], layer, temperature, tokens=[token])[0]


_KIND_CODE = {"kept": 0, "substituted": 1, "ondemand_fallback": 2, "dropped": 3}


def _plan_arrays(decision: RouterDecision, plan):
    """Executed ids and kinds for one decision under an optional plan (model.py:294-305)."""
    k = len(decision.topk)
    if plan is None:
        return decision.topk.astype(np.int64), np.zeros(k, np.uint8)
    ids = np.empty(k, dtype=np.int64)
    kinds = np.empty(k, dtype=np.uint8)
    for i, slot in enumerate(plan.slots):
        ids[i] = slot.executed
        kinds[i] = _KIND_CODE[slot.kind]
    return ids, kinds


def _grouped_forward(x, ids, kinds, weights, arena, E, d, f, h_in=False):
    dev = arena.device
    ex = torch.tensor(ids, dtype=torch.int32, device=dev)
    kd = torch.tensor(kinds, dtype=torch.uint8, device=dev)
    pr = torch.tensor(weights, dtype=torch.float64, device=dev)
    xd = torch.tensor(x, dtype=torch.float64, device=dev)
    perm = ops.permute(ex, kd, E)
    xp = ops.gather_rows(xd, perm, 0)
    yp = ops.expert_ffn_f32(xp, perm, arena, torch.arange(E, dtype=torch.int32, device=dev), d, f, ops.ACT_TANH)
    y = ops.combine(yp, perm, pr, kd, h_in=xd if h_in else None, residual_scale=_RESIDUAL_SCALE)
    return y.double().cpu().numpy()


def forward_batch(model: Model, x: np.ndarray, decisions, plans=None) -> np.ndarray:
    """K3 -> K4 (f64 SIMT, tanh) -> K5 over one layer (model.py:318-340):
    weights are the ORIGINAL p~, dropped slots contribute 0, no renormalisation."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    n = x.shape[0]
    if len(decisions) != n:
        raise InputError("decisions/batch size mismatch")
    layer = decisions[0].layer
    E = model.spec.experts_per_layer
    k = len(decisions[0].topk)
    ids = np.empty((n, k), dtype=np.int64)
    kinds = np.empty((n, k), dtype=np.uint8)
    weights = np.empty((n, k))
    for i, d in enumerate(decisions):
        if d.layer != layer:
            raise InputError("mixed layers in one forward batch")
        ids[i], kinds[i] = _plan_arrays(d, None if plans is None else plans[i])
        weights[i] = d.probs_renorm
    if ids.min() < 0 or ids.max() >= E:
        raise InternalError("plan references expert outside the layer")
    return _grouped_forward(x, ids, kinds, weights, model.device_arena(layer), E, model.spec.hidden_dim,
                            model.spec.ffn_dim)


def forward_layer(model: Model, x: np.ndarray, decision: RouterDecision, plan=None) -> np.ndarray:
    return forward_batch(model, np.asarray(x)[None, :], [decision], None if plan is None else [plan])[0]


def layer_update(h: np.ndarray, y: np.ndarray) -> np.ndarray:
    """(h + 0.5 y) / max(rms, 1e-12) (model.py:343-347) through K5's epilogue."""
    h = np.atleast_2d(np.asarray(h, dtype=np.float64))
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    dev = _dev()
    B, d = h.shape
    yd = torch.tensor(y, dtype=torch.float64, device=dev)
    hd = torch.tensor(h, dtype=torch.float64, device=dev)
    perm = ops.Permutation(None, None, None, torch.arange(B, dtype=torch.int32, device=dev), B)
    out = ops.combine(yd, perm, torch.ones(B, 1, dtype=torch.float64, device=dev),
                      torch.zeros(B, 1, dtype=torch.uint8, device=dev), h_in=hd, residual_scale=_RESIDUAL_SCALE)
    return out.double().cpu().numpy()
