"""The reference's deterministic synthetic MoE substrate (host-side input
generation, not the hot path).

Restates ``model.py:38-222, 350-382`` of the reference so that a
``buddysim`` user who builds a model from a ``ModelSpec`` and a token
stream from a seed gets bit-identical float64 weights and embeddings here.
The hot path never runs in numpy: these arrays are uploaded to HBM once
(``Model.device_layer``) and every route/remap/forward runs in CUDA.
Pinned by ``tests/test_substrate.py`` against ``tests/golden/substrate.npz``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ConfigurationError, InputError

# rng domain tags (model.py:21-28)
_TAG_CLUSTER_DIR, _TAG_GATE_JITTER, _TAG_BIAS_RANK = 11, 12, 13
_TAG_EXPERT_BASE, _TAG_EXPERT_DELTA, _TAG_STREAM, _TAG_READOUT = 14, 15, 16, 17
# texture constants (model.py:33-37)
_GATE_GAIN, _GATE_JITTER, _STREAM_NOISE, _MIXTURE_EXPONENT = 1.5, 0.25, 0.6, 2.25


def _rng(*entropy: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(list(entropy)))


def _unit_rows(m: np.ndarray) -> np.ndarray:
    return m / np.linalg.norm(m, axis=-1, keepdims=True)


@dataclass(frozen=True)
class ModelSpec:
    """Shape and seeding of the synthetic model (model.py:47-82)."""

    num_layers: int = 24
    experts_per_layer: int = 64
    top_k: int = 6
    hidden_dim: int = 32
    ffn_dim: int = 64
    seed: int = 7
    skew: float = 0.8
    num_clusters: int = 8
    cluster_spread: float = 0.1

    def validate(self) -> "ModelSpec":
        if self.num_layers < 1:
            raise ConfigurationError("num_layers must be >= 1")
        if self.experts_per_layer < 1:
            raise ConfigurationError("experts_per_layer must be >= 1")
        if self.top_k < 1:
            raise ConfigurationError("top_k must be >= 1")
        if self.top_k > self.experts_per_layer:
            raise ConfigurationError(
                f"top_k={self.top_k} exceeds experts_per_layer={self.experts_per_layer}")
        if self.hidden_dim < 1 or self.ffn_dim < 1:
            raise ConfigurationError("hidden_dim and ffn_dim must be >= 1")
        if not (1 <= self.num_clusters <= self.experts_per_layer):
            raise ConfigurationError("num_clusters must be in [1, experts_per_layer]")
        if self.skew < 0:
            raise ConfigurationError("skew must be nonnegative")
        if self.cluster_spread < 0:
            raise ConfigurationError("cluster_spread must be nonnegative")
        if not (0 <= self.seed < 2**63):
            raise ConfigurationError("seed must be a nonnegative 64-bit integer")
        return self


def cluster_popularity(spec: ModelSpec):
    """(cluster_order, expert_rank), model.py:205-222."""
    E, C = spec.experts_per_layer, spec.num_clusters
    g = _rng(spec.seed, _TAG_BIAS_RANK)
    cluster_of = (np.arange(E) * C) // E
    cluster_order = g.permutation(C)
    expert_rank = np.empty(E, dtype=np.int64)
    nxt = 1
    for c in cluster_order:
        members = g.permutation(np.flatnonzero(cluster_of == c))
        expert_rank[members] = np.arange(nxt, nxt + members.size)
        nxt += members.size
    return cluster_order, expert_rank


def cluster_dirs(spec: ModelSpec) -> np.ndarray:
    """Unit cluster directions [C, d] shared across depth (model.py:131-134)."""
    return _unit_rows(_rng(spec.seed, _TAG_CLUSTER_DIR).standard_normal((spec.num_clusters, spec.hidden_dim)))


def gate_weights(spec: ModelSpec):
    """Router weights gate_w[L,E,d], gate_b[L,E] (model.py:122-150)."""
    E, d, C, L = spec.experts_per_layer, spec.hidden_dim, spec.num_clusters, spec.num_layers
    cluster_of = (np.arange(E) * C) // E
    dirs = cluster_dirs(spec)
    _, rank = cluster_popularity(spec)
    bias = spec.skew * np.log(E / rank)
    gate_w = np.empty((L, E, d))
    gate_b = np.empty((L, E))
    for layer in range(L):
        jitter = _rng(spec.seed, _TAG_GATE_JITTER, layer).standard_normal((E, d))
        rows = dirs[cluster_of] + _GATE_JITTER * jitter / np.sqrt(d)
        gate_w[layer] = _GATE_GAIN * _unit_rows(rows)
        gate_b[layer] = bias
    return gate_w, gate_b


def expert_weights(spec: ModelSpec, layer: int, expert_id: int):
    """One expert's (w_in[d,f], w_out[f,d]), model.py:161-171."""
    d, f = spec.hidden_dim, spec.ffn_dim
    c = int((expert_id * spec.num_clusters) // spec.experts_per_layer)
    base = _rng(spec.seed, _TAG_EXPERT_BASE, layer, c)
    w_in = base.standard_normal((d, f)) / np.sqrt(d)
    w_out = base.standard_normal((f, d)) / np.sqrt(f)
    delta = _rng(spec.seed, _TAG_EXPERT_DELTA, layer, expert_id)
    w_in = w_in + spec.cluster_spread * delta.standard_normal((d, f)) / np.sqrt(d)
    w_out = w_out + spec.cluster_spread * delta.standard_normal((f, d)) / np.sqrt(f)
    return w_in, w_out


def layer_stack(spec: ModelSpec, layer: int):
    """(w_in[E,d,f], w_out[E,f,d]) for one layer, model.py:173-186."""
    E = spec.experts_per_layer
    w_in = np.empty((E, spec.hidden_dim, spec.ffn_dim))
    w_out = np.empty((E, spec.ffn_dim, spec.hidden_dim))
    for e in range(E):
        w_in[e], w_out[e] = expert_weights(spec, layer, e)
    return w_in, w_out


def token_stream(spec: ModelSpec, seed: int, num_tokens: int) -> np.ndarray:
    """Gaussian-mixture embedding stream, RMS-normalised (model.py:350-375)."""
    if num_tokens < 1:
        raise ConfigurationError("num_tokens must be >= 1")
    if not (0 <= seed < 2**63):
        raise ConfigurationError("stream seed must be a nonnegative 64-bit integer")
    spec.validate()
    dirs = _unit_rows(_rng(spec.seed, _TAG_CLUSTER_DIR).standard_normal(
        (spec.num_clusters, spec.hidden_dim)))
    order, _ = cluster_popularity(spec)
    pos = np.arange(1, spec.num_clusters + 1, dtype=np.float64)
    weights = pos ** (-_MIXTURE_EXPONENT * spec.skew)
    probs = np.empty(spec.num_clusters)
    probs[order] = weights / weights.sum()
    g = _rng(seed, _TAG_STREAM)
    comp = g.choice(spec.num_clusters, size=num_tokens, p=probs)
    noise = g.standard_normal((num_tokens, spec.hidden_dim)) / np.sqrt(spec.hidden_dim)
    x = dirs[comp] + _STREAM_NOISE * noise
    rms = np.sqrt(np.mean(np.square(x), axis=1, keepdims=True))
    return x / np.maximum(rms, 1e-12)


def readout_head(spec: ModelSpec, num_classes: int = 16) -> np.ndarray:
    """model.py:378-382."""
    if num_classes < 2:
        raise ConfigurationError("num_classes must be >= 2")
    return _rng(spec.seed, _TAG_READOUT).standard_normal((num_classes, spec.hidden_dim))


def check_layer(spec: ModelSpec, layer: int) -> None:
    if not (0 <= layer < spec.num_layers):
        raise InputError(f"layer {layer} out of range")
