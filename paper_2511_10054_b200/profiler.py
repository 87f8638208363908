"""Streaming co-activation statistics — the reference ``profiler`` API
(profiler.py:1-214) with counters in HBM.

CoActivationStats keeps integer u64 counters on the GPU (main range and
warm-up range separately) plus f64 weighted mass; ``observe_batch`` is the
hot path (K6 over a whole batch of decisions), ``observe`` the one-token
reference signature. The float64 views ``counts`` / ``pair_counts`` are
materialised with the reference's exact sequential accumulation order
(bm_counts_to_f64), assuming warm-up tokens are observed before the rest
(as in a stream). BSST v1 files are byte-identical to the reference's.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import DegeneratePivotError, FormatError, InputError
from . import _native as N

_STATS_MAGIC = b"BSST"
_STATS_VERSION = 1


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


class CoActivationStats:
    def __init__(self, layer: int, num_experts: int, warmup_steps: int = 256, warmup_weight: float = 0.0,
                 laplace_eps: float = 1e-3, tokens_seen: int = 0, counts=None, pair_counts=None, pair_weights=None):
        E = num_experts
        if E < 1:
            raise InputError("num_experts must be >= 1")
        if laplace_eps < 0:
            raise InputError("laplace_eps must be nonnegative")
        if not (0.0 <= warmup_weight <= 1.0):
            raise InputError("warmup_weight must be in [0, 1]")
        if warmup_steps < 0:
            raise InputError("warmup_steps must be nonnegative")
        self.layer, self.num_experts = layer, E
        self.warmup_steps, self.warmup_weight, self.laplace_eps = warmup_steps, warmup_weight, laplace_eps
        self.tokens_seen = tokens_seen
        dev = _dev()
        self._c = torch.zeros(E, dtype=torch.int64, device=dev)
        self._p = torch.zeros(E, E, dtype=torch.int64, device=dev)
        self._wc = torch.zeros(E, dtype=torch.int64, device=dev)
        self._wp = torch.zeros(E, E, dtype=torch.int64, device=dev)
        self._pw = torch.zeros(E, E, dtype=torch.float64, device=dev)
        # float matrices given explicitly (load_stats / merge of foreign stats)
        self._f64 = None
        self._host = None
        if counts is not None or pair_counts is not None or pair_weights is not None:
            self._f64 = (np.zeros(E) if counts is None else np.array(counts, np.float64),
                         np.zeros((E, E)) if pair_counts is None else np.array(pair_counts, np.float64),
                         np.zeros((E, E)) if pair_weights is None else np.array(pair_weights, np.float64))
            self._pw = torch.tensor(self._f64[2], device=dev)

    def config_tuple(self) -> tuple:
        return (self.layer, self.num_experts, self.warmup_steps, self.warmup_weight, self.laplace_eps)

    # reference-visible float64 views ------------------------------------
    # The reference's stats are plain numpy arrays that callers may edit in
    # place (tests poke ties into pair_counts). The views below are therefore
    # materialised once into host arrays that stay writable; the next device
    # operation folds them back: unchanged views are dropped (the integer
    # counters stay authoritative), edited ones become the stats' float state.
    def _views(self):
        if self._f64 is not None:
            return self._f64
        if self._host is None:
            c = ops.counts_to_f64(self._c, self._wc, self.warmup_weight).cpu().numpy()
            p = ops.counts_to_f64(self._p, self._wp, self.warmup_weight).cpu().numpy()
            w = self._pw.cpu().numpy()
            self._host = ((c, p, w), (c.copy(), p.copy(), w.copy()))
        return self._host[0]

    def _sync(self):
        if self._host is None:
            return
        views, snap = self._host
        self._host = None
        if all(np.array_equal(v, s0) for v, s0 in zip(views, snap)):
            return
        self._f64 = views
        self._pw = torch.tensor(views[2], device=_dev())

    @property
    def counts(self) -> np.ndarray:
        return self._views()[0]

    @counts.setter
    def counts(self, value):
        np.copyto(self._views()[0], np.asarray(value, np.float64))

    @property
    def pair_counts(self) -> np.ndarray:
        return self._views()[1]

    @pair_counts.setter
    def pair_counts(self, value):
        np.copyto(self._views()[1], np.asarray(value, np.float64))

    @property
    def pair_weights(self) -> np.ndarray:
        return self._views()[2]

    @pair_weights.setter
    def pair_weights(self, value):
        np.copyto(self._views()[2], np.asarray(value, np.float64))

    def device_matrix(self, mode: str) -> torch.Tensor:
        self._sync()
        if self._f64 is not None:
            return torch.tensor(self._f64[2] if mode == "weighted" else self._f64[1], device=_dev())
        if mode == "weighted":
            return self._pw
        return ops.counts_to_f64(self._p, self._wp, self.warmup_weight)

    # accumulation ------------------------------------------------------------
    def observe_tensors(self, topk: torch.Tensor, probs: torch.Tensor | None, first_step: int) -> None:
        """K6 over rows of a batch whose global steps are first_step, first_step+1, ..."""
        self._sync()
        if self._f64 is not None:
            raise InputError("stats loaded from floats cannot accumulate further")
        n = topk.shape[0]
        warm_end = max(0, min(n, self.warmup_steps - first_step))
        if warm_end > 0 and self.warmup_weight != 0.0:
            ops.coact_count(topk[:warm_end].contiguous(), self.num_experts, self._wc, self._wp)
            if probs is not None:
                ops.coact_weighted(topk[:warm_end].contiguous(), probs[:warm_end].contiguous(), self.num_experts,
                                   self.warmup_weight, self._pw)
        if warm_end < n:
            ops.coact_count(topk[warm_end:].contiguous(), self.num_experts, self._c, self._p)
            if probs is not None:
                ops.coact_weighted(topk[warm_end:].contiguous(), probs[warm_end:].contiguous(), self.num_experts,
                                   1.0, self._pw)
        self.tokens_seen += n


@dataclass(frozen=True)
class ConditionalRow:
    pivot: int
    q: np.ndarray


def _validate(stats, decision):
    if decision.layer != stats.layer:
        raise InputError(f"decision layer {decision.layer} != stats layer {stats.layer}")
    ids = [int(e) for e in decision.topk]
    if len(set(ids)) != len(ids):
        raise InputError("duplicate experts in selected set")
    if min(ids) < 0 or max(ids) >= stats.num_experts:
        raise InputError("expert id out of range")


def observe(stats: CoActivationStats, decision, step: int) -> None:
    """profiler.py:67-95 for one decision (K6 on one row)."""
    _validate(stats, decision)
    dev = _dev()
    tk = torch.tensor(np.asarray(decision.topk, np.int32)[None, :], device=dev)
    pr = torch.tensor(np.asarray(decision.probs_renorm, np.float32)[None, :], device=dev)
    stats.observe_tensors(tk, pr, int(step))


def observe_batch(stats: CoActivationStats, decisions, steps=None) -> None:
    """Fold a batch of decisions with consecutive (or given ascending) steps."""
    if not decisions:
        return
    for d in decisions:
        _validate(stats, d)
    dev = _dev()
    tk = torch.tensor(np.stack([np.asarray(d.topk, np.int32) for d in decisions]), device=dev)
    pr = torch.tensor(np.stack([np.asarray(d.probs_renorm, np.float32) for d in decisions]), device=dev)
    first = int(steps[0]) if steps is not None else int(decisions[0].token)
    stats.observe_tensors(tk, pr, first)


def conditional_row(stats: CoActivationStats, pivot: int, mode: str = "binary") -> ConditionalRow:
    """profiler.py:98-119 on the GPU (bm_conditional_rows)."""
    if not (0 <= pivot < stats.num_experts):
        raise InputError(f"pivot {pivot} out of range")
    if mode not in ("binary", "weighted"):
        raise InputError(f"unknown mode {mode!r}")
    M = stats.device_matrix(mode).contiguous()
    E = stats.num_experts
    q = torch.empty(E, E, dtype=torch.float64, device=M.device)
    deg = torch.empty(E, dtype=torch.uint8, device=M.device)
    N.call("bm_conditional_rows", M.data_ptr(), E, float(stats.laplace_eps), q.data_ptr(), deg.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    if int(deg[pivot].item()):
        raise DegeneratePivotError(f"pivot {pivot} has no co-activation mass and eps == 0")
    return ConditionalRow(pivot=pivot, q=q[pivot].cpu().numpy())


def merge(a: CoActivationStats, b: CoActivationStats) -> CoActivationStats:
    """Elementwise sum of shard statistics (profiler.py:122-137)."""
    if a.config_tuple() != b.config_tuple():
        raise InputError("cannot merge stats with different layer/shape/config")
    out = CoActivationStats(a.layer, a.num_experts, a.warmup_steps, a.warmup_weight, a.laplace_eps,
                            a.tokens_seen + b.tokens_seen)
    a._sync()
    b._sync()
    if a._f64 is None and b._f64 is None:
        for name in ("_c", "_p", "_wc", "_wp", "_pw"):
            setattr(out, name, getattr(a, name) + getattr(b, name))
    else:  # reference float semantics: a + b of the float views
        out._f64 = (a.counts + b.counts, a.pair_counts + b.pair_counts, a.pair_weights + b.pair_weights)
        out._pw = torch.tensor(out._f64[2], device=_dev())
    return out


_HEADER = struct.Struct("<4sIIIIddQ")


def save_stats(stats: CoActivationStats, path) -> None:
    """BSST v1 (profiler.py:140-160), byte-identical to the reference writer."""
    E = stats.num_experts
    with open(path, "wb") as f:
        f.write(_HEADER.pack(_STATS_MAGIC, _STATS_VERSION, stats.layer, E, stats.warmup_steps, stats.warmup_weight,
                             stats.laplace_eps, stats.tokens_seen))
        f.write(np.asarray(stats.counts).astype("<f8").tobytes())
        f.write(np.asarray(stats.pair_counts).astype("<f8").tobytes())
        f.write(np.asarray(stats.pair_weights).astype("<f8").tobytes())


def load_stats(path) -> CoActivationStats:
    """profiler.py:163-192."""
    with open(path, "rb") as f:
        raw = f.read()
    if len(raw) < _HEADER.size:
        raise FormatError(f"{path}: truncated stats file")
    magic, version, layer, E, wsteps, wweight, eps, seen = _HEADER.unpack_from(raw)
    if magic != _STATS_MAGIC:
        raise FormatError(f"{path}: not a co-activation stats file")
    if version != _STATS_VERSION:
        raise FormatError(f"{path}: unsupported stats version {version}")
    if len(raw) != _HEADER.size + 8 * (E + 2 * E * E):
        raise FormatError(f"{path}: wrong payload size")
    off = _HEADER.size
    counts = np.frombuffer(raw, dtype="<f8", count=E, offset=off).copy()
    off += 8 * E
    pc = np.frombuffer(raw, dtype="<f8", count=E * E, offset=off).reshape(E, E).copy()
    off += 8 * E * E
    pw = np.frombuffer(raw, dtype="<f8", count=E * E, offset=off).reshape(E, E).copy()
    return CoActivationStats(layer, E, wsteps, wweight, eps, seen, counts=counts, pair_counts=pc, pair_weights=pw)


def export_coactivation_csv(stats: CoActivationStats, path, mode: str = "binary") -> None:
    if mode not in ("binary", "weighted"):
        raise InputError(f"unknown mode {mode!r}")
    m = stats.pair_counts if mode == "binary" else stats.pair_weights
    with open(path, "w") as f:
        for row in m:
            f.write(",".join(repr(float(v)) for v in row))
            f.write("\n")


def gini(counts) -> float:
    """profiler.py:206-214 (host helper)."""
    x = np.sort(np.asarray(counts, dtype=np.float64))
    n = x.size
    total = x.sum()
    if n == 0 or total <= 0:
        return 0.0
    cum = np.cumsum(x)
    return float((n + 1 - 2 * (cum / total).sum()) / n)
