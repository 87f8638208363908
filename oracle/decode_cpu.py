"""TEST / BASELINE INFRASTRUCTURE: the reference's offloaded-MoE decode step
on the host cores, for bench.py's CPU reference arm and in-line cpu_baseline.

It runs the algorithm of the reference's run_simulation inner loop
(harness.py:315-393) with this package's numpy restatements, in float64 like
the reference, on the same synthetic inputs as the GPU arm:

  * gate weights and token streams of the reference substrate
    (paper_2511_10054_b200.substrate, numpy), rounded to float32 where the GPU
    arm rounds them, so both arms route the same numbers;
  * expert weights from the counter-based generator (oracle/c/synth_host.c,
    bit-identical to the GPU arm's bm_synth_bf16), widened to float64;
  * buddy tables and tau built here from the profile stream (K1/K6/K7/tau
    semantics: route -> observe -> build_table -> calibrate_tau), with the
    stream pushed through each layer's experts in f64 like cmd_profile
    (harness.py:93-101), or the GPU arm's tables passed in.

Per (step, layer): route_batch (model.py:231-280) -> evaluate_gates
(gating.py:148-165) -> substitute_batch (substitution.py:193-208) -> cache
replay (memtier access, harness.py:363-382) -> forward_batch combine
semantics (model.py:318-340; SwiGLU experts, the rows of each executed expert
as one GEMM, spread over the host threads) -> layer_update (model.py:343-347).

The work is layer-major: one layer's float64 experts (11.3 GB at the Mixtral
shape) are generated untimed, then every step's batch passes through that
layer, each (step, layer) timed on its own. A layer's cache state evolves in
step order exactly as step-major; only the cross-layer prefetch/settle
interleaving of the shared clock is dropped, and its predictor does not fire
at these batch sizes (capacity - distinct executed <= 0). A
step's time is the sum of its layers' times: a measured sum, not an
extrapolation.
"""

from __future__ import annotations

import hashlib
import math
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import buddy_oracle as O
from . import synth_host


def _tau(probs, percentile):
    t = np.array([O.tae(p) for p in probs])
    s = np.sort(t)
    idx = max(1, math.ceil(percentile * s.size / 100.0)) - 1
    return float(s[min(idx, s.size - 1)])


def tables_digest(ids, lens) -> str:
    h = hashlib.sha256()
    for l in range(len(ids)):
        h.update(np.ascontiguousarray(ids[l], np.int32).tobytes())
        h.update(np.ascontiguousarray(lens[l], np.int32).tobytes())
    return h.hexdigest()[:16]


class CpuDecode:
    """One replica's decode over `layers` layers of a BASELINE shape."""

    def __init__(self, model: str, layers: int, batch: int, profile_tokens: int = 4096, alpha: float = 0.95,
                 tau_percentile: float = 15.0, rho: int = 3, seed: int = 0, threads: int | None = None,
                 cache_rate: float | None = None, stream_seed: int = 2, stream_tokens: int | None = None,
                 profile: str = "forward", tables=None, clustered: bool = True,
                 clusters: int | None = None):
        """profile: how the buddy tables and tau are built when ``tables`` is not
        given, as workload.build does on the GPU: "forward" pushes the profile
        stream through every layer's experts (full residency, f64 here),
        "route" routes the same profile tokens at every layer. tables: (ids
        [L,E,K], lens [L,E], taus [L]) to reuse instead (e.g. the GPU arm's)."""
        from paper_2511_10054_b200 import substrate, synth
        E, k, d, f, rate = synth.SHAPES[model]
        self.rate = float(cache_rate) if cache_rate is not None else rate
        self.E, self.k, self.d, self.f, self.S = E, k, d, f, synth.SHARED.get(model, 0)
        self.cap = int(math.floor(self.rate * E))
        self.k_max = min(16, E - 1)
        self.L, self.B, self.rho, self.seed = layers, batch, rho, seed
        self.alpha, self.tau_percentile = alpha, tau_percentile
        self.threads = threads or len(os.sched_getaffinity(0))
        C = clusters if clusters is not None else (synth.CLUSTERS[model] if clustered else min(E, 8))
        self.clustered = clustered
        self.cl_of = synth.cluster_of(E, C) if clustered else None
        spec = substrate.ModelSpec(num_layers=layers, experts_per_layer=E, top_k=k, hidden_dim=d, ffn_dim=f,
                                   num_clusters=C, seed=7)
        self.spec = spec
        gw, gb = substrate.gate_weights(spec)
        # the GPU arm routes fp32-rounded gates and tokens
        self.gw = gw.astype(np.float32).astype(np.float64)
        self.gb = gb.astype(np.float32).astype(np.float64)
        self.synth = synth
        self.stream_seed, self.stream_tokens = stream_seed, stream_tokens
        self.pool = ThreadPoolExecutor(max_workers=self.threads)
        self.profile = profile
        self.profile_s = 0.0
        self.gen_s = 0.0
        if tables is not None:
            ids, lens, taus = tables
            self.ids = [np.asarray(ids[l], np.int32) for l in range(layers)]
            self.lens = [np.asarray(lens[l], np.int32) for l in range(layers)]
            self.taus = [float(t) for t in taus]
        else:
            self.ids, self.lens, self.taus = [None] * layers, [None] * layers, [None] * layers
            self.xp = substrate.token_stream(spec, 1, profile_tokens).astype(np.float32).astype(np.float64)
            if profile == "route":
                for l in range(layers):
                    self._profile_layer(l, None)

    @property
    def digest(self) -> str:
        return tables_digest(self.ids, self.lens)

    def _profile_layer(self, l: int, experts):
        """Table + tau of layer l from the profile stream (K1 -> K6 with warm-up
        weight 0 -> K7, nearest-rank tau); "forward" then pushes the stream
        through the layer's experts with every slot kept (identity plans)."""
        t0 = time.perf_counter()
        warm = min(256, self.xp.shape[0])
        _, topk, probs = O.route(self.xp, self.gw[l], self.gb[l], self.k)
        _, pairs, _, _ = O.coact_count(topk, None, self.E, 0, warm, 0.0)
        ids, _, lens = O.build_table(pairs, 1e-3, self.alpha, self.k_max)
        self.ids[l], self.lens[l], self.taus[l] = ids, lens, _tau(probs, self.tau_percentile)
        if self.profile == "forward":
            kd = np.zeros(topk.shape, np.uint8)
            self.xp = O.layer_update(self.xp, self._combine(self.xp, topk, kd, probs, experts))
        self.profile_s += time.perf_counter() - t0

    def tokens(self, n: int) -> np.ndarray:
        from paper_2511_10054_b200 import substrate
        x = substrate.token_stream(self.spec, self.stream_seed, self.stream_tokens or n)
        return x[:n].astype(np.float32).astype(np.float64)

    def layer_experts(self, l: int):
        """float64 (W1 [f,d], W3 [f,d], W2 [d,f]) of every expert of layer l (untimed),
        all matrices' chunks spread over the thread pool."""
        s, d, f = self.synth, self.d, self.f
        luts16 = [np.ascontiguousarray(s.lut_bf16(s.matrix_scale(d, f, m))) for m in (s.W1, s.W3, s.W2)]
        luts = [np.ascontiguousarray(s.bf16_to_f64(t)) for t in luts16]
        out, tasks = {}, []
        for e in range(self.E + self.S):
            mats = []
            for m, shape in ((s.W1, (f, d)), (s.W3, (f, d)), (s.W2, (d, f))):
                a = np.empty(shape, np.float64)
                if self.clustered and e < self.E:  # base_cluster + spread * delta_e (model.py:161-171)
                    tasks += synth_host.fill_mix_tasks(s.base_key(self.seed, l, int(self.cl_of[e]), m),
                                                       s.matrix_key(self.seed, l, e, m), s.SPREAD, d * f, luts16[m],
                                                       a.reshape(-1))
                else:
                    tasks += synth_host.fill_tasks(s.matrix_key(self.seed, l, e, m), d * f, luts[m], a.reshape(-1))
                mats.append(a)
            out[e] = tuple(mats)
        list(self.pool.map(lambda t: t(), tasks))
        return out

    def _ffn_rows(self, groups):
        """{expert: (x_rows, (w1, w3, w2))} -> {expert: y_rows}, GEMMs split over
        column blocks so every host thread streams its own slice of weights."""
        per = max(1, -(-2 * self.threads // max(1, len(groups))))
        f, d = self.f, self.d
        hs = {e: np.empty((x.shape[0], f)) for e, (x, _) in groups.items()}
        ys = {e: np.empty((x.shape[0], d)) for e, (x, _) in groups.items()}

        def g1(task):
            e, a, b = task
            x, (w1, w3, _) = groups[e]
            u = x @ w1[a:b].T
            hs[e][:, a:b] = (u / (1.0 + np.exp(-u))) * (x @ w3[a:b].T)

        def g2(task):
            e, a, b = task
            _, (_, _, w2) = groups[e]
            ys[e][:, a:b] = hs[e] @ w2[a:b].T

        t1 = [(e, f * i // per, f * (i + 1) // per) for e in groups for i in range(per)]
        list(self.pool.map(g1, t1))
        t2 = [(e, d * i // per, d * (i + 1) // per) for e in groups for i in range(per)]
        list(self.pool.map(g2, t2))
        return ys

    def layer_step(self, l: int, h: np.ndarray, res: O.Residency, clock: O.Clock, experts, tokens, method="buddy"):
        """One (step, layer) of the reference loop; returns the new hidden state."""
        E, k = self.E, self.k
        z, topk, probs = O.route(h, self.gw[l], self.gb[l], k)
        mask = res.mask.copy()
        if method == "buddy":
            _, _, ok, _, batch_ok = O.gate_batch(probs, topk, mask, self.taus[l], None, 1.0)
            ex, kd, _ = O.remap_batch(topk, z, mask, self.ids[l], np.zeros(self.ids[l].shape), self.lens[l],
                                      ok & batch_ok, self.k_max, self.rho)
        else:
            ex, kd, _ = O.ondemand_plan(topk, mask)
        nslots = 0
        for b in range(h.shape[0]):  # cache replay in (token, slot) order
            for s in range(k):
                if kd[b, s] == O.KIND_DROPPED:
                    continue
                if kd[b, s] == O.KIND_SUBSTITUTED:
                    O.access(res, int(topk[b, s]), clock, 9.5, 0.0, 0, True, int(tokens[b]))
                O.access(res, int(ex[b, s]), clock, 9.5, 0.0, 0, False, int(tokens[b]))
                nslots += 1
        clock.now += 0.5 * nslots
        return O.layer_update(h, self._combine(h, ex, kd, probs, experts))

    def _combine(self, h, ex, kd, probs, experts):
        """forward_batch combine (model.py:318-340): each executed expert's rows as
        one GEMM over the host threads, slots added in slot order with the
        original probabilities, dropped slots 0; shared experts weight 1."""
        E, k = self.E, ex.shape[1]
        live = kd != O.KIND_DROPPED
        groups, rows_of = {}, {}
        for e in np.unique(ex[live]):
            rows = np.flatnonzero(np.any((ex == e) & live, axis=1))
            rows_of[int(e)] = rows
            groups[int(e)] = (h[rows], experts[int(e)])
        for sx in range(self.S):
            groups[E + sx] = (h, experts[E + sx])
        ys = self._ffn_rows(groups)
        y = np.zeros_like(h)
        for s in range(k):
            for b in np.flatnonzero(live[:, s]):
                e = int(ex[b, s])
                y[b] += probs[b, s] * ys[e][int(np.searchsorted(rows_of[e], b))]
        for sx in range(self.S):
            y += ys[E + sx]
        return y

    def run(self, steps: int, timed_from: int, layers_run: int | None = None, method: str = "buddy", log=None):
        """Layer-major decode of `steps` batches; returns per-step seconds of
        the steps >= timed_from (each the sum of its layers' times)."""
        from paper_2511_10054_b200.synth import initial_residents
        layers_run = self.L if layers_run is None else layers_run
        B = self.B
        x = self.tokens(steps * B)
        H = [x[j * B:(j + 1) * B].copy() for j in range(steps)]
        per_step = np.zeros(steps)
        clock = O.Clock()
        gen_s = 0.0
        for l in range(layers_run):
            t0 = time.perf_counter()
            experts = self.layer_experts(l)
            gen_s += time.perf_counter() - t0
            if self.ids[l] is None:  # this layer's table from the profile stream (untimed)
                self._profile_layer(l, experts)
            res = O.Residency(self.E, self.cap, O.POLICY_LRU, initial_residents(self.E, self.cap, 0, l), None, l)
            for j in range(steps):
                t1 = time.perf_counter()
                H[j] = self.layer_step(l, H[j], res, clock, experts, np.arange(j * B, (j + 1) * B), method)
                per_step[j] += time.perf_counter() - t1
            del experts
            if log:
                log(f"cpu layer {l}: {per_step[timed_from:].sum() * 1e3:.0f} ms timed so far, gen {gen_s:.1f}s")
        self.gen_s = gen_s
        return per_step[timed_from:], H

    def close(self):
        self.pool.shutdown()
