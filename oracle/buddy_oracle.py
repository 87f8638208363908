"""numpy restatement of the reference BuddyMoE hot path (TEST INFRASTRUCTURE).

See ``oracle/__init__.py`` for the rules. File:line citations refer to the
reference package ``pkg/src/buddysim/`` (read-only, not shipped here).

Array conventions shared with the CUDA path (``include/bmoe.h``):
  * routing:   logits[B,E] f64, topk[B,k] int (descending, ties -> lower id),
               probs[B,k] f64 (renormalised over the selected set);
  * plans:     executed[B,k] int, kind[B,k] uint8 with
               KIND_KEPT=0, KIND_SUBSTITUTED=1, KIND_ONDEMAND=2, KIND_DROPPED=3,
               used[B] int;
  * buddy table (dense): ids[E,K] int32 padded with -1, weights[E,K] f64,
               lens[E] int32 (a pivot's list is ids[p, :lens[p]]).
"""

from __future__ import annotations

import math

import numpy as np

KIND_KEPT, KIND_SUBSTITUTED, KIND_ONDEMAND, KIND_DROPPED = 0, 1, 2, 3
KIND_NAMES = ("kept", "substituted", "ondemand_fallback", "dropped")
FALLBACK_PREFETCH, FALLBACK_DROP = 0, 1

_COVER_TOL = 1e-9          # buddies.py:25
_ZCLAMP = 3.0              # substitution.py:33
_RESIDUAL_SCALE = 0.5      # model.py:36


# --------------------------------------------------------------- routing
def softmax(z: np.ndarray) -> np.ndarray:
    """model.py:225-228."""
    z = z - z.max(axis=-1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=-1, keepdims=True)


def select_topk(z: np.ndarray, k: int, temperature: float = 1.0):
    """Selection + renormalisation from given logits, model.py:259-263.

    Stable argsort of -z: descending, ties toward the lower expert index;
    selection is temperature independent, only the probabilities change.
    """
    z = np.atleast_2d(np.asarray(z, dtype=np.float64))
    p = softmax(z / temperature)
    order = np.argsort(-z, axis=1, kind="stable")[:, :k]
    p_sel = np.take_along_axis(p, order, axis=1)
    p_sel = p_sel / p_sel.sum(axis=1, keepdims=True)
    return order.astype(np.int64), p_sel


def route(x, gate_w, gate_b, k: int, temperature: float = 1.0):
    """route_batch arithmetic, model.py:231-280 (f64 GEMM at :258)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    z = x @ np.asarray(gate_w, dtype=np.float64).T + np.asarray(gate_b, dtype=np.float64)
    topk, probs = select_topk(z, k, temperature)
    return z, topk, probs


# ----------------------------------------------------------------- gates
def tae(p: np.ndarray) -> float:
    """Normalised selected-set entropy, gating.py:71-83."""
    p = np.asarray(p, dtype=np.float64)
    k = p.size
    if k == 1:
        return 0.0
    nz = p[p > 0.0]
    h = -float(np.sum(nz * np.log(nz))) / math.log(k)
    return min(1.0, max(0.0, h))


def margin(p: np.ndarray) -> float:
    """Top-2 gap, gating.py:86-92."""
    p = np.asarray(p, dtype=np.float64)
    if p.size == 1:
        return 1.0
    top2 = np.sort(p)[-2:]
    return float(top2[1] - top2[0])


def token_gate(p, tau: float, gamma=None) -> bool:
    """gating.py:95-108: forbidden iff TAE <= tau or margin >= gamma."""
    if tae(p) <= tau:
        return False
    if gamma is not None and margin(p) >= gamma:
        return False
    return True


def distribution_gate(requested, mask, beta: float):
    """gating.py:126-145 — delta over requested slots, duplicates counted."""
    req = np.asarray(requested, dtype=np.int64).ravel()
    mask = np.asarray(mask, dtype=bool)
    delta = float(np.mean(~mask[req]))
    return delta, not (delta >= beta)


def calibrate_tau(samples, percentile: float) -> float:
    """Nearest-rank percentile, gating.py:111-123."""
    x = np.sort(np.asarray(list(samples), dtype=np.float64))
    n = x.size
    if n < 100:
        raise ValueError("need >= 100 samples")
    idx = max(1, math.ceil(percentile * n / 100.0)) - 1
    return float(x[min(idx, n - 1)])


def gate_batch(probs, topk, mask, tau, gamma=None, beta=1.0):
    """evaluate_gates, gating.py:148-165 → (tae[B], margin[B], token_ok[B], delta, batch_ok)."""
    probs = np.atleast_2d(probs)
    delta, batch_ok = distribution_gate(np.asarray(topk).ravel(), mask, beta)
    t = np.array([tae(p) for p in probs])
    m = np.array([margin(p) for p in probs])
    ok = np.array([token_gate(p, tau, gamma) for p in probs], dtype=bool)
    return t, m, ok, delta, batch_ok


# ----------------------------------------------------- substitution (Alg. 1)
def zscore(logits, j: int) -> float:
    """substitution.py:98-104."""
    z = np.asarray(logits, dtype=np.float64)
    sd = float(z.std())
    if sd <= 0.0:
        return 0.0
    v = (float(z[j]) - float(z.mean())) / sd
    return min(_ZCLAMP, max(-_ZCLAMP, v))


def _candidates(pivot, logits, ids, weights, lens, h, eta, kappa, partition_of, hop,
                use_local_logit=True):
    """_ordered_candidates, substitution.py:133-143 (+ psi_score :107-130).

    The diversity factor is omitted: it only rescales already-chosen
    candidates, which are in the assigned set and are skipped regardless
    (SURVEY §0 fact 4), so the relative order of viable candidates is
    unchanged under the stable sort.
    """
    n = min(int(lens[pivot]), h)
    cand = [int(j) for j in ids[pivot, :n]]
    if eta == 0.0 and kappa == 0.0:
        return cand
    scores = []
    for r, j in enumerate(cand):
        q = float(weights[pivot, r])
        zh = zscore(logits, j) if use_local_logit else 0.0
        hops = 0.0
        if partition_of is not None and partition_of[pivot] != partition_of[j]:
            hops = hop
        scores.append(q * (1.0 + eta * zh) * (1.0 - kappa * hops))
    order = np.argsort(-np.asarray(scores, dtype=np.float64), kind="stable")
    return [cand[i] for i in order]


def remap_token(topk, logits, mask, ids, weights, lens, allowed, h, rho,
                fallback=FALLBACK_PREFETCH, eta=0.0, kappa=0.0, partition_of=None,
                hop=1.0, use_local_logit=True):
    """substitute_token, substitution.py:146-190.

    rho < 0 (or None) means unlimited. Returns (executed[k], kind[k], used).
    """
    mask = np.asarray(mask, dtype=bool)
    budget = math.inf if (rho is None or rho < 0) else rho
    fb = KIND_ONDEMAND if fallback == FALLBACK_PREFETCH else KIND_DROPPED
    assigned = {int(e) for e in topk}
    k = len(topk)
    executed = np.empty(k, dtype=np.int64)
    kind = np.empty(k, dtype=np.uint8)
    used = 0
    for s, orig in enumerate(int(e) for e in topk):
        if mask[orig]:
            executed[s], kind[s] = orig, KIND_KEPT
            continue
        picked = None
        if allowed and used < budget:
            for j in _candidates(orig, logits, ids, weights, lens, h, eta, kappa,
                                 partition_of, hop, use_local_logit):
                if mask[j] and j not in assigned:
                    picked = j
                    break
        if picked is None:
            executed[s], kind[s] = orig, fb
        else:
            executed[s], kind[s] = picked, KIND_SUBSTITUTED
            assigned.add(picked)
            used += 1
    return executed, kind, used


def remap_batch(topk, logits, mask, ids, weights, lens, allowed, h, rho, **kw):
    """substitute_batch, substitution.py:193-208 (tokens are independent)."""
    topk = np.atleast_2d(topk)
    B, k = topk.shape
    ex = np.empty((B, k), dtype=np.int64)
    kd = np.empty((B, k), dtype=np.uint8)
    used = np.empty(B, dtype=np.int64)
    for b in range(B):
        lg = None if logits is None else logits[b]
        ex[b], kd[b], used[b] = remap_token(topk[b], lg, mask, ids, weights, lens,
                                            bool(allowed[b]), h, rho, **kw)
    return ex, kd, used


def ondemand_plan(topk, mask):
    """substitution.py:217-224 — the "without buddy" arm."""
    topk = np.atleast_2d(topk)
    mask = np.asarray(mask, dtype=bool)
    kind = np.where(mask[topk], KIND_KEPT, KIND_ONDEMAND).astype(np.uint8)
    return topk.astype(np.int64).copy(), kind, np.zeros(topk.shape[0], dtype=np.int64)


# --------------------------------------------------- co-activation profiling
def random_plan(topk, mask, rng):
    """substitution.py:227-248 for a batch, one shared numpy Generator in
    token order (harness.py:358-359): kept if resident, else a uniform draw
    rng.integers(0, n) from the resident experts not yet assigned to the
    token (ascending), else ondemand. Returns (executed, kind, used)."""
    topk = np.asarray(topk)
    mask = np.asarray(mask, bool)
    B, k = topk.shape
    ex = topk.astype(np.int64).copy()
    kd = np.zeros((B, k), np.uint8)
    used = np.zeros(B, np.int64)
    res = np.flatnonzero(mask)
    for b in range(B):
        taken = np.zeros(mask.size, bool)
        taken[topk[b]] = True
        for s in range(k):
            o = int(topk[b, s])
            if mask[o]:
                continue
            pool = res[~taken[res]]
            if pool.size == 0:
                kd[b, s] = KIND_ONDEMAND
                continue
            j = int(pool[rng.integers(0, pool.size)])
            ex[b, s], kd[b, s] = j, KIND_SUBSTITUTED
            taken[j] = True
            used[b] += 1
    return ex, kd, used


def coact_count(topk, probs, num_experts, tok0=0, warmup_steps=256, warmup_weight=0.0):
    """observe() folded over a trace, profiler.py:67-95.

    Token t (global index tok0+t) has weight warmup_weight if its index is
    below warmup_steps, else 1. np.bincount accumulates each cell strictly
    in input order, which is the reference's per-cell order (token, a, b),
    so all three outputs are bit-identical to repeated observe() calls.
    Returns (counts[E], pair_counts[E,E], pair_weights[E,E], tokens_seen).
    """
    topk = np.asarray(topk, dtype=np.int64)
    N, k = topk.shape
    E = int(num_experts)
    step = tok0 + np.arange(N)
    w = np.where(step < warmup_steps, float(warmup_weight), 1.0)
    counts = np.zeros(E)
    pairs = np.zeros(E * E)
    pw = np.zeros(E * E)
    live = w != 0.0                       # profiler.py:83-84: w == 0 returns early
    tk, ww = topk[live], w[live]
    if tk.size:
        counts += np.bincount(tk.ravel(), weights=np.repeat(ww, k), minlength=E)
        a_idx, b_idx = np.triu_indices(k, 1)
        i, j = tk[:, a_idx], tk[:, b_idx]
        # interleave (i,j) and (j,i) per pair so each cell sees token order
        cells = np.stack([i * E + j, j * E + i], axis=-1).ravel()
        wrep = np.repeat(ww, 2 * a_idx.size)
        pairs += np.bincount(cells, weights=wrep, minlength=E * E)
        if probs is not None:
            p = np.asarray(probs, dtype=np.float64)[live]
            m = ww[:, None] * np.minimum(p[:, a_idx], p[:, b_idx])
            mrep = np.repeat(m.ravel(), 2)
            pw += np.bincount(cells, weights=mrep, minlength=E * E)
    return counts, pairs.reshape(E, E), pw.reshape(E, E), N


def pairwise_sum(a) -> float:
    """numpy's pairwise summation for a contiguous float64 vector
    (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE=128), restated so
    the CUDA ranking kernel can follow the same order."""
    a = [float(v) for v in a]

    def rec(lo, n):
        if n < 8:
            res = 0.0
            for i in range(n):
                res += a[lo + i]
            return res
        if n <= 128:
            r = a[lo:lo + 8]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[lo + i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[lo + i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return rec(lo, n2) + rec(lo + n2, n - n2)

    return rec(0, len(a))


def conditional_row(pair_matrix, pivot: int, eps: float):
    """profiler.py:98-119. Returns q or None for a degenerate pivot."""
    row = np.asarray(pair_matrix[pivot], dtype=np.float64).copy()
    row += eps
    row[pivot] = 0.0
    total = row.sum()
    if total <= 0.0:
        return None
    return row / total


def build_table(pair_matrix, eps: float, alpha: float, k_max: int):
    """build_table + cft_prefix, buddies.py:79-129 → dense (ids, weights, lens)."""
    M = np.asarray(pair_matrix, dtype=np.float64)
    E = M.shape[0]
    ids = np.full((E, k_max), -1, dtype=np.int32)
    wts = np.zeros((E, k_max), dtype=np.float64)
    lens = np.zeros(E, dtype=np.int32)
    for p in range(E):
        q = conditional_row(M, p, eps)
        if q is None:
            continue
        order = np.argsort(-q, kind="stable")
        sq = q[order]
        nnz = int(np.count_nonzero(sq))
        cum = np.cumsum(sq[:nnz])
        t = int(np.searchsorted(cum, alpha - _COVER_TOL, side="left")) + 1
        n = min(min(t, nnz), k_max)
        ids[p, :n] = order[:n]
        wts[p, :n] = q[order[:n]]
        lens[p] = n
    return ids, wts, lens


def build_table_scalar(pair_matrix, eps: float, alpha: float, k_max: int):
    """The same table through the scalar recipe the CUDA kernel follows
    (SURVEY App. B.5): numpy-order pairwise total, sort key (-q, j),
    sequential cumsum, first index with cum >= alpha - 1e-9."""
    M = np.asarray(pair_matrix, dtype=np.float64)
    E = M.shape[0]
    ids = np.full((E, k_max), -1, dtype=np.int32)
    wts = np.zeros((E, k_max), dtype=np.float64)
    lens = np.zeros(E, dtype=np.int32)
    for p in range(E):
        row = [float(M[p, j]) + eps for j in range(E)]
        row[p] = 0.0
        total = pairwise_sum(row)
        if total <= 0.0:
            continue
        q = [v / total for v in row]
        order = sorted(range(E), key=lambda j: (-q[j], j))
        nnz = sum(1 for v in q if v != 0.0)
        cum, t = 0.0, nnz
        for r in range(nnz):
            cum += q[order[r]]
            if cum >= alpha - _COVER_TOL:
                t = r + 1
                break
        n = min(t, k_max)
        for r in range(n):
            ids[p, r] = order[r]
            wts[p, r] = q[order[r]]
        lens[p] = n
    return ids, wts, lens


def table_from_lists(ids_list, w_list, k_max):
    """Dense (ids, weights, lens) from per-pivot arrays (BuddyTable._ids)."""
    E = len(ids_list)
    ids = np.full((E, k_max), -1, dtype=np.int32)
    wts = np.zeros((E, k_max), dtype=np.float64)
    lens = np.zeros(E, dtype=np.int32)
    for p in range(E):
        n = min(len(ids_list[p]), k_max)
        ids[p, :n] = np.asarray(ids_list[p][:n])
        wts[p, :n] = np.asarray(w_list[p][:n])
        lens[p] = n
    return ids, wts, lens


# ------------------------------------------------------------ expert FFN
def ffn_tanh(x, w_in, w_out):
    """Expert.__call__, model.py:85-99: tanh(x @ w_in) @ w_out, w_in[d,f], w_out[f,d]."""
    return np.tanh(np.asarray(x, np.float64) @ w_in) @ w_out


def silu(v):
    return v / (1.0 + np.exp(-v))


def ffn_swiglu(x, w1, w3, w2):
    """SwiGLU expert (Mixtral/Qwen3/DSV2 convention; no reference oracle —
    parity pinned by restatement only): w1,w3 [f,d], w2 [d,f]."""
    x = np.asarray(x, np.float64)
    return (silu(x @ w1.T) * (x @ w3.T)) @ w2.T


def forward(x, executed, kind, probs, expert_fn):
    """forward_batch combine semantics, model.py:318-340: weights are the
    ORIGINAL renormalised probabilities, dropped slots contribute 0 and the
    remaining mass is not renormalised. expert_fn(e, x_rows) -> y_rows."""
    x = np.atleast_2d(np.asarray(x, np.float64))
    B, k = np.asarray(executed).shape
    y = np.zeros_like(x)
    for b in range(B):
        for s in range(k):
            if kind[b][s] == KIND_DROPPED:
                continue
            y[b] += probs[b][s] * expert_fn(int(executed[b][s]), x[b:b + 1])[0]
    return y


def layer_update(h, y):
    """model.py:343-347."""
    h = h + _RESIDUAL_SCALE * y
    rms = np.sqrt(np.mean(np.square(h), axis=-1, keepdims=True))
    return h / np.maximum(rms, 1e-12)


# ------------------------------------------------------ expert cache replica
POLICY_LRU, POLICY_LFU, POLICY_FREQ_STATIC = 0, 1, 2
EV_HIT, EV_MISS_ONDEMAND, EV_MISS_SUBSTITUTED = 0, 1, 2
EV_PREFETCH_ISSUE, EV_PREFETCH_COMPLETE, EV_EVICT, EV_DROP = 3, 4, 5, 6
EV_NAMES = ("hit", "miss_ondemand", "miss_substituted", "prefetch_issue",
            "prefetch_complete", "evict", "drop")


def initial_residents(num_experts, capacity, policy, seed=0, layer=0, static_freq=None):
    """ResidencyState.__init__ initial set, memtier.py:127-140."""
    if capacity <= 0:
        return []
    if policy == POLICY_FREQ_STATIC:
        order = np.lexsort((np.arange(num_experts), -np.asarray(static_freq, np.float64)))
        initial = order[:capacity]
    else:
        rng = np.random.default_rng(np.random.SeedSequence([seed, 21, layer]))
        initial = rng.permutation(num_experts)[:capacity]
    return sorted(int(v) for v in initial)


class Residency:
    """ResidencyState replica, memtier.py:96-198."""

    def __init__(self, num_experts, capacity, policy, initial, static_freq=None, layer=0):
        self.E, self.capacity, self.policy, self.layer = num_experts, capacity, policy, layer
        self.mask = np.zeros(num_experts, dtype=bool)
        self.last_use = np.zeros(num_experts, dtype=np.int64)
        self.freq = np.zeros(num_experts)
        self.static = None if static_freq is None else np.asarray(static_freq, np.float64)
        self.tick = 0
        self.unused_prefetch = np.zeros(num_experts, dtype=bool)
        self.pending = []
        self.waste_evictions = 0
        for e in initial:
            self.mask[e] = True
            self.touch(e)

    def touch(self, e):                                     # memtier.py:156-160
        self.tick += 1
        self.last_use[e] = self.tick
        self.freq[e] += 1.0
        self.unused_prefetch[e] = False

    def victim(self):                                       # memtier.py:162-170
        res = np.flatnonzero(self.mask)
        if self.policy == POLICY_LRU:
            sc = self.last_use[res]
        elif self.policy == POLICY_LFU:
            sc = self.freq[res]
        else:
            sc = self.static[res]
        return int(res[int(np.argmin(sc))])

    def insert(self, e, via_prefetch=False):                # memtier.py:172-195
        if self.capacity == 0:
            return None
        victim = None
        if not self.mask[e]:
            if int(self.mask.sum()) >= self.capacity:
                victim = self.victim()
                self.mask[victim] = False
                if self.unused_prefetch[victim]:
                    self.waste_evictions += 1
                    self.unused_prefetch[victim] = False
                self.freq[victim] = 0.0
            self.mask[e] = True
        if via_prefetch:
            self.freq[e] = 0.0
            self.tick += 1
            self.last_use[e] = self.tick
            self.unused_prefetch[e] = True
        else:
            self.touch(e)
        return victim


class Clock:
    """SimClock + PcieChannel, memtier.py:72-93."""

    def __init__(self):
        self.now = 0.0
        self.free_at = 0.0

    def acquire(self, now, dur):
        start = max(now, self.free_at)
        done = start + dur
        self.free_at = done
        return done


def access(st: Residency, e, clock: Clock, load_ms, hit_ms, expert_bytes,
           substituted_away=False, token=-1, log=None):
    """memtier.py:217-254. Events are (time, kind, layer, token, expert, bytes, stall)."""
    start = clock.now
    if st.mask[e]:
        st.touch(e)
        clock.now += hit_ms
        ev = (start, EV_HIT, st.layer, token, e, 0, hit_ms)
    elif substituted_away:
        clock.now += hit_ms
        ev = (start, EV_MISS_SUBSTITUTED, st.layer, token, e, 0, hit_ms)
    else:
        done = clock.acquire(start, load_ms)
        stall = done - start
        clock.now = done
        victim = st.insert(e)
        ev = (start, EV_MISS_ONDEMAND, st.layer, token, e, expert_bytes, stall)
        if log is not None:
            log.append(ev)
            if victim is not None:
                log.append((clock.now, EV_EVICT, st.layer, -1, victim, 0, 0.0))
        return ev
    if log is not None:
        log.append(ev)
    return ev


def prefetch(st: Residency, experts, clock: Clock, prefetch_ms, log=None):
    """memtier.py:257-280."""
    inflight = {e for _, e in st.pending}
    for e in experts:
        e = int(e)
        if st.mask[e] or e in inflight:
            continue
        done = clock.acquire(clock.now, prefetch_ms)
        st.pending.append((done, e))
        inflight.add(e)
        if log is not None:
            log.append((clock.now, EV_PREFETCH_ISSUE, st.layer, -1, e, 0, 0.0))


def settle(st: Residency, clock: Clock, expert_bytes, log=None):
    """memtier.py:283-300."""
    remaining = []
    for done, e in st.pending:
        if done <= clock.now:
            victim = st.insert(e, via_prefetch=True)
            if log is not None:
                log.append((done, EV_PREFETCH_COMPLETE, st.layer, -1, e, expert_bytes, 0.0))
                if victim is not None:
                    log.append((done, EV_EVICT, st.layer, -1, victim, 0, 0.0))
        else:
            remaining.append((done, e))
    st.pending = remaining


def predict_for_layer(capacity, prev_counts: dict):
    """_predict_for_layer, harness.py:209-218."""
    if not prev_counts:
        return []
    m = max(0, capacity - len(prev_counts))
    if m == 0:
        return []
    ranked = sorted(prev_counts.items(), key=lambda kv: (-kv[1], kv[0]))
    return [e for e, _ in ranked[:m]]
