"""Engine decisions under every cache policy and plan option, checked
against the oracle replay of harness.py:315-393 driven by the routing the
GPU produced (engine trace): LRU / LFU / freq_static eviction, capacity 0
and full, drop fallback (drop events, dropped slots skip compute), rho = 0
and unlimited, prefetch on/off, method original. Bit-exact event logs."""

import numpy as np
import pytest
import torch

import oracle as O
from paper_2511_10054_b200 import ops, substrate
from paper_2511_10054_b200.engine import DecodeEngine, EngineSpec, HostMirror

pytestmark = pytest.mark.gpu

SPEC = substrate.ModelSpec(num_layers=3, experts_per_layer=16, top_k=3, hidden_dim=128, ffn_dim=128,
                           num_clusters=4)
E, K, D, F, L = 16, 3, 128, 128, 3
POL = {"lru": O.POLICY_LRU, "lfu": O.POLICY_LFU, "freq_static": O.POLICY_FREQ_STATIC}


def _tables(rng):
    ids = np.full((L, E, 8), -1, np.int32)
    lens = np.zeros((L, E), np.int32)
    for l in range(L):
        for p in range(E):
            n = int(rng.integers(0, 9))
            c = rng.permutation([j for j in range(E) if j != p])[:n]
            ids[l, p, :n] = c
            lens[l, p] = n
    return ids, lens


def _run(policy="lru", rate=0.5, fallback=0, rho=2, prefetch=True, method="buddy", B=8, steps=6, seed=0):
    rng = np.random.default_rng(seed)
    gw, gb = substrate.gate_weights(SPEC)
    mirrors = []
    for l in range(L):
        w_in, w_out = substrate.layer_stack(SPEC, l)
        a = np.concatenate([np.transpose(w_in, (0, 2, 1)).reshape(E, -1),
                            np.transpose(w_out, (0, 2, 1)).reshape(E, -1)], axis=1).astype(np.float32)
        m = HostMirror(a.nbytes)
        m.as_tensor(torch.float32).copy_(torch.from_numpy(a).view(-1))
        mirrors.append(m)
    ids, lens = _tables(rng)
    static = rng.random((L, E)) if policy == "freq_static" else None
    cap = int(np.floor(rate * E))
    initial = [O.initial_residents(E, cap, POL[policy], 0, l, None if static is None else static[l]) for l in range(L)]
    taus = [0.3, 0.5, 0.7]
    es = EngineSpec(num_layers=L, num_experts=E, top_k=K, d=D, f=F, capacity=cap, max_batch=B, act=ops.ACT_TANH,
                    method=method, policy=policy, search_rank_h=6, rho=rho, fallback=fallback, prefetch=prefetch,
                    fp32_weights=True, expert_bytes=2 * D * F * 8, load_ms=9.5, hit_ms=0.25, compute_ms=0.5,
                    pcie_bw_bytes_per_s=4.0e8)
    eng = DecodeEngine(es, mirrors, torch.tensor(gw, dtype=torch.float32, device="cuda"),
                       torch.tensor(gb, dtype=torch.float32, device="cuda"), torch.from_numpy(ids).cuda(),
                       torch.from_numpy(lens).cuda(), taus, initial, static)
    eng.set_trace(True)
    x = torch.from_numpy(substrate.token_stream(SPEC, 3, steps * B).astype(np.float32)).cuda()
    for s in range(steps):
        eng.step(x[s * B:(s + 1) * B], np.arange(s * B, (s + 1) * B))
    torch.cuda.synchronize()
    ev, tr = eng.events(), eng.trace()
    # ---- oracle replay of the same decisions ----
    st = [O.Residency(E, cap, POL[policy], initial[l], None if static is None else static[l], l) for l in range(L)]
    clock, log, prev = O.Clock(), [], [dict() for _ in range(L)]
    ebytes, pre_ms = es.expert_bytes, 1000.0 * es.expert_bytes / es.pcie_bw_bytes_per_s
    i = 0
    for s in range(steps):
        toks = np.arange(s * B, (s + 1) * B)
        for l in range(L):
            rec = tr[i]
            i += 1
            if prefetch:
                t = (l + 1) % L
                O.prefetch(st[t], O.predict_for_layer(cap, prev[t]), clock, pre_ms, log)
            O.settle(st[l], clock, ebytes, log)
            assert np.array_equal(rec["mask"], st[l].mask)
            if method == "buddy":
                _, bok = O.distribution_gate(rec["topk"].ravel(), st[l].mask, 1.0)
                ex, kd, _ = O.remap_batch(rec["topk"], None, st[l].mask, ids[l], np.zeros(ids[l].shape), lens[l],
                                          rec["allowed"] & bok, 6, -1 if rho is None else rho, fallback=fallback)
            else:
                ex, kd, _ = O.ondemand_plan(rec["topk"], st[l].mask)
            assert np.array_equal(ex, rec["executed"]) and np.array_equal(kd, rec["kind"])
            slots = 0
            for b in range(B):
                for sl in range(K):
                    if kd[b, sl] == O.KIND_DROPPED:
                        log.append((clock.now, O.EV_DROP, l, int(toks[b]), int(rec["topk"][b, sl]), 0, 0.0))
                        continue
                    if kd[b, sl] == O.KIND_SUBSTITUTED:
                        O.access(st[l], int(rec["topk"][b, sl]), clock, 9.5, 0.25, ebytes, True, int(toks[b]), log)
                    O.access(st[l], int(ex[b, sl]), clock, 9.5, 0.25, ebytes, False, int(toks[b]), log)
                    slots += 1
            clock.now += 0.5 * slots
            cnt = {}
            for b in range(B):
                for sl in range(K):
                    if kd[b, sl] != O.KIND_DROPPED:
                        cnt[int(ex[b, sl])] = cnt.get(int(ex[b, sl]), 0) + 1
            prev[l] = cnt
    ref = np.array(log, np.float64).reshape(-1, 7)
    eng.close()
    return ev, ref, x


@pytest.mark.parametrize("kw", [
    dict(policy="lru"), dict(policy="lfu"), dict(policy="freq_static"),
    dict(fallback=1), dict(rho=0), dict(rho=None), dict(prefetch=False), dict(rate=1.0), dict(rate=0.0625),
    dict(method="original"), dict(B=1, steps=12), dict(rate=0.25),
])
def test_engine_policy_matches_oracle(cuda_ok, kw):
    ev, ref, x = _run(**kw)
    assert ev.shape == ref.shape, (ev.shape, ref.shape)
    assert np.array_equal(ev, ref)
    assert np.isfinite(x.cpu().numpy()).all()
