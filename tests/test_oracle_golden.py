"""Pin the CPU oracle to the reference's own outputs (golden vectors made by
tests/golden/make_golden.py, which imports the reference). CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import golden


def _corpus(name):
    g = golden(name)
    n = g["E"].shape[0]
    for i in range(n):
        E, k = int(g["E"][i]), int(g["k"][i])
        yield dict(E=E, k=k, topk=g["topk"][i, :k], logits=g["logits"][i, :E], mask=g["mask"][i, :E],
                   ids=g["ids"][i], w=g["w"][i], lens=g["lens"][i], h=int(g["h"][i]),
                   rho=int(g["rho"][i]), allowed=bool(g["allowed"][i]), eta=float(g["eta"][i]),
                   kappa=float(g["kappa"][i]),
                   part=g["part"][i, :E] if g["has_part"][i] else None,
                   fallback=int(g["fallback"][i]), executed=g["executed"][i, :k],
                   kind=g["kind"][i, :k], used=int(g["used"][i]))


@pytest.mark.parametrize("name", ["remap_corpus_20260819.npz", "remap_corpus_1234.npz"])
def test_remap_oracle_matches_reference_corpus(name):
    n = 0
    for c in _corpus(name):
        ex, kd, used = O.remap_token(c["topk"], c["logits"], c["mask"], c["ids"], c["w"], c["lens"],
                                     c["allowed"], c["h"], c["rho"], fallback=c["fallback"],
                                     eta=c["eta"], kappa=c["kappa"], partition_of=c["part"], hop=1.0)
        assert list(ex) == list(c["executed"]) and list(kd) == list(c["kind"]) and used == c["used"]
        n += 1
    assert n in (1000, 300)


@pytest.mark.parametrize("name", ["routing_tiny.npz", "routing_default.npz", "routing_e128.npz"])
def test_route_oracle_matches_reference(name):
    g = golden(name)
    k = g["topk"].shape[1]
    z, tk, pr = O.route(g["x"], g["gate_w"], g["gate_b"], k, float(g["T"]))
    np.testing.assert_allclose(z, g["logits"], rtol=0, atol=1e-12)
    assert np.array_equal(tk, g["topk"])
    np.testing.assert_allclose(pr, g["probs"], rtol=1e-12, atol=0)
    # selection from the reference's own logits is exactly the reference's
    tk2, pr2 = O.select_topk(g["logits"], k, float(g["T"]))
    assert np.array_equal(tk2, g["topk"]) and np.array_equal(pr2, g["probs"])
    t = np.array([O.tae(p) for p in g["probs"]])
    m = np.array([O.margin(p) for p in g["probs"]])
    assert np.array_equal(t, g["tae"]) and np.array_equal(m, g["margin"])


def test_gate_known_answers():
    # reference tests/test_gating.py:25-69 and test_acceptance.py:112-128
    assert O.tae(np.full(6, 1 / 6)) == pytest.approx(1.0, abs=1e-9)
    assert O.tae(np.array([1.0, 0.0])) == 0.0
    assert O.tae(np.array([0.75, 0.25])) == pytest.approx(0.8113, abs=1e-4)
    assert O.tae(np.array([1.0])) == 0.0
    assert O.margin(np.array([0.75, 0.25])) == pytest.approx(0.5, abs=1e-12)
    mask = np.zeros(8, bool)
    mask[[0, 1, 2]] = True
    assert O.distribution_gate([0, 1, 2, 3, 4, 5], mask, 0.6) == (0.5, True)
    assert O.distribution_gate([0, 1, 2, 3, 4, 5], mask, 0.5) == (0.5, False)
    assert O.distribution_gate([3, 3, 0], mask, 1.0)[0] == pytest.approx(2 / 3)
    # nearest-rank tau (test_gating.py:94-104)
    s = np.arange(1, 101) / 100.0
    assert O.calibrate_tau(s, 15.0) == 0.15
    assert O.calibrate_tau(s, 0.0) == 0.01
    assert O.calibrate_tau(s, 100.0) == 1.0


@pytest.mark.parametrize("name", ["coact_tiny.npz", "coact_default_w05.npz", "coact_e128.npz",
                                  "coact_e160_noeps.npz"])
def test_coact_and_table_oracle_match_reference(name):
    g = golden(name)
    E = int(g["E"])
    c, pc, pw, seen = O.coact_count(g["topk"], g["probs"], E, 0, int(g["warmup_steps"]),
                                    float(g["warmup_weight"]))
    assert seen == int(g["tokens_seen"])
    assert np.array_equal(c, g["counts"]) and np.array_equal(pc, g["pairs"])
    assert np.array_equal(pw, g["pw"])          # bincount keeps the per-cell order
    for i in range(int(g["nbuild"])):
        alpha, kmax, mode = float(g[f"b{i}_alpha"]), int(g[f"b{i}_kmax"]), str(g[f"b{i}_mode"])
        M = g["pairs"] if mode == "binary" else g["pw"]
        ids, w, lens = O.build_table(M, float(g["eps"]), alpha, kmax)
        assert np.array_equal(ids, g[f"b{i}_ids"]) and np.array_equal(lens, g[f"b{i}_lens"])
        assert np.array_equal(w, g[f"b{i}_w"])
        if E <= 128:    # the scalar recipe is slow in Python; E=160 runs it on a subset below
            ids2, w2, lens2 = O.build_table_scalar(M, float(g["eps"]), alpha, kmax)
            assert np.array_equal(ids2, ids) and np.array_equal(w2, w) and np.array_equal(lens2, lens)


def test_pairwise_sum_matches_numpy():
    rng = np.random.default_rng(0)
    for n in list(range(0, 300)) + [511, 512, 513, 1000, 1024, 4099]:
        a = rng.standard_normal(n) * 10 ** rng.uniform(-3, 3, n)
        assert O.pairwise_sum(a) == float(a.sum()), n


def test_sharded_counts_merge_equals_single_pass():
    # profiler.merge contract (test_profiler.py:116-132): shards sum to the whole
    g = golden("coact_e128.npz")
    E = int(g["E"])
    tk, pr = g["topk"], g["probs"]
    cut = [0, 700, 1900, tk.shape[0]]
    tot = np.zeros((E, E))
    seen = 0
    for a, b in zip(cut[:-1], cut[1:]):
        _, pc, _, n = O.coact_count(tk[a:b], pr[a:b], E, a, int(g["warmup_steps"]), 0.0)
        tot += pc
        seen += n
    assert np.array_equal(tot, g["pairs"]) and seen == int(g["tokens_seen"])


@pytest.mark.parametrize("idx,pol", [(0, "lru"), (1, "lfu"), (2, "freq_static"), (3, "lru")])
def test_memtier_oracle_replays_reference_events(idx, pol):
    g = golden(f"memtier_{idx}_{pol}.npz")
    E, rate, policy, seed, layer = int(g["E"]), float(g["rate"]), int(g["policy"]), int(g["seed"]), int(g["layer"])
    cap = int(np.floor(rate * E))
    static = g["static"] if policy == O.POLICY_FREQ_STATIC else None
    st = O.Residency(E, cap, policy, O.initial_residents(E, cap, policy, seed, layer, static),
                     static, layer)
    clock, log = O.Clock(), []
    load_ms, hit_ms, nbytes = 9.5, 0.25, 32768
    pre_ms = 1000.0 * nbytes / 4.0e6
    buf, tok = [], 0
    for op, a, b in g["prog"]:
        tok += 1
        if op == 0:
            O.access(st, int(a), clock, load_ms, hit_ms, nbytes, token=tok, log=log)
        elif op == 1:
            O.access(st, int(a), clock, load_ms, hit_ms, nbytes, substituted_away=True, token=tok, log=log)
        elif op == 2:
            if a < 0:
                O.prefetch(st, buf, clock, pre_ms, log=log)
                buf = []
            else:
                buf.append(int(a))
        elif op == 3:
            O.settle(st, clock, nbytes, log=log)
        else:
            clock.now += b / 2.0
    ev = np.array(log, np.float64).reshape(-1, 7)
    assert ev.shape == g["events"].shape
    assert np.array_equal(ev, g["events"])
    assert np.array_equal(st.mask, g["final_mask"]) and np.array_equal(st.last_use, g["final_last_use"])
    assert np.array_equal(st.freq, g["final_freq"]) and st.waste_evictions == int(g["waste"])


@pytest.mark.parametrize("name", ["mixtral", "qwen3", "dsv2"])
def test_oracle_at_baseline_shapes(name):
    """The oracle's f64 routing reproduces the reference's at the BASELINE
    shapes (first 512 tokens, regenerated by the substrate restatement), and
    its counts / table over the reference's routing are bit-exact."""
    from paper_2511_10054_b200 import substrate
    g = golden(f"routing_{name}.npz")
    E, k, d = int(g["E"]), int(g["k"]), int(g["d"])
    spec = substrate.ModelSpec(num_layers=1, experts_per_layer=E, top_k=k, hidden_dim=d, ffn_dim=64,
                               num_clusters=min(E, 8), seed=7)
    gw, gb = substrate.gate_weights(spec)
    x = substrate.token_stream(spec, 2, int(g["n"]))[:512]
    z, tk, pr = O.route(x, gw[0], gb[0], k)
    np.testing.assert_allclose(z, g["logits"][:512], rtol=0, atol=1e-12)
    assert np.array_equal(tk, g["topk"][:512].astype(np.int64))
    c, p, _, _ = O.coact_count(g["topk"].astype(np.int64), None, E, 0, 256, 0.0)
    assert np.array_equal(c, g["counts"]) and np.array_equal(p, g["pairs"])
    ids, w, lens = O.build_table(p, 1e-3, 0.95, min(16, E - 1))
    assert np.array_equal(ids, g["ids"]) and np.array_equal(w, g["w"]) and np.array_equal(lens, g["lens"])
