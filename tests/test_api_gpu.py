"""API conformance: the reference-named modules (model, gating,
substitution, profiler, buddies) behave like the reference on its own
known-answer cases, while computing on the GPU kernels."""

import os

import numpy as np
import pytest

import oracle as O
from conftest import golden
from paper_2511_10054_b200 import buddies, gating, model, profiler, substitution
from paper_2511_10054_b200.errors import CalibrationError, DegeneratePivotError, InputError, InternalError

pytestmark = pytest.mark.gpu


def _dec(topk, probs=None, logits=None, E=None, token=0, layer=0):
    topk = np.asarray(topk, np.int64)
    k = topk.size
    probs = np.full(k, 1.0 / k) if probs is None else np.asarray(probs, np.float64)
    E = int(topk.max()) + 1 if E is None else E
    logits = np.zeros(E) if logits is None else np.asarray(logits, np.float64)
    return model.RouterDecision(token, layer, logits, topk, probs, 1.0)


def _table(E, lists, k_max=16):
    ids = [np.array([e for e, _ in lists.get(p, [])], np.int64) for p in range(E)]
    w = [np.array([x for _, x in lists.get(p, [])], np.float64) for p in range(E)]
    return buddies.BuddyTable(0, E, 0.95, k_max, ids, w)


def test_model_routing_and_forward(cuda_ok):
    spec = model.ModelSpec(num_layers=2, experts_per_layer=8, top_k=2, hidden_dim=128, ffn_dim=256, num_clusters=8)
    m = model.build_model(spec)
    x = model.token_stream(spec, 2, 32)
    ds = model.route_batch(m, x, 1, temperature=0.7)
    for d in ds:
        tk, pr = O.select_topk(d.logits[None, :], 2, 0.7)   # selection consistent with returned logits
        assert np.array_equal(d.topk, tk[0]) and np.allclose(d.probs_renorm, pr[0], rtol=1e-12)
        assert abs(d.probs_renorm.sum() - 1.0) < 1e-12
    g = golden("routing_tiny.npz")                            # vs the reference's own f64 routing
    agree = np.mean([np.array_equal(d.topk, t) for d, t in
                     zip(model.route_batch(m, g["x"], 0), g["topk"])])
    assert agree >= 0.99
    # forward = sum_s p~[s] FFN_s(x), original weights, dropped -> 0 (model.py:318-340)
    w_in, w_out = m.layer_stack(1)
    plans = []
    for d in ds:
        slots = (substitution.PlanSlot(int(d.topk[0]), int(d.topk[0]), "kept"),
                 substitution.PlanSlot(int(d.topk[1]), (int(d.topk[1]) + 1) % 8 if (int(d.topk[1]) + 1) % 8 != int(d.topk[0]) else (int(d.topk[1]) + 2) % 8, "substituted"))
        plans.append(substitution.ReplacementPlan(d.token, 1, slots, 1))
    plans[3] = substitution.ReplacementPlan(3, 1, (plans[3].slots[0], substitution.PlanSlot(
        plans[3].slots[1].original, plans[3].slots[1].original, "dropped")), 0)
    y = model.forward_batch(m, x, ds, plans)
    ex = np.array([[s.executed for s in p.slots] for p in plans])
    kd = np.array([[("kept", "substituted", "ondemand_fallback", "dropped").index(s.kind) for s in p.slots]
                   for p in plans])
    ref = O.forward(x, ex, kd, np.stack([d.probs_renorm for d in ds]),
                    lambda e, xr: O.ffn_tanh(xr, w_in[e], w_out[e]))
    # the Python API forward runs the f64 SIMT kernels: the reference's precision
    assert np.max(np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)) <= 1e-12
    h = model.layer_update(x, y)
    assert np.allclose(np.sqrt(np.mean(h ** 2, axis=1)), 1.0, atol=1e-12)
    np.testing.assert_allclose(h, O.layer_update(x, y), rtol=0, atol=1e-13)
    bad = [substitution.ReplacementPlan(0, 1, (substitution.PlanSlot(0, 9, "substituted"),
                                               substitution.PlanSlot(1, 1, "kept")), 1)] + plans[1:]
    with pytest.raises(InternalError):
        model.forward_batch(m, x, ds, bad)
    # ties select the lower index (test_model.py:115-120 analogue)
    tk, _ = O.select_topk(np.zeros((1, 8)), 4)
    assert tk.tolist() == [[0, 1, 2, 3]]


def test_gating_known_answers(cuda_ok):
    assert gating.tae(_dec([0, 1, 2, 3, 4, 5])) == pytest.approx(1.0, abs=1e-9)
    assert gating.tae(_dec([0, 1], [1.0, 0.0])) == 0.0
    assert gating.tae(_dec([0, 1], [0.75, 0.25])) == pytest.approx(0.8113, abs=1e-4)
    assert gating.tae(_dec([3], [1.0])) == 0.0
    assert gating.margin(_dec([0, 1], [0.75, 0.25])) == pytest.approx(0.5, abs=1e-12)
    cfg = gating.GateConfig(tau=gating.tae(_dec([0, 1], [0.75, 0.25])), tau_percentile=None)
    assert not gating.token_gate(_dec([0, 1], [0.75, 0.25]), cfg)        # h <= tau is inclusive
    mask = np.zeros(8, bool)
    mask[[0, 1, 2]] = True
    assert gating.distribution_gate([0, 1, 2, 3, 4, 5], mask, 0.6) == (0.5, True)
    assert gating.distribution_gate([0, 1, 2, 3, 4, 5], mask, 0.5) == (0.5, False)
    assert gating.distribution_gate([3, 3, 0], mask, 1.0)[0] == pytest.approx(2 / 3)
    s = np.arange(1, 101) / 100.0
    assert gating.calibrate_tau(s, 15.0) == 0.15 and gating.calibrate_tau(s, 0.0) == 0.01
    assert gating.calibrate_tau(s, 100.0) == 1.0
    with pytest.raises(CalibrationError):
        gating.calibrate_tau(s[:99], 15.0)
    g = golden("routing_default.npz")
    ds = [_dec(t, p, z, 64) for t, p, z in zip(g["topk"], g["probs"], g["logits"])]
    outs = gating.evaluate_gates(ds, np.arange(64) % 3 == 0, gating.GateConfig(tau=0.5, tau_percentile=None))
    t, m, ok, delta, bok = O.gate_batch(g["probs"], g["topk"], np.arange(64) % 3 == 0, 0.5)
    assert np.allclose([o.tae for o in outs], t, atol=1e-12) and [o.token_allowed for o in outs] == list(ok)
    assert all(o.delta == delta and o.batch_allowed == bok for o in outs)


def test_substitution_matches_reference_corpus(cuda_ok):
    g = golden("remap_corpus_1234.npz")
    for i in range(g["E"].shape[0]):
        E, k = int(g["E"][i]), int(g["k"][i])
        lists = {p: list(zip(g["ids"][i, p, :g["lens"][i, p]].tolist(), g["w"][i, p, :g["lens"][i, p]].tolist()))
                 for p in range(E)}
        table = _table(E, lists)
        d = _dec(g["topk"][i, :k], None, g["logits"][i, :E], E)
        cfg = substitution.SubstitutionConfig(int(g["h"][i]), None if g["rho"][i] < 0 else int(g["rho"][i]),
                                              ("prefetch_original", "drop_expert")[int(g["fallback"][i])])
        params = substitution.PsiParams(eta=float(g["eta"][i]), kappa=float(g["kappa"][i]))
        topo = substitution.Topology(g["part"][i, :E] if g["has_part"][i] else None, 1.0)
        gates = gating.GateOutcome(bool(g["allowed"][i]), True, 1.0, 0.0, 0.0)
        plan = substitution.substitute_token(d, g["mask"][i, :E], table, gates, cfg, params, topo)
        assert [s.executed for s in plan.slots] == list(g["executed"][i, :k])
        kinds = ("kept", "substituted", "ondemand_fallback", "dropped")
        assert [s.kind for s in plan.slots] == [kinds[c] for c in g["kind"][i, :k]]
        assert plan.replacements_used == int(g["used"][i])
        substitution.check_plan(plan, d, g["mask"][i, :E], table, cfg)
    d = _dec([3, 1, 4], E=8)
    mask = np.zeros(8, bool)
    mask[[1, 2]] = True
    assert [s.kind for s in substitution.ondemand_plan(d, mask).slots] == ["ondemand_fallback", "kept",
                                                                           "ondemand_fallback"]
    assert all(s.kind == "kept" for s in substitution.identity_plan(d).slots)


def test_profiler_and_buddies(cuda_ok, tmp_path):
    g = golden("coact_default_w05.npz")
    E = int(g["E"])
    st = profiler.CoActivationStats(0, E, int(g["warmup_steps"]), float(g["warmup_weight"]), float(g["eps"]))
    ds = [_dec(t, p, None, E, token=i) for i, (t, p) in enumerate(zip(g["topk"], g["probs"]))]
    profiler.observe_batch(st, ds[:700])
    for i in range(700, 710):
        profiler.observe(st, ds[i], i)
    profiler.observe_batch(st, ds[710:])
    assert np.array_equal(st.counts, g["counts"]) and np.array_equal(st.pair_counts, g["pairs"])
    assert np.allclose(st.pair_weights, g["pw"], rtol=1e-5) and st.tokens_seen == int(g["tokens_seen"])
    q = profiler.conditional_row(st, 5).q
    assert np.array_equal(q, O.conditional_row(g["pairs"], 5, float(g["eps"])))
    for i in range(int(g["nbuild"])):
        alpha, kmax, mode = float(g[f"b{i}_alpha"]), int(g[f"b{i}_kmax"]), str(g[f"b{i}_mode"])
        if mode != "binary":
            continue
        t = buddies.build_table(st, alpha, kmax, mode)
        for p in range(E):
            n = int(g[f"b{i}_lens"][p])
            assert np.array_equal(t.ids(p), g[f"b{i}_ids"][p, :n]) and np.array_equal(t.weights(p), g[f"b{i}_w"][p, :n])
        assert t.k_max == kmax
    # cft_prefix vs brute force (test_buddies.py:29-57 analogue)
    rng = np.random.default_rng(0)
    for _ in range(50):
        qv = rng.random(12) * (rng.random(12) < 0.7)
        qv /= qv.sum()
        alpha = float(rng.uniform(0.1, 1.0))
        t = buddies.cft_prefix(profiler.ConditionalRow(0, qv), alpha)
        top = np.sort(qv)[::-1]
        assert top[:t].sum() >= alpha - 1e-9 - 1e-15 or t == np.count_nonzero(qv)
        assert t == 1 or top[:t - 1].sum() < alpha - 1e-9
    # BSST / BSBT round trips
    p = tmp_path / "s.bin"
    profiler.save_stats(st, p)
    st2 = profiler.load_stats(p)
    assert np.array_equal(st2.pair_counts, st.pair_counts) and st2.tokens_seen == st.tokens_seen
    t = buddies.build_table(st2, 0.95, 16)
    buddies.save_table(t, tmp_path / "t.bin")
    t2 = buddies.load_table(tmp_path / "t.bin")
    assert all(np.array_equal(t.ids(p), t2.ids(p)) for p in range(E))
    # merge == single stream (profiler.merge contract)
    a = profiler.CoActivationStats(0, E, 256, 0.5, 1e-3)
    b = profiler.CoActivationStats(0, E, 256, 0.5, 1e-3)
    profiler.observe_batch(a, ds[:256])
    profiler.observe_batch(b, ds[256:])
    m = profiler.merge(a, b)
    assert np.array_equal(m.pair_counts, g["pairs"])
    # degenerate pivot with eps = 0
    z = profiler.CoActivationStats(0, 8, 0, 0.0, 0.0)
    profiler.observe(z, _dec([0, 1], E=8), 0)
    with pytest.raises(DegeneratePivotError):
        profiler.conditional_row(z, 5)
    with pytest.raises(InputError):
        profiler.observe(z, _dec([2, 2], E=8), 1)
