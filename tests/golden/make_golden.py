"""Generate golden vectors by running the REFERENCE ``buddysim`` package.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src (and the reference
test helpers from /root/reference/pkg/tests) and writes small ``.npz``
fixtures next to this script. Nothing on the GPU box reads /root/reference;
the committed fixtures are what travels. Every fixture is produced by the
reference's own functions, so the oracle (``oracle/``) and the CUDA path are
both pinned to the reference, not to each other.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = os.environ.get("BUDDYSIM_REF", "/root/reference/pkg")
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))

import buddysim  # noqa: E402
from buddysim import buddies, gating, harness, memtier, profiler, substitution  # noqa: E402
from buddysim.config import default_config, parse_config_text  # noqa: E402
from buddysim.gating import GateOutcome  # noqa: E402
from buddysim.model import ModelSpec, build_model, forward_batch, layer_update, route_batch, token_stream  # noqa: E402
from buddysim.substitution import PsiParams, SubstitutionConfig, Topology  # noqa: E402
from conftest import make_decision, random_instance  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
KIND = {"kept": 0, "substituted": 1, "ondemand_fallback": 2, "dropped": 3}
EV = {"hit": 0, "miss_ondemand": 1, "miss_substituted": 2, "prefetch_issue": 3,
      "prefetch_complete": 4, "evict": 5, "drop": 6}
POL = {"lru": 0, "lfu": 1, "freq_static": 2}

EMAX, KMAXI, HMAX = 32, 6, 16


def remap_corpus(seed: int, n: int) -> dict:
    """random_instance corpus (reference tests/conftest.py:129-171) planned by
    the reference substitute_token (substitution.py:146-190)."""
    rng = np.random.default_rng(seed)
    f = {k: [] for k in ("E", "k", "topk", "logits", "mask", "ids", "w", "lens", "h", "rho",
                         "allowed", "eta", "kappa", "part", "has_part", "fallback",
                         "executed", "kind", "used")}
    for _ in range(n):
        inst = random_instance(rng)
        d, mask, table = inst["decision"], inst["mask"], inst["table"]
        E, k = table.num_experts, len(d.topk)
        gates = GateOutcome(inst["allowed"], True, 1.0, 0.0, 0.0)
        cfg = SubstitutionConfig(search_rank_h=inst["h"], rho=inst["rho"], fallback=inst["fallback"])
        plan = substitution.substitute_token(
            d, mask, table, gates, cfg, PsiParams(eta=inst["eta"], kappa=inst["kappa"]),
            Topology(partition_of=inst["partition_of"], hop=1.0))
        ids = np.full((EMAX, HMAX), -1, np.int32)
        w = np.zeros((EMAX, HMAX))
        lens = np.zeros(EMAX, np.int32)
        for p in range(E):
            li = table.ids(p)
            ids[p, :len(li)] = li
            w[p, :len(li)] = table.weights(p)
            lens[p] = len(li)
        pad = lambda a, n, v, dt: np.concatenate([np.asarray(a, dt), np.full(n - len(a), v, dt)])
        f["E"].append(E); f["k"].append(k)
        f["topk"].append(pad(d.topk, KMAXI, -1, np.int32))
        f["logits"].append(pad(d.logits, EMAX, 0.0, np.float64))
        f["mask"].append(pad(mask, EMAX, False, bool))
        f["ids"].append(ids); f["w"].append(w); f["lens"].append(lens)
        f["h"].append(inst["h"]); f["rho"].append(-1 if inst["rho"] is None else inst["rho"])
        f["allowed"].append(inst["allowed"]); f["eta"].append(inst["eta"]); f["kappa"].append(inst["kappa"])
        po = inst["partition_of"]
        f["has_part"].append(po is not None)
        f["part"].append(pad([] if po is None else po, EMAX, 0, np.int32))
        f["fallback"].append(0 if inst["fallback"] == substitution.FALLBACK_PREFETCH else 1)
        f["executed"].append(pad([s.executed for s in plan.slots], KMAXI, -1, np.int32))
        f["kind"].append(pad([KIND[s.kind] for s in plan.slots], KMAXI, 255, np.uint8))
        f["used"].append(plan.replacements_used)
    return {k: np.asarray(v) for k, v in f.items()}


def routing_case(spec: ModelSpec, stream_seed: int, n: int, layer: int = 0, T: float = 1.0) -> dict:
    """route_batch (model.py:231-280) on the reference's own substrate."""
    m = build_model(spec)
    x = token_stream(spec, stream_seed, n)
    ds = route_batch(m, x, layer, T)
    probs = np.stack([d.probs_renorm for d in ds])
    return dict(x=x, gate_w=m.gate_w[layer], gate_b=m.gate_b[layer], T=T,
                logits=np.stack([d.logits for d in ds]), topk=np.stack([d.topk for d in ds]),
                probs=probs, tae=np.array([gating.tae(d) for d in ds]),
                margin=np.array([gating.margin(d) for d in ds]))


def routing_shape_case(E: int, k: int, d: int, n: int, n_logits: int = 1024) -> dict:
    """route_batch at a BASELINE shape (Mixtral 8/2/4096, Qwen3 128/8/2048,
    DSV2-Lite 64/6/2048) on the reference substrate with the bench's router
    spec (seed 7, min(E, 8) clusters; token stream seed 2), then observe over
    every routed token (warm-up 256, weight 0) and build_table (alpha 0.95,
    k_max 16). The tokens are not stored: substrate.token_stream regenerates
    them bit-identically. Logits/probs are kept for the first n_logits rows."""
    spec = ModelSpec(num_layers=1, experts_per_layer=E, top_k=k, hidden_dim=d, ffn_dim=64,
                     num_clusters=min(E, 8), seed=7)
    m = build_model(spec)
    x = token_stream(spec, 2, n)
    ds = route_batch(m, x, 0)
    st = profiler.CoActivationStats(layer=0, num_experts=E, warmup_steps=256, warmup_weight=0.0, laplace_eps=1e-3)
    for dd in ds:
        profiler.observe(st, dd, step=dd.token)
    t = buddies.build_table(st, alpha=0.95, k_max=min(16, E - 1))
    K = min(16, E - 1)
    ids = np.full((E, K), -1, np.int32); w = np.zeros((E, K)); lens = np.zeros(E, np.int32)
    for p in range(E):
        li = t.ids(p); ids[p, :len(li)] = li; w[p, :len(li)] = t.weights(p); lens[p] = len(li)
    return dict(E=E, k=k, d=d, n=n, topk=np.stack([dd.topk for dd in ds]).astype(np.int16),
                logits=np.stack([dd.logits for dd in ds[:n_logits]]),
                probs=np.stack([dd.probs_renorm for dd in ds[:n_logits]]),
                tae=np.array([gating.tae(dd) for dd in ds[:n_logits]]),
                counts=st.counts, pairs=st.pair_counts, ids=ids, w=w, lens=lens)


def coact_case(spec: ModelSpec, n: int, warmup_steps: int, warmup_weight: float, eps: float,
               builds, stream_seed: int = 1) -> dict:
    """observe (profiler.py:67-95) over a routed stream, then build_table
    (buddies.py:102-129) at several (alpha, k_max, mode)."""
    m = build_model(spec)
    x = token_stream(spec, stream_seed, n)
    ds = route_batch(m, x, 0)
    st = profiler.CoActivationStats(layer=0, num_experts=spec.experts_per_layer,
                                    warmup_steps=warmup_steps, warmup_weight=warmup_weight,
                                    laplace_eps=eps)
    for d in ds:
        profiler.observe(st, d, step=d.token)
    out = dict(topk=np.stack([d.topk for d in ds]), probs=np.stack([d.probs_renorm for d in ds]),
               counts=st.counts, pairs=st.pair_counts, pw=st.pair_weights,
               tokens_seen=st.tokens_seen, warmup_steps=warmup_steps,
               warmup_weight=warmup_weight, eps=eps, E=spec.experts_per_layer)
    for i, (alpha, kmax, mode) in enumerate(builds):
        t = buddies.build_table(st, alpha, kmax, mode)
        ids = np.full((t.num_experts, kmax), -1, np.int32)
        w = np.zeros((t.num_experts, kmax))
        lens = np.zeros(t.num_experts, np.int32)
        for p in range(t.num_experts):
            li = t.ids(p)
            ids[p, :len(li)] = li
            w[p, :len(li)] = t.weights(p)
            lens[p] = len(li)
        out[f"b{i}_alpha"], out[f"b{i}_kmax"], out[f"b{i}_mode"] = alpha, kmax, mode
        out[f"b{i}_ids"], out[f"b{i}_w"], out[f"b{i}_lens"] = ids, w, lens
    out["nbuild"] = len(builds)
    return out


def coact_random_case(E: int, k: int, n: int, seed: int, builds, eps=1e-3) -> dict:
    """Skewed random routing at large E (exercises the >128 pairwise-sum split)."""
    rng = np.random.default_rng(seed)
    pop = 1.0 / np.arange(1, E + 1) ** 0.8
    pop /= pop.sum()
    st = profiler.CoActivationStats(layer=0, num_experts=E, warmup_steps=16, warmup_weight=0.0,
                                    laplace_eps=eps)
    tk = np.empty((n, k), np.int64)
    pr = np.empty((n, k))
    for t in range(n):
        ids = rng.choice(E, size=k, replace=False, p=pop)
        p = rng.random(k) + 0.05
        p /= p.sum()
        d = make_decision(ids, p, num_experts=E)
        profiler.observe(st, d, step=t)
        tk[t], pr[t] = ids, p
    out = dict(topk=tk, probs=pr, counts=st.counts, pairs=st.pair_counts, pw=st.pair_weights,
               tokens_seen=st.tokens_seen, warmup_steps=16, warmup_weight=0.0, eps=eps, E=E)
    for i, (alpha, kmax, mode) in enumerate(builds):
        t = buddies.build_table(st, alpha, kmax, mode)
        ids = np.full((E, kmax), -1, np.int32)
        w = np.zeros((E, kmax))
        lens = np.zeros(E, np.int32)
        for p in range(E):
            li = t.ids(p)
            ids[p, :len(li)] = li
            w[p, :len(li)] = t.weights(p)
            lens[p] = len(li)
        out[f"b{i}_alpha"], out[f"b{i}_kmax"], out[f"b{i}_mode"] = alpha, kmax, mode
        out[f"b{i}_ids"], out[f"b{i}_w"], out[f"b{i}_lens"] = ids, w, lens
    out["nbuild"] = len(builds)
    return out


def memtier_case(seed: int, E: int, rate: float, policy: str, nops: int) -> dict:
    """Random access/prefetch/settle program against ResidencyState
    (memtier.py:96-300); records the reference's event log."""
    rng = np.random.default_rng(seed)
    static = rng.random(E) if policy == "freq_static" else None
    st = memtier.init_residency(E, rate, policy, seed=seed, static_freq=static, layer=3)
    cost = memtier.CostModel(expert_load_ms=9.5, hit_ms=0.25, expert_compute_ms=0.5,
                             pcie_bw_bytes_per_s=4.0e6, expert_bytes=32768)
    clock = memtier.SimClock()
    log: list = []
    prog = []  # (op, a, b): op 0 access ondemand, 1 access substituted, 2 prefetch list, 3 settle, 4 advance
    for _ in range(nops):
        r = rng.random()
        if r < 0.55:
            e = int(rng.integers(E)); prog.append((0, e, 0))
            memtier.access(st, e, clock, cost, token=len(prog), log=log)
        elif r < 0.7:
            e = int(rng.integers(E)); prog.append((1, e, 0))
            memtier.access(st, e, clock, cost, mode="substituted_away", token=len(prog), log=log)
        elif r < 0.8:
            es = rng.choice(E, size=int(rng.integers(1, 4)), replace=False)
            for e in es:
                prog.append((2, int(e), 0))
            prog.append((2, -1, 0))  # end of one prefetch call
            memtier.prefetch(st, [int(e) for e in es], clock, cost, log=log)
        elif r < 0.9:
            prog.append((3, 0, 0))
            memtier.settle(st, clock, cost, log=log)
        else:
            ms = float(rng.integers(0, 40)) * 0.5
            prog.append((4, 0, int(ms * 2)))
            clock.advance(ms)
    ev = np.array([(e.time_ms, EV[e.kind], e.layer, e.token, e.expert, e.bytes, e.stall_ms)
                   for e in log], dtype=np.float64).reshape(-1, 7)
    return dict(E=E, rate=rate, policy=POL[policy], seed=seed, layer=3,
                static=np.zeros(E) if static is None else static,
                prog=np.array(prog, np.int64).reshape(-1, 3), events=ev,
                final_mask=st.mask.copy(), final_last_use=st._last_use.copy(),
                final_freq=st._freq.copy(), waste=st.waste_evictions, now=clock.now)


def forward_case(spec: ModelSpec, n: int, seed: int) -> dict:
    """forward_batch + layer_update (model.py:318-347) with a random plan
    that mixes kept / substituted / dropped slots."""
    m = build_model(spec)
    x = token_stream(spec, seed, n)
    ds = route_batch(m, x, 0)
    rng = np.random.default_rng(seed)
    E, k = spec.experts_per_layer, spec.top_k
    plans, ex, kd = [], np.empty((n, k), np.int64), np.empty((n, k), np.uint8)
    for i, d in enumerate(ds):
        slots, used = [], 0
        avail = [e for e in range(E) if e not in set(int(v) for v in d.topk)]
        for s, o in enumerate(int(v) for v in d.topk):
            r = rng.random()
            if r < 0.5 or not avail:
                slots.append(substitution.PlanSlot(o, o, "kept"))
            elif r < 0.8:
                j = avail.pop(int(rng.integers(len(avail))))
                slots.append(substitution.PlanSlot(o, j, "substituted")); used += 1
            else:
                slots.append(substitution.PlanSlot(o, o, "dropped"))
            ex[i, s], kd[i, s] = slots[-1].executed, KIND[slots[-1].kind]
        plans.append(substitution.ReplacementPlan(d.token, 0, tuple(slots), used))
    y = forward_batch(m, x, ds, plans)
    return dict(x=x, topk=np.stack([d.topk for d in ds]),
                probs=np.stack([d.probs_renorm for d in ds]), executed=ex, kind=kd,
                y=y, h=layer_update(x, y))


TINY_SIM = """
model.layers = 4
model.experts = 8
model.top_k = 2
model.hidden_dim = 128
model.ffn_dim = 256
model.clusters = 8
stream.num_tokens = 2000
stream.batch = 16
builder.k_max = 7
sub.h = 7
cache.rate = 0.5
"""


def sim_case() -> dict:
    """BASELINE config 1 (tiny, E=8 k=2 d=128, f=256, 4 layers) through the
    reference pipeline: cmd_profile -> cmd_build -> run_simulation for the
    buddy and original methods at c=0.5 (harness.py:70-424)."""
    cfg = parse_config_text(TINY_SIM)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        pdir, bdir = os.path.join(td, "p"), os.path.join(td, "b")
        harness.cmd_profile(cfg, pdir)
        cfg.set("io.profile_dir", pdir)
        harness.cmd_build(cfg, bdir)
        L = cfg["model.layers"]
        tables = [buddies.load_table(os.path.join(bdir, f"buddies_L{l:02d}.bin")) for l in range(L)]
        samples = harness.load_tae_samples(os.path.join(pdir, "tae_samples.txt"))
        taus = [gating.calibrate_tau(samples[l], 15.0) for l in range(L)]
        stats = [profiler.load_stats(os.path.join(pdir, f"stats_L{l:02d}.bin")) for l in range(L)]
        for l in range(L):
            out[f"pairs_L{l}"] = stats[l].pair_counts
            out[f"counts_L{l}"] = stats[l].counts
            ids = np.full((8, 7), -1, np.int32); w = np.zeros((8, 7)); lens = np.zeros(8, np.int32)
            for p in range(8):
                li = tables[l].ids(p); ids[p, :len(li)] = li; w[p, :len(li)] = tables[l].weights(p); lens[p] = len(li)
            out[f"ids_L{l}"], out[f"w_L{l}"], out[f"lens_L{l}"] = ids, w, lens
            out[f"tae_L{l}"] = np.asarray(samples[l])
        out["taus"] = np.asarray(taus)
        for method in ("buddy", "original"):
            c = parse_config_text(TINY_SIM)
            c.set("method", method); c.set("stream.seed", "2"); c.set("stream.num_tokens", "320")
            c.set("sub.rho", "3")
            r = harness.run_simulation(c, tables=tables if method == "buddy" else None,
                                       tau_by_layer=taus if method == "buddy" else None)
            ev = np.array([(e.time_ms, EV[e.kind], e.layer, e.token, e.expert, e.bytes, e.stall_ms)
                           for e in r.events], np.float64).reshape(-1, 7)
            out[f"{method}_events"] = ev
            out[f"{method}_outputs"] = r.outputs
            mt = r.metrics
            out[f"{method}_metrics"] = np.array([mt.tokens_per_s, mt.stall_ms, mt.compute_ms, mt.hits,
                                                 mt.misses_ondemand, mt.misses_substituted, mt.drops,
                                                 mt.prefetch_issued, mt.prefetch_completed,
                                                 mt.evictions, mt.read_bytes, mt.substitutions,
                                                 mt.gate_token_forbidden, mt.gate_batch_bypassed,
                                                 mt.fidelity_cosine, mt.fidelity_argmax])
            out[f"{method}_gates"] = np.array([g[:8] for g in r.gate_records], np.float64).reshape(-1, 8)
    return out


def files_case() -> dict:
    """The raw bytes of every file the reference's cmd_profile -> cmd_build
    write for the tiny config (harness.py:70-157: stats_LXX.bin (BSST v1),
    coact_LXX.csv, tae_samples.txt, buddies_LXX.bin (BSBT v1), buddies_LXX.csv),
    so the GPU pipeline's files can be compared byte for byte."""
    cfg = parse_config_text(TINY_SIM)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        pdir, bdir = os.path.join(td, "p"), os.path.join(td, "b")
        harness.cmd_profile(cfg, pdir)
        cfg.set("io.profile_dir", pdir)
        harness.cmd_build(cfg, bdir)
        for tag, d in (("p", pdir), ("b", bdir)):
            for name in sorted(os.listdir(d)):
                with open(os.path.join(d, name), "rb") as fh:
                    out[f"{tag}/{name}"] = np.frombuffer(fh.read(), np.uint8)
    return out


def sim_beta_case() -> dict:
    """The tiny pipeline's buddy simulation with the adaptive distribution
    gate (gate.pcie_budget_bytes set -> gating.BetaController,
    harness.py:293-297, 354-357): 1,280 tokens = 320 gate records, so beta
    is re-derived 5 times; the budget admits ~1.5 expert misses per record."""
    cfg = parse_config_text(TINY_SIM)
    out = {}
    with tempfile.TemporaryDirectory() as td:
        pdir, bdir = os.path.join(td, "p"), os.path.join(td, "b")
        harness.cmd_profile(cfg, pdir)
        cfg.set("io.profile_dir", pdir)
        harness.cmd_build(cfg, bdir)
        L = cfg["model.layers"]
        tables = [buddies.load_table(os.path.join(bdir, f"buddies_L{l:02d}.bin")) for l in range(L)]
        samples = harness.load_tae_samples(os.path.join(pdir, "tae_samples.txt"))
        taus = [gating.calibrate_tau(samples[l], 15.0) for l in range(L)]
        for budget in (1.5, 0.5):
            c = parse_config_text(TINY_SIM)
            c.set("method", "buddy"); c.set("stream.seed", "2"); c.set("stream.num_tokens", "1280")
            c.set("sub.rho", "3")
            ebytes = 2 * 128 * 256 * 8
            c.set("gate.pcie_budget_bytes", str(budget * ebytes))
            r = harness.run_simulation(c, tables=tables, tau_by_layer=taus)
            tag = f"b{int(budget * 10)}"
            out[f"{tag}_events"] = np.array([(e.time_ms, EV[e.kind], e.layer, e.token, e.expert, e.bytes, e.stall_ms)
                                             for e in r.events], np.float64).reshape(-1, 7)
            out[f"{tag}_gates"] = np.array([g[:8] for g in r.gate_records], np.float64).reshape(-1, 8)
            mt = r.metrics
            out[f"{tag}_metrics"] = np.array([mt.misses_ondemand, mt.substitutions, mt.gate_token_forbidden,
                                              mt.gate_batch_bypassed])
            out[f"{tag}_budget"] = np.float64(budget * ebytes)
    return out


def sim_random_case() -> dict:
    """The paper's Random baseline (substitution.random_plan through
    run_simulation(method="random"), harness.py:299-300, 358-359) on the tiny
    config at two cache rates and two run seeds: event logs, outputs and
    metrics, so the engine's host PCG64 replica is pinned draw for draw."""
    out = {}
    for rate, seed in ((0.5, 0), (0.375, 5), (0.75, 11)):
        c = parse_config_text(TINY_SIM)
        c.set("method", "random"); c.set("stream.seed", "2"); c.set("stream.num_tokens", "320")
        c.set("cache.rate", str(rate)); c.set("run.seed", str(seed))
        r = harness.run_simulation(c)
        tag = f"c{int(rate * 1000)}_s{seed}"
        out[f"{tag}_events"] = np.array([(e.time_ms, EV[e.kind], e.layer, e.token, e.expert, e.bytes, e.stall_ms)
                                         for e in r.events], np.float64).reshape(-1, 7)
        out[f"{tag}_outputs"] = r.outputs
        mt = r.metrics
        out[f"{tag}_metrics"] = np.array([mt.tokens_per_s, mt.stall_ms, mt.compute_ms, mt.hits,
                                          mt.misses_ondemand, mt.misses_substituted, mt.drops,
                                          mt.prefetch_issued, mt.prefetch_completed, mt.evictions,
                                          mt.read_bytes, mt.substitutions, mt.fidelity_cosine,
                                          mt.fidelity_argmax])
        out[f"{tag}_cfg"] = np.array([rate, seed])
    return out


def substrate_case() -> dict:
    """Samples of the reference's synthetic substrate (model.py:122-222,
    350-382) so the framework's restatement can be pinned without storing
    whole weight stacks."""
    out = {}
    for name, spec in (("tiny", ModelSpec(num_layers=4, experts_per_layer=8, top_k=2, hidden_dim=128,
                                          ffn_dim=256, num_clusters=8)),
                       ("dflt", ModelSpec()),
                       ("odd", ModelSpec(num_layers=2, experts_per_layer=12, top_k=3, hidden_dim=20,
                                         ffn_dim=36, num_clusters=5, skew=0.0, seed=99,
                                         cluster_spread=0.3))):
        m = build_model(spec)
        out[f"{name}_gate_w"], out[f"{name}_gate_b"] = m.gate_w, m.gate_b
        L = spec.num_layers
        wi, wo = m.layer_stack(L - 1)
        out[f"{name}_w_in_e0"], out[f"{name}_w_out_elast"] = wi[0], wo[-1]
        out[f"{name}_w_in_sum"] = wi.sum(axis=(1, 2))
        out[f"{name}_w_out_sum"] = wo.sum(axis=(1, 2))
        out[f"{name}_stream"] = token_stream(spec, 5, 64)
        out[f"{name}_readout"] = buddysim.model.readout_head(spec, 16)
    return out


def main() -> None:
    if sys.argv[1:] == ["beta"]:  # regenerate only the adaptive-beta fixture
        np.savez_compressed(os.path.join(OUT, "sim_tiny_beta.npz"), **sim_beta_case())
        return
    if sys.argv[1:] == ["shapes"]:  # routing + tables at the BASELINE shapes
        for name, E, k, d, n in (("mixtral", 8, 2, 4096, 16384), ("qwen3", 128, 8, 2048, 32768),
                                 ("dsv2", 64, 6, 2048, 32768)):
            np.savez_compressed(os.path.join(OUT, f"routing_{name}.npz"), **routing_shape_case(E, k, d, n))
        return
    if sys.argv[1:] == ["files"]:  # regenerate only the profile/build file bytes
        np.savez_compressed(os.path.join(OUT, "files_tiny.npz"), **files_case())
        return
    if sys.argv[1:] == ["random"]:  # regenerate only the Random-arm fixture
        np.savez_compressed(os.path.join(OUT, "sim_tiny_random.npz"), **sim_random_case())
        return
    np.savez_compressed(os.path.join(OUT, "remap_corpus_20260819.npz"), **remap_corpus(20260819, 1000))
    np.savez_compressed(os.path.join(OUT, "remap_corpus_1234.npz"), **remap_corpus(1234, 300))
    tiny = ModelSpec(num_layers=2, experts_per_layer=8, top_k=2, hidden_dim=128, ffn_dim=256,
                     num_clusters=8)
    dflt = ModelSpec()
    big = ModelSpec(num_layers=1, experts_per_layer=128, top_k=8, hidden_dim=64, ffn_dim=32,
                    num_clusters=16)
    np.savez_compressed(os.path.join(OUT, "routing_tiny.npz"), **routing_case(tiny, 2, 256))
    np.savez_compressed(os.path.join(OUT, "routing_default.npz"), **routing_case(dflt, 2, 256, layer=5, T=0.7))
    np.savez_compressed(os.path.join(OUT, "routing_e128.npz"), **routing_case(big, 3, 256))
    builds_small = [(0.95, 7, "binary"), (0.75, 4, "binary"), (0.99, 2, "binary"), (1.0, 500, "binary"),
                    (0.95, 7, "weighted")]
    np.savez_compressed(os.path.join(OUT, "coact_tiny.npz"),
                        **coact_case(tiny, 2000, 256, 0.0, 1e-3, builds_small))
    np.savez_compressed(os.path.join(OUT, "coact_default_w05.npz"),
                        **coact_case(dflt, 1500, 256, 0.5, 1e-3,
                                     [(0.95, 16, "binary"), (0.75, 4, "binary"), (1.0, 64, "binary"),
                                      (0.95, 16, "weighted")]))
    np.savez_compressed(os.path.join(OUT, "coact_e128.npz"),
                        **coact_random_case(128, 8, 3000, 7, [(0.95, 16, "binary"), (0.5, 16, "binary"),
                                                              (1.0, 200, "binary")]))
    np.savez_compressed(os.path.join(OUT, "coact_e160_noeps.npz"),
                        **coact_random_case(160, 6, 600, 9, [(0.95, 16, "binary"), (0.8, 32, "weighted")],
                                            eps=0.0))
    for i, (pol, rate, E) in enumerate([("lru", 0.5, 16), ("lfu", 0.375, 24), ("freq_static", 0.25, 32),
                                        ("lru", 0.75, 64)]):
        np.savez_compressed(os.path.join(OUT, f"memtier_{i}_{pol}.npz"), **memtier_case(100 + i, E, rate, pol, 400))
    np.savez_compressed(os.path.join(OUT, "forward_tiny.npz"), **forward_case(tiny, 32, 5))
    np.savez_compressed(os.path.join(OUT, "sim_tiny.npz"), **sim_case())
    np.savez_compressed(os.path.join(OUT, "substrate.npz"), **substrate_case())
    np.savez_compressed(os.path.join(OUT, "sim_tiny_random.npz"), **sim_random_case())
    np.savez_compressed(os.path.join(OUT, "files_tiny.npz"), **files_case())
    print("golden fixtures written to", OUT, "with buddysim", buddysim.__version__)


if __name__ == "__main__":
    main()
