"""Drivers of the reference harness on the B200 kernels:
``run_profile`` (cmd_profile, harness.py:70-117: routing + K6 co-activation
counts + entropy samples over the profiling stream, BSST / CSV /
tae_samples.txt files), ``run_build`` (cmd_build, :134-157: K7 tables, BSBT /
CSV files), ``calibrate_taus`` (the tau step of cmd_simulate, :476-484),
``run_simulation`` (:221-424), ``run_oracle`` (:175-186) and ``fidelity``
(:189-206).

The reference's entry points keep their names and signatures: ``cmd_profile``
/ ``cmd_build`` / ``cmd_simulate`` (artifact files as the reference writes
them), ``run_simulation`` / ``run_oracle`` / ``fidelity`` /
``_predict_for_layer``; ``run_profile`` / ``run_build`` are their tensor-level
forms. A configuration is either the reference's ExperimentConfig (used
duck-typed: ``.values``, ``.explicit``, ``validate_run()``; the config system
itself is out of scope) or a plain dict of its dotted keys (defaults from
config.py:64-111). ``run_simulation`` builds the synthetic model and replays
the evaluation stream through ``DecodeEngine`` (fp32 parity mode with the
reference's tanh experts), so its event log, counters, gate records,
bandwidth series and outputs compare one to one with the reference's
SimResult. The CLI and ``cmd_report`` table formatting are not here.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

import os

from . import _native as N
from . import buddies, gating, memtier, ops, profiler, substrate
from .engine import DecodeEngine, EngineSpec, HostMirror
from .errors import CalibrationError, ConfigurationError, FormatError, InvariantViolation

DEFAULTS = {
    "model.layers": 24, "model.experts": 64, "model.top_k": 6, "model.hidden_dim": 32, "model.ffn_dim": 64,
    "model.seed": 7, "model.skew": 0.8, "model.clusters": 8, "model.cluster_spread": 0.1,
    "stream.seed": 1, "stream.num_tokens": 10000, "stream.batch": 16, "cache.rate": 0.75, "cache.policy": "lru",
    "cost.expert_load_ms": 9.5, "cost.hit_ms": 0.0, "cost.expert_compute_ms": 0.5,
    "cost.pcie_bw_bytes_per_s": 4.0e6, "gate.temperature": 1.0, "gate.beta": 1.0, "gate.margin_gamma": None,
    "gate.pcie_budget_bytes": None,
    "sub.h": 16, "sub.rho": None, "sub.fallback": "prefetch_original", "prefetch.enabled": True,
    "method": "buddy", "run.seed": 0, "fidelity.readout_classes": 16,
    "stream.warmup_steps": 256, "profile.laplace_eps": 1e-3, "profile.warmup_weight": 0.0,
    "builder.alpha": "0.95", "builder.k_max": 16, "builder.mode": "binary", "gate.tau_percentile": 15.0,
    "gate.tau": None, "sub.eta": 0.0, "sub.kappa": 0.0, "sub.diversity_factor": 0.5, "sub.use_local_logit": True,
    "topology.partitions": 1, "topology.hop": 1.0,
    "io.profile_dir": "out/profile", "io.build_dir": "out/build", "io.run_dir": "out/run",
}


def _cfg(cfg) -> dict:
    """Dotted-key dict of a configuration: the reference's ExperimentConfig
    (validated like its own callers do, harness.py:73,138,232) or a dict."""
    c = dict(DEFAULTS)
    if cfg is not None and isinstance(getattr(cfg, "values", None), dict):
        if hasattr(cfg, "validate_run"):
            cfg.validate_run()
        c.update(cfg.values)
        c["__explicit__"] = set(getattr(cfg, "explicit", ()))
    else:
        c.update(cfg or {})
        c["__explicit__"] = set((cfg or {}).keys())
    return c


def _fixed_tau(c):
    """gate.tau when it supersedes the percentile (ExperimentConfig.gate_config, config.py:150-175)."""
    tau, pct, ex = c["gate.tau"], c["gate.tau_percentile"], c["__explicit__"]
    if "gate.tau" in ex and "gate.tau_percentile" in ex and tau is not None and pct is not None:
        raise ConfigurationError("set gate.tau or gate.tau_percentile, not both")
    if tau is not None and "gate.tau_percentile" not in ex:
        return float(tau), None
    if tau is None and pct is None:
        raise ConfigurationError("one of gate.tau / gate.tau_percentile must be set")
    return None, pct


# file names of the reference harness (harness.py:47-65)
def stats_path(out_dir, layer):
    return os.path.join(out_dir, f"stats_L{layer:02d}.bin")


def coact_path(out_dir, layer):
    return os.path.join(out_dir, f"coact_L{layer:02d}.csv")


def table_path(out_dir, layer):
    return os.path.join(out_dir, f"buddies_L{layer:02d}.bin")


def table_csv_path(out_dir, layer):
    return os.path.join(out_dir, f"buddies_L{layer:02d}.csv")


def tae_path(out_dir):
    return os.path.join(out_dir, "tae_samples.txt")


@dataclass
class SimResult:
    """harness.py:163-172, plus the engine's per layer-step trace."""
    metrics: memtier.RunMetrics
    outputs: np.ndarray
    events: list
    gate_records: list
    tau_by_layer: list
    beta_final: float
    bandwidth_series: list  # (step, read_bytes) per outer batch step
    trace: list = field(default_factory=list)


def _spec(c) -> substrate.ModelSpec:
    return substrate.ModelSpec(num_layers=c["model.layers"], experts_per_layer=c["model.experts"],
                               top_k=c["model.top_k"], hidden_dim=c["model.hidden_dim"], ffn_dim=c["model.ffn_dim"],
                               seed=c["model.seed"], skew=c["model.skew"], num_clusters=c["model.clusters"],
                               cluster_spread=c["model.cluster_spread"]).validate()


def _tanh_arena(spec, layer):
    w_in, w_out = substrate.layer_stack(spec, layer)
    E = w_in.shape[0]
    return np.concatenate([np.transpose(w_in, (0, 2, 1)).reshape(E, -1),
                           np.transpose(w_out, (0, 2, 1)).reshape(E, -1)], axis=1).astype(np.float32)


def run_oracle(model, x: np.ndarray, temperature: float = 1.0, batch: int = 256) -> np.ndarray:
    """Full-residency forward (identity plans) through K1, K3-K5 (harness.py:175-186).
    ``model``: a model.Model (as the reference passes) or its ModelSpec."""
    spec = model.spec if hasattr(model, "spec") else model
    dev = torch.device("cuda", torch.cuda.current_device())
    gw, gb = substrate.gate_weights(spec)
    gw = torch.tensor(gw, dtype=torch.float32, device=dev)
    gb = torch.tensor(gb, dtype=torch.float32, device=dev)
    arenas = [torch.tensor(_tanh_arena(spec, l), device=dev) for l in range(spec.num_layers)]
    E, k, d, f = spec.experts_per_layer, spec.top_k, spec.hidden_dim, spec.ffn_dim
    bufs = torch.arange(E, dtype=torch.int32, device=dev)
    out = np.empty_like(x)
    for b0 in range(0, x.shape[0], batch):
        h = torch.tensor(x[b0:b0 + batch], dtype=torch.float32, device=dev)
        for l in range(spec.num_layers):
            r = ops.gate_topk(h, gw[l], gb[l], k, temperature)
            kept = torch.zeros_like(r.topk, dtype=torch.uint8)
            perm = ops.permute(r.topk, kept, E)
            yp = ops.expert_ffn_f32(ops.gather_rows(h, perm, 0), perm, arenas[l], bufs, d, f, ops.ACT_TANH)
            h = ops.combine(yp, perm, r.probs, kept, h_in=h)
        out[b0:b0 + batch] = h.double().cpu().numpy()
    return out


def fidelity(outputs: np.ndarray, oracle: np.ndarray, readout: np.ndarray) -> tuple:
    """(mean cosine, argmax agreement) on the GPU (harness.py:189-206);
    bitwise-equal rows score exactly 1.0."""
    if outputs.shape != oracle.shape:
        raise ConfigurationError("fidelity shapes do not match")
    dev = torch.device("cuda", torch.cuda.current_device())
    a = torch.tensor(outputs, dtype=torch.float64, device=dev)
    b = torch.tensor(oracle, dtype=torch.float64, device=dev)
    r = torch.tensor(readout, dtype=torch.float64, device=dev)
    denom = torch.clamp(torch.linalg.norm(a, dim=1) * torch.linalg.norm(b, dim=1), min=1e-30)
    cos = torch.clamp((a * b).sum(1) / denom, -1.0, 1.0)
    cos = torch.where((a == b).all(1), torch.ones_like(cos), cos)
    agree = ((a @ r.T).argmax(1) == (b @ r.T).argmax(1)).double().mean()
    return float(cos.mean().item()), float(agree.item())


def events_array(events) -> np.ndarray:
    """SimEvents as an [n,7] float64 array (time, kind code, layer, token,
    expert, bytes, stall), the layout of the golden fixtures."""
    code = {k: i for i, k in enumerate(memtier._EV_BY_CODE)}
    return np.array([(e.time_ms, code[e.kind], e.layer, e.token, e.expert, e.bytes, e.stall_ms) for e in events],
                    np.float64).reshape(-1, 7)


def _predict_for_layer(state, prev_counts: dict) -> list:
    """Previous-step top-m frequency predictor (harness.py:209-218), decided by
    the C++ control plane's predictor (bm_cache_predict) that the engine uses:
    m = capacity - distinct experts of the previous step, ranked by count
    desc then id asc."""
    import ctypes
    E = state.num_experts
    counts = np.zeros(E, np.int32)
    for e, n in prev_counts.items():
        counts[int(e)] = int(n)
    preds = np.zeros(max(E, 1), np.int32)
    n = ctypes.c_int64()
    N.call("bm_cache_predict", state._h, 0, counts.ctypes.data, preds.ctypes.data, ctypes.byref(n))
    return [int(v) for v in preds[:n.value]]


def _dense_tables(tables, L, E):
    """(ids [L,E,K] int32, lens [L,E] int32, weights [L,E,K] f64 | None) from a
    list of buddies.BuddyTable or a dense (ids, lens[, weights]) tuple."""
    if isinstance(tables, (list, tuple)) and len(tables) and hasattr(tables[0], "ids"):
        K = max(1, max(len(t.ids(p)) for t in tables for p in range(E)))
        ids = np.full((L, E, K), -1, np.int32)
        lens = np.zeros((L, E), np.int32)
        w = np.zeros((L, E, K), np.float64)
        for l, t in enumerate(tables):
            for p in range(E):
                n = len(t.ids(p))
                ids[l, p, :n] = t.ids(p)
                w[l, p, :n] = t.weights(p)
                lens[l, p] = n
        return ids, lens, w
    ids, lens = np.asarray(tables[0], np.int32), np.asarray(tables[1], np.int32)
    w = np.asarray(tables[2], np.float64) if len(tables) > 2 else None
    return ids, lens, w


def run_simulation(cfg, tables=None, tau_by_layer=None, static_freq=None, oracle_outputs=None,
                   collect_events: bool = True) -> SimResult:
    """The reference decode replay (harness.py:221-424) on the engine.
    ``tables``: a list of buddies.BuddyTable (one per layer) or dense
    (ids[L,E,K], lens[L,E][, weights[L,E,K]]); ``tau_by_layer``: calibrated
    thresholds (ignored when gate.tau is fixed); ``static_freq``: per-layer
    profiling frequencies for the freq_static policy."""
    c = _cfg(cfg)
    spec = _spec(c)
    L, E = spec.num_layers, spec.experts_per_layer
    method = c["method"]
    if method not in ("buddy", "original", "random"):
        raise ConfigurationError(f"unknown method {method!r} (buddy|original|random)")
    if not (0.0 < c["cache.rate"] <= 1.0):
        raise ConfigurationError("cache_rate must be in (0, 1]")
    if c["cache.policy"] not in memtier.POLICIES:
        raise ConfigurationError(f"unknown eviction policy {c['cache.policy']!r}")
    cap = int(np.floor(c["cache.rate"] * E))
    dev = torch.device("cuda", torch.cuda.current_device())
    ids = lens = w = None
    taus = [-1.0] * L
    psi = method == "buddy" and (c["sub.eta"] != 0.0 or c["sub.kappa"] != 0.0)
    if method == "buddy":
        if tables is None or (isinstance(tables, list) and len(tables) != L):
            raise ConfigurationError("buddy method needs one buddy table per layer")
        if isinstance(tables, list) and hasattr(tables[0], "ids"):
            for t in tables:
                if t.num_experts != E:
                    raise ConfigurationError(f"buddy table shape {t.num_experts} does not match model {E}")
                if c["sub.h"] > t.k_max:
                    raise ConfigurationError("sub.h exceeds the table's k_max")
        ids, lens, w = _dense_tables(tables, L, E)
        if psi and w is None:
            raise ConfigurationError("Psi ordering (sub.eta / sub.kappa) needs the table weights")
        fixed, _ = _fixed_tau(c)
        if fixed is not None:
            taus = [fixed] * L
        elif tau_by_layer is None or len(tau_by_layer) != L:
            raise ConfigurationError("buddy method needs a calibrated tau per layer")
        else:
            taus = [float(t) for t in tau_by_layer]
    sf = None
    if c["cache.policy"] == memtier.POLICY_FREQ_STATIC:
        if static_freq is None or len(static_freq) != L:
            raise ConfigurationError("freq_static policy needs profiling frequencies per layer")
        sf = np.stack([np.asarray(v, np.float64) for v in static_freq])
    P = int(c["topology.partitions"])
    partition_of = (np.arange(E) * P) // E if P > 1 else None
    mirrors = []
    for l in range(L):
        a = _tanh_arena(spec, l)
        m = HostMirror(a.nbytes)
        m.as_tensor(torch.float32).copy_(torch.from_numpy(a).view(-1))
        mirrors.append(m)
    gw, gb = substrate.gate_weights(spec)
    ebytes = 2 * spec.hidden_dim * spec.ffn_dim * 8
    es = EngineSpec(num_layers=L, num_experts=E, top_k=spec.top_k, d=spec.hidden_dim, f=spec.ffn_dim,
                    capacity=cap, max_batch=c["stream.batch"], act=ops.ACT_TANH, method=method,
                    policy=c["cache.policy"], search_rank_h=c["sub.h"], rho=c["sub.rho"],
                    fallback=0 if c["sub.fallback"] == "prefetch_original" else 1, beta=c["gate.beta"],
                    temperature=c["gate.temperature"], gamma=c["gate.margin_gamma"], prefetch=c["prefetch.enabled"],
                    fp32_weights=True, expert_bytes=ebytes,
                    load_ms=c["cost.expert_load_ms"], hit_ms=c["cost.hit_ms"], compute_ms=c["cost.expert_compute_ms"],
                    pcie_bw_bytes_per_s=c["cost.pcie_bw_bytes_per_s"],
                    pcie_budget_bytes=c["gate.pcie_budget_bytes"] if method == "buddy" else None,
                    run_seed=c["run.seed"])
    initial = [memtier.initial_residents(E, cap, c["cache.policy"], c["run.seed"], l,
                                         None if sf is None else sf[l]) for l in range(L)]
    eng = DecodeEngine(es, mirrors, torch.tensor(gw, dtype=torch.float32, device=dev),
                       torch.tensor(gb, dtype=torch.float32, device=dev),
                       None if ids is None else torch.tensor(ids, device=dev),
                       None if lens is None else torch.tensor(lens, device=dev), taus, initial, sf)
    if psi:
        eng.set_psi(torch.tensor(w, device=dev), c["sub.eta"], c["sub.kappa"], c["sub.use_local_logit"],
                    None if partition_of is None else torch.tensor(partition_of, dtype=torch.int32, device=dev),
                    c["topology.hop"])
    eng.set_trace(True)
    n, B = c["stream.num_tokens"], c["stream.batch"]
    x = substrate.token_stream(spec, c["stream.seed"], n)
    h = torch.tensor(x, dtype=torch.float32, device=dev)
    bandwidth, n_seen = [], 0
    for step, b0 in enumerate(range(0, n, B)):
        eng.step(h[b0:b0 + B], np.arange(b0, min(n, b0 + B)))
        # step bytes as the reference counts them (harness.py:327-329, 374-378): prefetch
        # completions and on-demand misses of routed slots (a substituted slot's stand-in
        # that misses is not counted), from this step's slice of the control-plane log
        ev = eng.events(n_seen)
        n_seen += len(ev)
        kinds = ev[:, 1].astype(np.int64)
        after_sub = np.zeros(len(ev), bool)
        after_sub[1:] = kinds[:-1] == 2
        counted = (kinds == 4) | ((kinds == 1) & ~after_sub)
        bandwidth.append((step, int(ev[counted, 5].sum())))
    torch.cuda.synchronize()
    eng.finish()
    events = memtier.events_from_array(eng.sorted_events())
    st = eng.stats()
    waste = 0  # wasted prefetches (harness.py:400): evicted unused + still-unused residents
    cache = N.lib().bm_engine_cache(eng._h)
    sc = np.zeros(4, np.int64)
    for l in range(L):
        N.call("bm_cache_layer_state", cache, l, None, None, sc.ctypes.data)
        waste += int(sc[2] + sc[3])
    m = memtier.step_metrics(events, tokens=n, compute_ms=c["cost.expert_compute_ms"] * st["executed_slots"],
                             waste_bytes=waste * es.expert_bytes)
    m.substitutions = st["substitutions"]
    m.gate_token_forbidden = st["gate_forbidden"]
    m.gate_batch_bypassed = st["batch_bypassed"]
    if m.read_bytes != ebytes * (m.misses_ondemand + m.prefetch_completed):
        raise InvariantViolation("transfer byte conservation failed")
    outputs = h.double().cpu().numpy()
    if oracle_outputs is None:
        oracle_outputs = run_oracle(spec, x, c["gate.temperature"], batch=B)
    m.fidelity_cosine, m.fidelity_argmax = fidelity(outputs, oracle_outputs,
                                                    substrate.readout_head(spec, c["fidelity.readout_classes"]))
    trace = eng.trace()
    gate_records = []
    if method == "buddy":  # (step, layer, token, tae, margin, delta, token_allowed, batch_allowed), harness.py:345-350
        for i, r in enumerate(trace):
            b0 = (i // L) * B
            for j in range(r["topk"].shape[0]):
                gate_records.append((i // L, r["layer"], b0 + j, float(r["tae"][j]), float(r["margin"][j]),
                                     r["delta"], bool(r["allowed"][j]), bool(r["batch_ok"])))
    beta_final = st["beta"] if (method == "buddy" and c["gate.pcie_budget_bytes"] is not None) else c["gate.beta"]
    eng.close()
    for mm in mirrors:
        mm.close()
    return SimResult(metrics=m, outputs=outputs, events=events if collect_events else [], gate_records=gate_records,
                     tau_by_layer=list(taus) if method == "buddy" else [], beta_final=beta_final,
                     bandwidth_series=bandwidth, trace=trace)


# ------------------------------------------------------------------ profile


@dataclass
class ProfileResult:
    stats: list            # profiler.CoActivationStats per layer (device counters)
    tae_samples: list      # float64 CUDA tensor of entropy samples per layer, token order
    paths: dict


def run_profile(cfg: dict, out_dir: str | None = None) -> ProfileResult:
    """cmd_profile (harness.py:70-117) on the GPU: the full-residency forward
    over the profiling stream (K1 router, identity plans, K3-K5 fp32 tanh
    experts), K6 co-activation counting per layer with the global token index
    as the step (warm-up by global index, profiler.py:81-95) and the K1
    entropy (TAE) of every token collected on the device. With ``out_dir``
    the reference's files are written: stats_LXX.bin (BSST v1),
    coact_LXX.csv and tae_samples.txt ("bsim/1", one `layer value` line per
    sample in routing order)."""
    c = _cfg(cfg)
    spec = _spec(c)
    L, E, k, d, f = spec.num_layers, spec.experts_per_layer, spec.top_k, spec.hidden_dim, spec.ffn_dim
    T = float(c["gate.temperature"])
    dev = torch.device("cuda", torch.cuda.current_device())
    gw, gb = substrate.gate_weights(spec)
    gw = torch.tensor(gw, dtype=torch.float32, device=dev)
    gb = torch.tensor(gb, dtype=torch.float32, device=dev)
    arenas = [torch.tensor(_tanh_arena(spec, l), device=dev) for l in range(L)]
    bufs = torch.arange(E, dtype=torch.int32, device=dev)
    stats = [profiler.CoActivationStats(layer=l, num_experts=E, warmup_steps=c["stream.warmup_steps"],
                                        warmup_weight=c["profile.warmup_weight"],
                                        laplace_eps=c["profile.laplace_eps"]) for l in range(L)]
    # pair weights are always accumulated, like observe() does (profiler.py:81-95): the
    # BSST files carry them whichever builder mode reads them later
    weighted = True
    n, B = c["stream.num_tokens"], c["stream.batch"]
    x = substrate.token_stream(spec, c["stream.seed"], n)
    xd = torch.tensor(x, dtype=torch.float32, device=dev)
    tae = [[] for _ in range(L)]
    for b0 in range(0, n, B):
        h = xd[b0:b0 + B]
        for l in range(L):
            r = ops.gate_topk(h, gw[l], gb[l], k, T)
            stats[l].observe_tensors(r.topk, r.probs if weighted else None, b0)
            tae[l].append(r.tae)
            kept = torch.zeros_like(r.topk, dtype=torch.uint8)
            perm = ops.permute(r.topk, kept, E)
            yp = ops.expert_ffn_f32(ops.gather_rows(h, perm, 0), perm, arenas[l], bufs, d, f, ops.ACT_TANH)
            h = ops.combine(yp, perm, r.probs, kept, h_in=h)
    samples = [torch.cat(t) for t in tae]
    paths = {}
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        paths = {"stats": [], "coact": [], "tae": tae_path(out_dir)}
        for l, st in enumerate(stats):
            profiler.save_stats(st, stats_path(out_dir, l))
            profiler.export_coactivation_csv(st, coact_path(out_dir, l), mode="binary")
            paths["stats"].append(stats_path(out_dir, l))
            paths["coact"].append(coact_path(out_dir, l))
        save_tae_samples(samples, paths["tae"])
    return ProfileResult(stats=stats, tae_samples=samples, paths=paths)


def save_tae_samples(samples, path) -> None:
    """tae_samples.txt (harness.py:112-116): "bsim/1" then `layer repr(value)`."""
    with open(path, "w") as fh:
        fh.write("bsim/1\n")
        for l, t in enumerate(samples):
            vals = t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t, np.float64)
            fh.writelines(f"{l} {float(v)!r}\n" for v in vals)


def load_tae_samples(path) -> dict:
    """harness.load_tae_samples (harness.py:120-129)."""
    out: dict = {}
    with open(path) as fh:
        if fh.readline().strip() != "bsim/1":
            raise FormatError(f"{path}: bad or missing version header")
        for line in fh:
            layer, value = line.split()
            out.setdefault(int(layer), []).append(float(value))
    return out


def calibrate_taus(samples, percentile: float = 15.0) -> list:
    """Per-layer tau by nearest rank over a GPU sort (gating.calibrate_tau,
    gating.py:111-123; the tau step of cmd_simulate, harness.py:476-484).
    ``samples``: list (layer order) or dict layer -> samples; CUDA tensors
    stay on the device."""
    if isinstance(samples, dict):
        layers = sorted(samples)
        if layers != list(range(len(layers))):
            missing = next(l for l in range(len(layers) + 1) if l not in samples)
            raise CalibrationError(f"no entropy samples for layer {missing}")
        samples = [samples[l] for l in layers]
    return [gating.calibrate_tau(s, percentile) for s in samples]


def _alphas(c, L) -> list:
    parts = [p.strip() for p in str(c["builder.alpha"]).split(",") if p.strip()]
    try:
        vals = [float(p) for p in parts]
    except ValueError:
        raise ConfigurationError(f"bad builder.alpha {c['builder.alpha']!r}") from None
    if len(vals) == 1:
        vals = vals * L
    if len(vals) != L:
        raise ConfigurationError(f"builder.alpha needs 1 or {L} values, got {len(vals)}")
    if not all(0.0 < v <= 1.0 for v in vals):
        raise ConfigurationError("builder.alpha values must be in (0, 1]")
    return vals


def run_build(cfg: dict, stats=None, profile_dir: str | None = None, out_dir: str | None = None) -> list:
    """cmd_build (harness.py:134-157): one K7 buddy table per layer from the
    profiled stats (given, or loaded from profile_dir's BSST files); with
    ``out_dir`` writes buddies_LXX.bin (BSBT v1) and buddies_LXX.csv."""
    c = _cfg(cfg)
    L = c["model.layers"]
    if stats is None:
        if profile_dir is None:
            raise ConfigurationError("run_build needs stats or a profile_dir")
        stats = [profiler.load_stats(stats_path(profile_dir, l)) for l in range(L)]
    alphas = _alphas(c, L)
    tables = [buddies.build_table(stats[l], alphas[l], c["builder.k_max"], c["builder.mode"]) for l in range(L)]
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        for l, t in enumerate(tables):
            buddies.save_table(t, table_path(out_dir, l))
            buddies.export_table_csv(t, table_csv_path(out_dir, l))
    return tables


# ------------------------------------------------------------ file-level commands
def cmd_profile(cfg, out_dir: str) -> dict:
    """harness.cmd_profile (harness.py:70-117): run_profile writing
    stats_LXX.bin, coact_LXX.csv and tae_samples.txt; returns the paths."""
    return run_profile(cfg, out_dir).paths


def cmd_build(cfg, out_dir: str) -> dict:
    """harness.cmd_build (harness.py:135-157): one K7 table per layer from the
    BSST files under io.profile_dir; returns the paths and the size report."""
    c = _cfg(cfg)
    tables = run_build(c, profile_dir=c["io.profile_dir"], out_dir=out_dir)
    L = c["model.layers"]
    paths = {"tables": [table_path(out_dir, l) for l in range(L)],
             "csv": [table_csv_path(out_dir, l) for l in range(L)]}
    paths["report"] = "\n".join(f"layer {l}: {buddies.table_size_report(t).format().splitlines()[0]}"
                                for l, t in enumerate(tables))
    return paths


def _echo(c) -> list:
    """The configuration echo of a metrics file (harness.py:427-440)."""
    rho = c["sub.rho"]
    return [("method", c["method"]), ("cache_rate", repr(c["cache.rate"])), ("cache_policy", c["cache.policy"]),
            ("alpha", str(c["builder.alpha"])), ("k_max", str(c["builder.k_max"])),
            ("rho", "unlimited" if rho is None else str(rho)), ("run_seed", str(c["run.seed"])),
            ("stream_seed", str(c["stream.seed"])), ("num_tokens", str(c["stream.num_tokens"])),
            ("batch", str(c["stream.batch"]))]


def write_metrics(metrics, cfg, path) -> None:
    """metrics.csv: "metric,value" then RunMetrics rows and the config echo."""
    rows = metrics.as_rows() + _echo(_cfg(cfg))
    with open(path, "w") as fh:
        fh.write("metric,value\n" + "".join(f"{k},{v}\n" for k, v in rows))


def read_metrics(path) -> dict:
    with open(path) as fh:
        lines = fh.read().splitlines()
    if not lines or lines[0].strip() != "metric,value":
        raise FormatError(f"{path}: not a metrics file")
    out = dict(line.strip().partition(",")[::2] for line in lines[1:])
    if out.get("format") != "bsim/1":
        raise FormatError(f"{path}: bad or missing format version")
    return out


def cmd_simulate(cfg, out_dir: str):
    """harness.cmd_simulate (harness.py:462-512): tables from io.build_dir, tau
    from io.profile_dir's entropy samples (unless gate.tau is fixed),
    freq_static frequencies from the profiled counts, run_simulation on the
    engine, then metrics.csv, events.log, bandwidth.csv (and gates.log)."""
    c = _cfg(cfg)
    L, method, pdir = c["model.layers"], c["method"], c["io.profile_dir"]
    tables = taus = static = None
    if method == "buddy":
        tables = [buddies.load_table(table_path(c["io.build_dir"], l)) for l in range(L)]
        fixed, pct = _fixed_tau(c)
        if fixed is None:
            taus = calibrate_taus(load_tae_samples(tae_path(pdir)), pct) if L else []
    if c["cache.policy"] == memtier.POLICY_FREQ_STATIC:
        static = [profiler.load_stats(stats_path(pdir, l)).counts for l in range(L)]
    r = run_simulation(cfg, tables=tables, tau_by_layer=taus, static_freq=static)
    os.makedirs(out_dir, exist_ok=True)
    paths = {k: os.path.join(out_dir, v) for k, v in
             (("metrics", "metrics.csv"), ("events", "events.log"), ("bandwidth", "bandwidth.csv"))}
    write_metrics(r.metrics, cfg, paths["metrics"])
    memtier.save_events(r.events, paths["events"])
    with open(paths["bandwidth"], "w") as fh:
        fh.write("step,read_bytes\n" + "".join(f"{s},{b}\n" for s, b in r.bandwidth_series))
    if method == "buddy":
        paths["gates"] = os.path.join(out_dir, "gates.log")
        with open(paths["gates"], "w") as fh:
            fh.write("bsim/1\n")
            fh.writelines(f"{st} {ly} {tk} {h!r} {mg!r} {dl!r} {int(ok)} {int(bok)}\n"
                          for st, ly, tk, h, mg, dl, ok, bok in r.gate_records)
    return r.metrics, paths


_REPORT_COLUMNS = ("method", "cache_rate", "alpha", "k_max", "rho", "fidelity_cosine", "fidelity_argmax",
                   "tokens_per_s", "read_bytes")
_REPORT_FLOATS = {"fidelity_cosine", "fidelity_argmax", "tokens_per_s", "cache_rate"}


def cmd_report(metrics_paths, out_dir: str | None = None) -> str:
    """Comparison table of metrics files (harness.py:522-559): one aligned row
    per file (floats to 4 decimals), optionally report.csv with the raw values."""
    if not metrics_paths:
        raise ConfigurationError("report needs at least one metrics file")
    raw = []
    for p in metrics_paths:
        m = read_metrics(p)
        missing = [col for col in _REPORT_COLUMNS if col not in m]
        if missing:
            raise FormatError(f"{p}: missing metrics {missing}")
        raw.append([m[col] for col in _REPORT_COLUMNS])

    def cell(v, col):
        if col not in _REPORT_FLOATS:
            return v
        try:
            return f"{float(v):.4f}"
        except ValueError:
            return v

    grid = [list(_REPORT_COLUMNS)] + [[cell(v, col) for v, col in zip(r, _REPORT_COLUMNS)] for r in raw]
    width = [max(len(row[i]) for row in grid) for i in range(len(_REPORT_COLUMNS))]
    table = "\n".join("  ".join(v.ljust(w) for v, w in zip(row, width)).rstrip() for row in grid)
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, "report.csv"), "w") as fh:
            fh.write("\n".join(",".join(r) for r in [list(_REPORT_COLUMNS)] + raw) + "\n")
    return table
