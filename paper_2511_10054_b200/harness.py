"""Drivers of the reference harness on the B200 kernels:
``run_profile`` (cmd_profile, harness.py:70-117: routing + K6 co-activation
counts + entropy samples over the profiling stream, BSST / CSV /
tae_samples.txt files), ``run_build`` (cmd_build, :134-157: K7 tables, BSBT /
CSV files), ``calibrate_taus`` (the tau step of cmd_simulate, :476-484),
``run_simulation`` (:221-424), ``run_oracle`` (:175-186) and ``fidelity``
(:189-206).

Only the hot-path parts of the reference harness are here (SURVEY §8 rows
R6, R17-R22 and §8(f) rows 1-2); the CLI, config-file parsing and report
formatting are out of scope.
``run_simulation`` takes the reference's dotted configuration keys as a
dict (defaults from config.py:64-111), builds the synthetic model, and
replays the evaluation stream through ``DecodeEngine`` (fp32 parity mode with
the reference's tanh experts), so its event log, counters and outputs are
comparable one to one with the reference's SimResult.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import os

from . import _native as N
from . import buddies, gating, memtier, ops, profiler, substrate
from .engine import DecodeEngine, EngineSpec, HostMirror
from .errors import CalibrationError, ConfigurationError, FormatError

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
}


def _cfg(cfg: dict) -> dict:
    c = dict(DEFAULTS)
    c.update(cfg or {})
    return c


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
    metrics: memtier.RunMetrics
    outputs: np.ndarray
    events: list
    tau_by_layer: list
    trace: list


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


def run_oracle(spec: substrate.ModelSpec, x: np.ndarray, temperature: float = 1.0, batch: int = 256) -> np.ndarray:
    """Full-residency forward (identity plans) through K1, K3-K5 (harness.py:175-186)."""
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


def run_simulation(cfg: dict, tables=None, tau_by_layer=None, oracle_outputs=None) -> SimResult:
    """The reference decode replay (harness.py:221-424) on the engine.
    ``tables``: dense (ids[L,E,K] int32, lens[L,E] int32) or a list of
    buddies.BuddyTable; ``tau_by_layer``: calibrated thresholds."""
    c = dict(DEFAULTS)
    c.update(cfg)
    spec = _spec(c)
    L, E = spec.num_layers, spec.experts_per_layer
    method = c["method"]
    if method not in ("buddy", "original", "random"):
        raise ConfigurationError(f"unknown method {method!r} (buddy|original|random)")
    cap = int(np.floor(c["cache.rate"] * E))
    dev = torch.device("cuda", torch.cuda.current_device())
    mirrors = []
    for l in range(L):
        a = _tanh_arena(spec, l)
        m = HostMirror(a.nbytes)
        m.as_tensor(torch.float32).copy_(torch.from_numpy(a).view(-1))
        mirrors.append(m)
    gw, gb = substrate.gate_weights(spec)
    ids = lens = None
    if method == "buddy":
        if tables is None or tau_by_layer is None:
            raise ConfigurationError("buddy method needs one buddy table and one tau per layer")
        table_objs = isinstance(tables, (list, tuple)) and hasattr(tables[0], "ids")
        if table_objs:
            K = max(max([len(t.ids(p)) for t in tables for p in range(E)]), 1)
            ids_np = np.full((L, E, K), -1, np.int32)
            lens_np = np.zeros((L, E), np.int32)
            for l, t in enumerate(tables):
                for p in range(E):
                    n = len(t.ids(p))
                    ids_np[l, p, :n] = t.ids(p)
                    lens_np[l, p] = n
        else:
            ids_np, lens_np = tables
        ids = torch.tensor(np.asarray(ids_np, np.int32), device=dev)
        lens = torch.tensor(np.asarray(lens_np, np.int32), device=dev)
        if table_objs and c["sub.h"] > tables[0].k_max:
            raise ConfigurationError("sub.h exceeds the table's k_max")
    taus = list(tau_by_layer) if method == "buddy" else [-1.0] * L
    es = EngineSpec(num_layers=L, num_experts=E, top_k=spec.top_k, d=spec.hidden_dim, f=spec.ffn_dim,
                    capacity=cap, max_batch=c["stream.batch"], act=ops.ACT_TANH, method=method,
                    policy=c["cache.policy"], search_rank_h=c["sub.h"], rho=c["sub.rho"],
                    fallback=0 if c["sub.fallback"] == "prefetch_original" else 1, beta=c["gate.beta"],
                    temperature=c["gate.temperature"], gamma=c["gate.margin_gamma"], prefetch=c["prefetch.enabled"],
                    fp32_weights=True, expert_bytes=2 * spec.hidden_dim * spec.ffn_dim * 8,
                    load_ms=c["cost.expert_load_ms"], hit_ms=c["cost.hit_ms"], compute_ms=c["cost.expert_compute_ms"],
                    pcie_bw_bytes_per_s=c["cost.pcie_bw_bytes_per_s"],
                    pcie_budget_bytes=c["gate.pcie_budget_bytes"] if method == "buddy" else None,
                    run_seed=c["run.seed"])
    initial = [memtier.initial_residents(E, cap, c["cache.policy"], c["run.seed"], l) for l in range(L)]
    eng = DecodeEngine(es, mirrors, torch.tensor(gw, dtype=torch.float32, device=dev),
                       torch.tensor(gb, dtype=torch.float32, device=dev), ids, lens, taus, initial)
    eng.set_trace(True)
    n, B = c["stream.num_tokens"], c["stream.batch"]
    x = substrate.token_stream(spec, c["stream.seed"], n)
    h = torch.tensor(x, dtype=torch.float32, device=dev)
    for b0 in range(0, n, B):
        eng.step(h[b0:b0 + B], np.arange(b0, min(n, b0 + B)))
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
    outputs = h.double().cpu().numpy()
    if oracle_outputs is None:
        oracle_outputs = run_oracle(spec, x, c["gate.temperature"], batch=B)
    m.fidelity_cosine, m.fidelity_argmax = fidelity(outputs, oracle_outputs,
                                                    substrate.readout_head(spec, c["fidelity.readout_classes"]))
    trace = eng.trace()
    eng.close()
    for mm in mirrors:
        mm.close()
    return SimResult(metrics=m, outputs=outputs, events=events, tau_by_layer=taus, trace=trace)


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
    weighted = c["builder.mode"] == "weighted" or c["profile.warmup_weight"] != 0.0
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
