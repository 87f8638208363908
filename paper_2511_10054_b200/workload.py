"""Synthetic offloaded-MoE workloads at the BASELINE shapes.

Weights are random-init N(0, 1/fan_in) in bf16 (no checkpoints), generated
on the GPU per expert and copied into per-layer pinned host mirrors. The
router follows the reference's substrate recipe (unit cluster directions,
Zipf-like bias, Gaussian-mixture token stream; substrate.py restating
model.py:122-222, 350-375) at the named d/E, so routing is skewed and
clustered the way the paper's buddy tables assume.

Profiling (the paper's offline stage) runs on the GPU, layer-major: route
the profile stream (K1), count co-activations (K6), forward with every
expert resident (K3-K5), then rank buddies (K7) and calibrate tau from the
TAE samples — cmd_profile + cmd_build (harness.py:70-158) over tensors.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import ops, substrate, synth
from .engine import DecodeEngine, EngineSpec, HostMirror, SharedMirror, coded_mirror_from_device, fill_mirror_from_device

SHAPES, SHARED = synth.SHAPES, synth.SHARED
initial_residents = synth.initial_residents  # seeded-permutation prefix (memtier.py:132-140)


host_mem_available = synth.host_mem_available


@dataclass
class ShareSpec:
    """Node-shared expert mirrors for replicas of one model: the owner
    (local rank 0) writes /dev/shm/<tag>_L<l>, ``barrier()`` orders the
    writes before the other local ranks attach."""
    tag: str
    owner: bool
    barrier: object
    directory: str = "/dev/shm"

    def path(self, layer: int) -> str:
        return os.path.join(self.directory, f"{self.tag}_L{layer:03d}")


def shm_bytes_free(directory: str = "/dev/shm") -> int:
    try:
        st = os.statvfs(directory)
        return st.f_bavail * st.f_frsize
    except OSError:
        return 0


@dataclass
class Workload:
    name: str
    spec: substrate.ModelSpec
    eng: EngineSpec
    mirrors: list
    gate_w: torch.Tensor
    gate_b: torch.Tensor
    tbl_ids: torch.Tensor
    tbl_len: torch.Tensor
    taus: list
    initial: list
    profile_seconds: float = 0.0
    mean_buddies: float = 0.0
    extra: dict = field(default_factory=dict)

    def engine(self, method: str = "buddy", **overrides) -> DecodeEngine:
        kw = dict(self.eng.__dict__)
        kw.update(overrides)
        kw["method"] = method
        es = EngineSpec(**kw)
        initial = self.initial
        if "capacity" in overrides:
            initial = [initial_residents(es.num_experts, es.capacity, 0, l) for l in range(es.num_layers)]
        return DecodeEngine(es, self.mirrors, self.gate_w, self.gate_b,
                            self.tbl_ids if method == "buddy" else None,
                            self.tbl_len if method == "buddy" else None,
                            self.taus, initial)

    def tokens(self, seed: int, n: int) -> np.ndarray:
        return substrate.token_stream(self.spec, seed, n).astype(np.float32)

    def close(self):
        for m in self.mirrors:
            m.close()


def _synth_expert(luts, seed: int, layer: int, expert: int, d: int, f: int, out: torch.Tensor,
                  cluster: int | None = None, spread: float = synth.SPREAD) -> torch.Tensor:
    """One SwiGLU expert [W1 [f,d] | W3 [f,d] | W2 [d,f]] bf16, row-major, from
    the counter-based generator (synth.py; the CPU reference arm regenerates
    the same bits on the host): N(0, 1/fan_in) values, or with ``cluster``
    the clustered recipe base_cluster + spread * delta_expert."""
    n = d * f
    for m in (synth.W1, synth.W3, synth.W2):
        dst = out[m * n:(m + 1) * n]
        if cluster is None:
            ops.synth_bf16(luts[m], synth.matrix_key(seed, layer, expert, m), dst)
        else:
            N.call("bm_synth_mix_bf16", luts[m].data_ptr(), synth.base_key(seed, layer, cluster, m),
                   synth.matrix_key(seed, layer, expert, m), float(spread), n, dst.data_ptr(),
                   torch.cuda.current_stream().cuda_stream)
    return out


def profile_tables(x: torch.Tensor, gate_w, gate_b, k: int, E: int, alpha: float, k_max: int, tau_percentile: float,
                   warm: int = 256):
    """Buddy table + tau of one layer from the profile tokens ``x`` routed by
    that layer's gate: K1 -> K6 (warm-up weight 0, config.py:80) -> K7, and
    the nearest-rank tau over the TAE samples (calibrate_tau, gating.py:111-123)."""
    r = ops.gate_topk(x, gate_w, gate_b, k)
    warm = min(warm, x.shape[0])
    wc, wp = ops.coact_count(r.topk[:warm], E)
    mc, mp = ops.coact_count(r.topk[warm:], E)
    t = ops.buddy_rank(ops.counts_to_f64(mp, wp, 0.0), 1e-3, alpha, k_max)
    s, _ = torch.sort(r.tae)
    idx = max(1, math.ceil(tau_percentile * s.numel() / 100.0)) - 1
    return r, t, float(s[min(idx, s.numel() - 1)])


def build(name: str = "mixtral", layers: int = 32, max_batch: int = 16, seed: int = 0,
          profile_tokens: int = 4096, alpha: float = 0.95, k_max: int | None = None, tau_percentile: float = 15.0,
          clusters: int | None = None, n_tile: int = 128, device: str = "cuda", rho: int | None = 3,
          codec: int = 1, share: ShareSpec | None = None, log=None, cache_rate: float | None = None,
          profile: str = "forward", clustered: bool = True) -> Workload:
    """codec 1 keeps the pinned mirrors exponent-coded (bm_xfer_*: ~0.67 of
    the bf16 bytes cross PCIe per miss, rebuilt bit-exactly in HBM); 0 raw.
    share: one node-shared mirror per layer for all local replicas (only the
    writing rank generates the weights).
    profile: "forward" (default) pushes the profile stream through every
    layer's experts (full residency) and builds each layer's buddy table and
    tau from the routing it sees there, like the reference's cmd_profile
    (harness.py:93-101); "route" routes the same profile tokens at every layer
    (no expert forward; the CPU twin then builds bit-identical tables).
    clustered: experts follow the reference's clustered recipe on
    `clusters` clusters shared with the router (default synth.CLUSTERS[name],
    the reference's default model.clusters = 8 capped at E), else independent
    N(0, 1/fan_in) experts and min(E, 8) router clusters."""
    import time
    E, k, d, f, rate = SHAPES[name]
    if cache_rate is not None:
        rate = float(cache_rate)
    S = SHARED.get(name, 0)
    cap = int(math.floor(rate * E))
    k_max = k_max if k_max is not None else min(16, E - 1)
    if clusters is None:
        clusters = synth.CLUSTERS[name] if clustered else min(E, 8)
    spec = substrate.ModelSpec(num_layers=layers, experts_per_layer=E, top_k=k, hidden_dim=d, ffn_dim=f,
                               num_clusters=clusters, seed=7)
    cl_of = synth.cluster_of(E, clusters) if clustered else None
    gw, gb = substrate.gate_weights(spec)
    gate_w = torch.from_numpy(gw.astype(np.float32)).to(device)
    gate_b = torch.from_numpy(gb.astype(np.float32)).to(device)
    buf_elems = 3 * d * f
    buf_bytes = buf_elems * 2
    t0 = time.time()
    mirrors = []
    if profile not in ("route", "forward"):
        raise ValueError(f"profile must be 'route' or 'forward', got {profile!r}")
    luts = [torch.from_numpy(synth.lut_bf16(synth.matrix_scale(d, f, m)).view(np.int16)).to(device)
            for m in (synth.W1, synth.W3, synth.W2)]
    row = torch.empty(buf_elems, device=device, dtype=torch.bfloat16)
    writer = share is None or share.owner
    arena = torch.empty(E + S, buf_elems, device=device, dtype=torch.bfloat16)
    ids_all = torch.full((layers, E, k_max), -1, device=device, dtype=torch.int32)
    len_all = torch.zeros(layers, E, device=device, dtype=torch.int32)
    taus = []
    x = torch.from_numpy(substrate.token_stream(spec, 1, profile_tokens).astype(np.float32)).to(device)
    ws = None
    mean_len = []
    for l in range(layers):
        if writer or profile == "forward":
            for e in range(E + S):  # row-major N(0, 1/fan_in) (synth.py), then the UMMA-tiled HBM layout
                w = _synth_expert(luts, seed, l, e, d, f, row,
                                  None if cl_of is None or e >= E else int(cl_of[e]))
                ops.pack_expert_bf16(w[: f * d].view(f, d), w[f * d: 2 * f * d].view(f, d),
                                     w[2 * f * d:].view(d, f), ops.ACT_SWIGLU, arena[e])
        if not writer:
            m = None  # attached after the owner has written every layer
        else:
            make = HostMirror if share is None else (lambda n, _l=l: SharedMirror(share.path(_l), n, create=True))
            if codec:
                m = coded_mirror_from_device(arena, make)
            else:
                m = make((E + S) * buf_bytes)
                fill_mirror_from_device(m, arena)
        mirrors.append(m)
        # ---- profile this layer ----
        r, t, tau = profile_tables(x, gate_w[l], gate_b[l], k, E, alpha, k_max, tau_percentile)
        ids_all[l], len_all[l] = t.ids, t.lens
        mean_len.append(float(t.lens.float().mean()))
        taus.append(tau)
        if log:
            log(f"layer {l}: mirror {(m.nbytes if m else 0) / 2**30:.2f} GiB, tau {taus[-1]:.4f}, "
                f"mean buddies {mean_len[-1]:.2f}, {time.time() - t0:.1f}s")
        if profile == "route":
            continue
        kept = torch.zeros_like(r.topk, dtype=torch.uint8)  # identity plan: full residency
        ex, kd, pr = r.topk, kept, r.probs
        if S:
            ex, kd, pr = ops.append_shared(ex, kd, pr, E, S)
        perm = ops.permute(ex, kd, E + S)
        if ws is None or ws.r_max < perm.r_max:
            ws = ops.FfnWorkspace(E + S, d, f, perm.r_max, 256, device)
        xp = ops.gather_rows(x, perm, 1)
        yp = ops.expert_ffn_bf16(xp, perm, arena, torch.arange(E + S, device=device, dtype=torch.int32), d, f,
                                 ops.ACT_SWIGLU, ws)
        x = ops.combine(yp, perm, pr, kd, h_in=x)
    torch.cuda.synchronize()
    del arena, ws, row
    if share is not None:
        share.barrier()
        if not share.owner:
            mirrors = [SharedMirror(share.path(l)) for l in range(layers)]
        share.barrier()  # every rank has mapped every layer: drop the names, so a crash cannot leak /dev/shm
        if share.owner:
            for m in mirrors:
                m.unlink()
    initial = [initial_residents(E, cap, 0, l) for l in range(layers)]
    es = EngineSpec(num_layers=layers, num_experts=E, top_k=k, d=d, f=f, capacity=cap, max_batch=max_batch,
                    act=ops.ACT_SWIGLU, search_rank_h=k_max, rho=rho, n_tile=n_tile, expert_bytes=buf_bytes,
                    num_shared=S)
    return Workload(name, spec, es, mirrors, gate_w, gate_b, ids_all, len_all, taus, initial,
                    profile_seconds=time.time() - t0, mean_buddies=float(np.mean(mean_len)),
                    extra={"cache_rate": rate, "profile": profile, "seed": seed, "alpha": alpha,
                           "clusters": clusters, "clustered": clustered, "spread": synth.SPREAD if clustered else None,
                           "tau_percentile": tau_percentile, "profile_tokens": profile_tokens})
