"""The paper's Random baseline on the engine (method="random"), pinned to the
REFERENCE's run_simulation(method="random") (harness.py:299-300, 358-359;
substitution.py:227-248) on the tiny config at three cache rates and run
seeds: the engine draws from a host replica of numpy's PCG64 stream, so the
event log must equal the reference's bit for bit, the counters exactly, and
the outputs (fp32 parity mode) within 1e-4 relative of the reference's f64.

Also here: the data-plane hazard of a speculative fetch still in flight when
its expert is evicted unused (LFU + prefetch), checked on outputs."""

import numpy as np
import pytest
import torch

from conftest import golden
from paper_2511_10054_b200 import harness, ops, substrate
from paper_2511_10054_b200.engine import DecodeEngine, EngineSpec, HostMirror

pytestmark = pytest.mark.gpu

TINY = {"model.layers": 4, "model.experts": 8, "model.top_k": 2, "model.hidden_dim": 128, "model.ffn_dim": 256,
        "model.clusters": 8, "stream.batch": 16, "sub.h": 7, "stream.seed": 2, "stream.num_tokens": 320,
        "method": "random"}


@pytest.mark.parametrize("tag", ["c500_s0", "c375_s5", "c750_s11"])
def test_random_arm_equals_reference(cuda_ok, tag):
    g = golden("sim_tiny_random.npz")
    rate, seed = g[f"{tag}_cfg"]
    r = harness.run_simulation(dict(TINY, **{"cache.rate": float(rate), "run.seed": int(seed)}))
    ref = g[f"{tag}_events"]
    got = harness.events_array(r.events)
    assert got.shape == ref.shape, (got.shape, ref.shape)
    assert np.array_equal(got, ref)
    m = r.metrics
    vals = np.array([m.tokens_per_s, m.stall_ms, m.compute_ms, m.hits, m.misses_ondemand, m.misses_substituted,
                     m.drops, m.prefetch_issued, m.prefetch_completed, m.evictions, m.read_bytes, m.substitutions])
    assert np.array_equal(vals, g[f"{tag}_metrics"][:12]), (vals, g[f"{tag}_metrics"][:12])
    ro = g[f"{tag}_outputs"]
    rel = np.linalg.norm(r.outputs - ro, axis=1) / np.linalg.norm(ro, axis=1)
    assert rel.max() <= 1e-4, rel.max()
    assert abs(m.fidelity_cosine - g[f"{tag}_metrics"][12]) <= 1e-6


def _bf16_mirrors(L, E, d, f, seed):
    gen = torch.Generator(device="cuda")
    mirrors = []
    for l in range(L):
        gen.manual_seed(seed + l)
        tiled = torch.empty(E, 3 * d * f, dtype=torch.bfloat16, device="cuda")
        for e in range(E):
            w = torch.empty(3 * d * f, device="cuda", dtype=torch.bfloat16)
            w[: 2 * d * f].normal_(0.0, d ** -0.5, generator=gen)
            w[2 * d * f:].normal_(0.0, f ** -0.5, generator=gen)
            ops.pack_expert_bf16(w[: f * d].view(f, d), w[f * d: 2 * f * d].view(f, d), w[2 * f * d:].view(d, f),
                                 ops.ACT_SWIGLU, tiled[e])
        m = HostMirror(tiled.numel() * 2)
        m.as_tensor(torch.bfloat16).copy_(tiled.view(-1).cpu())
        mirrors.append(m)
    return mirrors


@pytest.mark.parametrize("policy,B,steps", [("lfu", 1, 96), ("lru", 8, 24)])
def test_speculative_fetch_evicted_unused_keeps_weights_intact(cuda_ok, policy, B, steps):
    """method=original executes every routed expert exactly, so its outputs do
    not depend on the cache at all: a small LFU/LRU cache with prefetch on and
    25 MB experts (copies long enough to be in flight when their expert is
    evicted unused) must give the outputs of a cache that holds every expert.
    A buffer reused while its speculative copy still lands would corrupt an
    expert (relative error ~1, far above the 1e-2 allowed for the different
    grouping of the FFN launches: bf16 intermediates, measured <= 1.1e-3).
    LFU at B=1 makes the predictor fire: an expert executed early in a step is
    evicted by a later miss of the same step, gets prefetched, lands with
    frequency 0 and is the next victim, possibly before its copy finished."""
    spec = substrate.ModelSpec(num_layers=3, experts_per_layer=8, top_k=2, hidden_dim=1024, ffn_dim=4096,
                               num_clusters=8)
    L, E, k, d, f = 3, 8, 2, 1024, 4096
    mirrors = _bf16_mirrors(L, E, d, f, 123)
    gw, gb = substrate.gate_weights(spec)
    gwt = torch.tensor(gw, dtype=torch.float32, device="cuda")
    gbt = torch.tensor(gb, dtype=torch.float32, device="cuda")
    x0 = torch.from_numpy(substrate.token_stream(spec, 4, B * steps).astype(np.float32)).cuda()
    outs, rel = {}, None
    for cap in (4 if B == 1 else 2, E):
        es = EngineSpec(num_layers=L, num_experts=E, top_k=k, d=d, f=f, capacity=cap, max_batch=B,
                        method="original", policy=policy, prefetch=True, expert_bytes=3 * d * f * 2,
                        load_ms=9.5, hit_ms=0.0, compute_ms=0.5, pcie_bw_bytes_per_s=4.0e9)
        eng = DecodeEngine(es, mirrors, gwt, gbt, None, None, [-1.0] * L,
                           [list(range(cap))] * L)
        x = x0.clone()
        for s in range(steps):
            eng.step(x[s * B:(s + 1) * B], np.arange(s * B, (s + 1) * B))
        torch.cuda.synchronize()
        st = eng.stats()
        eng.close()
        outs[cap] = (x.double().cpu().numpy(), st)
    small = min(outs)
    a, b = outs[small][0], outs[E][0]
    rel = np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)
    st = outs[small][1]
    print(f"{policy}: physical fetches {st['physical_fetches']}, prefetch copies {st['prefetch_copies']}, "
          f"in-flight releases {st['inflight_releases']}, max rel {rel.max():.2e}")
    assert st["physical_fetches"] > 0
    if policy == "lfu":
        assert st["prefetch_copies"] > 0
    assert rel.max() <= 1e-2, rel.max()
    for m in mirrors:
        m.close()
