"""Size-independent parity at the BASELINE shapes (Mixtral-8x7B, Qwen3-30B-A3B,
DeepSeek-V2-Lite routed experts), bf16 tensor-core engine with few layers:

* every layer-step's remap plan equals the oracle planner run on the very
  routing, gates and residency snapshot the GPU saw (bit-exact);
* the control plane's full event log equals the oracle cache replica
  replaying those plans (bit-exact), i.e. hit/miss/evict/prefetch decisions;
* the delta/batch gate equals the oracle's on the same snapshot;
* buffers: the engine never exceeds its HBM pool (no InvariantViolation).
"""

import numpy as np
import pytest
import torch

import oracle as O
from paper_2511_10054_b200 import workload as W

pytestmark = pytest.mark.gpu


def _oracle_replay(wl, trace, B, n_steps, L):
    """Replay harness.py:315-393 decisions with the oracle: plans from the
    traced routing, then the memtier replica; returns the event array."""
    E, cap = wl.eng.num_experts, wl.eng.capacity
    st = [O.Residency(E, cap, O.POLICY_LRU, O.initial_residents(E, cap, O.POLICY_LRU, 0, l), None, l)
          for l in range(L)]
    clock, log = O.Clock(), []
    prev = [dict() for _ in range(L)]
    ebytes = wl.eng.expert_bytes
    pre_ms = 1000.0 * ebytes / wl.eng.pcie_bw_bytes_per_s
    ids_all = wl.tbl_ids.cpu().numpy()
    lens_all = wl.tbl_len.cpu().numpy()
    i = 0
    for step in range(n_steps):
        toks = np.arange(step * B, (step + 1) * B)
        for l in range(L):
            rec = trace[i]
            i += 1
            assert rec["layer"] == l
            t = (l + 1) % L
            O.prefetch(st[t], O.predict_for_layer(cap, prev[t]), clock, pre_ms, log)
            O.settle(st[l], clock, ebytes, log)
            assert np.array_equal(rec["mask"], st[l].mask), "snapshot differs"
            delta, bok = O.distribution_gate(rec["topk"].ravel(), st[l].mask, wl.eng.beta)
            assert bok == rec["batch_ok"]
            ex, kd, _ = O.remap_batch(rec["topk"], None, st[l].mask, ids_all[l], np.zeros(ids_all[l].shape),
                                      lens_all[l], rec["allowed"] & bok, wl.eng.search_rank_h,
                                      -1 if wl.eng.rho is None else wl.eng.rho)
            assert np.array_equal(ex, rec["executed"]) and np.array_equal(kd, rec["kind"]), f"plan differs at {i}"
            slots = 0
            for b in range(B):
                for s in range(rec["topk"].shape[1]):
                    if kd[b, s] == O.KIND_SUBSTITUTED:
                        O.access(st[l], int(rec["topk"][b, s]), clock, wl.eng.load_ms, wl.eng.hit_ms, ebytes, True,
                                 int(toks[b]), log)
                    O.access(st[l], int(ex[b, s]), clock, wl.eng.load_ms, wl.eng.hit_ms, ebytes, False,
                             int(toks[b]), log)
                    slots += 1
            clock.now += wl.eng.compute_ms * slots
            cnt = {}
            for e in ex.ravel():
                cnt[int(e)] = cnt.get(int(e), 0) + 1
            prev[l] = cnt
    return np.array(log, np.float64).reshape(-1, 7)


def test_dsv2_shared_experts_numerics(cuda_ok):
    """DeepSeek-V2-Lite shape: 64 routed (top-6) + 2 always-resident shared
    experts. One layer-step of the bf16 engine vs an fp32 torch reference that
    applies the engine's own plan plus both shared experts with weight 1,
    then layer_update: rel 2e-2 per token."""
    wl = W.build("dsv2lite", layers=1, max_batch=8, profile_tokens=512)
    E, S, d, f = 64, 2, 2048, 1408
    from paper_2511_10054_b200 import synth
    luts = [torch.from_numpy(synth.lut_bf16(synth.matrix_scale(d, f, m)).view(np.int16)).cuda() for m in range(3)]
    # workload seed 0, layer 0: regenerate the row-major weights
    # the workload's clustered recipe (routed experts only; the shared ones are independent)
    cl_of = synth.cluster_of(E, wl.extra["clusters"])
    experts = [W._synth_expert(luts, 0, 0, e, d, f, torch.empty(3 * d * f, dtype=torch.bfloat16, device="cuda"),
                               int(cl_of[e]) if e < E else None).float()
               for e in range(E + S)]
    eng = wl.engine("buddy")
    eng.set_trace(True)
    x = torch.from_numpy(wl.tokens(2, 8)).cuda()
    h0 = x.clone()
    eng.step(x, np.arange(8))
    torch.cuda.synchronize()
    rec = eng.trace()[0]
    from paper_2511_10054_b200 import ops
    r = ops.gate_topk(h0, wl.gate_w[0], wl.gate_b[0], 6)
    probs = r.probs.cpu().numpy()
    assert np.array_equal(r.topk.cpu().numpy(), rec["topk"])
    xb = h0.to(torch.bfloat16).float()

    def ffn(e, v):
        w = experts[e]
        W1, W3, W2 = w[: f * d].view(f, d), w[f * d: 2 * f * d].view(f, d), w[2 * f * d:].view(d, f)
        hh = torch.nn.functional.silu(v @ W1.T) * (v @ W3.T)
        return hh.to(torch.bfloat16).float() @ W2.T

    y = torch.zeros_like(h0)
    for b in range(8):
        for s in range(6):
            if rec["kind"][b, s] != 3:
                y[b] += float(probs[b, s]) * ffn(int(rec["executed"][b, s]), xb[b:b + 1])[0]
        for sx in range(S):
            y[b] += ffn(E + sx, xb[b:b + 1])[0]
    ref = h0 + 0.5 * y
    ref = ref / ref.pow(2).mean(1, keepdim=True).sqrt()
    rel = (torch.linalg.norm(x - ref, dim=1) / torch.linalg.norm(ref, dim=1)).max().item()
    assert rel <= 2e-2, rel
    eng.close()
    wl.close()


@pytest.mark.parametrize("name,layers,B", [("mixtral", 2, 16), ("qwen3", 3, 16), ("dsv2lite", 3, 8),
                                           ("qwen3", 2, 512)])  # the last one is a prefill-sized batch
def test_engine_decisions_bit_exact_at_baseline_shapes(cuda_ok, name, layers, B):
    wl = W.build(name, layers=layers, max_batch=B, profile_tokens=2048)
    eng = wl.engine("buddy")
    eng.set_trace(True)
    steps = 4
    x = torch.from_numpy(wl.tokens(2, steps * B)).cuda()
    for s in range(steps):
        eng.step(x[s * B:(s + 1) * B], np.arange(s * B, (s + 1) * B))
    torch.cuda.synchronize()
    ev = eng.events()
    ref = _oracle_replay(wl, eng.trace(), B, steps, layers)
    assert ev.shape == ref.shape and np.array_equal(ev, ref)
    st = eng.stats()
    assert st["tokens"] == steps * B and np.isfinite(x.cpu().numpy()).all()
    eng.close()
    wl.close()


@pytest.mark.parametrize("model", ["qwen3", "dsv2lite"])
def test_engine_fused_combine_equals_separate_launch(model):
    """The engine's layer-step runs K5 inside its last fused FFN launch
    (post1 when nothing is fetched, else post2; DSV2: the shared experts'
    slots ride along); with BMOE_FUSE_COMBINE=0 it is its own launch. Hidden
    states bitwise equal, event logs equal, one kernel launch fewer per decode
    layer-step."""
    import os
    wl = W.build(model, layers=3, max_batch=16, profile_tokens=1024)
    outs, evs, launches = [], [], []
    old = os.environ.get("BMOE_FUSE_COMBINE")
    try:
        for flag in ("0", "1"):
            os.environ["BMOE_FUSE_COMBINE"] = flag
            eng = wl.engine("buddy")
            x = torch.from_numpy(wl.tokens(2, 64)).cuda()
            for s in range(4):
                eng.step(x[s * 16:(s + 1) * 16], np.arange(s * 16, (s + 1) * 16))
            torch.cuda.synchronize()
            outs.append(x.cpu().numpy())
            evs.append(eng.events())
            launches.append(eng.stats()["kernel_launches"])
            eng.close()
    finally:
        if old is None:
            os.environ.pop("BMOE_FUSE_COMBINE", None)
        else:
            os.environ["BMOE_FUSE_COMBINE"] = old
        wl.close()
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    assert np.array_equal(evs[0], evs[1])
    assert launches[0] - launches[1] == 3 * 4, launches


def test_engine_varying_batch_sizes_graphs_equal_eager():
    """One engine serving decode batches of different sizes (16, 64, 8, 64,
    16 tokens: token tiles 16 / 64 / 16, graphs captured per (layer, B)) over
    one FFN workspace: hidden states bitwise equal to the same sequence run
    eagerly without graphs, and event logs equal."""
    import os
    wl = W.build("qwen3", layers=2, max_batch=64, profile_tokens=1024)
    sizes = (16, 64, 8, 64, 16, 16, 64)
    outs, evs = [], []
    old = os.environ.get("BMOE_GRAPHS")
    try:
        for graphs in ("1", "0"):
            os.environ["BMOE_GRAPHS"] = graphs
            eng = wl.engine("buddy")
            x = torch.from_numpy(wl.tokens(5, sum(sizes))).cuda()
            o = 0
            for B in sizes:
                eng.step(x[o:o + B], np.arange(o, o + B))
                o += B
            torch.cuda.synchronize()
            outs.append(x.cpu().numpy())
            evs.append(eng.events())
            eng.close()
    finally:
        if old is None:
            os.environ.pop("BMOE_GRAPHS", None)
        else:
            os.environ["BMOE_GRAPHS"] = old
        wl.close()
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    assert np.array_equal(evs[0], evs[1])


def test_engine_zero_copy_plan_equals_copies():
    """The remap reads the residency snapshot and writes the packed plan
    through mapped pinned memory (no upload / readback copy on the host round
    trip); BMOE_ZERO_COPY=0 restores the copies. Same decisions, events and
    hidden states bit for bit, with the buddy and the Random method."""
    import os
    wl = W.build("qwen3", layers=3, max_batch=16, profile_tokens=1024)
    old = os.environ.get("BMOE_ZERO_COPY")
    try:
        for method in ("buddy", "random", "original"):
            outs, evs = [], []
            for zc in ("1", "0"):
                os.environ["BMOE_ZERO_COPY"] = zc
                eng = wl.engine(method)
                x = torch.from_numpy(wl.tokens(4, 80)).cuda()
                for s, B in enumerate((16, 16, 1, 16, 8)):
                    o = sum((16, 16, 1, 16, 8)[:s])
                    eng.step(x[o:o + B], np.arange(o, o + B))
                torch.cuda.synchronize()
                outs.append(x.cpu().numpy())
                evs.append(eng.events())
                eng.close()
            assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32)), method
            assert np.array_equal(evs[0], evs[1]), method
    finally:
        if old is None:
            os.environ.pop("BMOE_ZERO_COPY", None)
        else:
            os.environ["BMOE_ZERO_COPY"] = old
        wl.close()
