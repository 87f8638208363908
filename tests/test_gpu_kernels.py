"""Parity of every CUDA kernel against the oracle / reference golden vectors.

All tests call through the C-ABI (libbmoe.so via ctypes). Bit-exact for
integer / index / table work; tolerances are stated where floating point
differs (fp32 mode rel 1e-5, bf16 mode rel 2e-2 vs an fp32 reference).
"""

import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden
from paper_2511_10054_b200 import ops
from paper_2511_10054_b200.errors import InputError

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _t(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def _corpus(name):
    g = golden(name)
    for i in range(g["E"].shape[0]):
        E, k = int(g["E"][i]), int(g["k"][i])
        yield dict(E=E, k=k, topk=g["topk"][i, :k], logits=g["logits"][i, :E], mask=g["mask"][i, :E],
                   ids=g["ids"][i, :E], w=g["w"][i, :E], lens=g["lens"][i, :E], h=int(g["h"][i]),
                   rho=int(g["rho"][i]), allowed=bool(g["allowed"][i]), eta=float(g["eta"][i]),
                   kappa=float(g["kappa"][i]), part=g["part"][i, :E] if g["has_part"][i] else None,
                   fallback=int(g["fallback"][i]), executed=g["executed"][i, :k], kind=g["kind"][i, :k],
                   used=int(g["used"][i]))


@pytest.mark.parametrize("name", ["remap_corpus_20260819.npz", "remap_corpus_1234.npz"])
def test_remap_kernel_bit_exact_on_reference_corpus(cuda_ok, name):
    """K2 vs the reference planner on the acceptance (1000, seed 20260819) and
    fuzz (300, seed 1234) corpora, incl. Psi ordering, rho, H, drop fallback."""
    n = 0
    for c in _corpus(name):
        table = ops.DeviceTable(_t(c["ids"]), _t(c["w"]), _t(c["lens"]))
        plan = ops.buddy_remap(
            _t(c["topk"][None, :], torch.int32), _t(np.array([c["allowed"]], np.uint8)),
            ops.bitmap_from_mask(c["mask"], DEV), table, H=c["h"], rho=None if c["rho"] < 0 else c["rho"],
            fallback=c["fallback"], beta=2.0, eta=c["eta"], kappa=c["kappa"],
            partition_of=None if c["part"] is None else _t(c["part"], torch.int32), hop=1.0,
            logits=_t(c["logits"][None, :]))
        ex = plan.executed.cpu().numpy()[0]
        kd = plan.kind.cpu().numpy()[0]
        assert list(ex) == list(c["executed"]), (n, ex, c)
        assert list(kd) == list(c["kind"]), (n, kd, c)
        assert int(plan.used.cpu()[0]) == c["used"]
        n += 1
    assert n in (1000, 300)


def test_remap_batch_gates_and_methods(cuda_ok):
    """Batch semantics: delta over requested slots (duplicates counted), the
    beta bypass, ondemand_plan and identity_plan (gating.py:126-165,
    substitution.py:211-224) against the oracle on a random batch."""
    rng = np.random.default_rng(3)
    E, k, B = 64, 6, 48
    topk = np.stack([rng.choice(E, k, replace=False) for _ in range(B)])
    mask = rng.random(E) < 0.5
    lists_ids = [rng.permutation([j for j in range(E) if j != p])[:16] for p in range(E)]
    ids, w, lens = O.table_from_lists(lists_ids, [np.sort(rng.random(16))[::-1] for _ in range(E)], 16)
    allowed = rng.random(B) < 0.8
    table = ops.DeviceTable(_t(ids), _t(w), _t(lens))
    bm = ops.bitmap_from_mask(mask, DEV)
    for beta in (1.0, 0.5, 0.3):
        delta, batch_ok = O.distribution_gate(topk.ravel(), mask, beta)
        plan = ops.buddy_remap(_t(topk, torch.int32), _t(allowed.astype(np.uint8)), bm, table, H=8, rho=2,
                               beta=beta)
        ex_o, kd_o, used_o = O.remap_batch(topk, None, mask, ids, w, lens, allowed & batch_ok, 8, 2)
        assert np.array_equal(plan.executed.cpu().numpy(), ex_o)
        assert np.array_equal(plan.kind.cpu().numpy(), kd_o)
        assert np.array_equal(plan.used.cpu().numpy(), used_o)
        assert float(plan.delta.cpu()[0]) == delta and bool(plan.batch_allowed.cpu()[0]) == batch_ok
    ex_o, kd_o, _ = O.ondemand_plan(topk, mask)
    plan = ops.buddy_remap(_t(topk, torch.int32), None, bm, None, method=ops.METHOD_ORIGINAL, num_experts=E)
    assert np.array_equal(plan.executed.cpu().numpy(), ex_o) and np.array_equal(plan.kind.cpu().numpy(), kd_o)
    plan = ops.buddy_remap(_t(topk, torch.int32), None, bm, None, method=ops.METHOD_IDENTITY, num_experts=E)
    assert np.array_equal(plan.executed.cpu().numpy(), topk) and not plan.kind.cpu().numpy().any()


@pytest.mark.parametrize("name", ["routing_tiny.npz", "routing_default.npz", "routing_e128.npz"])
def test_select_from_reference_logits_bit_exact(cuda_ok, name):
    """Identical logits give identical indices (model.py:259-263)."""
    g = golden(name)
    k = g["topk"].shape[1]
    r = ops.select_topk_f64(_t(g["logits"]), k, float(g["T"]))
    assert np.array_equal(r.topk.cpu().numpy(), g["topk"])
    np.testing.assert_allclose(r.probs64.cpu().numpy(), g["probs"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(r.tae.cpu().numpy(), g["tae"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(r.margin.cpu().numpy(), g["margin"], rtol=0, atol=1e-12)


def test_select_ties_to_lower_index(cuda_ok):
    # test_model.py:115-120: all-equal logits select [0,1,2,3]
    r = ops.select_topk_f64(torch.zeros(3, 8, dtype=torch.float64, device=DEV), 4)
    assert r.topk.cpu().numpy().tolist() == [[0, 1, 2, 3]] * 3
    z = torch.tensor([[1.0, 3.0, 3.0, 2.0, 3.0]], dtype=torch.float64, device=DEV)
    assert ops.select_topk_f64(z, 3).topk.cpu().numpy().tolist() == [[1, 2, 4]]


@pytest.mark.parametrize("name", ["routing_tiny.npz", "routing_default.npz", "routing_e128.npz"])
def test_fused_gate_fp32(cuda_ok, name):
    """K1 fp32 GEMV: logits within normwise 1e-5 of the f64 reference; given
    its own fp32 logits the selection/gates equal the oracle bit-exactly."""
    g = golden(name)
    k = g["topk"].shape[1]
    T = float(g["T"])
    x, wg, b = g["x"], g["gate_w"], g["gate_b"]
    r = ops.gate_topk(_t(x, torch.float32), _t(wg, torch.float32), _t(b, torch.float32), k, T, tau=0.5)
    z = r.logits.cpu().numpy().astype(np.float64)
    scale = np.linalg.norm(x, axis=1)[:, None] * np.linalg.norm(wg, axis=1).max()
    assert np.all(np.abs(z - g["logits"]) <= 1e-5 * scale)
    tk, pr = O.select_topk(z, k, T)
    assert np.array_equal(r.topk.cpu().numpy(), tk)
    np.testing.assert_allclose(r.probs.cpu().numpy(), pr, rtol=1e-6, atol=1e-7)
    tae_o = np.array([O.tae(p) for p in pr])
    np.testing.assert_allclose(r.tae.cpu().numpy(), tae_o, rtol=0, atol=1e-12)
    exempt = np.abs(tae_o - 0.5) < 1e-12
    ok_o = np.array([O.token_gate(p, 0.5) for p in pr])
    assert np.array_equal(r.allowed.cpu().numpy().astype(bool)[~exempt], ok_o[~exempt])
    # routing agreement with the f64 reference end to end (reported)
    agree = np.mean(np.all(r.topk.cpu().numpy() == g["topk"], axis=1))
    assert agree >= 0.99


@pytest.mark.parametrize("name", ["coact_tiny.npz", "coact_default_w05.npz", "coact_e128.npz",
                                  "coact_e160_noeps.npz"])
def test_coact_and_rank_bit_exact(cuda_ok, name):
    """K6 counts and K7 tables vs the reference's observe + build_table."""
    g = golden(name)
    E, ws, ww = int(g["E"]), int(g["warmup_steps"]), float(g["warmup_weight"])
    topk = _t(g["topk"], torch.int32)
    warm_c, warm_p = ops.coact_count(topk[:ws], E)
    main_c, main_p = ops.coact_count(topk[ws:], E)
    counts = ops.counts_to_f64(main_c, warm_c, ww).cpu().numpy()
    pairs = ops.counts_to_f64(main_p, warm_p, ww).cpu().numpy()
    assert np.array_equal(counts, g["counts"]) and np.array_equal(pairs, g["pairs"])
    pw = ops.coact_weighted(topk[ws:], _t(g["probs"][ws:], torch.float32), E, 1.0)
    if ww:
        ops.coact_weighted(topk[:ws], _t(g["probs"][:ws], torch.float32), E, ww, pw)
    np.testing.assert_allclose(pw.cpu().numpy(), g["pw"], rtol=1e-5, atol=1e-9)
    for i in range(int(g["nbuild"])):
        alpha, kmax, mode = float(g[f"b{i}_alpha"]), int(g[f"b{i}_kmax"]), str(g[f"b{i}_mode"])
        M = _t(g["pairs"] if mode == "binary" else g["pw"])
        t = ops.buddy_rank(M, float(g["eps"]), alpha, kmax)
        assert np.array_equal(t.ids.cpu().numpy(), g[f"b{i}_ids"]), (name, i)
        assert np.array_equal(t.lens.cpu().numpy(), g[f"b{i}_lens"]), (name, i)
        assert np.array_equal(t.weights.cpu().numpy(), g[f"b{i}_w"]), (name, i)


def test_coact_counts_large_random_vs_oracle(cuda_ok):
    """Many CTAs + the k=8 vector path: 2M tokens, E=128 (bincount oracle)."""
    rng = np.random.default_rng(11)
    N, E, k = 2_000_000, 128, 8
    pop = 1.0 / np.arange(1, E + 1) ** 0.8
    pop /= pop.sum()
    # distinct ids per row: Gumbel top-k over log-popularity
    gumb = rng.gumbel(size=(N, E)).astype(np.float32) + np.log(pop).astype(np.float32)
    topk = np.argpartition(-gumb, k, axis=1)[:, :k].astype(np.int32)
    del gumb
    c, p = ops.coact_count(_t(topk), E)
    oc, op, _, _ = O.coact_count(topk, None, E, 0, 0, 0.0)
    assert np.array_equal(c.cpu().numpy().astype(np.float64), oc)
    assert np.array_equal(p.cpu().numpy().astype(np.float64), op)


def test_coact_full_64m_trace_vs_one_hot_products(cuda_ok):
    """BASELINE configs[4] at full size: the 64M-token, E=128, k=8 bench
    trace. K6's counts and pair matrix equal an independent count — the
    one-hot products X^T X of 4M-token slices (fp32 tensor products of 0/1
    matrices, exact below 2^24 per slice) summed in int64 — and satisfy the
    size-independent identities (symmetry, zero diagonal, row sums =
    (k-1) * counts, total = N * k * (k-1))."""
    import bench
    N, E, k = 64 * 1024 * 1024, 128, 8
    trace = bench.gen_trace(N, E, k, 0, N, "cuda")
    c, p = ops.coact_count(trace, E)
    ref = torch.zeros(E, E, dtype=torch.int64, device="cuda")
    step = 4 * 1024 * 1024
    for a in range(0, N, step):
        oh = torch.zeros(min(step, N - a), E, dtype=torch.float32, device="cuda")
        oh.scatter_(1, trace[a:a + step].long(), 1.0)
        ref += (oh.T @ oh).round().to(torch.int64)
        del oh
    assert torch.equal(c, torch.diagonal(ref))
    ref.fill_diagonal_(0)
    assert torch.equal(p, ref)
    assert torch.equal(p, p.T) and int(torch.diagonal(p).abs().sum()) == 0
    assert torch.equal(p.sum(1), (k - 1) * c)
    assert int(p.sum()) == N * k * (k - 1) and int(c.sum()) == N * k


@pytest.mark.parametrize("k", [1, 3, 8])
def test_coact_rejects_bad_rows(cuda_ok, k):
    """Rows with repeated / out-of-range ids are rejected (profiler.py:76-80);
    the valid rows are still counted exactly (k=1 exercises the counted
    diagonal, k>=2 the derived one)."""
    rng = np.random.default_rng(5 + k)
    E, N = 16, 4096
    topk = np.stack([rng.permutation(E)[:k] for _ in range(N)]).astype(np.int32)
    bad = np.zeros(N, bool)
    bad[rng.choice(N, 40, replace=False)] = True
    for t in np.flatnonzero(bad):
        if k > 1 and t % 2:
            topk[t, 1] = topk[t, 0]          # duplicate
        else:
            topk[t, k - 1] = E + (t % 3)      # out of range
    with pytest.raises(InputError):
        ops.coact_count(_t(topk), E)
    c, p = ops.coact_count(_t(topk), E, check=False)
    oc, op, _, _ = O.coact_count(topk[~bad], None, E, 0, 0, 0.0)
    assert np.array_equal(c.cpu().numpy().astype(np.float64), oc)
    assert np.array_equal(p.cpu().numpy().astype(np.float64), op)


def _arena_tanh(w_in, w_out):
    # buffer layout TANH: [Win^T (f x d) | Wout^T (d x f)]
    E = w_in.shape[0]
    return np.concatenate([np.transpose(w_in, (0, 2, 1)).reshape(E, -1),
                           np.transpose(w_out, (0, 2, 1)).reshape(E, -1)], axis=1)


def test_forward_tanh_fp32_vs_reference(cuda_ok):
    """permute -> gather -> fp32 FFN -> combine (+layer_update) vs the
    reference forward_batch on the same plan (model.py:318-347): rel 1e-5."""
    from paper_2511_10054_b200 import substrate as S
    g = golden("forward_tiny.npz")
    spec = S.ModelSpec(num_layers=2, experts_per_layer=8, top_k=2, hidden_dim=128, ffn_dim=256, num_clusters=8)
    w_in, w_out = S.layer_stack(spec, 0)
    arena = _t(_arena_tanh(w_in, w_out), torch.float32)
    E, d, f = 8, 128, 256
    ex, kd = _t(g["executed"], torch.int32), _t(g["kind"], torch.uint8)
    perm = ops.permute(ex, kd, E)
    xs = _t(g["x"], torch.float32)
    xp = ops.gather_rows(xs, perm, 0)
    y_perm = ops.expert_ffn_f32(xp, perm, arena, _t(np.arange(E, dtype=np.int32)), d, f, ops.ACT_TANH)
    probs = _t(g["probs"], torch.float32)
    y = ops.combine(y_perm, perm, probs, kd).cpu().numpy()
    # a token whose slots are all dropped has y == 0 exactly (no renormalisation)
    rel = np.linalg.norm(y - g["y"], axis=1) / np.maximum(np.linalg.norm(g["y"], axis=1), 1.0)
    assert rel.max() <= 1e-5, rel.max()
    h = ops.combine(y_perm, perm, probs, kd, h_in=xs).cpu().numpy()
    relh = np.linalg.norm(h - g["h"], axis=1) / np.linalg.norm(g["h"], axis=1)
    assert relh.max() <= 1e-5, relh.max()


def _rand_swiglu(rng, E, d, f, dtype=np.float32):
    w1 = (rng.standard_normal((E, f, d)) / np.sqrt(d)).astype(dtype)
    w3 = (rng.standard_normal((E, f, d)) / np.sqrt(d)).astype(dtype)
    w2 = (rng.standard_normal((E, d, f)) / np.sqrt(f)).astype(dtype)
    return w1, w3, w2


def _plan(rng, B, E, k, drop=0.1):
    topk = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
    kind = np.where(rng.random((B, k)) < drop, 3, 0).astype(np.uint8)
    p = rng.random((B, k)) + 0.05
    return topk, kind, (p / p.sum(1, keepdims=True)).astype(np.float32)


def test_forward_swiglu_fp32_vs_oracle(cuda_ok):
    rng = np.random.default_rng(5)
    E, d, f, B, k = 8, 256, 384, 24, 2
    w1, w3, w2 = _rand_swiglu(rng, E, d, f)
    arena = _t(np.concatenate([w1.reshape(E, -1), w3.reshape(E, -1), w2.reshape(E, -1)], axis=1))
    topk, kind, probs = _plan(rng, B, E, k)
    x = rng.standard_normal((B, d)).astype(np.float32)
    perm = ops.permute(_t(topk), _t(kind), E)
    xp = ops.gather_rows(_t(x), perm, 0)
    yp = ops.expert_ffn_f32(xp, perm, arena, _t(np.arange(E, dtype=np.int32)), d, f, ops.ACT_SWIGLU)
    y = ops.combine(yp, perm, _t(probs), _t(kind)).cpu().numpy()
    ref = O.forward(x, topk, kind, probs.astype(np.float64),
                    lambda e, xr: O.ffn_swiglu(xr, w1[e].astype(np.float64), w3[e].astype(np.float64),
                                               w2[e].astype(np.float64)))
    rel = np.linalg.norm(y - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
    assert rel.max() <= 1e-5, rel.max()


def _bf16_case(rng, E, d, f, B, k, act, n_tile=64, bufs=None, drop=0.1):
    topk, kind, probs = _plan(rng, B, E, k, drop)
    x = rng.standard_normal((B, d)).astype(np.float32)
    nb = E if bufs is None else bufs
    gen = torch.Generator(device=DEV)
    gen.manual_seed(int(rng.integers(1 << 30)))
    nmat = 3 if act == ops.ACT_SWIGLU else 2
    arena = torch.empty(nb, nmat * d * f, device=DEV, dtype=torch.bfloat16)
    for bb in range(nb):  # N(0, 1/fan_in) per matrix, generated on the device
        row = arena[bb]
        for m in range(nmat):
            fan_in = f if m == nmat - 1 else d
            row[m * d * f:(m + 1) * d * f].copy_(
                torch.randn(d * f, device=DEV, generator=gen).mul_(fan_in ** -0.5))
    buf_of = rng.permutation(nb)[:E].astype(np.int32)
    perm = ops.permute(_t(topk), _t(kind), E)
    xs = _t(x)
    xp = ops.gather_rows(xs, perm, 1)
    ws = ops.FfnWorkspace(E, d, f, perm.r_max, n_tile)
    tiled = ops.pack_arena_bf16(arena, d, f, act)
    yp = ops.expert_ffn_bf16(xp, perm, tiled, _t(buf_of), d, f, act, ws)
    y = ops.combine(yp, perm, _t(probs), _t(kind))
    # fp32 torch reference over the same bf16-rounded weights and inputs;
    # H is rounded to bf16 like the kernel's GEMM2 operand
    xr = xs.to(torch.bfloat16).float()
    ref = torch.zeros(B, d, device=DEV)
    for e in range(E):
        sel = [(b, s) for b in range(B) for s in range(k) if topk[b, s] == e and kind[b, s] != 3]
        if not sel:
            continue
        row = arena[int(buf_of[e])].float()
        xb = xr[[b for b, _ in sel]]
        if act == ops.ACT_SWIGLU:
            W1, W3, W2 = row[: f * d].view(f, d), row[f * d: 2 * f * d].view(f, d), row[2 * f * d:].view(d, f)
            h = torch.nn.functional.silu(xb @ W1.T) * (xb @ W3.T)
        else:
            Wi, W2 = row[: f * d].view(f, d), row[f * d:].view(d, f)
            h = torch.tanh(xb @ Wi.T)
        out = h.to(torch.bfloat16).float() @ W2.T
        for i, (b, s) in enumerate(sel):
            ref[b] += float(probs[b, s]) * out[i]
        del row
    return y, ref, (xp, perm, tiled, buf_of, ws)


@pytest.mark.parametrize("E,d,f,B,k,act,n_tile", [
    (8, 128, 256, 16, 2, ops.ACT_SWIGLU, 64),     # tiny
    (8, 128, 256, 16, 2, ops.ACT_TANH, 64),       # the reference expert
    (8, 4096, 14336, 1, 2, ops.ACT_SWIGLU, 64),   # Mixtral decode B=1
    (8, 4096, 14336, 32, 2, ops.ACT_SWIGLU, 64),  # Mixtral decode B=32
    (128, 2048, 768, 64, 8, ops.ACT_SWIGLU, 64),  # Qwen3-shaped
    (64, 2048, 1408, 16, 6, ops.ACT_SWIGLU, 32),  # DSV2-shaped, narrow n tile
    (4, 256, 512, 200, 2, ops.ACT_SWIGLU, 64),    # many tokens per expert: N chunking
    (4, 256, 512, 200, 2, ops.ACT_SWIGLU, 256),   # widest tile, single TMEM stage
    (8, 4096, 14336, 600, 2, ops.ACT_SWIGLU, 256),  # Mixtral prefill: data-parallel tiles, epilogue-finished
    (128, 2048, 768, 1024, 8, ops.ACT_SWIGLU, 128),  # Qwen3 prefill, double-buffered accumulator
    (8, 128, 256, 300, 2, ops.ACT_TANH, 128),     # the reference expert, prefill width
])
def test_bf16_tcgen05_ffn_vs_fp32_reference(cuda_ok, E, d, f, B, k, act, n_tile):
    """K4 bf16 tensor-core grouped FFN: rel 2e-2 (normwise per token) vs fp32."""
    rng = np.random.default_rng(E * 1000 + B)
    y, ref, _ = _bf16_case(rng, E, d, f, B, k, act, n_tile)
    rel = (torch.linalg.norm(y - ref, dim=1) / torch.linalg.norm(ref, dim=1).clamp_min(1e-30)).max().item()
    assert rel <= 2e-2, rel


def test_bf16_ffn_deterministic_and_buffer_indirection(cuda_ok):
    """Two runs are bitwise identical (no split-K atomics); experts live in
    arbitrary arena buffers (buf_of_expert indirection, 12 buffers for 8)."""
    rng = np.random.default_rng(9)
    y, ref, (xp, perm, arena, buf_of, ws) = _bf16_case(rng, 8, 512, 1024, 40, 2, ops.ACT_SWIGLU, bufs=12)
    rel = (torch.linalg.norm(y - ref, dim=1) / torch.linalg.norm(ref, dim=1)).max().item()
    assert rel <= 2e-2
    d, f = 512, 1024
    rows = int(perm.offset[-1])  # rows past the last segment are never written
    y1 = ops.expert_ffn_bf16(xp, perm, arena, _t(buf_of), d, f, ops.ACT_SWIGLU, ws)[:rows]
    y2 = ops.expert_ffn_bf16(xp, perm, arena, _t(buf_of), d, f, ops.ACT_SWIGLU, ws)[:rows]
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("E,d,f,B,k,act,n_tile", [
    (8, 4096, 14336, 16, 2, ops.ACT_SWIGLU, 16),  # Mixtral decode, one expert per few CTAs
    (8, 4096, 14336, 1, 1, ops.ACT_SWIGLU, 16),   # a single expert, one token
    (128, 2048, 768, 64, 8, ops.ACT_SWIGLU, 64),  # Qwen3-shaped, many small experts
    (64, 2048, 1408, 16, 6, ops.ACT_SWIGLU, 32),  # DSV2-shaped (GEMM2 K/64 = 22)
    (8, 128, 256, 16, 2, ops.ACT_TANH, 64),       # the reference expert
])
def test_fused_single_launch_equals_multi_kernel(cuda_ok, E, d, f, B, k, act, n_tile):
    """The one-launch decode FFN (in-kernel split-tile reduction + grid
    barrier) sums the same partials in the same CTA order as the GEMM +
    fixup kernels, so its output is bitwise identical; 30 repeats catch
    ordering races in the arrival counters / barrier (self-cleaning state)."""
    import os
    rng = np.random.default_rng(E + B + d)
    _, _, (xp, perm, arena, buf_of, ws) = _bf16_case(rng, E, d, f, B, k, act, n_tile)
    rows = int(perm.offset[-1])
    bo = _t(buf_of)
    saved = {v: os.environ.get(v) for v in ("BMOE_FUSED", "BMOE_KPS", "BMOE_FFN_GROUPS", "BMOE_FFN_MIN_ITERS")}
    try:
        os.environ["BMOE_KPS"] = "2"  # same k-steps per stage -> same stream-K split in both paths
        os.environ["BMOE_FFN_GROUPS"] = "1"  # one stream-K range per GEMM over all CTAs, as the separate kernels
        os.environ["BMOE_FFN_MIN_ITERS"] = "1"
        os.environ["BMOE_FUSED"] = "0"
        ref = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, act, ws)[:rows].clone()
        os.environ["BMOE_FUSED"] = "1"
        for _ in range(30):
            y = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, act, ws)[:rows]
            assert torch.equal(y, ref)
    finally:
        for v, val in saved.items():
            if val is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = val


@pytest.mark.parametrize("E,d,f,B,k,act", [
    (8, 1024, 2048, 700, 2, ops.ACT_SWIGLU),
    (4, 512, 1536, 1000, 2, ops.ACT_SWIGLU),
    (16, 512, 1024, 333, 3, ops.ACT_TANH),
    (4, 4096, 1024, 300, 2, ops.ACT_SWIGLU),  # K = 4096: SwiGLU GEMM1 on W1|W3-split pairs
])
def test_prefill_2sm_pairs_equal_single_cta(cuda_ok, E, d, f, B, k, act):
    """Prefill GEMMs on CTA pairs (cta_group::2, M = 256, the token half of
    each chunk in each CTA, GEMM2 at 256-token tiles) against the single-CTA
    kernels: every output element accumulates the same K = 16 MMA steps in
    the same order, so the results match bitwise; and both stay within the
    bf16 tolerance of the fp32 reference."""
    import os
    rng = np.random.default_rng(B + d)
    y, ref32, (xp, perm, arena, buf_of, ws) = _bf16_case(rng, E, d, f, B, k, act, 128)
    rows = int(perm.offset[-1])
    bo = _t(buf_of)
    old = {v: os.environ.get(v) for v in ("BMOE_2SM",)}
    try:
        os.environ["BMOE_2SM"] = "0"
        single = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, act, ws)[:rows].clone()
        # GEMM2 on pairs (+ W1|W3-split GEMM1 at K >= 4096: default); both GEMMs as two-m-tile pairs
        for mode in ("1", "2"):
            os.environ["BMOE_2SM"] = mode
            for _ in range(3):
                pair = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, act, ws)[:rows]
                assert torch.equal(pair, single), mode
    finally:
        for v, val in old.items():
            if val is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = val
    rel = (torch.linalg.norm(y - ref32, dim=1) / torch.linalg.norm(ref32, dim=1).clamp_min(1e-30)).max().item()
    assert rel <= 2e-2, rel


@pytest.mark.parametrize("tm", ["1", "2"], ids=["single_cta", "cta_pair"])
@pytest.mark.parametrize("E,d,f,B,k", [(16, 2048, 768, 1500, 8), (8, 2048, 1408, 900, 6), (4, 1024, 512, 77, 2),
                                       (4, 4096, 1024, 600, 2)])
def test_prefill_token_major_gemm1_bitwise(cuda_ok, monkeypatch, tm, E, d, f, B, k):
    """The token-major SwiGLU GEMM1 tiles (tokens as the MMA's A, [W1 ; W3]
    as one N = 256 B operand; BMOE_TM=1 single CTAs, =2 CTA pairs with the
    B operand split W1 | W3 across the pair) give every real row bitwise the
    result of the weight-major tiles (BMOE_TM=0): each output element is the
    same K = 16 step chain."""
    rng = np.random.default_rng(B + f)
    monkeypatch.setenv("BMOE_TM", tm)
    y, ref32, (xp, perm, arena, buf_of, ws) = _bf16_case(rng, E, d, f, B, k, ops.ACT_SWIGLU, 128)
    real = perm.row_token >= 0
    out = []
    for tm in ("0", tm):
        monkeypatch.setenv("BMOE_TM", tm)
        out.append(ops.expert_ffn_bf16(xp, perm, arena, _t(buf_of), d, f, ops.ACT_SWIGLU, ws)[real].clone())
    assert torch.equal(out[0], out[1])
    rel = (torch.linalg.norm(y - ref32, dim=1) / torch.linalg.norm(ref32, dim=1).clamp_min(1e-30)).max().item()
    assert rel <= 2e-2, rel


@pytest.mark.parametrize("B,E,d,k", [(16, 128, 2048, 8), (5, 100, 96, 6), (7, 9, 33, 2), (3, 256, 512, 8),
                                     (600, 64, 256, 6), (16, 8, 4096, 2), (2051, 128, 2048, 8), (603, 10, 36, 3)])
def test_gate_cluster_split_bitwise(cuda_ok, monkeypatch, B, E, d, k):
    """K1 splits a token over a CTA cluster (DSMEM logits) at small B and
    gives a CTA 8 tokens at large B: every output is bitwise equal to one CTA
    per token (BMOE_GATE_SPLIT=1, BMOE_GATE_WIDE=0), and the logits match a
    float64 GEMV within fp32 rounding."""
    g = torch.Generator(device="cpu").manual_seed(B * 1000 + E)
    x = torch.randn(B, d, generator=g).to(DEV)
    wg = (torch.randn(E, d, generator=g) * d ** -0.5).to(DEV)
    b = (torch.randn(E, generator=g) * 0.1).to(DEV)
    outs = []
    for split, wide in (("0", "1"), ("1", "0"), ("3", "0")):
        monkeypatch.setenv("BMOE_GATE_SPLIT", split)
        monkeypatch.setenv("BMOE_GATE_WIDE", wide)
        outs.append(ops.gate_topk(x, wg, b, k, 1.0, tau=0.4, gamma=0.9))
    for r in outs[1:]:
        for name in ("logits", "topk", "probs", "tae", "margin", "allowed"):
            assert torch.equal(getattr(outs[0], name), getattr(r, name)), name
    z64 = x.double() @ wg.double().T + b.double()
    scale = x.double().norm(dim=1, keepdim=True) * wg.double().norm(dim=1).max()
    assert bool(((outs[0].logits.double() - z64).abs() <= 1e-5 * scale).all())


def test_empty_inputs(cuda_ok):
    """Empty batches and traces (the reference handles an empty decision list
    in route_batch / substitute_batch / observe_batch / forward_batch): every
    kernel accepts zero tokens, launches nothing harmful and returns empty or
    zero results; δ of an empty batch is 0 (batch allowed)."""
    E, k, d, f = 8, 2, 128, 256
    x = torch.empty(0, d, device=DEV)
    wg = torch.randn(E, d, device=DEV)
    r = ops.gate_topk(x, wg, torch.zeros(E, device=DEV), k, tau=0.3)
    assert r.topk.shape == (0, k) and r.logits.shape == (0, E)
    ids = torch.full((E, 4), -1, dtype=torch.int32, device=DEV)
    t = ops.DeviceTable(ids, torch.zeros(E, 4, dtype=torch.float64, device=DEV),
                        torch.zeros(E, dtype=torch.int32, device=DEV))
    plan = ops.buddy_remap(r.topk, r.allowed, ops.bitmap_from_mask(np.ones(E, bool), DEV), t, H=4, rho=3)
    assert plan.executed.shape == (0, k)
    perm = ops.permute(plan.executed, plan.kind, E)
    assert int(perm.count.sum()) == 0
    c, p = ops.coact_count(torch.empty(0, k, dtype=torch.int32, device=DEV), E)
    assert int(c.sum()) == 0 and int(p.sum()) == 0
    w = (torch.randn(E, 3 * d * f, device=DEV) * 0.05).to(torch.bfloat16)
    arena = ops.pack_arena_bf16(w, d, f, ops.ACT_SWIGLU)
    ws = ops.FfnWorkspace(E, d, f, max(perm.r_max, 16), 64)
    xp = ops.gather_rows(x, perm, 1)
    ops.expert_ffn_bf16(xp, perm, arena, torch.arange(E, dtype=torch.int32, device=DEV), d, f, ops.ACT_SWIGLU, ws)
    torch.cuda.synchronize()


def test_split_gemm1_dsmem_exchange_under_timing_stress(cuda_ok):
    """The CTA-pair SwiGLU GEMM1 exchanges its W1/W3 halves through DSMEM,
    ordered by cluster-scope mbarriers (racecheck does not model those and
    reports the 4 exchanges as hazards, profiles/r1e_sanitizer.txt). A real
    race would make the result depend on timing: 40 launches, each with a
    different background load on a second stream skewing when the two CTAs of
    a pair reach the exchange, must all equal the single-CTA result bitwise."""
    import os
    rng = np.random.default_rng(77)
    E, d, f, B, k = 4, 4096, 1024, 300, 2
    y, ref32, (xp, perm, arena, buf_of, ws) = _bf16_case(rng, E, d, f, B, k, ops.ACT_SWIGLU, 128)
    rows = int(perm.offset[-1])
    bo = _t(buf_of)
    old = os.environ.get("BMOE_2SM")
    side = torch.cuda.Stream()
    junk = torch.randn(8 << 20, device=DEV)
    try:
        os.environ["BMOE_2SM"] = "0"
        single = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows].clone()
        os.environ.pop("BMOE_2SM")  # default: W1|W3-split GEMM1 on CTA pairs at K >= 4096
        for i in range(40):
            with torch.cuda.stream(side):
                for _ in range(i % 5):
                    junk.mul_(1.0000001)  # occupies some SMs while the pairs start
            out = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows]
            assert torch.equal(out, single), i
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("BMOE_2SM", None)
        else:
            os.environ["BMOE_2SM"] = old


@pytest.mark.parametrize("B,k,E,drop", [(2048, 8, 128, 0.0), (2051, 8, 128, 0.1), (8192, 8, 128, 0.0),
                                        (700, 6, 66, 0.2), (4096, 2, 8, 0.05), (513, 8, 256, 0.0)])
def test_multi_cta_permute_equals_single_cta(cuda_ok, B, k, E, drop):
    """Prefill-size plans take the three-kernel multi-CTA permute (chunk
    histograms, chunk bases, scatter); every output — counts, padded offsets,
    row tokens (padding -1) and slot rows — must equal the single-CTA kernel's
    bit for bit, dropped slots included."""
    from paper_2511_10054_b200 import _native as N
    rng = np.random.default_rng(B + E)
    ex = torch.tensor(np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32), device=DEV)
    kd = torch.tensor((rng.random((B, k)) < drop).astype(np.uint8) * 3, device=DEV)
    multi = ops.permute(ex, kd, E)
    single = ops.Permutation(torch.empty_like(multi.count), torch.empty_like(multi.offset),
                             torch.full_like(multi.row_token, -7), torch.empty_like(multi.slot_row), multi.r_max)
    N.call("bm_permute", ex.data_ptr(), kd.data_ptr(), B, k, E, 16, single.count.data_ptr(),
           single.offset.data_ptr(), single.row_token.data_ptr(), single.slot_row.data_ptr(),
           torch.cuda.current_stream().cuda_stream)
    rows = int(single.offset[-1])
    assert torch.equal(multi.count, single.count) and torch.equal(multi.offset, single.offset)
    assert torch.equal(multi.slot_row, single.slot_row)
    assert torch.equal(multi.row_token[:rows], single.row_token[:rows])


@pytest.mark.parametrize("E,d,f,B,k,n_tile", [
    (8, 4096, 14336, 16, 2, 16),   # Mixtral decode
    (128, 2048, 768, 16, 8, 16),   # Qwen3 decode (k = 8 slots per token)
    (64, 2048, 1408, 200, 6, 64),  # more tokens than CTAs: CTAs combine several tokens
    (8, 512, 1024, 300, 2, 128),   # prefill width: GEMM kernels, then the separate combine
])
def test_ffn_combine_one_launch_equals_two(cuda_ok, E, d, f, B, k, n_tile):
    """bm_expert_ffn_bf16_combine (north_star (c): the grouped FFN with the
    gate-weighted combine fused) runs K5 + layer_update after a second grid
    barrier of the fused decode launch, with combine_kernel's own code: h is
    bitwise identical to expert_ffn_bf16 followed by combine(h_in=h), over
    repeats (the barrier generations advance twice per launch)."""
    seed = E * 7 + B
    topk, kind, probs = _plan(np.random.default_rng(seed), B, E, k)
    _, _, (xp, perm, arena, buf_of, ws) = _bf16_case(np.random.default_rng(seed), E, d, f, B, k, ops.ACT_SWIGLU,
                                                     n_tile)
    bo, pr, kd = _t(buf_of), _t(probs), _t(kind)
    h0 = torch.randn(B, d, device=DEV, generator=torch.Generator(device=DEV).manual_seed(seed))
    y = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)
    ref = ops.combine(y, perm, pr, kd, h_in=h0.clone(), residual_scale=0.5)
    for _ in range(10):
        h = h0.clone()
        ops.expert_ffn_bf16_combine(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws, pr, kd, h, 0.5)
        assert torch.equal(h, ref)


def test_fused_workspace_shared_across_token_tiles(cuda_ok):
    """One workspace serves decode calls of different token tiles (an engine's
    batches of 16 and 64 tokens): the barrier count, launch count, H readiness
    and arrival counters live at offsets independent of n_tile, so interleaved
    calls with n_tile 64 / 16 / 32 on one buffer give exactly what fresh
    workspaces give."""
    import copy
    E, d, f, B, k = 16, 1024, 2048, 48, 2
    seed = 91
    _, _, (xp, perm, arena, buf_of, ws) = _bf16_case(np.random.default_rng(seed), E, d, f, B, k, ops.ACT_SWIGLU, 64)
    bo = _t(buf_of)
    rows = int(perm.offset[-1])
    shared = ops.FfnWorkspace(E, d, f, perm.r_max, 64)
    for nt in (64, 16, 32, 16, 64, 32):
        fresh = ops.FfnWorkspace(E, d, f, perm.r_max, nt)
        ref = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, fresh)[:rows].clone()
        view = copy.copy(shared)
        view.n_tile = nt
        got = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, view)[:rows]
        assert torch.equal(got, ref), nt



@pytest.mark.parametrize("E,d,f,B,k,n_tile", [
    (8, 4096, 14336, 16, 2, 16),   # Mixtral decode: 2-4 experts, one per group
    (128, 2048, 768, 16, 8, 16),   # Qwen3 decode: many small experts, 3 groups
    (64, 2048, 1408, 64, 6, 64),   # DSV2-shaped (GEMM2 K/64 = 22), wider tile
])
def test_fused_expert_groups(cuda_ok, E, d, f, B, k, n_tile):
    """Interleaved expert-group phases (G1(0), G1(1), G2(0), ..., BMOE_FFN_GROUPS,
    forced here at every size with BMOE_FFN_GROUP_ITERS=0) change where the
    stream-K ranges split tiles, so GEMM1's partial sums meet in another
    order and an H value near a bf16 rounding boundary can round the other
    way: within 5e-3 of the one-range kernel (the bf16 tolerance is 2e-2),
    and bitwise repeatable."""
    import os
    rng = np.random.default_rng(E + B + d + 1)
    y, ref32, (xp, perm, arena, buf_of, ws) = _bf16_case(rng, E, d, f, B, k, ops.ACT_SWIGLU, n_tile)
    rows = int(perm.offset[-1])
    bo = _t(buf_of)
    saved = {v: os.environ.get(v) for v in ("BMOE_FFN_GROUPS", "BMOE_FFN_GROUP_ITERS")}
    try:
        os.environ["BMOE_FFN_GROUP_ITERS"] = "0"
        os.environ["BMOE_FFN_GROUPS"] = "1"
        one = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows].clone()
        for g in ("2", "3", "4"):
            os.environ["BMOE_FFN_GROUPS"] = g
            first = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows].clone()
            for _ in range(5):
                assert torch.equal(ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows], first)
            rel = ((first - one).norm(dim=1) / one.norm(dim=1).clamp_min(1e-30)).max().item()
            assert rel <= 5e-3, (g, rel)
    finally:
        for v, val in saved.items():
            if val is None:
                os.environ.pop(v, None)
            else:
                os.environ[v] = val


def test_kernel_timing_spans(cuda_ok):
    """The bench's FFN timing hook: every fused decode call gets a CUDA-event
    duration and an on-device span (first CTA in to last CTA out) with
    0 < span <= events; prefill-width calls report span 0."""
    from paper_2511_10054_b200 import _native as N
    E, d, f, B, k = 8, 1024, 2048, 16, 2
    _, _, (xp, perm, arena, buf_of, ws) = _bf16_case(np.random.default_rng(3), E, d, f, B, k, ops.ACT_SWIGLU, 16)
    bo = _t(buf_of)
    _, _, (xp2, perm2, arena2, buf_of2, ws2) = _bf16_case(np.random.default_rng(4), E, d, f, 300, k,
                                                          ops.ACT_SWIGLU, 128)
    N.lib().bm_set_kernel_timing(1)
    try:
        for _ in range(3):
            ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)
        ops.expert_ffn_bf16(xp2, perm2, arena2, _t(buf_of2), d, f, ops.ACT_SWIGLU, ws2)
        times = np.zeros(16, np.float32)
        n = int(N.lib().bm_kernel_times(times.ctypes.data, times.size))
        spans = np.zeros(8, np.float32)
        m = int(N.lib().bm_kernel_spans(spans.ctypes.data, spans.size))
    finally:
        N.lib().bm_set_kernel_timing(0)
    assert n == 8 and m == 4
    ev = times[0:n:2]
    assert np.all(spans[:3] > 0) and np.all(spans[:3] <= ev[:3] + 1e-3), (spans, ev)
    assert spans[3] == 0.0


def test_ffn_phase_trace(cuda_ok, monkeypatch):
    """BMOE_FFN_TRACE: the fused decode kernel's per-CTA phase stamps are
    ordered (entry <= setup <= exit) and every CTA stamps its entry and exit."""
    from paper_2511_10054_b200 import _native as N
    monkeypatch.setenv("BMOE_FFN_TRACE", "1")
    E, d, f, B, k = 8, 1024, 2048, 16, 2
    _, _, (xp, perm, arena, buf_of, ws) = _bf16_case(np.random.default_rng(8), E, d, f, B, k, ops.ACT_SWIGLU, 16)
    ops.expert_ffn_bf16(xp, perm, arena, _t(buf_of), d, f, ops.ACT_SWIGLU, ws)
    torch.cuda.synchronize()
    G = torch.cuda.get_device_properties(0).multi_processor_count
    st = np.zeros(G * 12, np.uint64)
    n = int(N.lib().bm_ffn_trace_read(st.ctypes.data, st.size))
    assert n == G * 12
    st = st[:n].reshape(-1, 12).astype(np.int64)
    assert np.all(st[:, 0] > 0) and np.all(st[:, 7] > 0)
    assert np.all(st[:, 0] <= st[:, 1]) and np.all(st[:, 1] <= st[:, 7])


@pytest.mark.parametrize("tc", ["1", "2", "2:0xFFF", "2:0xAAA"], ids=["i8", "mxf4", "mxf4_tb_build", "mxf4_mixed_build"])
@pytest.mark.parametrize("E,k,n", [(128, 8, 300_001), (64, 6, 100_003), (100, 3, 50_000), (8, 2, 20_000),
                                   (128, 8, 255), (128, 16, 70_001)])
def test_coact_tensor_core_path_bit_exact(cuda_ok, monkeypatch, tc, E, k, n):
    """K6's tensor-core paths (BMOE_COACT_TC=1: tcgen05 kind::i8, =2: kind::mxf4
    with e2m1 one-hots, built by shared-memory ORs, or by register bit
    transposes in the builder warps of BMOE_COACT_TB_MASK (0xFFF: all, 0xAAA:
    every other one); unit block scales, X^T X over one-hot tiles in TMEM)
    give exactly the shared-memory-atomics kernel's counts, pairs and
    rejected-row count, rejected rows (duplicates, out-of-range ids) included."""
    rng = np.random.default_rng(E * 31 + k)
    topk = np.stack([rng.choice(E, k, replace=False) for _ in range(n)]).astype(np.int32)
    bad = rng.choice(n, 50, replace=False)
    topk[bad[:25], 0] = topk[bad[:25], -1]  # duplicate ids
    topk[bad[25:], 1] = E + 3               # out of range
    t = _t(topk)
    out = []
    for mode in ("0", tc):
        mode, _, mask = mode.partition(":")
        monkeypatch.setenv("BMOE_COACT_TC", mode)
        if mask:
            monkeypatch.setenv("BMOE_COACT_TB_MASK", mask)
        else:
            monkeypatch.delenv("BMOE_COACT_TB_MASK", raising=False)
        c = torch.zeros(E, dtype=torch.int64, device=DEV)
        p = torch.zeros(E, E, dtype=torch.int64, device=DEV)
        badc = torch.zeros(1, dtype=torch.int32, device=DEV)
        from paper_2511_10054_b200 import _native as N
        N.call("bm_coact_count", t.data_ptr(), n, k, E, c.data_ptr(), p.data_ptr(), badc.data_ptr(),
               torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        out.append((c.cpu(), p.cpu(), int(badc.item())))
    assert out[0][2] == out[1][2] == 50
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])
