"""Small invocation of every kernel, for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import __graft_entry__  # noqa: E402

if __name__ == "__main__":
    __graft_entry__.smoke()
    import numpy as np
    import torch
    from paper_2511_10054_b200 import ops
    # remap with Psi ordering and H > 32 (multi-chunk ballots), E not a multiple of 32
    rng = np.random.default_rng(1)
    E, k, B, K = 100, 6, 40, 64
    topk = np.stack([rng.choice(E, k, replace=False) for _ in range(B)]).astype(np.int32)
    ids = np.stack([rng.permutation([j for j in range(E) if j != p])[:K] for p in range(E)]).astype(np.int32)
    w = np.sort(rng.random((E, K)), axis=1)[:, ::-1].copy()
    t = ops.DeviceTable(torch.from_numpy(ids).cuda(), torch.from_numpy(w).cuda(),
                        torch.full((E,), K, dtype=torch.int32).cuda())
    plan = ops.buddy_remap(torch.from_numpy(topk).cuda(), torch.ones(B, dtype=torch.uint8).cuda(),
                           ops.bitmap_from_mask(rng.random(E) < 0.3, "cuda"), t, H=50, rho=None, eta=0.2, kappa=0.1,
                           partition_of=torch.from_numpy((np.arange(E) * 3 // E).astype(np.int32)).cuda(),
                           logits=torch.randn(B, E, dtype=torch.float64).cuda())
    torch.cuda.synchronize()
    # router split over CTA clusters (logits pushed to CTA 0 over DSMEM), E=128 and a ragged E
    for E_, B_ in ((128, 16), (100, 5)):
        r = ops.gate_topk(torch.randn(B_, 256).cuda(), torch.randn(E_, 256).cuda() * 0.06, torch.zeros(E_).cuda(), 8)
    torch.cuda.synchronize()
    # fused decode FFN with many split tiles (n_tile 16, 148 CTAs over a small
    # problem) and the multi-kernel path on the same inputs: bitwise equal
    E2, d, f, B2 = 8, 512, 1024, 40
    tk = np.stack([rng.choice(E2, 2, replace=False) for _ in range(B2)]).astype(np.int32)
    perm = ops.permute(torch.from_numpy(tk).cuda(), torch.zeros(B2, 2, dtype=torch.uint8).cuda(), E2)
    xp = ops.gather_rows(torch.randn(B2, d).cuda(), perm, 1)
    w = (torch.randn(E2, 3 * d * f).cuda() * 0.03).to(torch.bfloat16)
    arena = ops.pack_arena_bf16(w, d, f, ops.ACT_SWIGLU)
    ws = ops.FfnWorkspace(E2, d, f, perm.r_max, 16)
    bo = torch.arange(E2, dtype=torch.int32).cuda()
    rows = int(perm.offset[-1])
    os.environ["BMOE_KPS"] = "2"
    os.environ["BMOE_FFN_MIN_ITERS"] = "1"  # every CTA in the stream-K range, as the separate kernels
    y1 = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows].clone()
    os.environ["BMOE_FUSED"] = "0"
    y0 = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows].clone()
    del os.environ["BMOE_FUSED"], os.environ["BMOE_KPS"], os.environ["BMOE_FFN_MIN_ITERS"]
    torch.cuda.synchronize()
    assert torch.equal(y0, y1)
    # interleaved expert-group phases (forced) and the combine fused behind the FFN
    os.environ["BMOE_FFN_GROUP_ITERS"] = "0"
    os.environ["BMOE_FFN_GROUPS"] = "3"
    y3 = ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)[:rows].clone()
    pr = torch.rand(B2, 2).cuda()
    h = torch.randn(B2, d).cuda()
    ops.expert_ffn_bf16_combine(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws, pr,
                                torch.zeros(B2, 2, dtype=torch.uint8).cuda(), h, 0.5)
    del os.environ["BMOE_FFN_GROUP_ITERS"], os.environ["BMOE_FFN_GROUPS"]
    torch.cuda.synchronize()
    assert torch.isfinite(y3).all() and torch.isfinite(h).all()
    # prefill width: data-parallel tiles finished in the GEMM epilogue (n_tile 128, > 1 chunk per expert)
    B3 = 300
    tk = np.stack([rng.choice(E2, 2, replace=False) for _ in range(B3)]).astype(np.int32)
    perm = ops.permute(torch.from_numpy(tk).cuda(), torch.zeros(B3, 2, dtype=torch.uint8).cuda(), E2)
    xp = ops.gather_rows(torch.randn(B3, d).cuda(), perm, 1)
    ws = ops.FfnWorkspace(E2, d, f, perm.r_max, 128)
    ops.expert_ffn_bf16(xp, perm, arena, bo, d, f, ops.ACT_SWIGLU, ws)  # GEMM2 on CTA pairs
    # K = 4096: SwiGLU GEMM1 on CTA pairs too (W1 | W3 split, DSMEM exchange)
    E3, d3, f3 = 4, 4096, 1024
    tk = np.stack([rng.choice(E3, 2, replace=False) for _ in range(B3)]).astype(np.int32)
    perm = ops.permute(torch.from_numpy(tk).cuda(), torch.zeros(B3, 2, dtype=torch.uint8).cuda(), E3)
    xp = ops.gather_rows(torch.randn(B3, d3).cuda(), perm, 1)
    w3 = (torch.randn(E3, 3 * d3 * f3).cuda() * 0.02).to(torch.bfloat16)
    arena3 = ops.pack_arena_bf16(w3, d3, f3, ops.ACT_SWIGLU)
    ws = ops.FfnWorkspace(E3, d3, f3, perm.r_max, 128)
    ops.expert_ffn_bf16(xp, perm, arena3, torch.arange(E3, dtype=torch.int32).cuda(), d3, f3, ops.ACT_SWIGLU, ws)
    torch.cuda.synchronize()
    # decode engine over exponent-coded mirrors (staging ring + piece decoder + prefetch stream)
    from paper_2511_10054_b200 import workload as W
    wl = W.build("tiny", layers=2, max_batch=16, profile_tokens=512, codec=1)
    eng = wl.engine("buddy")
    x = torch.from_numpy(wl.tokens(2, 48)).cuda()
    for s in range(3):
        eng.step(x[s * 16:(s + 1) * 16], np.arange(s * 16, (s + 1) * 16))
    torch.cuda.synchronize()
    assert eng.stats()["wire_bytes"] > 0
    eng.close()
    wl.close()
    # fetch codec v3 and v2 (the v3 decoder reads up to 3 words past a lane's stream: piece slack)
    for fmt in ("3", "2"):
        os.environ["BMOE_XFER_FORMAT"] = fmt
        xv = (torch.randn(3 * 8192 + 2048).cuda() * 0.02).to(torch.bfloat16)
        assert torch.equal(ops.xfer_decode(ops.xfer_encode(xv), xv.numel()).view(torch.int16), xv.view(torch.int16))
    os.environ.pop("BMOE_XFER_FORMAT")
    # K6 on every path (mxf4 tensor cores, i8 tensor cores, atomics), k = 8 and a general k
    from paper_2511_10054_b200 import _native as N
    for kk, EE, n in ((8, 128, 5000), (3, 100, 777)):
        tk6 = torch.from_numpy(np.stack([rng.choice(EE, kk, replace=False) for _ in range(n)]).astype(np.int32)).cuda()
        res = []
        for mode in ("2", "1", "0"):
            os.environ["BMOE_COACT_TC"] = mode
            c = torch.zeros(EE, dtype=torch.int64).cuda()
            pp = torch.zeros(EE, EE, dtype=torch.int64).cuda()
            bad = torch.zeros(1, dtype=torch.int32).cuda()
            N.call("bm_coact_count", tk6.data_ptr(), n, kk, EE, c.data_ptr(), pp.data_ptr(), bad.data_ptr(),
                   torch.cuda.current_stream().cuda_stream)
            res.append((c.cpu(), pp.cpu()))
        assert all(torch.equal(res[0][0], r[0]) and torch.equal(res[0][1], r[1]) for r in res)
    os.environ.pop("BMOE_COACT_TC")
    torch.cuda.synchronize()
    print("sanitize smoke ok")
