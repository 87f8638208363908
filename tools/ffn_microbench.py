"""Microbenchmark of the bf16 grouped expert FFN (K4) alone, decode-shaped.

    python tools/ffn_microbench.py [--experts-active 4] [--tokens 16] [--iters 50]

Builds a Mixtral-shaped arena (8 experts, d=4096, f=14336, UMMA-tiled bf16),
routes `tokens` tokens top-2 over the first `experts-active` experts, and
times bm_expert_ffn_bf16's two GEMM kernels with CUDA events (the library's
kernel-timing hook). Each iteration rotates through 4 arena copies so the
weights are never L2-resident (126 MB L2 vs 1.4 GB per call).
Prints one JSON line: per-kernel ms, algorithmic GB/s, fraction of measured HBM,
and (prefill shapes) TFLOP/s of the whole call.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_10054_b200 import _native as N  # noqa: E402
from paper_2511_10054_b200 import ops  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--experts-active", type=int, default=4)
    ap.add_argument("--tokens", type=int, default=16)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--f", type=int, default=14336)
    ap.add_argument("--E", type=int, default=8)
    ap.add_argument("--n-tile", type=int, default=16)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--k", type=int, default=2, help="slots per token (top-k)")
    ap.add_argument("--trace", action="store_true",
                    help="phase trace of the fused decode kernel (needs BMOE_FFN_TRACE=1): per-CTA globaltimer "
                         "stamps of single graph replays, as microseconds after the first CTA's entry")
    args = ap.parse_args()
    E, d, f, B, A = args.E, args.d, args.f, args.tokens, args.experts_active
    dev = "cuda"
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    arenas = []
    for _ in range(args.copies):
        ar = torch.empty(E, 3 * d * f, device=dev, dtype=torch.bfloat16)
        for e in range(E):
            w = torch.randn(3 * d * f, device=dev, generator=g).to(torch.bfloat16)
            ops.pack_expert_bf16(w[: f * d].view(f, d), w[f * d: 2 * f * d].view(f, d), w[2 * f * d:].view(d, f),
                                 ops.ACT_SWIGLU, ar[e])
        arenas.append(ar)
    rng = np.random.default_rng(0)
    topk = np.stack([rng.choice(A, args.k, replace=False) for _ in range(B)]).astype(np.int32)
    kind = np.zeros_like(topk, dtype=np.uint8)
    perm = ops.permute(torch.from_numpy(topk).to(dev), torch.from_numpy(kind).to(dev), E)
    x = torch.randn(B, d, device=dev)
    xp = ops.gather_rows(x, perm, 1)
    ws = ops.FfnWorkspace(E, d, f, perm.r_max, args.n_tile)
    bufs = torch.arange(E, device=dev, dtype=torch.int32)
    for i in range(5):
        ops.expert_ffn_bf16(xp, perm, arenas[i % len(arenas)], bufs, d, f, ops.ACT_SWIGLU, ws)
    torch.cuda.synchronize()
    N.lib().bm_set_kernel_timing(1)
    for i in range(args.iters):
        ops.expert_ffn_bf16(xp, perm, arenas[i % len(arenas)], bufs, d, f, ops.ACT_SWIGLU, ws)
    buf = np.zeros(2 * args.iters + 4, np.float32)
    n = int(N.lib().bm_kernel_times(buf.ctypes.data, buf.size))
    N.lib().bm_set_kernel_timing(0)
    g1, g2 = float(np.median(buf[0:n:2])), float(np.median(buf[1:n:2]))
    # whole call (both GEMMs + any fixup work) replayed from CUDA graphs, as
    # the engine runs it, with CUDA events around each replay
    graphs = []
    for ar in arenas:
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            ops.expert_ffn_bf16(xp, perm, ar, bufs, d, f, ops.ACT_SWIGLU, ws)
        graphs.append(gr)
    for gr in graphs:
        gr.replay()
    evs = []
    for i in range(args.iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        graphs[i % len(graphs)].replay()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    call = float(np.median([a.elapsed_time(b) for a, b in evs]))
    n_exp = int((perm.count > 0).sum())
    b1 = n_exp * 2 * d * f * 2 + B * args.k * d * 2
    b2 = n_exp * d * f * 2 + B * args.k * f * 2
    flops1, flops2 = 2.0 * B * args.k * d * f * 2, 2.0 * B * args.k * d * f  # 6*d*f per (token, slot)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    out = {"experts": n_exp, "tokens": B, "k": args.k, "n_tile": args.n_tile, "gemm1_ms": g1, "gemm2_ms": g2, "call_ms": call,
           "call_gbs": (b1 + b2) / call / 1e6, "call_frac": (b1 + b2) / call / 1e6 / peak,
           "tflops_pair": (flops1 + flops2) / (g1 + g2) / 1e9,
           "call_tflops": (flops1 + flops2) / call / 1e9,
           "pair_gbs": (b1 + b2) / (g1 + g2) / 1e6, "peak_gbs": peak,
           # a decode-width call is one fused kernel: the timing hook reports it as "gemm1" and 0 for gemm2
           "gemm1_frac": (b1 + (b2 if g2 == 0 else 0)) / g1 / 1e6 / peak, "gemm2_frac": b2 / g2 / 1e6 / peak if g2 else None,
           "env": {k: v for k, v in os.environ.items() if k.startswith("BMOE_")}}
    if args.trace:
        names = ["entry", "setup", "g1_loads_issued", "g1_mma_done", "g1_epi_done", "h_ready_seen", "g2_epi_done",
                 "exit", "g1_last_acc_ready", "g1_split_arrivals_seen", "g2_first_stage", "g2_mma_done"]
        NP = len(names)
        G = torch.cuda.get_device_properties(0).multi_processor_count
        rows = []
        for i in range(20):
            graphs[i % len(graphs)].replay()
            torch.cuda.synchronize()
            st = np.zeros(G * NP, np.uint64)
            n = int(N.lib().bm_ffn_trace_read(st.ctypes.data, st.size))
            st = st[:n].reshape(-1, NP).astype(np.float64)
            t0 = st[:, 0].min()
            rel = np.where(st > 0, (st - t0) / 1000.0, np.nan)
            rows.append([[np.nanmin(rel[:, j]), np.nanmedian(rel[:, j]), np.nanmax(rel[:, j])] for j in range(NP)])
        med = np.median(np.array(rows), axis=0)
        out["trace_us"] = {nm: {"min": round(float(a), 2), "med": round(float(b), 2), "max": round(float(c), 2)}
                           for nm, (a, b, c) in zip(names, med)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
