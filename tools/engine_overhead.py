"""Decode-step overhead of the engine with every expert resident (no H2D):
ms per layer-step vs the sum of kernel times from an ncu-free CUDA-event
breakdown. Usage: python tools/engine_overhead.py [--layers 4] [--batch 16]"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_10054_b200 import _native as N  # noqa: E402
from paper_2511_10054_b200 import workload as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--shape", default="mixtral")
    args = ap.parse_args()
    wl = W.build(args.shape, layers=args.layers, max_batch=args.batch, profile_tokens=1024)
    E = wl.eng.num_experts
    eng = wl.engine("buddy", capacity=E, staging=E)
    B = args.batch
    x = torch.from_numpy(wl.tokens(2, (args.steps + 3) * B)).cuda()
    for s in range(3):
        eng.step(x[s * B:(s + 1) * B], np.arange(B))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for s in range(3, 3 + args.steps):
        eng.step(x[s * B:(s + 1) * B], np.arange(B))
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    N.lib().bm_set_kernel_timing(1)
    for s in range(3, 3 + args.steps):
        eng.step(x[s * B:(s + 1) * B], np.arange(B))
    buf = np.zeros(6 * args.steps * args.layers, np.float32)
    n = int(N.lib().bm_kernel_times(buf.ctypes.data, buf.size))
    N.lib().bm_set_kernel_timing(0)
    gemm = float(buf[:n].sum()) / args.steps
    st = eng.stats()
    print(json.dumps({"shape": args.shape, "layers": args.layers, "batch": B, "ms_per_step": ms,
                      "ms_per_layer_step": ms / args.layers, "gemm_ms_per_layer_step": gemm / args.layers,
                      "physical_fetches": st["physical_fetches"], "experts_per_ffn": st["ffn_experts"] / max(1, st["ffn_calls"])}))


if __name__ == "__main__":
    main()
