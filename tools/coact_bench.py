"""K6 microbenchmark: bm_coact_count over a synthetic top-k trace (default the
configs[4] shape, 64M tokens x top-8 of 128 experts) with the shared-memory
atomics kernel (BMOE_COACT_TC=0), the kind::i8 path (=1) and the kind::mxf4
path (=2); checks the three give identical counts and prints one JSON line per
mode (ms by CUDA events, median of --iters, and trace-read GB/s).

    python tools/coact_bench.py [--tokens 67108864] [--experts 128] [--k 8]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=64 * 1024 * 1024)
    ap.add_argument("--experts", type=int, default=128)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--modes", default="0,1,2")
    args = ap.parse_args()
    n, E, k = args.tokens, args.experts, args.k
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    # k distinct experts per token: top-k of random keys
    topk = torch.empty(n, k, dtype=torch.int32, device="cuda")
    step = 1 << 22
    for s in range(0, n, step):
        m = min(step, n - s)
        topk[s:s + m] = torch.rand(m, E, generator=g, device="cuda").topk(k, dim=1).indices.to(torch.int32)
    stream = torch.cuda.current_stream().cuda_stream
    ref = None
    for mode in args.modes.split(","):
        os.environ["BMOE_COACT_TC"] = mode
        c = torch.zeros(E, dtype=torch.int64, device="cuda")
        p = torch.zeros(E, E, dtype=torch.int64, device="cuda")
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")

        def run():
            c.zero_(); p.zero_(); bad.zero_()
            N.call("bm_coact_count", topk.data_ptr(), n, k, E, c.data_ptr(), p.data_ptr(), bad.data_ptr(), stream)

        run()
        torch.cuda.synchronize()
        out = (c.clone(), p.clone(), int(bad.item()))
        if ref is None:
            ref = out
        same = torch.equal(ref[0], out[0]) and torch.equal(ref[1], out[1]) and ref[2] == out[2]
        ts = []
        for _ in range(args.iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c.zero_(); p.zero_(); bad.zero_()
            a.record()
            N.call("bm_coact_count", topk.data_ptr(), n, k, E, c.data_ptr(), p.data_ptr(), bad.data_ptr(), stream)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        print(json.dumps({"mode": {"0": "atomics", "1": "tc_i8", "2": "tc_mxf4"}[mode], "tokens": n, "experts": E,
                          "k": k, "ms": ms, "trace_gbs": n * k * 4 / ms / 1e6, "equal_to_atomics": same,
                          "total_pairs": int(out[1].sum().item())}))


if __name__ == "__main__":
    main()
