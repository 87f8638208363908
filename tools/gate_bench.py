"""Router (K1) latency at decode batch sizes: graph-replayed gate_topk calls
timed with CUDA events, per cluster split (BMOE_GATE_SPLIT), with the router
weights cold (a fresh copy per call from a rotating set larger than L2)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_10054_b200 import ops  # noqa: E402


def main():
    out = []
    for E, d, k in ((128, 2048, 8), (64, 2048, 6), (8, 4096, 2)):
        copies = max(2, int(256e6 // (E * d * 4)))
        ws = [torch.randn(E, d, device="cuda") * d ** -0.5 for _ in range(copies)]
        b = torch.zeros(E, device="cuda")
        for B in (1, 16):
            x = torch.randn(B, d, device="cuda")
            for split in ("1", "4", "8", "16", "0"):
                os.environ["BMOE_GATE_SPLIT"] = split
                for w in ws[:3]:
                    ops.gate_topk(x, w, b, k, 1.0, tau=0.3)
                torch.cuda.synchronize()
                ev = []
                for i in range(60):
                    a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    ops.gate_topk(x, ws[i % copies], b, k, 1.0, tau=0.3)
                    c.record()
                    ev.append((a, c))
                torch.cuda.synchronize()
                t = sorted(a.elapsed_time(c) for a, c in ev)[len(ev) // 2]
                out.append({"E": E, "d": d, "k": k, "B": B, "split": split, "us": round(t * 1000, 2)})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
