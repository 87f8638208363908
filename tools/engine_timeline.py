"""Where an engine step's time goes: runs the engine for a few steps under the
CUDA activity profiler (CUPTI through torch.profiler) and reports the H2D
copy-engine busy fraction, the gaps between copies and the GPU work and host
phases that fill them. Usage:
    python tools/engine_timeline.py --model qwen3 --layers 12 --steps 4
"""

import argparse
import json
import os
import re
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2511_10054_b200 import workload as W  # noqa: E402


def _union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen3")
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--trace", default="")
    args = ap.parse_args()
    wl = W.build(args.model, layers=args.layers, max_batch=args.batch, profile_tokens=4096, codec=1)
    eng = wl.engine("buddy")
    B = args.batch
    x = torch.from_numpy(wl.tokens(1, (args.warmup + args.steps) * B)).cuda()
    for s in range(args.warmup):
        eng.step(x[s * B:(s + 1) * B], np.arange(s * B, (s + 1) * B))
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for s in range(args.warmup, args.warmup + args.steps):
            eng.step(x[s * B:(s + 1) * B], np.arange(s * B, (s + 1) * B))
        torch.cuda.synchronize()
    if args.trace:
        prof.export_chrome_trace(args.trace)
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    h2d = [(e.time_range.start, e.time_range.end) for e in ev if "HtoD" in e.name or "Memcpy HtoD" in e.name]
    kern = [(e.time_range.start, e.time_range.end, e.name) for e in ev if "Memcpy" not in e.name and "Memset" not in e.name]
    t0 = min(a for a, _, _ in kern + [(a, b, "") for a, b in h2d])
    t1 = max(b for _, b, _ in kern + [(a, b, "") for a, b in h2d])
    busy = _union(h2d)
    busy_us = sum(b - a for a, b in busy)
    gaps = [(busy[i][1], busy[i + 1][0]) for i in range(len(busy) - 1) if busy[i + 1][0] - busy[i][1] > 5]
    gap_us = sum(b - a for a, b in gaps)
    # kernels by name inside the gaps (time overlapped with each gap)
    by = {}
    for a, b in gaps:
        for ka, kb, n in kern:
            o = min(b, kb) - max(a, ka)
            if o > 0:
                m = re.findall(r"(\w+)(?:<[^>]*>)?\(", n)
                short = m[0] if m else n[:40]
                by[short] = by.get(short, 0.0) + o
    kern_union = _union([(a, b) for a, b, _ in kern])
    gap_gpu_busy = 0.0
    for a, b in gaps:
        for ka, kb in kern_union:
            o = min(b, kb) - max(a, ka)
            if o > 0:
                gap_gpu_busy += o
    per = {}
    for a, b, n in kern:
        m = re.findall(r"(\w+)(?:<[^>]*>)?\(", n)
        key = m[0] if m else n[:40]
        c, t = per.get(key, (0, 0.0))
        per[key] = (c + 1, t + (b - a))
    hist = np.histogram([b - a for a, b in gaps], bins=[5, 20, 50, 100, 200, 500, 1e9])[0].tolist()
    out = {"model": args.model, "layers": args.layers, "steps": args.steps,
           "span_ms": (t1 - t0) / 1e3, "h2d_busy_ms": busy_us / 1e3, "h2d_busy_frac": busy_us / (t1 - t0),
           "n_copies": len(h2d), "gaps_gt5us": len(gaps), "gap_ms": gap_us / 1e3,
           "gap_per_layer_step_us": gap_us / (args.layers * args.steps),
           "gap_hist_us[5,20,50,100,200,500,inf]": hist,
           "gpu_busy_in_gaps_ms": gap_gpu_busy / 1e3,
           "kernels_in_gaps_ms": {k: round(v / 1e3, 3) for k, v in sorted(by.items(), key=lambda t: -t[1])[:12]},
           "kernels": {k: {"n": c, "avg_us": round(t / c, 1), "total_ms": round(t / 1e3, 3)}
                       for k, (c, t) in sorted(per.items(), key=lambda t: -t[1][1])}}
    # host-side ranges (engine step on the CPU timeline)
    cpu = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda"):
            cpu[e.name] = cpu.get(e.name, 0.0) + e.cpu_time_total
    out["cuda_api_ms"] = {k: round(v / 1e3, 2) for k, v in sorted(cpu.items(), key=lambda t: -t[1])[:10]}
    print(json.dumps(out, indent=1))
    eng.close()
    wl.close()


if __name__ == "__main__":
    main()
