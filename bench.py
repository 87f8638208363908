#!/usr/bin/env python
"""Benchmark: Mixtral-8x7B-shaped offloaded-MoE decode at a 50% expert-cache
budget on B200 (BASELINE.json configs[1]), tokens/s with buddy substitution
(headline) and without (on-demand fetch), expert-miss stall, plus the
grouped-expert-GEMM roofline and the CPU reference path timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step = one decode step: B tokens through all L MoE layers (gate, remap,
cache replay, H2D fetch of misses, grouped FFN, combine). Weights are
random-init bf16 of the named shapes (no checkpoints); routing is the
reference's synthetic clustered router; buddy tables come from an on-GPU
profiling pass over a separate token stream. Multi-GPU = independent
replicas (one process per GPU, disjoint token streams), no collective on
the data path; timing is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs: [1] Mixtral decode (the headline), [2] Qwen3 decode / prefill, [3] DSV2-Lite replicas
MODELS = {
    "mixtral": {"workload": "mixtral-8x7b-moe", "model": "Mixtral-8x7B-shaped MoE layers (random init)", "layers": 32},
    "qwen3": {"workload": "qwen3-30b-a3b-moe", "model": "Qwen3-30B-A3B-shaped MoE layers (random init)", "layers": 48},
    "dsv2lite": {"workload": "deepseek-v2-lite-moe",
                 "model": "DeepSeek-V2-Lite-shaped MoE layers, 64 routed + 2 shared experts (random init)",
                 "layers": 26},
}


def _shape(model: str):
    from paper_2511_10054_b200.workload import SHAPES, SHARED
    E, k, d, f, rate = SHAPES[model]
    return E, k, d, f, rate, SHARED.get(model, 0)


def _peaks(kind: str = "hbm"):
    """Roofline denominators: MEASURED_PEAKS.json (driver-written), else the
    profiling guide's fallback (6.65 TB/s, 1.59 PFLOP/s burst)."""
    key = {"hbm": "hbm_gbs", "tensor": "bf16_tflops"}[kind]
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p[key]), "measured"
    except Exception:
        return (6650.0 if kind == "hbm" else 1590.0), "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML from
    a thread in this process (the data nvidia-smi reports, without spawning
    a polling process beside the latency-sensitive host control loop), or
    `nvidia-smi -lms` when NVML is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    PERIOD_S = float(os.environ.get("BMOE_CLOCK_PERIOD", "0.25"))

    def __init__(self, index: int):
        self.rows = []
        self.p = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            bits = (pynvml.nvmlClocksThrottleReasonHwSlowdown, pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, pynvml.nvmlClocksThrottleReasonSwPowerCap)

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        self.rows.append([str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits])
                    except Exception:
                        pass
                    self._stop.wait(self.PERIOD_S)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.nvml = True
            return
        except Exception:
            self.nvml = False
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def ready(self, timeout: float = 5.0):
        """Block until nvidia-smi delivers its first row (it takes ~0.5 s to
        start), so a short timed region is not missed entirely; rows before
        this point are discarded."""
        t0 = time.time()
        while (self.nvml or self.p is not None) and not self.rows and time.time() - t0 < timeout:
            time.sleep(0.02)
        self.rows = self.rows[-1:]
        return self

    def stop(self):
        if not self.nvml and self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if len(self.rows) < 2:  # region shorter than the sampling period: one more row right at its end
            t0 = time.time()
            while len(self.rows) < 2 and time.time() - t0 < 1.0:
                time.sleep(0.02)
        if self.nvml:
            self._stop.set()
            self.t.join(timeout=2)
        else:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        sm, mx = [], []
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml" if self.nvml else "nvidia-smi"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _allmax(v: float, ws: int):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _mirror_bytes_per_layer(model: str, codec: int) -> float:
    E, _, d, f, _, S = _shape(model)
    return (E + S) * 3 * d * f * 2 * (0.72 if codec else 1.0)


def _layers_for_host(ws: int, requested: int | None, codec: int = 1, model: str = "mixtral") -> int:
    """The model's layer count when the pinned mirrors (one per replica, or
    one node-shared copy: ws=1) fit in 60% of host RAM, fewer otherwise
    (config.layers says which)."""
    from paper_2511_10054_b200.workload import host_mem_available
    fit = int(0.6 * host_mem_available() / (ws * _mirror_bytes_per_layer(model, codec)))
    L = min(MODELS[model]["layers"], max(1, fit))
    return min(L, requested) if requested else L


def _plan_mirrors(ws: int, local: int, args):
    """Replicas of one model on one node share ONE expert mirror in /dev/shm
    (SharedMirror: written by local rank 0, mapped + page-locked by every
    rank) when it fits there; otherwise every rank keeps a private pinned
    mirror and the layer count shrinks with the replica count."""
    from paper_2511_10054_b200.workload import ShareSpec, shm_bytes_free
    if ws == 1:
        return _layers_for_host(1, args.layers, args.codec, args.model), None
    L = _layers_for_host(1, args.layers, args.codec, args.model)
    if shm_bytes_free() >= 1.05 * L * _mirror_bytes_per_layer(args.model, args.codec):
        import torch.distributed as dist
        tag = f"bmoe_{os.environ.get('TORCHELASTIC_RUN_ID', 'run')}_{os.environ.get('MASTER_PORT', '0')}_{args.model}"
        return L, ShareSpec(tag=tag, owner=(local == 0), barrier=dist.barrier)
    return _layers_for_host(ws, args.layers, args.codec, args.model), None


# ------------------------------------------------------------------ CPU legs
def stage_layer_f64(wl, layer: int):
    """The reference holds float64 expert stacks (model.py:173-186); convert
    one layer's bf16 mirror once, outside any timed region."""
    from paper_2511_10054_b200.engine import mirror_expert
    E, d, f = wl.eng.num_experts + wl.eng.num_shared, wl.eng.d, wl.eng.f
    out = {}
    for e in range(E):
        m = mirror_expert(wl.mirrors[layer], e, 3 * d * f).view(3, -1).float().cpu().numpy().astype(np.float64)
        out[e] = (m[0].reshape(f, d), m[1].reshape(f, d), m[2].reshape(d, f))
    return out


def cpu_reference_sample(wl, layer: int, B: int, seed: int, stacks, method: str = "buddy") -> float:
    """The reference algorithm for one layer-step, run by the numpy oracle port
    (oracle/, f64 like the reference): route_batch -> evaluate_gates ->
    substitute_batch -> forward_batch (per token and slot, as model.py:338-340
    gathers weights per slot) -> layer_update (model.py:231-347,
    gating.py:148-165, substitution.py:193-208). Returns seconds."""
    import oracle as O
    from paper_2511_10054_b200.workload import initial_residents
    E, k, S = wl.eng.num_experts, wl.eng.top_k, wl.eng.num_shared
    x = wl.tokens(seed, B).astype(np.float64)
    gw = wl.gate_w[layer].double().cpu().numpy()
    gb = wl.gate_b[layer].double().cpu().numpy()
    ids = wl.tbl_ids[layer].cpu().numpy()
    lens = wl.tbl_len[layer].cpu().numpy()
    mask = np.zeros(E, bool)
    mask[initial_residents(E, wl.eng.capacity, 0, layer)] = True
    t0 = time.perf_counter()
    z, topk, probs = O.route(x, gw, gb, k)
    _, _, ok, _, batch_ok = O.gate_batch(probs, topk, mask, wl.taus[layer], None, 1.0)
    if method == "buddy":
        ex, kd, _ = O.remap_batch(topk, z, mask, ids, np.zeros(ids.shape), lens, ok & batch_ok,
                                  wl.eng.search_rank_h, wl.eng.rho if wl.eng.rho is not None else -1)
    else:
        ex, kd, _ = O.ondemand_plan(topk, mask)
    y = O.forward(x, ex, kd, probs, lambda e, xr: O.ffn_swiglu(xr, *stacks[e]))
    for sx in range(S):  # shared experts: every token, weight 1
        y = y + O.ffn_swiglu(x, *stacks[E + sx])
    O.layer_update(x, y)
    return time.perf_counter() - t0


def run_reference(args, ws, rank):
    """--impl reference: the reference's CPU path (oracle port; the reference
    is pure Python/numpy and has no GPU path) on the host cores."""
    if rank != 0:
        return
    import torch
    from paper_2511_10054_b200 import workload as W
    L = _layers_for_host(ws, args.layers, args.codec, args.model)
    # one layer's weights/tables suffice: the sample is one layer-step, the
    # metric extrapolates to the same L layers as the GPU arm
    wl = W.build(args.model, layers=1, max_batch=args.batch, profile_tokens=args.profile_tokens)
    cores = len(os.sched_getaffinity(0))
    Bs = args.cpu_tokens
    stacks = stage_layer_f64(wl, 0)
    times = []
    for i in range(args.warmup + args.steps):
        sec = cpu_reference_sample(wl, 0, Bs, 1000 + i, stacks)
        if i >= args.warmup:
            times.append(sec)
    per_layer = statistics.mean(times)
    tps = Bs / (per_layer * L)
    line = {"impl": "reference", "metric": _metric(args.batch),
            "value": tps, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": per_layer * L * 1000.0, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(args.model, wl, L, args.batch, "buddy"),
            "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": f"{Bs} tokens x 1 layer per step (f64 numpy oracle, BLAS threads={cores}), "
                                       f"extrapolated x{L} layers"},
            "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    wl.close()


def _metric(B: int) -> str:
    phase = "decode" if B <= 64 else "prefill"
    return f"MoE {phase} tokens/sec at fixed expert-cache budget; expert-miss stall (ms)"


def _config(model, wl, L, B, method):
    E, k, d, f, rate, S = _shape(model)
    phase = "decode" if B <= 64 else "prefill"
    cfg = {"workload": f"{MODELS[model]['workload']}-{phase}", "model": MODELS[model]["model"],
           "layers": L, "experts": E, "top_k": k, "d_model": d, "d_ff": f, "cache_rate": rate,
           "capacity_per_layer": wl.eng.capacity, "global_batch": B, "seq_len": 1, "method": method, "rho": 3,
           "search_rank_h": wl.eng.search_rank_h, "alpha": 0.95, "tau_percentile": 15, "policy": "lru",
           "parallelism": "replicas (one process per GPU, disjoint token streams, no collective)",
           "l2": f"inputs larger than L2 ({(E + S) * 3 * d * f * 2 / 1e9:.2f} GB of expert weights per layer)"}
    if S:
        cfg["shared_experts"] = S
    return cfg


def gen_trace(N: int, E: int, k: int, start: int, end: int, device: str, seed: int = 11):
    """Rows [start, end) of a seeded, Zipf-skewed routing trace with distinct
    ids per token (Gumbel top-k over log-popularity). Generated in globally
    indexed 1M-token chunks, so every world size sees the same trace."""
    import torch
    chunk = 1 << 20
    logpop = (-0.8 * torch.log(torch.arange(1, E + 1, device=device, dtype=torch.float32)))
    out = torch.empty(end - start, k, device=device, dtype=torch.int32)
    c = (start // chunk) * chunk
    while c < end:
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + c // chunk)
        n = min(chunk, N - c)
        u = torch.rand(n, E, generator=g, device=device).clamp_(1e-12, 1.0)
        idx = (logpop - torch.log(-torch.log(u))).topk(k, dim=1).indices.to(torch.int32)
        a, b = max(start, c), min(end, c + n)
        out[a - start:b - start] = idx[a - c:b - c]
        c += chunk
    return out


def run_profile_bench(args, ws, rank, local):
    """BASELINE configs[4]: co-activation profiling sweep, 64M-token trace,
    E=128, k=8, token-sharded with one NCCL all-reduce (strong scaling)."""
    import torch
    import oracle as O
    from paper_2511_10054_b200 import ops, profiling as P
    N, E, k = args.trace_tokens, 128, 8
    a, b = P.shard_range(N, rank, ws)
    trace = gen_trace(N, E, k, a, b, "cuda")
    torch.cuda.synchronize()
    group = None

    def one_pass(timing=None):
        if timing is not None:
            timing[0].record()
        wend = max(0, min(b - a, 256 - a))
        wc, wp = ops.coact_count(trace[:wend], E) if wend else (None, None)
        mc, mp = ops.coact_count(trace[wend:], E)
        if timing is not None:
            timing[1].record()
        z1 = torch.zeros(E, dtype=torch.int64, device="cuda")
        z2 = torch.zeros(E, E, dtype=torch.int64, device="cuda")
        c = P.CoactCounts(mc, mp, wc if wc is not None else z1, wp if wp is not None else z2, b - a)
        if ws > 1:
            buf = c.pack()
            torch.distributed.all_reduce(buf, group=group)
            c = P.CoactCounts.unpack(buf, E)
        _, pairs = P.to_f64(c, 0.0)
        return P.build_table(pairs, 1e-3, 0.95, 16)

    for _ in range(args.warmup):
        one_pass()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clk = ClockSampler(local).ready()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kt = []
    s.record()
    for _ in range(args.steps):
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        one_pass(ev)
        kt.append(ev)
    e.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = _allmax(s.elapsed_time(e), ws)
    k_ms = float(np.mean([x.elapsed_time(y) for x, y in kt]))
    bytes_k = (b - a) * k * 4
    peak, peak_kind = _peaks()
    ach = bytes_k / (k_ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        sample = trace[: 1 << 20].cpu().numpy()
        t0 = time.perf_counter()
        O.coact_count(sample, None, E, 0, 256, 0.0)
        dt = time.perf_counter() - t0
        cpu = {"value": sample.shape[0] / dt, "unit": "tokens/s", "cores": 1, "kind": "port",
               "sample": "1,048,576 tokens of the same trace through the numpy oracle's bincount restatement of "
                         "observe (bit-exact), 1 process"}
    line = {"metric": "co-activation profiling throughput (64M-token trace, E=128, k=8)", "value": N * args.steps / (ms / 1e3),
            "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32/u64 counters, f64 ranking",
            "data": "synthetic Zipf-skewed routing trace", "config": {"workload": "coact-profile-64M-E128-k8",
            "tokens": N, "experts": E, "top_k": k, "warmup_steps": 256, "alpha": 0.95, "k_max": 16,
            "parallelism": f"token-sharded x{ws} + NCCL all-reduce", "l2": "trace (2 GB) larger than L2"},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         # DRAM bytes of the one 64M-token launch captured with ncu --set full
                         "traffic": 2148022000 + 4829952 if N == 64 << 20 and ws == 1 else None,
                         "traffic_source": "profiles/r1_coact_count.ncu-rep (ncu --set full; the launch reads the "
                                           "2.147 GB trace once)",
                         "kernel": "coact_count_kernel", "algorithmic_bytes_per_launch": bytes_k,
                         "avg_launch_ms": k_ms, "peak_kind": peak_kind},
            "cpu_baseline": cpu, "e2e": None, "gpu_launches": 5 * args.steps, "clocks": clocks}
    if rank == 0:
        print(json.dumps(line), flush=True)


def measure_h2d(wl) -> float:
    """GB/s of cudaMemcpyAsync from the pinned host mirror into HBM (one
    expert at a time, 4 experts): the PCIe roofline of an expert fetch."""
    import torch
    from paper_2511_10054_b200 import _native as N
    nb = wl.eng.buf_bytes
    dst = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    best = 0.0
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for e in range(4):
            src = wl.mirrors[0].ptr + (e * nb) % max(1, wl.mirrors[0].nbytes - nb)
            N.call("bm_memcpy", dst.data_ptr(), src, nb, s.cuda_stream)
        b.record()
        torch.cuda.synchronize()
        best = max(best, 4 * nb / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def _timed(eng, x_work, B, steps, offset, torch):
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for i in range(steps):
        j = offset + i
        eng.step(x_work[j * B:(j + 1) * B], np.arange(j * B, (j + 1) * B))
    end.record()
    torch.cuda.synchronize()
    return start.elapsed_time(end)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--profile-tokens", type=int, default=4096)
    ap.add_argument("--cpu-tokens", type=int, default=2)
    ap.add_argument("--no-original", action="store_true", help="skip the without-buddy run")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="decode", choices=["decode", "profile"],
                    help="decode: the offloaded MoE step (a batch > 64 tokens is a prefill chunk); "
                         "profile: co-activation profiling sweep (configs[4])")
    ap.add_argument("--model", default="mixtral", choices=sorted(MODELS))
    ap.add_argument("--trace-tokens", type=int, default=64 * 1024 * 1024)
    ap.add_argument("--codec", type=int, default=1, choices=[0, 1],
                    help="1: exponent-coded pinned mirrors (lossless, fewer PCIe bytes per miss); 0: raw bf16")
    args = ap.parse_args()
    ws, rank, local = _dist()
    import torch
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    if args.workload == "profile":
        run_profile_bench(args, ws, rank, local)
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    from paper_2511_10054_b200 import _native as N
    from paper_2511_10054_b200 import workload as W
    log = (lambda m: print(f"[bench r{rank}] {m}", file=sys.stderr, flush=True))
    L, share = _plan_mirrors(ws, local, args)
    B, K, Wm = args.batch, args.steps, args.warmup
    E, k_top, d, f, rate, S = _shape(args.model)
    t0 = time.time()
    # replicas serve ONE model (same weights and tables on every rank) over disjoint token streams
    wl = W.build(args.model, layers=L, max_batch=B, profile_tokens=args.profile_tokens, seed=0, codec=args.codec,
                 share=share)
    log(f"built {L} layers in {time.time() - t0:.1f}s (mean buddies {wl.mean_buddies:.2f}, "
        f"mirror {'node-shared' if share else 'private'})")
    n_steps_total = Wm + 3 * K
    x_host = torch.from_numpy(wl.tokens(2 + rank, n_steps_total * B)).pin_memory()
    x_dev = x_host.to("cuda")

    # settle (untimed): stream every pinned mirror through the copy engine once
    # (the first DMA reads of freshly pinned host pages are slower), then a
    # throwaway engine runs a few steps (graph / allocator / host paths)
    # Sweeps repeat until two consecutive ones agree within 2% and reach 97% of
    # the best seen (at most 30 sweeps or 40 s): after another process freed tens of GB
    # of pinned memory, sweeps ran at 44-49 GB/s instead of 55 for a while, and
    # a run timed then lost 15% (profiles/README.md).
    from paper_2511_10054_b200 import _native as Nn
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cs = torch.cuda.current_stream().cuda_stream
    sweep_gbs = []
    t_sweep = time.time()
    for _ in range(int(os.environ.get("BMOE_SETTLE_SWEEPS", "30"))):
        if len(sweep_gbs) >= 2 and time.time() - t_sweep > 40.0:  # bounded: replicas may share one mirror
            break
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for m in wl.mirrors:
            for off in range(0, m.nbytes, scratch.numel()):
                Nn.call("bm_memcpy", scratch.data_ptr(), m.ptr + off, min(scratch.numel(), m.nbytes - off), cs)
        b.record()
        torch.cuda.synchronize()
        sweep_gbs.append(sum(m.nbytes for m in wl.mirrors) / (a.elapsed_time(b) / 1e3) / 1e9)
        if (len(sweep_gbs) >= 2 and abs(sweep_gbs[-1] - sweep_gbs[-2]) <= 0.02 * sweep_gbs[-1]
                and min(sweep_gbs[-2:]) >= 0.97 * max(sweep_gbs)):
            break
    log(f"settle sweeps GB/s: {[round(g, 2) for g in sweep_gbs]}")
    del scratch
    # The throwaway engine runs at least 5 s (and 5 steps, at most 60): with only
    # 5 steps the first timed engine of a process ran up to 2-3% slower than a
    # later one on the same batches (profiles/README.md), with 40 it matched.
    pre = wl.engine("buddy")
    x_pre = x_dev.clone()
    t_settle, n_settle = time.time(), 0
    settle_s = float(os.environ.get("BMOE_SETTLE_S", "5"))
    while n_settle < 60 and (n_settle < 5 or time.time() - t_settle < settle_s):
        j = n_settle % n_steps_total
        pre.step(x_pre[j * B:(j + 1) * B], np.arange(j * B, (j + 1) * B))
        n_settle += 1
        torch.cuda.synchronize()
    log(f"settle engine: {n_settle} steps in {time.time() - t_settle:.1f}s")
    pre.close()

    # ---------------- with buddy substitution (headline) ----------------
    eng = wl.engine("buddy")
    x_work = x_dev.clone()
    _timed(eng, x_work, B, Wm, 0, torch)
    eng.stats(reset=True)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local).ready()
    ms = _timed(eng, x_work, B, K, Wm, torch)
    clocks = clk.stop()
    st = eng.stats(reset=True)
    ms = _allmax(ms, ws)
    value = ws * K * B / (ms / 1000.0)

    # ---------------- kernel timing pass (roofline of the grouped FFN GEMM) ----------------
    # (copy timing too: per-fetch timing events on the copy stream cost the
    # copy engine ~6 us each, so the timed run above goes without them)
    N.lib().bm_set_kernel_timing(1)
    eng.set_copy_timing(True)
    _timed(eng, x_work, B, K, Wm + K, torch)
    st_k = eng.stats(reset=True)
    eng.set_copy_timing(False)
    buf = (np.zeros(6 * L * K + 8, np.float32))
    n = int(N.lib().bm_kernel_times(buf.ctypes.data, buf.size))
    N.lib().bm_set_kernel_timing(0)
    g1 = buf[0:n:2]
    g2 = buf[1:n:2]
    launches = max(len(g1), 1)
    fused = bool(len(g2)) and float(np.max(g2)) == 0.0  # the timing hook reports 0 for one-kernel calls
    n_exp = st_k["ffn_experts"] / launches
    rows = st_k["ffn_rows"] / launches
    g1_ms, g2_ms = float(np.mean(g1)), float(np.mean(g2))
    # Algorithmic bytes (every executed expert's W1+W3+W2 + the activations
    # read) and flops (6·d·f per executed row) of the pass; the FFN's bound is
    # whichever roofline gives the longer ideal time (decode and small-expert
    # prefill stream weights: HBM; wide prefill tiles: tensor pipe).
    tot_k = st_k["ffn_experts"] * 3 * d * f * 2 + st_k["ffn_rows"] * (d + f) * 2
    flops = 6.0 * d * f * st_k["ffn_rows"]
    hbm_peak, hbm_kind = _peaks("hbm")
    tc_peak, tc_kind = _peaks("tensor")
    hbm_bound = tot_k / (hbm_peak * 1e9) >= flops / (tc_peak * 1e12)
    if fused or hbm_bound:
        # Decode: Σ bytes / Σ FFN kernel time. A layer-step with misses issues
        # two grouped-FFN calls (resident experts overlapped with the fetch,
        # then the fetched ones), each ONE fused kernel at decode width.
        peak, peak_kind = hbm_peak, hbm_kind
        ach = tot_k / (float(np.sum(g1) + np.sum(g2)) / 1e3) / 1e9
        # DRAM bytes of one captured launch (ncu --set full, committed under
        # profiles/), with that launch's own algorithmic bytes beside it
        traffic, traffic_launch = None, None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "r1e_traffic.json")))
            l0 = tr["launches"][0]
            if args.model == "mixtral" and fused:
                traffic = l0["dram_read_bytes"] + l0["dram_write_bytes"]
                traffic_launch = {"experts": l0["experts"], "weight_bytes": l0["weight_bytes"],
                                  "dram_over_weight_bytes": traffic / l0["weight_bytes"], "source": tr["source"]}
        except (OSError, KeyError, ValueError):
            pass
        roofline = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "traffic": traffic, "traffic_launch": traffic_launch,
                    "kernel": "ffn_fused_kernel (one cooperative launch: W1|W3 swap-AB GEMM -> SwiGLU -> W2 GEMM, "
                              "stream-K)" if fused else
                              "ffn_gemm_kernel x2 (data-parallel tcgen05 tiles, SwiGLU / output in the epilogue)",
                    "algorithmic_bytes_per_launch": tot_k / launches, "avg_launch_ms": g1_ms, "peak_kind": peak_kind,
                    "experts_per_launch": n_exp, "rows_per_launch": rows}
    else:
        # Prefill, tensor-bound: Σ 6·d·f flops per executed (token, slot) row over Σ GEMM1 + GEMM2 time
        peak, peak_kind = tc_peak, tc_kind
        ach = flops / (float(np.sum(g1) + np.sum(g2)) / 1e3) / 1e12
        roofline = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": None,
                    "kernel": "ffn_gemm_kernel x2 (data-parallel tcgen05 tiles, SwiGLU / output in the epilogue)",
                    "flops_per_call": flops / launches, "avg_gemm1_ms": g1_ms, "avg_gemm2_ms": g2_ms,
                    "peak_kind": peak_kind + " (burst)", "experts_per_launch": n_exp, "rows_per_launch": rows}

    # ---------------- fetch roofline: measured pinned H2D copy rate ----------------
    h2d_peak = measure_h2d(wl)
    fetch_gbs = st_k["wire_bytes"] / (st_k["copy_ms"] / 1e3) / 1e9 if st_k["copy_ms"] > 0 else None
    fetch_eff = st_k["h2d_bytes"] / (st_k["copy_ms"] / 1e3) / 1e9 if st_k["copy_ms"] > 0 else None

    # ---------------- end to end through the public API, host buffers ----------------
    # A fresh engine replays the same warm-up and the same K batches as the
    # device-resident run, so both see identical misses and fetches; only the
    # per-step pinned host -> device input copy and device -> host result
    # read are added.
    eng.close()
    eng = wl.engine("buddy")
    _timed(eng, x_dev.clone(), B, Wm, 0, torch)
    eng.stats(reset=True)
    out_host = torch.empty_like(x_host)
    h = torch.empty(B, d, device="cuda")
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for i in range(K):
        j = Wm + i
        h.copy_(x_host[j * B:(j + 1) * B], non_blocking=True)
        eng.step(h, np.arange(j * B, (j + 1) * B))
        out_host[j * B:(j + 1) * B].copy_(h, non_blocking=True)
    end.record()
    torch.cuda.synchronize()
    e2e_ms = _allmax(start.elapsed_time(end), ws)
    e2e = ws * K * B / (e2e_ms / 1000.0)
    st_e = eng.stats(reset=True)
    eng.close()

    # ---------------- without buddy (method=original, on-demand fetch) ----------------
    orig, fidelity = None, None
    if not args.no_original:
        eo = wl.engine("original")
        x2 = x_dev.clone()
        _timed(eo, x2, B, Wm, 0, torch)
        eo.stats(reset=True)
        if ws > 1:
            torch.distributed.barrier()
        ms_o = _allmax(_timed(eo, x2, B, K, Wm, torch), ws)
        so = eo.stats(reset=True)
        eo.close()
        # fidelity of the buddy arm (the paper's accuracy axis; harness.fidelity,
        # harness.py:189-206): its outputs vs the exact on-demand arm's on the
        # same timed tokens, mean cosine + argmax agreement under the
        # reference's seeded readout head
        from paper_2511_10054_b200 import harness, substrate
        rows = slice(Wm * B, (Wm + K) * B)
        cos, agree = harness.fidelity(x_work[rows].double().cpu().numpy(), x2[rows].double().cpu().numpy(),
                                      substrate.readout_head(wl.spec, 16))
        fidelity = {"cosine_mean": cos, "argmax_agreement": agree, "tokens": K * B,
                    "vs": "method=original (every expert exact, fetched on demand)",
                    "note": "random-init experts share no function, so a substituted buddy is an unrelated "
                            "expert here; on the reference's clustered substrate the engine reproduces the "
                            "reference's own fidelity (tests/test_engine_gpu.py)"}
        orig = {"value": ws * K * B / (ms_o / 1000.0), "unit": "tokens/s", "ms_per_step": ms_o / K,
                "stall_ms_per_step": so["stall_ms"] / K, "ondemand_misses_per_step": so["ondemand_misses"] / K,
                "physical_fetches_per_step": so["physical_fetches"] / K,
                "h2d_gb_per_step": so["h2d_bytes"] / K / 1e9, "wire_gb_per_step": so["wire_bytes"] / K / 1e9}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        stacks = stage_layer_f64(wl, 0)
        times = [cpu_reference_sample(wl, 0, min(args.cpu_tokens, B), 5000 + i, stacks) for i in range(2)]
        del stacks
        per_layer = min(times)
        nb = min(args.cpu_tokens, B)
        cpu = {"value": nb / (per_layer * L), "unit": "tokens/s", "cores": len(os.sched_getaffinity(0)),
               "kind": "port", "sample": f"{nb} tokens x 1 layer-step (route, gates, remap, f64 forward, "
                                         f"layer_update) via the numpy oracle, best of 2, extrapolated x{L} layers"}

    line = {
        "metric": _metric(B),
        "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": K, "warmup": Wm,
        "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (random-init bf16 weights, reference-style clustered router/token stream)",
        "config": dict(_config(args.model, wl, L, B, "buddy"),
                       host_mirror="node-shared /dev/shm" if share else "private pinned",
                       fetch_codec="exponent-coded bf16" if args.codec else "raw bf16"),
        "stall_ms_per_step": st["stall_ms"] / K,
        "sim_stall_model": {"ondemand_misses_per_step": st["ondemand_misses"] / K,
                            "substitutions_per_step": st["substitutions"] / K},
        "physical_fetches_per_step": st["physical_fetches"] / K,
        "h2d_gb_per_step": st["h2d_bytes"] / K / 1e9,
        "wire_gb_per_step": st["wire_bytes"] / K / 1e9,
        "fetch_codec": "exponent-coded bf16 (lossless, bm_xfer)" if args.codec else "raw bf16",
        "without_buddy": orig,
        "fidelity": fidelity,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "fetch_roofline": {"bound": "pcie", "achieved": fetch_gbs, "peak": h2d_peak, "unit": "GB/s",
                           "frac": (fetch_gbs / h2d_peak) if fetch_gbs else None, "effective_gbs": fetch_eff,
                           "step_utilisation": st["wire_bytes"] / 1e9 / (ms / 1e3) / h2d_peak,
                           "note": "H2D wire bytes / copy-engine busy time (CUDA events around each fetch, in the "
                                   "kernel-timing pass) vs the best pinned copy rate of 4 expert-sized copies back to "
                                   "back; effective_gbs = decoded expert bytes over the same time; step_utilisation = "
                                   "wire bytes of the timed run / (its step time x the pinned rate)"},
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": B * d * 4,
                "d2h_bytes_per_step": B * d * 4, "ms_per_step": e2e_ms / K,
                "physical_fetches_per_step": st_e["physical_fetches"] / K,
                "note": "fresh engine, same warm-up and the same K batches as `value`; pinned host in/out per step"},
        "gpu_launches": int(st["kernel_launches"]),
        "clocks": clocks,
        "setup_s": time.time() - t0,
        "settle_sweeps_gbs": sweep_gbs,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    wl.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
