"""Co-activation profiling over a routing trace, token-sharded across GPUs.

The tensor form of cmd_profile's counting + cmd_build (harness.py:70-158):
K6 counts binary co-activations of a trace ``topk[N,k]`` on each rank's
contiguous token range; the single exchange is one sum all-reduce of the
packed u64 counters (E + E^2 for the main range, E + E^2 for the warm-up
range, + tokens_seen) over NCCL/NVLink; every rank then converts to f64
(exact reference accumulation order, bm_counts_to_f64) and ranks buddies
with K7 identically, so no broadcast is needed. Merging shards is the
reference's elementwise `merge` (profiler.py:122-137) on integers, hence
exact. Reference semantics: observe (profiler.py:67-95).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .errors import ConfigurationError, InputError


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous token range of one rank: [r*N/W, (r+1)*N/W)."""
    return (n * rank) // world, (n * (rank + 1)) // world


@dataclass
class CoactCounts:
    """Integer co-activation counters (stored in int64 tensors; values < 2^63)."""
    counts: torch.Tensor       # [E]   main range
    pairs: torch.Tensor        # [E,E] main range
    warm_counts: torch.Tensor  # [E]   warm-up range (global index < warmup_steps)
    warm_pairs: torch.Tensor   # [E,E]
    tokens_seen: int

    def pack(self) -> torch.Tensor:
        seen = torch.tensor([self.tokens_seen], dtype=torch.int64, device=self.counts.device)
        return torch.cat([self.counts.view(-1), self.pairs.view(-1), self.warm_counts.view(-1),
                          self.warm_pairs.view(-1), seen])

    @staticmethod
    def unpack(buf: torch.Tensor, E: int) -> "CoactCounts":
        o = 0
        c = buf[o:o + E]; o += E
        p = buf[o:o + E * E].view(E, E); o += E * E
        wc = buf[o:o + E]; o += E
        wp = buf[o:o + E * E].view(E, E); o += E * E
        return CoactCounts(c, p, wc, wp, int(buf[o].item()))


def count_kernel(topk: torch.Tensor, num_experts: int):
    """K6 on the device: (counts[E], pairs[E,E]) int64."""
    return ops.coact_count(topk.contiguous(), num_experts)


def count_shard(topk_shard: torch.Tensor, num_experts: int, global_start: int, warmup_steps: int,
                counter=count_kernel) -> CoactCounts:
    """Counts for tokens with global indices [global_start, global_start+n)."""
    n = topk_shard.shape[0]
    warm_end = max(0, min(n, warmup_steps - global_start))
    wc, wp = counter(topk_shard[:warm_end], num_experts) if warm_end > 0 else (None, None)
    mc, mp = counter(topk_shard[warm_end:], num_experts) if warm_end < n else (None, None)
    dev = topk_shard.device
    z1 = lambda: torch.zeros(num_experts, dtype=torch.int64, device=dev)  # noqa: E731
    z2 = lambda: torch.zeros(num_experts, num_experts, dtype=torch.int64, device=dev)  # noqa: E731
    return CoactCounts(mc if mc is not None else z1(), mp if mp is not None else z2(),
                       wc if wc is not None else z1(), wp if wp is not None else z2(), n)


def profile_trace(topk: torch.Tensor, num_experts: int, warmup_steps: int = 256, group=None, sharded=True,
                  counter=count_kernel, total_tokens: int | None = None) -> CoactCounts:
    """Count a trace and all-reduce the counters across the process group.

    sharded=True: every rank holds the whole trace and counts its
    shard_range. sharded=False: ``topk`` is this rank's own shard of a
    ``total_tokens``-token trace split by shard_range, so its first row has
    the global index shard_range(total_tokens, rank, world)[0] (warm-up
    weighting follows the global index, profiler.py:81-95)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    N = topk.shape[0]
    if sharded and world > 1:
        a, b = shard_range(N, rank, world)
        local = count_shard(topk[a:b], num_experts, a, warmup_steps, counter)
    elif world > 1:
        if total_tokens is None:
            raise ConfigurationError("profile_trace(sharded=False) on several ranks needs total_tokens")
        a, b = shard_range(int(total_tokens), rank, world)
        if b - a != N:
            raise InputError(f"rank {rank} holds {N} tokens, shard_range gives {b - a}")
        local = count_shard(topk, num_experts, a, warmup_steps, counter)
    else:
        local = count_shard(topk, num_experts, 0, warmup_steps, counter)
    if world == 1:
        return local
    buf = local.pack()
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)  # the one exchange step
    return CoactCounts.unpack(buf, num_experts)


def to_f64(c: CoactCounts, warmup_weight: float = 0.0):
    """Reference float64 statistics (counts, pair_counts) with the exact
    sequential warm-up accumulation order (bm_counts_to_f64)."""
    return (ops.counts_to_f64(c.counts.contiguous(), c.warm_counts.contiguous(), warmup_weight),
            ops.counts_to_f64(c.pairs.contiguous(), c.warm_pairs.contiguous(), warmup_weight))


def build_table(pairs_f64: torch.Tensor, eps: float = 1e-3, alpha: float = 0.95, k_max: int = 16):
    """K7: bit-exact buddies.build_table (buddies.py:102-129) on the device."""
    return ops.buddy_rank(pairs_f64.contiguous(), eps, alpha, k_max)
