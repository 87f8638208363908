"""Token-sharded profiling over a world-size-2 gloo group on CPU.

The counting kernel needs a GPU, so the test injects the oracle's counter;
what is under test is the multi-process plumbing: contiguous shard ranges,
global warm-up indices crossing the shard boundary, packing, the single
sum all-reduce, and unpacking — which must reproduce the reference's
single-stream statistics exactly (profiler.merge contract, test_profiler.py:116-132).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden


def _oracle_counter(topk, E):
    import oracle as O
    c, p, _, _ = O.coact_count(topk.numpy(), None, E, 0, 0, 0.0)
    return torch.from_numpy(c.astype(np.int64)), torch.from_numpy(p.astype(np.int64))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_10054_b200 import profiling as P
        g = golden("coact_default_w05.npz")   # warmup_steps 256 crosses no/one shard boundary
        E = int(g["E"])
        topk = torch.from_numpy(g["topk"].astype(np.int32))
        c = P.profile_trace(topk, E, int(g["warmup_steps"]), counter=_oracle_counter)
        if rank == 0:
            ww = float(g["warmup_weight"])
            pairs = ww * c.warm_pairs.double().numpy() + c.pairs.double().numpy()
            counts = ww * c.warm_counts.double().numpy() + c.counts.double().numpy()
            q.put((np.array_equal(pairs, g["pairs"]), np.array_equal(counts, g["counts"]),
                   c.tokens_seen == int(g["tokens_seen"])))
        # a trace whose warm-up range straddles the shard boundary
        topk2 = topk[:300]
        c2 = P.profile_trace(topk2, E, 200, counter=_oracle_counter)
        if rank == 0:
            import oracle as O
            _, p_main, _, _ = O.coact_count(g["topk"][200:300], None, E, 0, 0, 0.0)
            _, p_warm, _, _ = O.coact_count(g["topk"][:200], None, E, 0, 0, 0.0)
            q.put((np.array_equal(c2.pairs.double().numpy(), p_main),
                   np.array_equal(c2.warm_pairs.double().numpy(), p_warm), c2.tokens_seen == 300))
        # each rank holds only its own shard (sharded=False): global warm-up offsets
        a, b = P.shard_range(300, rank, world)
        c3 = P.profile_trace(topk2[a:b].clone(), E, 200, sharded=False, counter=_oracle_counter, total_tokens=300)
        if rank == 0:
            q.put((torch.equal(c3.pairs, c2.pairs), torch.equal(c3.warm_pairs, c2.warm_pairs),
                   c3.tokens_seen == 300))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sharded_profile_allreduce_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    r1, r2, r3 = q.get(timeout=5), q.get(timeout=5), q.get(timeout=5)
    assert all(r1) and all(r2) and all(r3), (r1, r2, r3)


def test_shard_ranges_cover_exactly():
    from paper_2511_10054_b200.profiling import shard_range
    for n in (0, 1, 7, 1000, 64_000_001):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
