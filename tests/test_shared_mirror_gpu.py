"""Replicas sharing one node-level expert mirror, on one GPU: two processes
(gloo world of 2, both on cuda:0) build the same Qwen3-shaped workload with
a ShareSpec; rank 0 writes the coded mirror into /dev/shm and page-locks it,
rank 1 attaches read-only (cudaHostRegisterReadOnly). Both engines then
decode the same tokens and must agree bitwise with each other (and rank 1's
fetches really went through the shared mapping)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2511_10054_b200 import workload as W
        from paper_2511_10054_b200.engine import SharedMirror
        share = W.ShareSpec(tag=f"bmoe_pytest_{port}", owner=rank == 0, barrier=dist.barrier)
        wl = W.build("qwen3", layers=2, max_batch=16, profile_tokens=512, share=share)
        eng = wl.engine("buddy")
        x = torch.from_numpy(wl.tokens(2, 48)).cuda()
        for s in range(3):
            eng.step(x[s * 16:(s + 1) * 16], np.arange(s * 16, (s + 1) * 16))
        torch.cuda.synchronize()
        st = eng.stats()
        q.put((rank, x.cpu().numpy(), eng.events(), st["physical_fetches"], st["wire_bytes"],
               all(isinstance(m, SharedMirror) and m.codec == 1 for m in wl.mirrors)))
        eng.close()
        dist.barrier()  # the owner unlinks only after every rank is done
        wl.close()
    finally:
        dist.destroy_process_group()


def test_two_replicas_share_one_mirror(cuda_ok):
    if W_free() < (1 << 30):
        pytest.skip("/dev/shm too small on this box")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    # read the results before joining: a child blocks in q.put until its
    # (large) payload is consumed
    pc = mp.start_processes(_worker, args=(2, port, q), nprocs=2, start_method="spawn", join=False)
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    while not pc.join(timeout=300):
        pass
    (_, x0, ev0, pf0, wb0, sh0), (_, x1, ev1, pf1, wb1, sh1) = res
    assert sh0 and sh1
    assert pf1 > 0 and wb1 > 0  # rank 1 fetched experts from the shared mapping
    assert np.array_equal(ev0, ev1) and np.array_equal(x0.view(np.uint32), x1.view(np.uint32))


def W_free():
    from paper_2511_10054_b200.workload import shm_bytes_free
    return shm_bytes_free()
