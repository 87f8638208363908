"""Node-shared expert mirror for replicas (engine.SharedMirror,
workload.ShareSpec) over a world-size-2 gloo group on CPU: local rank 0
creates and fills the /dev/shm file, the barrier orders the writes, rank 1
attaches and sees the very bytes (and the coded-image magic); the owner
unlinks on close. Page-locking (bm_host_register) needs a GPU and is off."""

import os
import socket
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, directory, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_10054_b200.engine import SharedMirror
        from paper_2511_10054_b200.workload import ShareSpec
        share = ShareSpec(tag="bmoe_test", owner=rank == 0, barrier=dist.barrier, directory=directory)
        payload = np.frombuffer(b"BXL1" + bytes(range(256)) * 40, np.uint8)
        if share.owner:
            m = SharedMirror(share.path(3), payload.size, create=True, register=False)
            m.as_tensor().copy_(torch.from_numpy(payload.copy()))
        share.barrier()
        if not share.owner:
            m = SharedMirror(share.path(3), register=False)
            got = m.as_tensor().numpy().copy()
            q.put((m.nbytes, m.codec, bool(np.array_equal(got, payload))))
        dist.barrier()
        m.close()
        dist.barrier()
        if share.owner:
            q.put(os.path.exists(share.path(3)))
    finally:
        dist.destroy_process_group()


def test_shared_mirror_two_ranks():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with tempfile.TemporaryDirectory() as d:
        pc = mp.start_processes(_worker, args=(2, port, d, q), nprocs=2, start_method="spawn", join=False)
        res = [q.get(timeout=60) for _ in range(2)]
        while not pc.join(timeout=60):
            pass
    attach = next(r for r in res if isinstance(r, tuple))
    exists = next(r for r in res if isinstance(r, bool))
    assert attach == (4 + 256 * 40, 1, True)
    assert exists is False
