"""CPU checks of bench.py plumbing: the profiling trace is identical however
it is sharded (so N-GPU runs count the same tokens), and the layer count
adapts to host memory."""

import numpy as np
import torch

import bench
from paper_2511_10054_b200.profiling import shard_range


def test_trace_shards_concatenate_to_the_full_trace():
    N, E, k = (1 << 20) + 12345, 128, 8
    full = bench.gen_trace(N, E, k, 0, N, "cpu")
    assert full.shape == (N, k) and full.dtype == torch.int32
    # distinct ids per token, all in range
    s, _ = torch.sort(full[:5000], dim=1)
    assert bool((s[:, 1:] != s[:, :-1]).all()) and int(full.min()) >= 0 and int(full.max()) < E
    for world in (2, 3):
        parts = [bench.gen_trace(N, E, k, *shard_range(N, r, world), "cpu") for r in range(world)]
        assert torch.equal(torch.cat(parts), full)


def test_trace_is_skewed():
    t = bench.gen_trace(1 << 20, 128, 8, 0, 1 << 20, "cpu")
    counts = np.bincount(t.numpy().ravel(), minlength=128)
    assert counts[0] > 3 * counts[-1]  # Zipf(0.8) popularity


def test_layers_for_host_scales_with_world_size():
    l1 = bench._layers_for_host(1, None)
    l8 = bench._layers_for_host(8, None)
    assert 1 <= l8 <= l1 <= 32
    assert bench._layers_for_host(1, 4) == min(4, l1)
