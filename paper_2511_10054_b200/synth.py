"""Synthetic expert weights for the benchmark workloads, reproducible
bit for bit on the GPU and on the host.

No checkpoints exist here, so the BASELINE shapes run on random-init
weights. They come from a counter-based hash rather than a stateful RNG so
that two very different consumers see the same numbers:

  * the GPU arm (``workload.build``) generates each expert matrix in HBM with
    ``bm_synth_bf16`` (csrc/synth.cu) and packs it into the UMMA-tiled
    layout;
  * the CPU reference arm of ``bench.py`` regenerates the same matrices with
    the numpy twin below (uint64 arithmetic wraps like the kernel's), as
    float64 like the reference's expert stacks, without loading libbmoe or
    touching a GPU.

Value ``i`` of a matrix is ``lut[(mix64(base + i // 4) >> 16 * (i % 4)) &
0xFFFF]`` with ``mix64`` the splitmix64 finaliser, ``base`` a per-(seed,
layer, expert, matrix) key and ``lut`` the 65,536 bf16 quantiles
``Phi^-1((u + 0.5) / 65536) * scale`` of N(0, scale^2), scale = fan_in^-0.5
(the usual N(0, 1/fan_in) init). This module is numpy-only on purpose.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from statistics import NormalDist

import numpy as np

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_LUTS: dict = {}

W1, W3, W2 = 0, 1, 2  # matrix ids inside a SwiGLU expert [W1 | W3 | W2]

SHAPES = {
    # name: (E, k, d, f, cache_rate) — BASELINE.json configs[1..3] (+ the tiny config 0)
    "mixtral": (8, 2, 4096, 14336, 0.5),
    "qwen3": (128, 8, 2048, 768, 0.25),
    "dsv2lite": (64, 6, 2048, 1408, 0.5),
    "tiny": (8, 2, 128, 256, 0.5),
}
SHARED = {"dsv2lite": 2}  # always-resident shared experts (outside the cache budget)
# Clustered synthetic experts (the reference's substrate recipe, model.py:161-171):
# expert e of cluster c = base_c + SPREAD * delta_e, with the router built on
# the same clusters (substrate.ModelSpec.num_clusters). The default cluster
# count is the reference's own default, model.clusters = 8 (config.py:72),
# capped at E as ModelSpec.validate requires (model.py:74-75): at the Mixtral
# shape (E = 8) every expert is its own cluster, exactly what the reference
# builds there. FIDELITY_CLUSTERS are coarser groupings (several mates per
# cluster) for the buddy-vs-random fidelity experiments (bench --clusters).
CLUSTERS = {"mixtral": 8, "qwen3": 8, "dsv2lite": 8, "tiny": 8}
FIDELITY_CLUSTERS = {"mixtral": 2, "qwen3": 8, "dsv2lite": 4, "tiny": 2}
SPREAD = 0.1  # model.cluster_spread default (config.py)


def host_mem_available() -> int:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 64 << 30


def initial_residents(num_experts: int, capacity: int, seed: int, layer: int):
    """Seeded-permutation prefix, nested across capacities (memtier.py:132-140)."""
    if capacity <= 0:
        return []
    rng = np.random.default_rng(np.random.SeedSequence([seed, 21, layer]))
    return sorted(int(v) for v in rng.permutation(num_experts)[:capacity])


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """float64 -> bf16 bit patterns, round to nearest even (via float32)."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def lut_bf16(scale: float) -> np.ndarray:
    """The 65,536-entry quantile table of N(0, scale^2) as bf16 bits."""
    key = float(scale)
    if key not in _LUTS:
        nd = NormalDist()
        q = np.array([nd.inv_cdf((u + 0.5) / 65536.0) for u in range(65536)]) * key
        _LUTS[key] = _bf16_bits(q)
    return _LUTS[key]


def bf16_to_f64(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def matrix_key(seed: int, layer: int, expert: int, matrix: int) -> int:
    """The hash base of one expert matrix (distinct streams for every
    (seed, layer, expert, matrix); keys are spaced 2^40 apart, far beyond
    any matrix's n/4 counters)."""
    k = (((seed * 1_000_003 + layer) * 4099 + expert) * 4 + matrix) & ((1 << 24) - 1)
    return (k << 40) & ((1 << 64) - 1)


def base_key(seed: int, layer: int, cluster: int, matrix: int) -> int:
    """Hash base of cluster ``cluster``'s base matrix: the expert-key space
    with the top bit set (expert keys stay below 2^63)."""
    k = matrix_key(seed, layer, cluster, matrix)
    if k >> 63:
        raise ValueError("seed too large for the synthetic key space")
    return k | (1 << 63)


def cluster_of(num_experts: int, clusters: int) -> np.ndarray:
    """Contiguous cluster blocks (model.py:126-130)."""
    return (np.arange(num_experts) * clusters) // num_experts


def mix_bits(base_bits: np.ndarray, delta_bits: np.ndarray, spread: float) -> np.ndarray:
    """bf16_rn(b + spread * e) with fp32 operations, each rounded (the kernel's
    __fadd_rn(b, __fmul_rn(spread, e)))."""
    b = (base_bits.astype(np.uint32) << np.uint32(16)).view(np.float32)
    e = (delta_bits.astype(np.uint32) << np.uint32(16)).view(np.float32)
    v = b + np.float32(spread) * e
    return _bf16_bits(v)


def matrix_scale(d: int, f: int, matrix: int) -> float:
    return (d if matrix in (W1, W3) else f) ** -0.5


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z + _GOLD
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def synth_bits(base: int, n: int, lut: np.ndarray, start: int = 0) -> np.ndarray:
    """Values [start, start+n) of a matrix as bf16 bits (start % 4 == 0)."""
    assert start % 4 == 0
    g = np.arange(start // 4, (start + n + 3) // 4, dtype=np.uint64) + np.uint64(base)
    z = _mix64(g)
    idx = np.empty((z.size, 4), np.uint16)
    for j in range(4):
        idx[:, j] = (z >> np.uint64(16 * j)).astype(np.uint16)
    return lut[idx.reshape(-1)[:n]]


def synth_f64(base: int, n: int, scale: float, threads: int | None = None, out: np.ndarray | None = None,
              chunk: int = 1 << 18) -> np.ndarray:
    """A whole matrix as float64 (the reference's dtype), generated in
    parallel cache-sized chunks on the host (numpy releases the GIL); the
    same values as synth_bits, gathered straight from a float64 table."""
    assert chunk % 4 == 0
    lut64 = bf16_to_f64(lut_bf16(scale))
    out = np.empty(n, np.float64) if out is None else out
    threads = threads or len(os.sched_getaffinity(0))
    starts = list(range(0, n - n % 4, chunk))

    def work(c0):
        m = min(chunk, n - n % 4 - c0) // 4
        z = np.arange(c0 // 4, c0 // 4 + m, dtype=np.uint64)
        z += np.uint64(base) + _GOLD
        t = np.empty_like(z)
        for sh, mul in ((30, _M1), (27, _M2)):
            np.right_shift(z, np.uint64(sh), out=t)
            z ^= t
            z *= mul
        np.right_shift(z, np.uint64(31), out=t)
        z ^= t
        dst = out[c0:c0 + 4 * m].reshape(m, 4)
        idx = np.empty(m, np.uint16)
        for j in range(4):
            np.copyto(idx, (z >> np.uint64(16 * j)) if j else z, casting="unsafe")
            np.take(lut64, idx, out=dst[:, j])

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, starts))
    if n % 4:  # ragged tail
        out[n - n % 4:] = lut64[synth_bits(base, n % 4, np.arange(65536, dtype=np.uint16), n - n % 4)]
    return out


def expert_f64(seed: int, layer: int, expert: int, d: int, f: int, threads: int | None = None):
    """(W1 [f,d], W3 [f,d], W2 [d,f]) float64 of one SwiGLU expert."""
    mats = []
    for m, shape in ((W1, (f, d)), (W3, (f, d)), (W2, (d, f))):
        mats.append(synth_f64(matrix_key(seed, layer, expert, m), d * f, matrix_scale(d, f, m), threads)
                    .reshape(shape))
    return tuple(mats)
