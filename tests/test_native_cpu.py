"""CPU-side checks of the C-ABI library: it builds, loads, exports every
symbol include/bmoe.h declares, and its host-only control plane (the exact
memtier replica) reproduces the reference's event logs bit for bit."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_2511_10054_b200 import _native as N
from paper_2511_10054_b200 import memtier as M
from paper_2511_10054_b200.errors import ConfigurationError, InputError, InvariantViolation, NativeLibraryError


@pytest.fixture(scope="module", autouse=True)
def lib():
    if not os.path.exists(N.lib_path()):
        from paper_2511_10054_b200.build import build_library
        build_library()
    return N.lib()


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "bmoe.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(bm_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 40
    import ctypes
    so = ctypes.CDLL(N.lib_path())
    missing = [n for n in sorted(names) if not hasattr(so, n)]
    assert not missing, missing
    # and the binding declares exactly the exported ABI
    assert names == set(N.exported_symbols()), names ^ set(N.exported_symbols())
    assert N.lib().bm_abi_version() == 1


def test_no_cpu_fallback_for_kernels():
    """Product entry points refuse CPU tensors instead of computing on the host."""
    import torch
    from paper_2511_10054_b200 import ops
    with pytest.raises(InputError):
        ops.gate_topk(torch.zeros(2, 8), torch.zeros(4, 8), None, 2)
    with pytest.raises(InputError):
        ops.coact_count(torch.zeros(4, 2, dtype=torch.int32), 8)


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "_LIB_PATH", "/nonexistent/libbmoe.so")
    with pytest.raises(NativeLibraryError):
        N.lib()


def _replay(g):
    E, rate, policy, seed, layer = int(g["E"]), float(g["rate"]), int(g["policy"]), int(g["seed"]), int(g["layer"])
    pol = ("lru", "lfu", "freq_static")[policy]
    st = M.init_residency(E, rate, pol, seed=seed, static_freq=g["static"] if pol == "freq_static" else None,
                          layer=layer)
    cost = M.CostModel(expert_load_ms=9.5, hit_ms=0.25, expert_compute_ms=0.5, pcie_bw_bytes_per_s=4.0e6,
                       expert_bytes=32768)
    clock, log, buf, tok = M.SimClock(), [], [], 0
    for op, a, b in g["prog"]:
        tok += 1
        if op == 0:
            M.access(st, int(a), clock, cost, token=tok, log=log)
        elif op == 1:
            M.access(st, int(a), clock, cost, mode="substituted_away", token=tok, log=log)
        elif op == 2:
            if a < 0:
                M.prefetch(st, buf, clock, cost, log=log)
                buf = []
            else:
                buf.append(int(a))
        elif op == 3:
            M.settle(st, clock, cost, log=log)
        else:
            clock.advance(b / 2.0)
    return st, clock, log


@pytest.mark.parametrize("idx,pol", [(0, "lru"), (1, "lfu"), (2, "freq_static"), (3, "lru")])
def test_cache_control_plane_replays_reference_events(idx, pol):
    """bm_cache (C++) vs the reference ResidencyState/access/prefetch/settle
    event log on random programs: bit-exact times, kinds, experts, bytes."""
    g = golden(f"memtier_{idx}_{pol}.npz")
    st, clock, log = _replay(g)
    codes = {k: i for i, k in enumerate(M._EV_BY_CODE)}
    ev = np.array([(e.time_ms, codes[e.kind], e.layer, e.token, e.expert, e.bytes, e.stall_ms) for e in log],
                  np.float64).reshape(-1, 7)
    assert ev.shape == g["events"].shape
    assert np.array_equal(ev, g["events"])
    assert np.array_equal(st.mask, g["final_mask"])
    assert np.array_equal(st._last_use, g["final_last_use"])
    assert np.array_equal(st._freq, g["final_freq"])
    assert st.waste_evictions == int(g["waste"]) and clock.now == float(g["now"])


def test_transfer_timing_known_answers():
    """Reference acceptance criterion 4 (test_acceptance.py:233-260)."""
    cost = M.CostModel()
    st = M.init_residency(64, 0.5, "lru", seed=0)
    clock = M.SimClock()
    missing = [int(e) for e in np.flatnonzero(~st.mask)[:4]]
    ev = M.access(st, missing[0], clock, cost)
    assert abs(ev.stall_ms - 9.5) <= 1e-9 and abs(clock.now - 9.5) <= 1e-9 and ev.bytes == 32768
    clock2 = M.SimClock()
    st2 = M.init_residency(64, 0.5, "lru", seed=0)
    M.prefetch(st2, missing[:2], clock2, cost)
    assert abs(st2.pending[0][0] - 8.192) <= 1e-9 and abs(st2.pending[1][0] - 2 * 8.192) <= 1e-9
    ev = M.access(st2, missing[2], clock2, cost)
    assert abs(ev.stall_ms - (2 * 8.192 + 9.5)) <= 1e-9
    before = clock.now
    ev = M.access(st, missing[3], clock, cost, mode="substituted_away")
    assert ev.bytes == 0 and clock.now == before + cost.hit_ms


def test_eviction_policies_ties_to_lowest_id():
    # test_memtier.py:122-158 style: LRU evicts least recent, LFU least frequent
    st = M.ResidencyState(8, 4, "lru")
    clock, cost = M.SimClock(), M.CostModel()
    res = [int(e) for e in np.flatnonzero(st.mask)]
    for e in res[1:]:
        M.access(st, e, clock, cost)
    miss = int(np.flatnonzero(~st.mask)[0])
    log = []
    M.access(st, miss, clock, cost, log=log)
    assert [e.kind for e in log] == ["miss_ondemand", "evict"] and log[1].expert == res[0]
    st = M.ResidencyState(8, 4, "lfu")
    res = [int(e) for e in np.flatnonzero(st.mask)]
    for e in res[1:]:
        M.access(st, e, clock, cost)
    log = []
    M.access(st, int(np.flatnonzero(~st.mask)[0]), clock, cost, log=log)
    assert log[1].expert == res[0]


def test_lru_recency_list_matches_argmin_scan():
    """The C++ LRU victim is the head of a recency list (O(1)); on a long
    thrashing stream (prefill-like: most accesses miss) it evicts exactly
    memtier's argmin(last_use), ties to the lowest id (memtier.py:162-170)."""
    rng = np.random.default_rng(5)
    E, cap = 64, 16
    st = M.ResidencyState(E, cap, "lru")
    clock, cost = M.SimClock(), M.CostModel()
    mask = st.mask.copy()
    last = np.where(mask, 0, -1).astype(np.int64)
    tick = 0
    for e in np.flatnonzero(mask):  # initial residents touched in id order
        tick += 1
        last[e] = tick
    for i in range(20000):
        e = int(rng.integers(E)) if i % 3 else int(rng.integers(8))
        log = []
        M.access(st, e, clock, cost, log=log)
        if not mask[e]:
            res = np.flatnonzero(mask)
            v = int(res[np.argmin(last[res])])
            assert [x.kind for x in log] == ["miss_ondemand", "evict"] and log[1].expert == v
            mask[v] = False
            mask[e] = True
        tick += 1
        last[e] = tick
    assert np.array_equal(st.mask, mask)


def test_policy_errors():
    with pytest.raises(ConfigurationError):
        M.ResidencyState(8, 9, "lru")
    with pytest.raises(ConfigurationError):
        M.ResidencyState(8, 4, "mru")
    with pytest.raises(ConfigurationError):
        M.ResidencyState(8, 4, "freq_static")
    st = M.ResidencyState(8, 4, "lru")
    with pytest.raises(InputError):
        M.access(st, 99, M.SimClock(), M.CostModel())
    with pytest.raises(InvariantViolation):
        M.SimClock().advance(-1.0)


def test_nesting_across_capacities():
    # initial contents nest across c for one seed (memtier.py:132-137)
    prev = set()
    for c in (0.25, 0.5, 0.75):
        cur = set(np.flatnonzero(M.init_residency(64, c, "lru", seed=3).mask))
        assert prev <= cur
        prev = cur


def test_random_plan_host_replica_equals_numpy_stream():
    """bm_random_plan (C++ PCG64 + Lemire bounded draws) makes the draws of
    numpy's Generator.integers (the reference's random_plan,
    substitution.py:227-248): plans equal the oracle's on shared seeds, and the
    generator state handed back equals the one numpy reaches."""
    import ctypes
    import oracle as O
    from paper_2511_10054_b200 import _native as N
    rng = np.random.default_rng(5)
    for case in range(300):
        E = int(rng.choice([4, 8, 33, 64, 128, 160]))
        k = int(rng.integers(1, min(8, E) + 1))
        B = int(rng.integers(1, 17))
        topk = np.stack([rng.permutation(E)[:k] for _ in range(B)]).astype(np.int32)
        mask = rng.random(E) < rng.random()
        seed = int(rng.integers(0, 2**31))
        ga = np.random.default_rng(np.random.SeedSequence([seed, 31]))
        gb = np.random.default_rng(np.random.SeedSequence([seed, 31]))
        if case % 4 == 1:  # leave a buffered 32-bit half in both
            ga.integers(0, 7), gb.integers(0, 7)
        ex_r, kd_r, used_r = O.random_plan(topk, mask, ga)
        st = N.Pcg64State.from_generator(gb)
        ex = np.empty((B, k), np.int32)
        kd = np.empty((B, k), np.uint8)
        used = np.empty(B, np.int32)
        m8 = mask.astype(np.uint8)
        N.call("bm_random_plan", topk.ctypes.data, B, k, m8.ctypes.data, E, ctypes.byref(st), ex.ctypes.data,
               kd.ctypes.data, used.ctypes.data)
        st.store_into(gb)
        assert np.array_equal(ex, ex_r) and np.array_equal(kd, kd_r) and np.array_equal(used, used_r), case
        assert ga.bit_generator.state == gb.bit_generator.state, case


def test_random_plan_api_matches_reference_semantics():
    """substitution.random_plan over the C-ABI advances the caller's numpy
    generator exactly like the reference function does."""
    from paper_2511_10054_b200.model import RouterDecision
    from paper_2511_10054_b200.substitution import random_plan
    import oracle as O
    g1 = np.random.default_rng(np.random.SeedSequence([3, 31]))
    g2 = np.random.default_rng(np.random.SeedSequence([3, 31]))
    mask = np.array([1, 0, 1, 0, 1, 1, 0, 0], bool)
    for t in range(50):
        topk = np.array([(t * 3) % 8, (t * 5 + 1) % 8 if (t * 5 + 1) % 8 != (t * 3) % 8 else (t * 5 + 2) % 8])
        d = RouterDecision(token=t, layer=0, logits=np.zeros(8), topk=topk, probs_renorm=np.array([0.6, 0.4]),
                           temperature=1.0)
        p = random_plan(d, mask, g1)
        ex, kd, used = O.random_plan(topk[None], mask, g2)
        assert [s.executed for s in p.slots] == list(ex[0]) and p.replacements_used == int(used[0])
    assert g1.bit_generator.state == g2.bit_generator.state
