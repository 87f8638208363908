"""Offloaded decode engine: Python handle over bm_engine (include/bmoe.h).

``DecodeEngine.step(h, tokens)`` is one decode step through every layer —
the tensor form of the reference's run_simulation inner loop
(harness.py:315-393) — with a real expert cache: HBM buffers under a
capacity budget, pinned-host fetches on copy streams, and the exact
memtier replica deciding hits, misses, evictions and prefetches.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .errors import ConfigurationError
from .ops import ACT_SWIGLU, FALLBACK_PREFETCH, METHOD_BUDDY

POLICIES = {"lru": 0, "lfu": 1, "freq_static": 2}
METHODS = {"buddy": 0, "original": 1, "identity": 2, "random": 3}
_RNG_TAG_RANDOM_METHOD = 31  # harness.py:44: the Random arm's stream is SeedSequence([run.seed, 31])


class HostMirror:
    """Pinned host memory holding every expert of one layer in the arena
    layout (cudaHostAlloc of the exact size, not torch's power-of-two pool)."""

    codec = 0  # 0: raw expert buffers back to back; 1: exponent-coded layer image

    def __init__(self, nbytes: int):
        ptr = C.c_void_p()
        N.call("bm_host_alloc", int(nbytes), C.byref(ptr))
        self.ptr = ptr.value
        self.nbytes = int(nbytes)

    def as_tensor(self, dtype=torch.uint8) -> torch.Tensor:
        buf = (C.c_uint8 * self.nbytes).from_address(self.ptr)
        return torch.frombuffer(buf, dtype=torch.uint8).view(dtype)

    def close(self):
        if self.ptr:
            N.lib().bm_host_free(self.ptr)
            self.ptr = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def fill_mirror_from_device(mirror: HostMirror, src: torch.Tensor, offset: int = 0):
    """Synchronous device -> pinned host copy into the mirror at a byte offset."""
    n = src.numel() * src.element_size()
    s = torch.cuda.current_stream()
    N.call("bm_memcpy", mirror.ptr + offset, src.data_ptr(), n, s.cuda_stream)
    s.synchronize()


class SharedMirror:
    """A layer mirror in a shared-memory file (``/dev/shm``) that every
    replica process on the node maps and page-locks (bm_host_register), so N
    replicas of one model hold ONE host copy of the experts instead of N.
    The owner (local rank 0) creates and fills it; the others attach
    read-only after a barrier. Same interface as HostMirror (ptr, nbytes,
    codec, close)."""

    def __init__(self, path: str, nbytes: int = 0, create: bool = False, register: bool = True):
        import mmap
        import os
        self.path, self.owner, self.registered = path, create, False
        fd = os.open(path, os.O_RDWR | (os.O_CREAT | os.O_TRUNC if create else 0), 0o600)
        try:
            if create:
                os.ftruncate(fd, int(nbytes))
            else:
                nbytes = os.fstat(fd).st_size
            self._mm = mmap.mmap(fd, int(nbytes), mmap.MAP_SHARED, mmap.PROT_READ | mmap.PROT_WRITE)
        finally:
            os.close(fd)
        self._buf = (C.c_char * int(nbytes)).from_buffer(self._mm)
        self.ptr = C.addressof(self._buf)
        self.nbytes = int(nbytes)
        self.codec = 1 if (not create and self.nbytes >= 4 and bytes(self._buf[:4]) == b"BXL1") else 0
        if register:
            N.call("bm_host_register", self.ptr, self.nbytes, 0 if create else 1)
            self.registered = True

    def as_tensor(self, dtype=torch.uint8) -> torch.Tensor:
        return torch.frombuffer(self._buf, dtype=torch.uint8).view(dtype)

    def unlink(self):
        """Remove the file name; the mappings stay valid until every process
        closes them (the kernel frees the pages then, even after a crash)."""
        import os
        if self.owner:
            try:
                os.unlink(self.path)
            except OSError:
                pass
            self.owner = False

    def close(self):
        import os
        if getattr(self, "_mm", None) is None:
            return
        if self.registered:
            N.lib().bm_host_unregister(self.ptr)
            self.registered = False
        self.ptr = None
        del self._buf
        self._mm.close()
        self._mm = None
        if self.owner:
            try:
                os.unlink(self.path)
            except OSError:
                pass

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def coded_mirror_from_device(arena: torch.Tensor, make_mirror=HostMirror):
    """Pinned host layer image of every expert of ``arena`` [count, elems]
    (bf16, device) in the exponent-coded transfer format: a
    bm_xfer_layer_header followed by one blob per expert (include/bmoe.h).
    The engine fetches it piece by piece and rebuilds the exact bf16 bytes
    in HBM, so fewer bytes cross PCIe per miss. ``make_mirror(nbytes)``
    allocates the host side (HostMirror, or a SharedMirror for replicas)."""
    from . import ops
    count, elems = arena.shape
    blobs = [ops.xfer_encode(arena[e]) for e in range(count)]
    head = 256 * ((24 + 8 * (count + 1) + 255) // 256)
    offs = [head]
    for b in blobs:
        offs.append(offs[-1] + 256 * ((b.numel() + 255) // 256))
    m = make_mirror(offs[-1])
    m.codec = 1
    hdr = np.zeros(head // 8, np.uint64)
    hdr[0] = np.uint64(0x314C5842 | (count << 32))  # magic "BXL1", count
    hdr[1] = np.uint64(elems * 2)
    hdr[2:3 + count] = np.asarray(offs, np.uint64)
    C.memmove(m.ptr, hdr.ctypes.data, head)
    s = torch.cuda.current_stream()
    for b, o in zip(blobs, offs):
        N.call("bm_memcpy", m.ptr + o, b.data_ptr(), b.numel(), s.cuda_stream)
    s.synchronize()
    return m


def mirror_expert(mirror: HostMirror, e: int, elems: int, device="cuda") -> torch.Tensor:
    """Expert e of a layer mirror as a bf16 device tensor [elems] (decoded
    when the mirror is coded) — for checks and the CPU reference legs."""
    from . import ops
    if mirror.codec == 0:
        raw = mirror.as_tensor(torch.bfloat16)[e * elems:(e + 1) * elems]
        return raw.to(device)
    words = (C.c_uint64 * (4 + e)).from_address(mirror.ptr)  # magic|count, raw_bytes, blob_off[...]
    lo, hi = int(words[2 + e]), int(words[3 + e])
    blob = torch.empty(hi - lo + 256, dtype=torch.uint8, device=device)
    off = (-blob.data_ptr()) % 256
    blob = blob[off:off + hi - lo]
    s = torch.cuda.current_stream()
    N.call("bm_memcpy", blob.data_ptr(), mirror.ptr + lo, hi - lo, s.cuda_stream)
    return ops.xfer_decode(blob, elems)


@dataclass
class EngineSpec:
    num_layers: int
    num_experts: int
    top_k: int
    d: int
    f: int
    capacity: int
    max_batch: int
    act: int = ACT_SWIGLU
    method: str = "buddy"
    policy: str = "lru"
    search_rank_h: int = 16
    rho: int | None = None
    fallback: int = FALLBACK_PREFETCH
    beta: float = 1.0
    temperature: float = 1.0
    gamma: float | None = None
    prefetch: bool = True
    n_tile: int = 128  # widest token tile; decode batches use min(B rounded to 16, n_tile)
    fp32_weights: bool = False
    staging: int = 0
    load_ms: float = 9.5
    hit_ms: float = 0.0
    compute_ms: float = 0.5
    prefetch_ms: float | None = None
    pcie_bw_bytes_per_s: float = 4.0e6
    expert_bytes: int | None = None
    num_shared: int = 0
    fetch_codec: int | None = None  # None: the mirrors' format (HostMirror.codec)
    pcie_budget_bytes: float | None = None  # adaptive beta (gating.BetaController) when set
    beta_bytes: str = "logical"  # adaptive beta prices a miss at expert_bytes ("logical", the reference's
    #                             cost model) or at the measured mean wire bytes of a fetch ("wire")
    run_seed: int = 0  # method "random": the plan stream of harness.py:299-300

    @property
    def buf_elems(self) -> int:
        return (3 if self.act == ACT_SWIGLU else 2) * self.d * self.f

    @property
    def buf_bytes(self) -> int:
        return self.buf_elems * (4 if self.fp32_weights else 2)


class DecodeEngine:
    def __init__(self, spec: EngineSpec, mirrors, gate_w: torch.Tensor, gate_b: torch.Tensor,
                 tbl_ids: torch.Tensor | None, tbl_len: torch.Tensor | None, taus, initial,
                 static_freq=None):
        if spec.method not in METHODS or spec.policy not in POLICIES:
            raise ConfigurationError(f"unknown method/policy {spec.method}/{spec.policy}")
        self.spec = spec
        self.mirrors = mirrors  # keep alive
        self.gate_w = gate_w.contiguous()
        self.gate_b = gate_b.contiguous()
        self.tbl_ids = None if tbl_ids is None else tbl_ids.contiguous()
        self.tbl_len = None if tbl_len is None else tbl_len.contiguous()
        cfg = N.EngineConfig()
        cfg.num_layers, cfg.num_experts, cfg.top_k = spec.num_layers, spec.num_experts, spec.top_k
        cfg.d, cfg.f, cfg.act = spec.d, spec.f, spec.act
        cfg.max_batch, cfg.capacity, cfg.staging = spec.max_batch, spec.capacity, spec.staging
        cfg.method, cfg.policy = METHODS[spec.method], POLICIES[spec.policy]
        cfg.search_rank_h, cfg.fallback = spec.search_rank_h, spec.fallback
        cfg.prefetch_enabled, cfg.n_tile = int(spec.prefetch), spec.n_tile
        cfg.fp32_weights = int(spec.fp32_weights)
        cfg.rho = -1 if spec.rho is None else int(spec.rho)
        cfg.beta, cfg.temperature = spec.beta, spec.temperature
        cfg.gamma = -1.0 if spec.gamma is None else spec.gamma
        ebytes = spec.expert_bytes if spec.expert_bytes is not None else spec.buf_bytes
        cfg.load_ms, cfg.hit_ms, cfg.compute_ms = spec.load_ms, spec.hit_ms, spec.compute_ms
        cfg.prefetch_ms = spec.prefetch_ms if spec.prefetch_ms is not None else \
            1000.0 * ebytes / spec.pcie_bw_bytes_per_s
        cfg.expert_bytes = ebytes
        cfg.num_shared = int(spec.num_shared)
        cfg.pcie_budget_bytes = -1.0 if spec.pcie_budget_bytes is None else float(spec.pcie_budget_bytes)
        if spec.beta_bytes not in ("logical", "wire"):
            raise ConfigurationError(f"beta_bytes must be 'logical' or 'wire', got {spec.beta_bytes!r}")
        cfg.beta_wire_bytes = int(spec.beta_bytes == "wire")
        cfg.rng = N.Pcg64State.from_generator(
            np.random.default_rng(np.random.SeedSequence([int(spec.run_seed), _RNG_TAG_RANDOM_METHOD])))
        cfg.fetch_codec = int(spec.fetch_codec if spec.fetch_codec is not None else getattr(mirrors[0], "codec", 0))
        L, E = spec.num_layers, spec.num_experts
        ptrs = (C.c_void_p * L)(*[m.ptr for m in mirrors])
        tau = (C.c_double * L)(*[(-1.0 if t is None else float(t)) for t in taus])
        cap = max(spec.capacity, 1)
        init = np.full((L, cap), -1, np.int32)
        for l, row in enumerate(initial):
            init[l, :len(row)] = row
        sf = None
        if static_freq is not None:
            sf = np.ascontiguousarray(np.asarray(static_freq, np.float64).reshape(L, E))
        h = C.c_void_p()
        N.call("bm_engine_create", C.byref(cfg), ptrs, self.gate_w.data_ptr(), self.gate_b.data_ptr(),
               None if self.tbl_ids is None else self.tbl_ids.data_ptr(),
               None if self.tbl_len is None else self.tbl_len.data_ptr(),
               0 if self.tbl_ids is None else int(self.tbl_ids.shape[-1]),
               tau, init.ctypes.data, None if sf is None else sf.ctypes.data, C.byref(h))
        self._h = h.value
        self._cfg = cfg

    def step(self, h: torch.Tensor, tokens) -> torch.Tensor:
        """One decode step (all layers) on h [B,d] fp32, in place."""
        B = h.shape[0]
        tok = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        N.call("bm_engine_step", self._h, h.data_ptr(), B, tok.ctypes.data, torch.cuda.current_stream().cuda_stream)
        return h

    def stats(self, reset: bool = False) -> dict:
        st = N.EngineStats()
        N.call("bm_engine_stats_get", self._h, C.byref(st), int(reset))
        return st.as_dict()

    def device_bytes(self) -> int:
        return int(N.lib().bm_engine_device_bytes(self._h))

    def events(self, start: int = 0):
        """The control plane's event log from index ``start`` on, in log order, as
        an [n,7] float64 array (time, kind, layer, token, expert, bytes, stall)."""
        c = N.lib().bm_engine_cache(self._h)
        n = max(0, int(N.lib().bm_cache_num_events(c)) - start)
        arr = (N.Event * max(n, 1))()
        if n:
            N.call("bm_cache_events", c, start, n, arr)
        return np.array([(e.time_ms, e.kind, e.layer, e.token, e.expert, e.bytes, e.stall_ms) for e in arr[:n]],
                        dtype=np.float64).reshape(-1, 7)

    def set_psi(self, tbl_w: torch.Tensor | None, eta: float = 0.0, kappa: float = 0.0, use_local_logit: bool = True,
                partition_of: torch.Tensor | None = None, hop: float = 1.0):
        """Psi candidate ordering in the remap (substitution.py:107-143): tbl_w
        [L,E,K] f64 device weights of the buddy table, partition_of [E] int32."""
        self._psi_keep = (tbl_w, partition_of)
        N.call("bm_engine_set_psi", self._h, None if tbl_w is None else tbl_w.data_ptr(), float(eta), float(kappa),
               int(bool(use_local_logit)), None if partition_of is None else partition_of.data_ptr(), float(hop))

    def raw_events(self):
        """The control plane's event log in log order (not time-sorted)."""
        return self.events()

    def set_copy_timing(self, enable: bool = True):
        """Time each fetch's copies (stats()["copy_ms"]); costs ~6 us of copy engine per fetch."""
        N.call("bm_engine_set_copy_timing", self._h, int(enable))

    def set_trace(self, enable: bool = True):
        N.call("bm_engine_set_trace", self._h, int(enable))

    def trace(self) -> list:
        """Per layer-step records: dict(layer, bitmap, batch_ok, topk, allowed, executed, kind)."""
        nr, nt = C.c_int64(), C.c_int64()
        N.call("bm_engine_trace_size", self._h, C.byref(nr), C.byref(nt))
        nr, nt = nr.value, nt.value
        k, words = self.spec.top_k, (self.spec.num_experts + 31) // 32
        lay = np.zeros(max(nr, 1), np.int32)
        Bs = np.zeros(max(nr, 1), np.int32)
        bms = np.zeros(max(nr, 1) * words, np.uint32)
        bok = np.zeros(max(nr, 1), np.uint8)
        tk = np.zeros(max(nt, 1) * k, np.int32)
        al = np.zeros(max(nt, 1), np.uint8)
        ex = np.zeros(max(nt, 1) * k, np.int32)
        kd = np.zeros(max(nt, 1) * k, np.uint8)
        N.call("bm_engine_trace_get", self._h, lay.ctypes.data, Bs.ctypes.data, bms.ctypes.data, bok.ctypes.data,
               tk.ctypes.data, al.ctypes.data, ex.ctypes.data, kd.ctypes.data)
        tae = np.zeros(max(nt, 1))
        mar = np.zeros(max(nt, 1))
        dl = np.zeros(max(nr, 1))
        N.call("bm_engine_trace_gates", self._h, tae.ctypes.data, mar.ctypes.data, dl.ctypes.data)
        out, t0 = [], 0
        for i in range(nr):
            B = int(Bs[i])
            bits = bms[i * words:(i + 1) * words]
            mask = np.array([(bits[e >> 5] >> (e & 31)) & 1 for e in range(self.spec.num_experts)], bool)
            out.append(dict(layer=int(lay[i]), mask=mask, batch_ok=bool(bok[i]),
                            topk=tk[t0 * k:(t0 + B) * k].reshape(B, k), allowed=al[t0:t0 + B].astype(bool),
                            executed=ex[t0 * k:(t0 + B) * k].reshape(B, k), kind=kd[t0 * k:(t0 + B) * k].reshape(B, k),
                            tae=tae[t0:t0 + B].copy(), margin=mar[t0:t0 + B].copy(), delta=float(dl[i])))
            t0 += B
        return out

    def finish(self):
        """Commit every in-flight transfer whose time has come, all layers —
        the reference's end-of-run settle (harness.py:395-396)."""
        c = N.lib().bm_engine_cache(self._h)
        for l in range(self.spec.num_layers):
            N.call("bm_cache_settle", c, l)

    def sorted_events(self):
        """Event log ordered by time, ties in log order (harness.py:397)."""
        ev = self.events()
        return ev[np.argsort(ev[:, 0], kind="stable")] if len(ev) else ev

    def snapshot(self, layer: int) -> np.ndarray:
        c = N.lib().bm_engine_cache(self._h)
        m = np.zeros(self.spec.num_experts, np.uint8)
        N.call("bm_cache_snapshot", c, layer, m.ctypes.data, None)
        return m.astype(bool)

    def close(self):
        if getattr(self, "_h", None):
            N.lib().bm_engine_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
