"""ctypes binding of libbmoe.so (include/bmoe.h).

There is no CPU fallback: if the library is missing or fails to load, every
product entry point raises NativeLibraryError. ``build()`` in
__graft_entry__.py (or ``python -m paper_2511_10054_b200.build``) produces it.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeLibraryError, raise_for

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libbmoe.so")

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
F64 = C.c_double
F32 = C.c_float


class Event(C.Structure):
    _fields_ = [("time_ms", C.c_double), ("kind", C.c_int32), ("layer", C.c_int32), ("token", C.c_int32),
                ("expert", C.c_int32), ("bytes", C.c_int64), ("stall_ms", C.c_double)]


class Pcg64State(C.Structure):
    """numpy's PCG64 bit-generator state (bm_pcg64)."""
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64), ("inc_hi", C.c_uint64), ("inc_lo", C.c_uint64),
                ("has_uint32", C.c_int32), ("uinteger", C.c_uint32)]

    @classmethod
    def from_generator(cls, rng) -> "Pcg64State":
        st = rng.bit_generator.state
        if st["bit_generator"] != "PCG64":
            raise TypeError(f"need a PCG64 generator, got {st['bit_generator']}")
        s, inc = st["state"]["state"], st["state"]["inc"]
        m = (1 << 64) - 1
        return cls(s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"]))

    def store_into(self, rng) -> None:
        """Write the advanced state back, so the numpy generator continues the same stream."""
        rng.bit_generator.state = {"bit_generator": "PCG64",
                                   "state": {"state": (self.state_hi << 64) | self.state_lo,
                                             "inc": (self.inc_hi << 64) | self.inc_lo},
                                   "has_uint32": int(self.has_uint32), "uinteger": int(self.uinteger)}


class BetaState(C.Structure):
    """bm_beta_state (adaptive distribution-gate beta)."""
    _fields_ = [("budget_bytes", C.c_double), ("expert_bytes", C.c_double), ("beta", C.c_double),
                ("decay", C.c_double), ("period", C.c_int64), ("steps", C.c_int64), ("n_grid", C.c_int32),
                ("pad_", C.c_int32), ("grid", C.c_double * 64), ("ema", C.c_double * 64)]


class EngineConfig(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_experts", C.c_int32), ("top_k", C.c_int32), ("d", C.c_int32),
                ("f", C.c_int32), ("act", C.c_int32), ("max_batch", C.c_int32), ("capacity", C.c_int32),
                ("staging", C.c_int32), ("method", C.c_int32), ("policy", C.c_int32),
                ("search_rank_h", C.c_int32), ("fallback", C.c_int32), ("prefetch_enabled", C.c_int32),
                ("n_tile", C.c_int32), ("fp32_weights", C.c_int32), ("rho", C.c_int64), ("beta", C.c_double),
                ("temperature", C.c_double), ("gamma", C.c_double), ("load_ms", C.c_double),
                ("hit_ms", C.c_double), ("compute_ms", C.c_double), ("prefetch_ms", C.c_double),
                ("expert_bytes", C.c_int64), ("num_shared", C.c_int32), ("fetch_codec", C.c_int32),
                ("pcie_budget_bytes", C.c_double), ("rng", Pcg64State), ("beta_wire_bytes", C.c_int32)]


class EngineStats(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("executed_slots", C.c_int64), ("ondemand_misses", C.c_int64),
                ("substitutions", C.c_int64), ("drops", C.c_int64), ("physical_fetches", C.c_int64),
                ("prefetch_copies", C.c_int64), ("h2d_bytes", C.c_int64), ("gate_forbidden", C.c_int64),
                ("batch_bypassed", C.c_int64), ("ffn_calls", C.c_int64), ("ffn_experts", C.c_int64),
                ("ffn_rows", C.c_int64), ("sim_now_ms", C.c_double), ("stall_ms", C.c_double),
                ("copy_ms", C.c_double), ("kernel_launches", C.c_int64), ("wire_bytes", C.c_int64),
                ("beta", C.c_double), ("inflight_releases", C.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


_SIGS = {
    "bm_engine_create": (C.c_int, [P, P, P, P, P, P, I32, P, P, P, P]),
    "bm_engine_destroy": (None, [P]),
    "bm_engine_step": (C.c_int, [P, P, I64, P, P]),
    "bm_engine_stats_get": (C.c_int, [P, P, I32]),
    "bm_engine_cache": (P, [P]),
    "bm_engine_set_trace": (C.c_int, [P, I32]),
    "bm_engine_set_copy_timing": (C.c_int, [P, I32]),
    "bm_engine_trace_size": (C.c_int, [P, P, P]),
    "bm_engine_trace_get": (C.c_int, [P, P, P, P, P, P, P, P, P]),
    "bm_engine_device_bytes": (I64, [P]),
    "bm_engine_trace_gates": (C.c_int, [P, P, P, P]),
    "bm_engine_set_psi": (C.c_int, [P, P, F64, F64, I32, P, F64]),
    "bm_host_alloc": (C.c_int, [I64, P]),
    "bm_host_free": (C.c_int, [P]),
    "bm_host_register": (C.c_int, [P, I64, I32]),
    "bm_host_unregister": (C.c_int, [P]),
    "bm_memcpy": (C.c_int, [P, P, I64, P]),
    "bm_xfer_blob_bound": (I64, [I64]),
    "bm_xfer_encode": (C.c_int, [P, I64, P, I64, P, P]),
    "bm_xfer_decode": (C.c_int, [P, P, I64, P]),
    "bm_xfer_decode_piece": (C.c_int, [P, P, I64, P]),
    "bm_xfer_decode_piece_ctas": (C.c_int, [P, P, I64, I32, P]),
    "bm_abi_version": (C.c_int, []),
    "bm_last_error": (C.c_char_p, []),
    "bm_device_sm_count": (C.c_int, []),
    "bm_gate_topk": (C.c_int, [P, P, P, I64, I64, I64, I64, F64, F64, F64, P, P, P, P, P, P, P]),
    "bm_select_topk_f64": (C.c_int, [P, I64, I64, I64, F64, F64, F64, P, P, P, P, P, P, P]),
    "bm_buddy_remap": (C.c_int, [P, P, P, I32, I64, I64, I64, P, P, P, P, I64, I64, I64, I32, I32, F64, F64, F64,
                                 I32, P, F64, P, P, P, P, P, P]),
    "bm_derive_beta": (C.c_int, [F64, F64, P, P, I32, F64, P]),
    "bm_beta_init": (C.c_int, [P, F64, F64, F64, P, I32, F64, I64]),
    "bm_beta_record": (C.c_int, [P, F64, I64, P]),
    "bm_random_plan": (C.c_int, [P, I64, I64, P, I64, P, P, P, P]),
    "bm_pcg64_integers": (C.c_int, [P, I64, I64, P]),
    "bm_synth_bf16": (C.c_int, [P, C.c_uint64, I64, P, P]),
    "bm_synth_mix_bf16": (C.c_int, [P, C.c_uint64, C.c_uint64, F32, I64, P, P]),
    "bm_permute_rows_max": (I64, [I64, I64, I64, I64]),
    "bm_append_shared": (C.c_int, [P, P, P, I64, I64, I64, I64, P, P, P, P]),
    "bm_split_counts": (C.c_int, [P, P, I64, P, P, P]),
    "bm_permute": (C.c_int, [P, P, I64, I64, I64, I64, P, P, P, P, P]),
    "bm_permute_scratch_elems": (C.c_int, [I64, I64, I64]),
    "bm_permute_ws": (C.c_int, [P, P, I64, I64, I64, I64, P, P, P, P, P, I64, P]),
    "bm_gather_rows": (C.c_int, [P, I64, I64, P, P, I64, I64, I32, P, P]),
    "bm_combine": (C.c_int, [P, P, P, P, I64, I64, I64, P, F32, P, P]),
    "bm_expert_ffn_f32": (C.c_int, [P, P, P, I64, I64, I64, I32, P, I64, P, I64, P, P, P]),
    "bm_expert_ffn_f64": (C.c_int, [P, P, P, I64, I64, I64, I32, P, I64, P, I64, P, P, P]),
    "bm_gather_rows_f64": (C.c_int, [P, I64, I64, P, P, I64, I64, P, P]),
    "bm_combine_f64": (C.c_int, [P, P, P, P, I64, I64, I64, P, F64, P, P]),
    "bm_pack_expert_bf16": (C.c_int, [P, P, P, I64, I64, I32, P, P]),
    "bm_expert_ffn_bf16_workspace": (I64, [I64, I64, I64, I64, I64]),
    "bm_expert_ffn_bf16": (C.c_int, [P, P, P, I64, I64, I64, I32, P, I64, P, I64, I64, P, I64, P, P]),
    "bm_expert_ffn_bf16_combine": (C.c_int, [P, P, P, I64, I64, I64, I32, P, I64, P, I64, I64, P, I64, P,
                                             P, P, P, I64, I64, P, F32, P]),
    "bm_set_kernel_timing": (C.c_int, [I32]),
    "bm_ffn_trace_read": (C.c_int64, [P, I64]),
    "bm_kernel_times": (I64, [P, I64]),
    "bm_kernel_spans": (I64, [P, I64]),
    "bm_kernel_timing_enabled": (C.c_int, []),
    "bm_coact_count": (C.c_int, [P, I64, I64, I64, P, P, P, P]),
    "bm_coact_weighted": (C.c_int, [P, P, I64, I64, I64, F64, P, P]),
    "bm_counts_to_f64": (C.c_int, [P, P, I64, F64, P, P]),
    "bm_buddy_rank": (C.c_int, [P, I64, F64, F64, I64, P, P, P, P]),
    "bm_conditional_rows": (C.c_int, [P, I64, F64, P, P, P]),
    "bm_cft_prefix": (C.c_int, [P, I64, I64, F64, P, P, P, P]),
    "bm_gate_from_probs": (C.c_int, [P, I64, I64, F64, F64, P, P, P, P]),
    "bm_distribution_gate": (C.c_int, [P, I64, P, F64, P, P, P]),
    "bm_cache_create": (C.c_int, [I32, I32, I32, I32, P, P, F64, F64, F64, I64, P]),
    "bm_cache_destroy": (None, [P]),
    "bm_cache_access": (C.c_int, [P, I32, I32, I32, I32, P]),
    "bm_cache_apply_plan": (C.c_int, [P, I32, I64, I64, P, P, P, P, P]),
    "bm_cache_prefetch": (C.c_int, [P, I32, P, I64]),
    "bm_cache_settle": (C.c_int, [P, I32]),
    "bm_cache_advance": (C.c_int, [P, F64]),
    "bm_cache_now": (C.c_int, [P, P]),
    "bm_cache_snapshot": (C.c_int, [P, I32, P, P]),
    "bm_cache_predict": (C.c_int, [P, I32, P, P, P]),
    "bm_cache_num_events": (I64, [P]),
    "bm_cache_events": (C.c_int, [P, I64, I64, P]),
    "bm_cache_clear_events": (None, [P]),
    "bm_cache_layer_state": (C.c_int, [P, I32, P, P, P]),
    "bm_cache_pending": (C.c_int, [P, I32, P, P, I64]),
    "bm_cache_set_clock": (C.c_int, [P, F64, F64]),
    "bm_cache_get_clock": (C.c_int, [P, P, P]),
    "bm_cache_set_costs": (C.c_int, [P, F64, F64, F64, I64]),
    "bm_cache_insert": (C.c_int, [P, I32, I32, I32, P]),
}

_lib = None


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """The loaded library; raises NativeLibraryError if it is unavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise NativeLibraryError(
                f"{_LIB_PATH} not built; run `python -m paper_2511_10054_b200.build` (no CPU fallback exists)")
        try:
            h = C.CDLL(_LIB_PATH)
        except OSError as e:  # pragma: no cover - environment specific
            raise NativeLibraryError(f"cannot load {_LIB_PATH}: {e}") from e
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name, None)
            if fn is None:
                raise NativeLibraryError(f"{_LIB_PATH} does not export {name}")
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def exported_symbols():
    return list(_SIGS)


def call(name: str, *args) -> int:
    """Call an int-returning ABI function and raise the mapped exception on error."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        raise_for(rc, f"{name}: {lib().bm_last_error().decode(errors='replace')}")
    return rc
