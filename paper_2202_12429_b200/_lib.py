"""ctypes binding of libbagpipe_b200.so (the C ABI of include/bagpipe_b200.h).

There is deliberately no fallback: if the library is missing or no CUDA device
is visible, :func:`lib` raises :class:`NativeUnavailable`.  Every hot-path call
of the package goes through these symbols.

PyTorch supplies device memory (CUDA tensors), streams and pinned host
buffers; the library receives raw pointers only.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import errors as E
from .traces import EmbeddingKey, unpack_key

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_native", "libbagpipe_b200.so")


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built or no GPU is present (no CPU fallback exists)."""


c_i32, c_i64, c_u64, c_f32, c_vp = C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_void_p


class ErrorT(C.Structure):
    _fields_ = [("code", c_i32), ("lock", c_i32), ("iteration", c_i64), ("index", c_i64), ("key", c_u64)]


class PrepView(C.Structure):
    _fields_ = [
        ("n_occ", c_i64), ("iteration", c_i64), ("num_ranks", c_i32), ("pad", c_i32),
        ("d_num_unique", c_vp), ("d_uniq_key_s", c_vp), ("d_uniq_id_s", c_vp), ("d_uniq_key_k", c_vp),
        ("d_perm_s2k", c_vp), ("d_perm_k2s", c_vp), ("d_seg_start", c_vp), ("d_occ_pos", c_vp),
        ("d_occ_label", c_vp), ("d_occ_k", c_vp), ("d_rank_bounds", c_vp),
    ]


class PlanBuffers(C.Structure):
    _fields_ = [
        ("d_prefetch_keys", c_vp), ("d_prefetch_ids", c_vp), ("d_prefetch_ttls", c_vp), ("d_ttl_k", c_vp),
        ("d_evict_keys", c_vp), ("d_evict_ids", c_vp), ("d_counts", c_vp),
    ]


class PlannerStats(C.Structure):
    _fields_ = [(n, c_i64) for n in (
        "tracked", "in_cache", "insertions", "removals", "peak_occupancy", "peak_projected",
        "last_projected", "last_prefetch", "last_evict", "registry_size")]


class CacheStats(C.Structure):
    _fields_ = [(n, c_i64) for n in ("occupancy", "insertions", "evictions", "peak_occupancy", "capacity",
                                     "registry_size")]


class EvictBuffers(C.Structure):
    _fields_ = [("d_keys", c_vp), ("d_ids", c_vp), ("d_rows", c_vp), ("d_dirty", c_vp), ("d_count", c_vp)]


class CacheView(C.Structure):
    _fields_ = [("capacity", c_i64), ("dim", c_i32), ("pad", c_i32), ("d_values", c_vp), ("d_ttl", c_vp),
                ("d_dirty", c_vp), ("d_used", c_vp), ("d_slot_key", c_vp)]


class PlannerDump(C.Structure):
    _fields_ = [("d_keys", c_vp), ("d_last", c_vp), ("d_flags", c_vp), ("d_count", c_vp)]


class EngineConfig(C.Structure):
    _fields_ = [("capacity", c_i64), ("max_occ", c_i64), ("seed", c_u64), ("dim", c_i32), ("num_ranks", c_i32),
                ("c_value", c_f32), ("c_label", c_f32), ("lr", c_f32), ("record_keys", c_i32),
                ("plan_slots", c_i32), ("chunk_slots", c_i32), ("prep_slots", c_i32), ("timing", c_i32),
                ("init_dims", c_i32), ("prep_flags", c_i32)]


class StepResult(C.Structure):
    _fields_ = [(n, c_i64) for n in ("unique", "inserted", "critical", "dirty_keys", "evicted", "evicted_dirty",
                                     "drained", "drained_dirty")] + [("err", ErrorT)]


class PeerXchg(C.Structure):  # bp_peer_xchg
    _fields_ = [("world", c_i32), ("rank", c_i32), ("bl", c_i64), ("t_global", c_i32), ("n_cols", c_i32),
                ("d_col_tables", c_vp), ("d_peer_rows", c_vp), ("d_peer_flags", c_vp), ("d_flags", c_vp)]


SGD_MAX_TENSORS = 32


class SgdTensors(C.Structure):  # bp_sgd_tensors
    _fields_ = [("n", c_i32), ("pad", c_i32), ("master", c_vp * SGD_MAX_TENSORS), ("lowp", c_vp * SGD_MAX_TENSORS),
                ("grad", c_vp * SGD_MAX_TENSORS), ("numel", c_i64 * SGD_MAX_TENSORS)]


class EngineParts(C.Structure):
    _fields_ = [("store", c_vp), ("cache", c_vp), ("planner", c_vp), ("compute_stream", c_vp),
                ("link_stream", c_vp)]


P = C.POINTER
_SIGS = {
    "bp_version": (C.c_char_p, []),
    "bp_abi_sizeof": (c_i64, [c_i32]),
    "bp_last_error_message": (C.c_char_p, []),
    "bp_ctx_create": (c_i32, [P(c_vp)]),
    "bp_ctx_destroy": (c_i32, [c_vp]),
    "bp_ctx_check": (c_i32, [c_vp, c_vp, P(ErrorT)]),
    "bp_schema_create": (c_i32, [c_i32, c_vp, c_i32, P(c_vp)]),
    "bp_schema_destroy": (c_i32, [c_vp]),
    "bp_schema_total_rows": (c_i64, [c_vp]),
    "bp_schema_ids": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bp_prep_create": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_vp,
                               P(c_vp)]),
    "bp_prep_destroy": (c_i32, [c_vp]),
    "bp_prep_get_view": (c_i32, [c_vp, P(PrepView)]),
    "bp_prep_num_unique": (c_i32, [c_vp, c_vp, P(c_i64)]),
    "bp_prep_key_rows": (c_i32, [c_vp, c_vp, c_vp]),
    "bp_planner_create": (c_i32, [c_vp, c_vp, c_i64, P(c_vp)]),
    "bp_planner_destroy": (c_i32, [c_vp]),
    "bp_planner_refill": (c_i32, [c_vp, c_vp, c_vp]),
    "bp_planner_pop": (c_i32, [c_vp, c_vp, P(PlanBuffers), c_vp]),
    "bp_planner_get_stats": (c_i32, [c_vp, c_vp, P(PlannerStats)]),
    "bp_planner_dump": (c_i32, [c_vp, P(PlannerDump), c_i64, c_vp]),
    "bp_cache_create": (c_i32, [c_vp, c_vp, c_i64, c_i32, P(c_vp)]),
    "bp_cache_destroy": (c_i32, [c_vp]),
    "bp_cache_get_stats": (c_i32, [c_vp, c_vp, P(CacheStats)]),
    "bp_cache_insert": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "bp_cache_set_ttl": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "bp_cache_resolve": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "bp_cache_apply_resolve": (c_i32, [c_vp, c_vp, c_vp, c_u64, c_i32, c_vp, c_vp]),
    "bp_cache_gather": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "bp_cache_update": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bp_cache_evict": (c_i32, [c_vp, c_i64, c_i32, P(EvictBuffers), c_i64, c_vp]),
    "bp_cache_evict_planned": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, P(EvictBuffers), c_vp]),
    "bp_cache_checksum": (c_i32, [c_vp, c_vp, c_vp]),
    "bp_cache_get_view": (c_i32, [c_vp, P(CacheView)]),
    "bp_store_create": (c_i32, [c_vp, c_vp, c_u64, c_vp, P(c_vp)]),
    "bp_store_destroy": (c_i32, [c_vp]),
    "bp_store_host_table": (c_vp, [c_vp]),
    "bp_store_written_bitmap": (c_vp, [c_vp]),
    "bp_store_fetch": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "bp_store_fetch_lazy": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "bp_store_link_counters": (c_i32, [c_vp, c_vp]),
    "bp_store_enable_log": (c_i32, [c_vp, c_i64, c_vp]),
    "bp_store_log_append": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "bp_store_compact": (c_i32, [c_vp, c_vp]),
    "bp_store_log_rows": (c_i64, [c_vp]),
    "bp_engine_set_write_log": (c_i32, [c_vp, c_i64]),
    "bp_engine_set_link_gate": (c_i32, [c_vp, c_i32]),
    "bp_store_write": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bp_store_write_masked": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bp_init_values": (c_i32, [c_u64, c_i32, c_vp, c_i64, c_vp, c_vp]),
    "bp_stub_step": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_f32, c_f32, c_f32, c_i32, c_vp, c_vp, c_i64,
                             c_vp, c_vp]),
    "bp_mark_ids": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "bp_add_at_rows": (c_i32, [c_vp, c_vp, c_i32, c_vp, c_vp]),
    "bp_sgd": (c_i32, [c_vp, c_vp, c_f32, c_i64, c_vp, c_vp]),
    "bp_sort_keys_u64": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp]),
    "bp_xor_checksum_rows": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp]),
    "bp_engine_create": (c_i32, [c_vp, c_vp, P(EngineConfig), P(c_vp)]),
    "bp_engine_destroy": (c_i32, [c_vp]),
    "bp_engine_parts": (c_i32, [c_vp, P(EngineParts)]),
    "bp_engine_add_batch": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i32, c_i32]),
    "bp_engine_add_batch_packed": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i32,
                                           c_i32]),
    "bp_engine_add_batch_columnar": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i32,
                                             c_i32]),
    "bp_prep_create_columnar": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i32, c_i64, c_i32, c_vp,
                                        P(c_vp)]),
    "bp_engine_prep": (c_i32, [c_vp, c_i64, P(c_vp)]),
    "bp_engine_release_batch": (c_i32, [c_vp, c_i64]),
    "bp_engine_refill": (c_i32, [c_vp, c_i64]),
    "bp_engine_pop": (c_i32, [c_vp, c_i64, P(c_i32)]),
    "bp_engine_plan_counts": (c_i32, [c_vp, c_i32, c_vp]),
    "bp_engine_plan_view": (c_i32, [c_vp, c_i32, P(PlanBuffers), P(c_vp)]),
    "bp_engine_fetch": (c_i32, [c_vp, c_i32]),
    "bp_engine_flush": (c_i32, [c_vp, c_vp, c_i32]),
    "bp_engine_train": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_u64, c_i32, c_i32, c_i32, P(StepResult)]),
    "bp_engine_chunk_keys": (c_i32, [c_vp, c_i32, c_vp, c_i64]),
    "bp_engine_chunk_view": (c_i32, [c_vp, c_i32, P(EvictBuffers)]),
    "bp_engine_sync": (c_i32, [c_vp]),
    "bp_debug_long_trace": (c_i32, [c_vp]),
    "bp_debug_skip_link": (c_i32, [c_i32]),
    "bp_debug_link_cb_stats": (c_i32, [c_vp]),
    "bp_ipc_alloc": (c_i32, [c_i64, P(c_vp), c_vp]),
    "bp_ipc_open": (c_i32, [c_vp, P(c_vp)]),
    "bp_ipc_close": (c_i32, [c_vp]),
    "bp_ipc_free": (c_i32, [c_vp]),
    "bp_peer_barrier": (c_i32, [c_vp, P(PeerXchg), C.c_uint32, c_vp]),
    "bp_embbag_forward_peer": (c_i32, [c_vp, c_vp, c_i32, c_vp, c_i32, P(PeerXchg), c_vp]),
    "bp_embbag_backward_peer": (c_i32, [c_vp, P(PeerXchg), c_f32, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_f32,
                                        c_f32, c_vp, c_vp]),
    "bp_engine_dlrm_forward_peer": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_u64, c_i32, c_i32, P(PeerXchg)]),
    "bp_engine_dlrm_backward_peer": (c_i32, [c_vp, c_i64, c_i32, P(PeerXchg), c_f32, c_i32, c_i32, c_f32, c_f32,
                                             c_i32, c_i32, P(StepResult)]),
    "bp_engine_dlrm_backward_peer_begin": (c_i32, [c_vp, c_i64, c_i32, P(PeerXchg), c_f32, c_i32, c_i32, c_f32,
                                                   c_f32, c_i32, c_i32]),
    "bp_host_rows_bench": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp]),
    "bp_trace_decode": (c_i32, [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bp_engine_set_link_mode": (c_i32, [c_vp, c_i32, c_i32]),
    "bp_engine_train_begin": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_u64, c_i32, c_i32, c_i32]),
    "bp_engine_train_end": (c_i32, [c_vp, P(StepResult)]),
    "bp_set_link_blocks": (c_i32, [c_i32]),
    "bp_set_link_config": (c_i32, [c_i32, c_i32, c_i32]),
    "bp_set_write_blocks": (c_i32, [c_i32]),
    "bp_set_stub_fork": (c_i32, [c_i32]),
    "bp_set_split_writeback": (c_i32, [c_i32]),
    "bp_set_green_link": (c_i32, [c_i32]),
    "bp_set_stub_short_ctas": (c_i32, [c_i32]),
    "bp_set_stub_carveout": (c_i32, [c_i32]),
    "bp_set_stub_long_threads": (c_i32, [c_i32]),
    "bp_set_stub_long_smem": (c_i32, [c_i32]),
    "bp_set_green_sms": (c_i32, [c_i32]),
    "bp_set_peer_sorted": (c_i32, [c_i32]),
    "bp_embbag_backward_peer_sorted": (c_i32, [c_vp, c_vp, c_f32, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_f32,
                                                c_f32, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "bp_green_info": (c_i32, [c_vp]),
    "bp_dlrm_master_sgd": (c_i32, [P(SgdTensors), c_f32, c_vp]),
    "bp_engine_dlrm_backward_begin": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_i32, c_i32, c_i32, c_f32, c_f32, c_i32,
                                              c_i32]),
    "bp_engine_plan_ready": (c_i32, [c_vp, c_i32, c_vp]),
    "bp_engine_join": (c_i32, [c_vp, c_vp]),
    "bp_engine_set_timing": (c_i32, [c_vp, c_i32]),
    "bp_engine_set_l2_flush": (c_i32, [c_vp, c_vp, c_i64, c_i32]),
    "bp_engine_stage_times": (c_i32, [c_vp, c_vp, c_vp]),
    "bp_engine_dlrm_forward": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_u64, c_i32, c_i32, c_vp]),
    "bp_engine_dlrm_backward": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_i32, c_i32, c_f32, c_f32, c_i32, c_i32,
                                        P(StepResult)]),
    "bp_dlrm_interact_forward": (c_i32, [c_vp, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp, c_i32, c_i32, c_vp]),
    "bp_dlrm_interact_backward": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp,
                                          c_vp]),
    "bp_embbag_forward": (c_i32, [c_vp, c_vp, c_i32, c_vp, c_i32, c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "bp_embbag_backward": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_f32, c_f32,
                                   c_vp, c_vp]),
    "bp_prep_occ_sorted_index": (c_i32, [c_vp, c_vp, c_vp]),
    "bp_prep_occ_rank": (c_i32, [c_vp, c_vp, c_vp]),
    "bp_embbag_bwd_scratch_bytes": (c_i64, [c_i64, c_i32]),
    "bp_embbag_backward_sorted_scratch": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_f32, c_f32,
                                                  c_vp, c_vp, c_i64, c_vp]),
    "bp_debug_bwd_variant": (c_i32, [c_i32]),
    "bp_debug_fwd_variant": (c_i32, [c_i32]),
    "bp_debug_prep_cluster": (c_i32, [c_i32]),
    "bp_debug_prep_shape": (c_i32, [c_i32]),
    "bp_debug_phase_trace": (c_i32, [c_i32, c_vp]),
    "bp_debug_pop_trace": (c_i32, [c_vp]),
    "bp_embbag_backward_sorted": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_i32, c_f32, c_f32, c_vp,
                                          c_vp]),
    "bp_dlrm_interact_backward_rows": (c_i32, [c_vp, c_i32, c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_vp,
                                               c_vp, c_vp, c_vp]),
    "bp_engine_dlrm_grad_rows": (c_i32, [c_vp, c_i64, c_vp]),
    "bp_engine_dlrm_backward_sorted": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_i32, c_i32, c_f32, c_f32, c_i32, c_i32,
                                               P(StepResult)]),
    "bp_store_create_ex": (c_i32, [c_vp, c_vp, c_u64, c_i32, c_vp, P(c_vp)]),
}

_lock = threading.Lock()
_lib = None


def exported_symbols() -> list:
    return sorted(_SIGS)


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """dlopen the library and declare signatures (no CUDA calls)."""
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib_ = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib_, name)
        fn.restype = res
        fn.argtypes = args
    structs = (ErrorT, PrepView, PlanBuffers, PlannerStats, CacheStats, EvictBuffers, CacheView, EngineConfig,
               StepResult, EngineParts, PlannerDump, PeerXchg, SgdTensors)
    for i, st in enumerate(structs):
        if lib_.bp_abi_sizeof(i) != C.sizeof(st):
            raise NativeUnavailable(f"ABI mismatch for {st.__name__}: library {lib_.bp_abi_sizeof(i)} bytes, "
                                    f"binding {C.sizeof(st)} bytes (rebuild the library)")
    return lib_


def lib() -> C.CDLL:
    """The loaded library; requires a CUDA device (there is no CPU path)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch

                if not torch.cuda.is_available():
                    raise NativeUnavailable("no CUDA device visible: the embedding path runs only on the GPU")
                torch.cuda.init()
                lb = load_library()
                # tuning knob: launch shape of the host-link kernels, "blocks,threads,smem_bytes"
                lc = os.environ.get("BAGPIPE_B200_LINK_CONFIG")
                if lc:
                    check(lb.bp_set_link_config(*[int(x) for x in lc.split(",")]), "bp_set_link_config")
                wb = os.environ.get("BAGPIPE_B200_WRITE_BLOCKS")  # tuning knob: write-back scatter grid
                if wb:
                    check(lb.bp_set_write_blocks(int(wb)), "bp_set_write_blocks")
                sk = os.environ.get("BAGPIPE_B200_DEBUG_SKIP_LINK")  # debug only: results become wrong
                if sk:
                    check(lb.bp_debug_skip_link(int(sk)), "bp_debug_skip_link")
                psr = os.environ.get("BAGPIPE_B200_PEER_SORTED")  # 0: reduce-by-key peer backward
                if psr:
                    check(lb.bp_set_peer_sorted(int(psr)), "bp_set_peer_sorted")
                gl = os.environ.get("BAGPIPE_B200_GREEN_LINK")  # the green partition's small part: link streams
                if gl:
                    check(lb.bp_set_green_link(int(gl)), "bp_set_green_link")
                gr = os.environ.get("BAGPIPE_B200_GREEN_SMS")  # tuning knob: SMs requested for the small partition (-1 auto, 0 off)
                if gr:
                    check(lb.bp_set_green_sms(int(gr)), "bp_set_green_sms")
                ls_ = os.environ.get("BAGPIPE_B200_STUB_LONG_SMEM")  # tuning knob: chain CTA smem pad (bytes)
                if ls_:
                    check(lb.bp_set_stub_long_smem(int(ls_)), "bp_set_stub_long_smem")
                lt = os.environ.get("BAGPIPE_B200_STUB_LONG_THREADS")  # tuning knob: hot-key chain CTA width
                if lt:
                    check(lb.bp_set_stub_long_threads(int(lt)), "bp_set_stub_long_threads")
                co = os.environ.get("BAGPIPE_B200_STUB_CARVEOUT")  # tuning knob: short kernel smem carveout %
                if co:
                    check(lb.bp_set_stub_carveout(int(co)), "bp_set_stub_carveout")
                sc_ = os.environ.get("BAGPIPE_B200_STUB_SHORT_CTAS")  # tuning knob: short trainer CTAs per SM
                if sc_:
                    check(lb.bp_set_stub_short_ctas(int(sc_)), "bp_set_stub_short_ctas")
                sw = os.environ.get("BAGPIPE_B200_SPLIT_WB")  # A/B switch: write-back on its own stream
                if sw:
                    check(lb.bp_set_split_writeback(int(sw)), "bp_set_split_writeback")
                sf = os.environ.get("BAGPIPE_B200_STUB_FORK")  # tuning knob: long trainer kernel beside the short
                if sf:
                    check(lb.bp_set_stub_fork(int(sf)), "bp_set_stub_fork")
                fv = os.environ.get("BAGPIPE_B200_FWD_VARIANT")  # tuning knob: EmbeddingBag forward shape
                if fv:
                    check(lb.bp_debug_fwd_variant(int(fv)), "bp_debug_fwd_variant")
                ps = os.environ.get("BAGPIPE_B200_PREP_IPT")  # tuning knob: cluster prep items per thread
                if ps:
                    check(lb.bp_debug_prep_shape(int(ps)), "bp_debug_prep_shape")
                pc = os.environ.get("BAGPIPE_B200_PREP_CLUSTER")  # 0: single-CTA column sort
                if pc:
                    check(lb.bp_debug_prep_cluster(int(pc)), "bp_debug_prep_cluster")
                bv = os.environ.get("BAGPIPE_B200_BWD_VARIANT")  # tuning knob: sorted backward launch shape
                if bv:
                    check(lb.bp_debug_bwd_variant(int(bv)), "bp_debug_bwd_variant")
                _lib = lb
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc == E.BP_OK:
        return
    cls = E.STATUS_TO_ERROR.get(rc, E.NativeError)
    msg = _lib.bp_last_error_message().decode() if _lib is not None and rc >= 100 else ""
    raise cls(f"{what} failed with status {rc}{': ' + msg if msg else ''}")


def ptr(t) -> int | None:
    """Device/host pointer of a tensor (None for None)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Context:
    """Per-process error record shared by all native objects (bp_ctx)."""

    _instance = None

    def __init__(self):
        h = c_vp()
        check(lib().bp_ctx_create(C.byref(h)), "bp_ctx_create")
        self.handle = h

    @classmethod
    def get(cls) -> "Context":
        if cls._instance is None:
            cls._instance = Context()
        return cls._instance

    def raise_pending(self, stream=None) -> None:
        """Synchronise ``stream`` and raise the first recorded device error."""
        err = ErrorT()
        code = lib().bp_ctx_check(self.handle, stream_ptr(stream), C.byref(err))
        if code == 0:
            return
        raise_error_record(err)


def raise_error_record(err: ErrorT) -> None:
    """Raise the reference exception for a device error record (code != 0)."""
    code = err.code
    key = unpack_key(err.key)
    it = None if err.iteration < 0 else int(err.iteration)
    index = int(err.index) & ((1 << 40) - 1)
    if code == 2:
        raise E.CacheMissError(key, it)
    if code == 3:
        raise E.CacheCapacityError(f"insert would exceed capacity at iteration {it}")
    if code == 4:
        raise E.CacheOrderingError(f"ordering violation for {key!r} (position {index}) at iteration {it}")
    if code == 5:
        raise E.StoreKeyError(f"key {key!r} outside the schema")
    if code == 7:
        raise E.EngineError(f"engine invariant violated at iteration {it} ({index})")
    cls = E.STATUS_TO_ERROR.get(code, E.NativeError)
    raise cls(f"device error {code} at iteration {it} for {key!r}")


def host_u64(keys) -> np.ndarray:
    """Packed u64 keys from EmbeddingKey sequences (or pass-through arrays)."""
    if isinstance(keys, np.ndarray):
        return np.ascontiguousarray(keys, dtype=np.uint64)
    n = len(keys)
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    arr = np.asarray(keys, dtype=np.int64).reshape(n, 2)
    return ((arr[:, 0].astype(np.uint64) << np.uint64(44)) | arr[:, 1].astype(np.uint64)).astype(np.uint64)


def to_device(arr: np.ndarray, stream=None):
    """Host numpy -> CUDA tensor (async from a pinned staging copy)."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(arr))
    if t.numel() == 0:
        return torch.empty(t.shape, dtype=t.dtype, device="cuda")
    t = t.pin_memory()
    with torch.cuda.stream(stream or torch.cuda.current_stream()):
        return t.to("cuda", non_blocking=True)


def to_host(t, n: int | None = None) -> np.ndarray:
    """CUDA tensor -> numpy copy (synchronising on the current stream)."""
    if n is not None:
        t = t[:n]
    return t.cpu().numpy()


__all__ = ["Context", "EmbeddingKey", "NativeUnavailable", "check", "lib", "load_library", "ptr", "stream_ptr"]
