"""ctypes binding of libpaste.so (the C ABI declared in include/paste.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2603_18897_b200.build``).  There is no fallback: if the
library or a CUDA device is missing, every hot-path call raises
:class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_int, c_int32, c_int64, c_void_p

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpaste.so")

PASTE_OK = 0
PASTE_ERR_INVALID = -1
PASTE_ERR_CUDA = -2
PASTE_ERR_UNSUPPORTED = -3


class NativeUnavailable(RuntimeError):
    """libpaste.so or the CUDA device it needs is not available."""


class PasteError(RuntimeError):
    pass


class PasteUnsupported(PasteError):
    pass


# ---------------------------------------------------------------------------
# struct mirrors (field order and types must match include/paste.h)
# ---------------------------------------------------------------------------

class PoolDesc(ctypes.Structure):
    _fields_ = [("n_patterns", c_int32), ("n_bucket_sigs", c_int32), ("k", c_int32),
                ("relation", c_int32), ("max_ctx", c_int32), ("max_bindings", c_int32),
                ("patterns", c_void_p), ("bindings", c_void_p), ("ctx_sig", c_void_p),
                ("steps", c_void_p), ("bucket_off", c_void_p), ("bucket_pat", c_void_p),
                ("bucket_scan_all", c_void_p), ("match_table", c_void_p), ("mt_k", c_int32),
                ("mt_g", c_int32)]


class AdmitDesc(ctypes.Structure):
    _fields_ = [("enabled", c_int32), ("n_tools", c_int32), ("allow", c_void_p),
                ("max_level", c_void_p), ("benefit", c_void_p)]


class WindowsDesc(ctypes.Structure):
    _fields_ = [("n_sessions", c_int64), ("capacity", c_int32), ("slot_major", c_int32),
                ("tok", c_void_p), ("evt", c_void_p), ("count", c_void_p),
                ("nodes", c_void_p), ("bytes", c_void_p), ("refs", c_void_p),
                ("new_tok", c_void_p), ("new_ref", c_void_p), ("new_evt_base", c_int64),
                ("new_byte_base", c_int64), ("stream_end", c_void_p), ("new_node", c_void_p),
                ("new_tok8", c_void_p), ("new_node16", c_void_p), ("new_node8", c_void_p),
                ("node_codes", c_void_p), ("event_codes", c_void_p)]


class PredictOut(ctypes.Structure):
    _fields_ = [("max_candidates", c_int32), ("max_bindings", c_int32),
                ("slot_major", c_int32), ("pad", c_int32), ("n_pred", c_void_p), ("pred_pat", c_void_p), ("pred_comp", c_void_p),
                ("pred_arg", c_void_p), ("n_act", c_void_p), ("act_pred", c_void_p),
                ("act_level", c_void_p), ("act_util", c_void_p), ("struct_err", c_void_p)]


class AdmitListsDesc(ctypes.Structure):
    _fields_ = [("n_lists", c_int64), ("list_off", c_void_p), ("tool", c_void_p),
                ("full", c_void_p), ("p", c_void_p), ("benefit", c_void_p),
                ("created_at", c_void_p), ("n_act", c_void_p), ("act_pred", c_void_p),
                ("act_level", c_void_p), ("act_util", c_void_p)]


class MineDesc(ctypes.Structure):
    _fields_ = [("n_sigs", c_int32), ("k", c_int32), ("relation", c_int32), ("pad", c_int32),
                ("tokens", c_void_p), ("n_tokens", c_int64), ("hist", c_void_p),
                ("tool_count", c_void_p), ("support", c_void_p), ("match", c_void_p),
                ("follow", c_void_p)]


class ColumnarDesc(ctypes.Structure):
    _fields_ = [("n_events", c_int64), ("session", c_void_p), ("seq", c_void_p),
                ("t_start", c_void_p), ("t_end", c_void_p), ("sig", c_void_p),
                ("inactivity_ms", ctypes.c_double), ("tokens_out", c_void_p),
                ("n_segments", c_void_p), ("n_unsorted", c_void_p)]


class OrderDesc(ctypes.Structure):
    _fields_ = [("n_events", c_int64), ("n_sessions", c_int32), ("pad", c_int32),
                ("session", c_void_p), ("seq", c_void_p), ("t_start", c_void_p),
                ("t_end", c_void_p), ("sig", c_void_p), ("inactivity_ms", ctypes.c_double),
                ("out_session", c_void_p), ("out_seq", c_void_p), ("out_t_start", c_void_p),
                ("out_t_end", c_void_p), ("out_sig", c_void_p), ("order", c_void_p),
                ("out_tok", c_void_p), ("n_out", c_void_p), ("n_segments", c_void_p), ("reordered", c_void_p),
                ("status", c_void_p)]


class JsonlSizes(ctypes.Structure):
    _fields_ = [(n, c_int64) for n in ("n_rows", "n_sessions", "n_errors", "n_lines", "n_nodes",
                                       "n_bytes", "n_keys", "key_names_len", "tool_names_len")] + \
        [("n_tools", c_int32), ("pad", c_int32)]


class JsonlOut(ctypes.Structure):
    _fields_ = [(n, c_void_p) for n in ("session", "seq", "t_start", "t_end", "sig",
                                        "error_lines", "error_codes", "error_seq", "tool_names",
                                        "nodes", "bytes", "refs", "key_names")]


class OccDesc(ctypes.Structure):
    _fields_ = [("n_tokens", c_int64), ("tok", c_void_p), ("n_cand", c_int32), ("k", c_int32),
                ("relation", c_int32), ("kmax", c_int32), ("n_sigs", c_int32),
                ("n_tools", c_int32), ("ctx", c_void_p), ("ctx_len", c_void_p),
                ("bucket_off", c_void_p), ("bucket", c_void_p), ("off", c_void_p),
                ("cursor", c_void_p), ("anchor", c_void_p), ("picked", c_void_p),
                ("overflow", c_void_p)]


PASTE_ORDER_NAN_T = 1
PASTE_ORDER_BAD_SESSION = 2


class SelectDesc(ctypes.Structure):
    _fields_ = [("n_jobs", c_int64), ("p", c_void_p), ("benefit", c_void_p), ("duration", c_void_p),
                ("cost", c_void_p), ("id", c_void_p), ("selected", c_void_p),
                ("n_selected", c_void_p)]


class LeafScanDesc(ctypes.Structure):
    _fields_ = [("n_queries", c_int64), ("node_budget", c_int64), ("nodes", c_void_p),
                ("bytes", c_void_p), ("refs", c_void_p), ("event", c_void_p),
                ("target_type", c_void_p), ("target_nan", c_void_p), ("target_off", c_void_p),
                ("target_bytes", c_void_p), ("out_off", c_void_p), ("out_nodes", c_void_p),
                ("n_out", c_void_p), ("truncated", c_void_p)]


class ResolveDesc(ctypes.Structure):
    _fields_ = [("n_queries", c_int64), ("bindings", c_void_p), ("steps", c_void_p),
                ("nodes", c_void_p), ("refs", c_void_p), ("src_event", c_void_p),
                ("hist_off", c_void_p), ("hist_tok", c_void_p), ("src_pos", c_void_p),
                ("result", c_void_p)]


class CompactDesc(ctypes.Structure):
    _fields_ = [("hdr", c_void_p), ("pred", c_void_p), ("arg", c_void_p), ("act", c_void_p),
                ("totals", c_void_p), ("format", c_int32), ("pad", c_int32)]


PASTE_CF_HDR8, PASTE_CF_PRED8, PASTE_CF_ARG16, PASTE_CF_ENTRY16, PASTE_CF_KEYS = 1, 2, 4, 8, 16
PASTE_CF_UNIQ = 32
PASTE_CF_KEY8 = 64
PASTE_COPY_H2D, PASTE_COPY_D2H, PASTE_COPY_D2D = 1, 2, 3
PASTE_INGEST_MISSING, PASTE_INGEST_T_ORDER, PASTE_INGEST_EMPTY_TOOL = 0x100, 0x200, 0x400


class HoldsDesc(ctypes.Structure):
    _fields_ = [("n_hyp", c_int64), ("n_occ", c_int64), ("n_ctx", c_int32), ("pad", c_int32)] + \
        [(name, c_void_p) for name in ("hyp", "steps", "fmt", "fmt_bytes", "nodes", "bytes", "refs",
                                       "occ_event", "src_pos", "hist_off", "hist_tok", "act_type",
                                       "act_nan", "act_off", "act_bytes", "hits", "unsure", "eq",
                                       "hist_end", "act_event", "act_node")]


class KeyLookupDesc(ctypes.Structure):
    _fields_ = [("n", c_int64), ("nodes", c_void_p), ("refs", c_void_p), ("tape", c_void_p),
                ("key", c_int32), ("pad", c_int32), ("out_node", c_void_p),
                ("n_scalar", c_void_p)]


class ReplayDesc(ctypes.Structure):
    _fields_ = [("n_calls", c_int64), ("capacity", c_int32), ("cand_limit", c_int32)] + \
        [(name, c_void_p) for name in ("ev_tok", "ev_evt", "call_pos", "call_len", "call_tool",
                                       "call_args", "call_keyset", "pat_keyset", "bind_key", "fmt",
                                       "fmt_bytes", "nodes", "bytes", "refs", "tallies", "unsure")]


class HashDesc(ctypes.Structure):
    _fields_ = [("n", c_int64)] + [(name, c_void_p) for name in (
        "nodes", "bytes", "refs", "key_bytes", "key_off", "key_rank", "digest", "unsure")]


class ActionKeysDesc(ctypes.Structure):
    _fields_ = [("n_sessions", c_int64), ("pool", PoolDesc), ("out", PredictOut)] + \
        [(name, c_void_p) for name in ("nodes", "bytes", "refs", "key_bytes", "key_off",
                                       "key_rank", "bind_key", "fmt", "fmt_bytes", "keys",
                                       "key_state")]


class ActionsDesc(ctypes.Structure):
    _fields_ = [("n_actions", c_int64), ("tool", c_void_p), ("level", c_void_p), ("p", c_void_p),
                ("key", c_void_p), ("n_tools", c_int32), ("pad", c_int32), ("mean", c_void_p),
                ("cost", c_void_p), ("warm_fraction", ctypes.c_double), ("r_total", c_int64),
                ("id_base", c_int64)]


class JobsOut(ctypes.Structure):
    _fields_ = [(name, c_void_p) for name in ("p", "benefit", "duration", "cost", "id", "action",
                                              "n_jobs", "next_id")]


class LiveActionsDesc(ctypes.Structure):
    _fields_ = [("n_sessions", c_int64), ("pool", PoolDesc), ("out", PredictOut)] + \
        [(name, c_void_p) for name in ("slot_keys", "tool", "level", "p", "key", "session",
                                       "slot", "n_actions")]


class LivePlan(ctypes.Structure):
    _fields_ = [("plan", c_void_p), ("max_candidates", c_int32), ("max_bindings", c_int32),
                ("walk", c_void_p), ("walk_nodes", c_int64)]


class IngestDesc(ctypes.Structure):
    _fields_ = [("capacity", c_int64), ("session", c_void_p), ("seq", c_void_p),
                ("t_start", c_void_p), ("t_end", c_void_p), ("sig", c_void_p),
                ("error_lines", c_void_p), ("error_capacity", c_int64), ("tool_names", c_void_p),
                ("tool_names_capacity", c_int64), ("n_events", c_int64), ("n_segments", c_int64),
                ("n_errors", c_int64), ("n_lines", c_int64), ("reordered_sessions", c_int64),
                ("tool_names_len", c_int64), ("n_tools", c_int32), ("pad", c_int32),
                ("error_codes", c_void_p), ("error_seq", c_void_p)]


# numpy mirrors of the element structs
PATTERN_DTYPE = np.dtype([("ctx_off", "i4"), ("ctx_len", "i4"), ("target_tool", "i4"),
                          ("bind_off", "i4"), ("n_bind", "i4"), ("flags", "i4"), ("p", "f8")])
BINDING_DTYPE = np.dtype([(name, "i4") for name in
                          ("kind", "ctx_pos", "step_off", "step_cnt", "suf_off", "suf_cnt",
                           "start_index", "fail_tool")])
assert PATTERN_DTYPE.itemsize == 32 and BINDING_DTYPE.itemsize == 32

# symbol -> (restype, argtypes); the list is checked against include/paste.h by tests
EXPORTS = {
    "paste_last_error": (c_char_p, []),
    "paste_abi_version": (c_int, []),
    "paste_last_launch_count": (c_int, []),
    "paste_memcpy_batch": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    "paste_predict_batch": (c_int, [POINTER(PoolDesc), POINTER(WindowsDesc),
                                    POINTER(AdmitDesc), POINTER(PredictOut), c_void_p]),
    "paste_admit_lists": (c_int, [POINTER(AdmitDesc), POINTER(AdmitListsDesc), c_void_p]),
    "paste_match_table_bytes": (c_int64, [POINTER(PoolDesc), c_int32, c_int32]),
    "paste_build_match_table": (c_int, [POINTER(PoolDesc), c_int32, c_int32, c_void_p, c_void_p]),
    "paste_mine_geometry": (c_int, [c_int32, c_int32, POINTER(c_int64), POINTER(c_int64)]),
    "paste_mine_count": (c_int, [POINTER(MineDesc), c_void_p]),
    "paste_holds": (c_int, [POINTER(HoldsDesc), c_void_p]),
    "paste_replay_score": (c_int, [POINTER(PoolDesc), POINTER(ReplayDesc), POINTER(PredictOut),
                                   c_void_p]),
    "paste_replay_fused": (c_int, [POINTER(PoolDesc), POINTER(ReplayDesc), c_int32, c_void_p]),
    "paste_compact_scratch_bytes": (c_int64, [c_int64]),
    "paste_live_plan_bytes": (c_int64, [POINTER(PoolDesc), c_int32, c_int32]),
    "paste_build_live_plan": (c_int, [POINTER(PoolDesc), POINTER(AdmitDesc), c_int32, c_int32,
                                      c_void_p, c_void_p]),
    "paste_live_walk_bytes": (c_int64, [c_int32, c_int64]),
    "paste_build_live_walk": (c_int, [POINTER(PoolDesc), c_int32, c_void_p, c_int64, c_void_p,
                                      c_void_p]),
    "paste_predict_live": (c_int, [POINTER(PoolDesc), POINTER(WindowsDesc), POINTER(AdmitDesc),
                                   POINTER(LivePlan), POINTER(PredictOut), c_void_p]),
    "paste_predict_live_compact_scratch_bytes": (c_int64, [c_int64, c_int32, c_int32]),
    "paste_predict_live_compact": (c_int, [POINTER(PoolDesc), POINTER(WindowsDesc),
                                           POINTER(AdmitDesc), POINTER(LivePlan), c_int32,
                                           POINTER(CompactDesc), c_void_p, c_int64, c_void_p]),
    "paste_canonical_hash": (c_int, [POINTER(HashDesc), c_void_p]),
    "paste_ingest_jsonl": (c_int, [c_char_p, c_int64, ctypes.c_double, POINTER(IngestDesc)]),
    "paste_jsonl_parse": (c_int, [c_char_p, c_int64, c_int32, POINTER(c_void_p)]),
    "paste_jsonl_sizes_of": (c_int, [c_void_p, POINTER(JsonlSizes)]),
    "paste_jsonl_copy": (c_int, [c_void_p, POINTER(JsonlOut)]),
    "paste_jsonl_destroy": (None, [c_void_p]),
    "paste_action_keys": (c_int, [POINTER(ActionKeysDesc), c_void_p]),
    "paste_action_jobs_scratch_bytes": (c_int64, [c_int64]),
    "paste_action_jobs": (c_int, [POINTER(ActionsDesc), POINTER(JobsOut), c_void_p, c_int64,
                                  c_void_p]),
    "paste_live_actions_scratch_bytes": (c_int64, [c_int64]),
    "paste_live_actions": (c_int, [POINTER(LiveActionsDesc), c_void_p, c_int64, c_void_p]),
    "paste_predict_compact_scratch_bytes": (c_int64, [c_int64]),
    "paste_predict_compact_supported": (c_int, [POINTER(PoolDesc), c_int, c_int, c_int, c_int]),
    "paste_predict_compact": (c_int, [POINTER(PoolDesc), POINTER(WindowsDesc), POINTER(AdmitDesc),
                                      c_int32, c_int32, POINTER(CompactDesc), c_void_p, c_void_p]),
    "paste_compact_records": (c_int, [POINTER(PredictOut), c_int64, POINTER(PoolDesc),
                                      POINTER(CompactDesc), c_void_p, c_void_p]),
    "paste_leaf_scan": (c_int, [POINTER(LeafScanDesc), c_void_p]),
    "paste_leaf_scan_shared_bytes": (c_int64, [c_int64, c_int64]),
    "paste_leaf_scan_shared": (c_int, [POINTER(LeafScanDesc), c_void_p, c_int64, c_void_p,
                                       c_void_p, c_void_p]),
    "paste_resolve": (c_int, [POINTER(ResolveDesc), c_void_p]),
    "paste_select_scratch_bytes": (c_int64, [c_int64]),
    "paste_select_greedy": (c_int, [POINTER(SelectDesc), c_int64, c_int64, c_void_p, c_int64,
                                    c_void_p]),
    "paste_select_victim": (c_int, [POINTER(SelectDesc), c_void_p, c_void_p, c_void_p]),
    "paste_mine_ingest_count": (c_int, [POINTER(ColumnarDesc), POINTER(MineDesc), c_void_p]),
    "paste_mine_expand": (c_int, [POINTER(MineDesc), c_void_p]),
    "paste_mine_slice_cols": (c_int32, [c_int32, c_int32]),
    "paste_mine_transpose_slices": (c_int, [POINTER(MineDesc), c_int32, c_void_p, c_void_p]),
    "paste_mine_expand_slice": (c_int, [POINTER(MineDesc), c_void_p, c_int32, c_int32, c_void_p]),
    "paste_mine_select": (c_int, [POINTER(MineDesc), c_int64, ctypes.c_double, c_int64, c_void_p,
                                  c_void_p, c_void_p]),
    "paste_mine_sort_scratch_bytes": (c_int64, [c_int64]),
    "paste_mine_stage_bytes": (c_int64, [c_int64, c_int32, c_int32]),
    "paste_mine_ingest_count_staged": (c_int, [POINTER(ColumnarDesc), POINTER(MineDesc), c_void_p,
                                               c_int64, c_void_p]),
    "paste_mine_occurrences": (c_int, [POINTER(OccDesc), c_void_p]),
    "paste_tape_key_lookup": (c_int, [POINTER(KeyLookupDesc), c_void_p]),
    "paste_ingest_order_scratch_bytes": (c_int64, [c_int64, c_int32]),
    "paste_ingest_order": (c_int, [POINTER(OrderDesc), c_void_p, c_int64, c_void_p]),
    "paste_mine_select_sorted": (c_int, [POINTER(MineDesc), c_int64, ctypes.c_double, c_int64,
                                         c_void_p, c_void_p, c_void_p, c_void_p]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libpaste.so and declare every export (no device needed)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: run __graft_entry__.build() to compile the sm_100a library")
    lib = ctypes.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.paste_abi_version() != 1:
        raise NativeUnavailable("libpaste ABI version mismatch")
    if path == LIB_PATH:
        _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    """The library, with a CUDA device required (hot-path entry)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the PASTE engine runs on B200 only "
                                "(there is no CPU fallback)")
    return load_library()


def check(status: int, lib_handle: ctypes.CDLL | None = None) -> None:
    if status == PASTE_OK:
        return
    handle = lib_handle or _lib
    msg = handle.paste_last_error().decode() if handle is not None else "unknown error"
    if status == PASTE_ERR_INVALID:
        raise ValueError(msg)
    if status == PASTE_ERR_UNSUPPORTED:
        raise PasteUnsupported(msg)
    raise PasteError(msg)


def ptr(t) -> int:
    """Device (or host) address of a torch tensor / numpy array, 0 for None."""
    if t is None:
        return 0
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()
