"""Host-side packing: signature interning, pool images, window batches.

Everything here turns reference-shaped Python objects into the flat arrays
the C ABI consumes (include/paste.h) and turns kernel outputs back into
reference objects.  No hot-path computation happens here.

Signature tokens: ``sig = 2 * tool_id + (1 if SUCCESS else 0)``.  Mining
interns tools in sorted name order so that sorting sig ids sorts
``(tool_type, status.value)`` pairs ("fail" < "success"), which is the
order the reference uses for targets and contexts (mining.py:264,276,105-111).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Any, Sequence

import numpy as np

from ._native import BINDING_DTYPE, PATTERN_DTYPE
from .events import Event, EventKind, EventSignature, Status
from .mappings import (FormatTemplate, IndexedFallback, PathLookup, expr_ctx_pos)
from .mining import MatchRelation, PatternPool
from .tape import KeyTable, TapeArena, leaf_str_of

X_PATH, X_FALLBACK, X_FORMAT = 0, 1, 2
PF_HAS_MAPPING, PF_STRUCT_ERR = 1, 2
C_FULL, C_PARTIAL, C_TOOL_ONLY = 0, 1, 2
INT32_MAX = 2**31 - 1


class SigTable:
    """tool name <-> tool id; sig = 2*id + success."""

    def __init__(self, tools: Sequence[str] = ()) -> None:
        self.tools: list[str] = []
        self.ids: dict[str, int] = {}
        for t in tools:
            self.tool(t)

    @classmethod
    def sorted_from(cls, tools) -> "SigTable":
        return cls(sorted(set(tools)))

    def tool(self, name: str) -> int:
        tid = self.ids.get(name)
        if tid is None:
            tid = len(self.tools)
            self.ids[name] = tid
            self.tools.append(name)
        return tid

    def sig(self, tool: str, status: Status) -> int:
        return 2 * self.tool(tool) + (1 if status is Status.SUCCESS else 0)

    def sig_of(self, s: EventSignature) -> int:
        return self.sig(s.tool_type, s.status)

    def signature(self, sig: int) -> EventSignature:
        return EventSignature(self.tools[sig >> 1], Status.SUCCESS if sig & 1 else Status.FAIL)

    @property
    def n_sigs(self) -> int:
        return 2 * len(self.tools)

    def __len__(self) -> int:
        return len(self.tools)


def _encode_steps(path, keys: KeyTable, out: list[int]) -> None:
    for step in path:
        if isinstance(step, int):  # bool included, as in the reference's isinstance test
            v = int(step)
            out += [1, v if 0 <= v <= INT32_MAX else -1]
        elif isinstance(step, str):
            out += [0, keys.intern(step)]
        else:  # a non-str, non-int key step can never be present in a JSON dict
            out += [0, -2]


def encode_binding(expr, sigs: SigTable, keys: KeyTable, steps: list[int]) -> tuple:
    """One ``paste_binding`` row for a mapping expression (steps appended)."""
    pos = expr_ctx_pos(expr)
    step_off = len(steps) // 2
    suf_off, suf_cnt, start, fail = 0, 0, -1, -1
    if isinstance(expr, PathLookup):
        kind, path = X_PATH, expr.path
    elif isinstance(expr, FormatTemplate):
        kind, path = X_FORMAT, expr.hole.path
    elif isinstance(expr, IndexedFallback):
        kind, path = X_FALLBACK, expr.path_prefix
        start = expr.start_index if expr.start_index <= INT32_MAX - 64 else -1
        fail = sigs.tool(expr.fail_tool)
    else:
        raise TypeError(f"unknown expression type: {type(expr)!r}")
    _encode_steps(path, keys, steps)
    step_cnt = len(steps) // 2 - step_off
    if kind == X_FALLBACK:
        suf_off = len(steps) // 2
        _encode_steps(expr.path_suffix, keys, steps)
        suf_cnt = len(steps) // 2 - suf_off
    return (kind, max(min(pos, INT32_MAX), -1), step_off, step_cnt, suf_off, suf_cnt, start, fail)


@dataclass
class PoolImage:
    """Compiled pattern pool: the arrays behind ``paste_pool_desc``."""

    pool: PatternPool
    sigs: SigTable
    keys: KeyTable
    patterns: np.ndarray        # PATTERN_DTYPE[P]
    bindings: np.ndarray        # BINDING_DTYPE[B]
    ctx_sig: np.ndarray         # i32
    steps: np.ndarray           # i32[2*S]
    bucket_off: np.ndarray      # i32[n_bucket_sigs+1]
    bucket_pat: np.ndarray      # i32
    bucket_scan_all: np.ndarray  # u8[n_bucket_sigs]
    pattern_ids: list[str]
    k: int
    relation: int
    max_ctx: int
    max_bindings: int
    max_bucket: int

    @property
    def n_bucket_sigs(self) -> int:
        return len(self.bucket_scan_all)

    @classmethod
    def compile(cls, pool: PatternPool, sigs: SigTable | None = None,
                keys: KeyTable | None = None) -> "PoolImage":
        sigs = SigTable() if sigs is None else sigs
        keys = KeyTable() if keys is None else keys
        # pool tools first (sorted), so their ids are stable and dense
        names = set()
        for pat in pool.patterns:
            names.update(s.tool_type for s in pat.context)
            names.add(pat.target)
            if pat.mapping is not None:
                names.update(b.expr.fail_tool for b in pat.mapping.bindings
                             if isinstance(b.expr, IndexedFallback))
        for name in sorted(names):
            sigs.tool(name)

        P = len(pool.patterns)
        pats = np.zeros(P, PATTERN_DTYPE)
        ctx_sig: list[int] = []
        binds: list[tuple] = []
        steps: list[int] = []
        for i, pat in enumerate(pool.patterns):
            flags = 0
            pats[i]["ctx_off"] = len(ctx_sig)
            pats[i]["ctx_len"] = len(pat.context)
            ctx_sig += [sigs.sig_of(s) for s in pat.context]
            pats[i]["target_tool"] = sigs.tool(pat.target)
            pats[i]["p"] = pat.p
            pats[i]["bind_off"] = len(binds)
            if pat.mapping is not None:
                flags |= PF_HAS_MAPPING
                for b in pat.mapping.bindings:
                    pos = expr_ctx_pos(b.expr)
                    if not 0 <= pos < len(pat.context):
                        flags |= PF_STRUCT_ERR  # mappings.py:164-169 raise
                    binds.append(encode_binding(b.expr, sigs, keys, steps))
            pats[i]["n_bind"] = len(binds) - pats[i]["bind_off"]
            pats[i]["flags"] = flags

        n_bucket = sigs.n_sigs
        order = sorted(range(P), key=lambda i: (-pool.patterns[i].p,
                                                pool.patterns[i].pattern_id, i))
        buckets: list[list[int]] = [[] for _ in range(n_bucket)]
        scan_all = np.zeros(max(n_bucket, 1), np.uint8)[:n_bucket]
        for i in order:
            last = ctx_sig[pats[i]["ctx_off"] + pats[i]["ctx_len"] - 1]
            buckets[last].append(i)
            if pats[i]["flags"] & PF_STRUCT_ERR:
                scan_all[last] = 1
        bucket_off = np.zeros(n_bucket + 1, np.int32)
        bucket_off[1:] = np.cumsum([len(b) for b in buckets]) if n_bucket else []
        bucket_pat = np.array([i for b in buckets for i in b] or [0], np.int32)
        binding_arr = np.array(binds, dtype=BINDING_DTYPE) if binds else np.zeros(1, BINDING_DTYPE)
        return cls(pool=pool, sigs=sigs, keys=keys, patterns=pats if P else np.zeros(1, PATTERN_DTYPE),
                   bindings=binding_arr, ctx_sig=np.array(ctx_sig or [0], np.int32),
                   steps=np.array(steps or [0, 0], np.int32), bucket_off=bucket_off,
                   bucket_pat=bucket_pat, bucket_scan_all=scan_all,
                   pattern_ids=[p.pattern_id for p in pool.patterns],
                   k=pool.config.k,
                   relation=0 if pool.config.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1,
                   max_ctx=max((len(p.context) for p in pool.patterns), default=0),
                   max_bindings=max((len(p.mapping.bindings) for p in pool.patterns
                                     if p.mapping is not None), default=0),
                   max_bucket=max((len(b) for b in buckets), default=0))


@dataclass
class WindowBatch:
    """Window rings for a batch of sessions + the payload arena they point at."""

    capacity: int
    tok: np.ndarray      # i32[n*W]
    evt: np.ndarray      # i32[n*W]
    count: np.ndarray    # i64[n]
    arena: TapeArena
    created: list[float | None]
    slot_major: int = 0

    @property
    def n(self) -> int:
        return len(self.count)


def pack_windows(windows: Sequence[Sequence[Event]], sigs: SigTable, keys: KeyTable,
                 capacity: int | None = None) -> WindowBatch:
    """Lay each window (oldest..newest events) into a ring with count = len,
    so slot i holds the i-th oldest event."""
    W = max(capacity or 0, max((len(w) for w in windows), default=0), 1)
    n = len(windows)
    tok = np.full(n * W, -1, np.int32)
    evt = np.full(n * W, -1, np.int32)
    count = np.zeros(n, np.int64)
    arena = TapeArena(keys)
    created: list[float | None] = []
    payloads: list = []  # tape i = payloads[i], encoded in one batch below
    for s, events in enumerate(windows):
        last_tool = None
        for i, ev in enumerate(events):
            if ev.kind is EventKind.TOOL_CALL:
                tok[s * W + i] = sigs.sig(ev.tool_type, ev.status)
                evt[s * W + i] = len(payloads)
                payloads.append(ev.result)
                last_tool = ev
        count[s] = len(events)
        created.append(last_tool.t_end if last_tool is not None else None)
    arena.add_many(payloads)
    return WindowBatch(W, tok, evt, count, arena, created)


def admit_tables(sigs: SigTable, policy, benefit) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Per-tool (allow, max_level, benefit) over the current tool table."""
    n = max(len(sigs), 1)
    allow = np.zeros(n, np.uint8)
    level = np.ones(n, np.uint8)
    bene = np.zeros(n, np.float64)
    for tid, name in enumerate(sigs.tools):
        rule = policy.rule_for(name)
        allow[tid] = 1 if rule.allow else 0
        level[tid] = int(rule.max_speculation)
        bene[tid] = float(benefit(name))
    return allow, level, bene


@dataclass
class PredictResult:
    """Host copies of ``paste_predict_out`` for one batch."""

    K: int
    B: int
    n_pred: np.ndarray
    pred_pat: np.ndarray
    pred_comp: np.ndarray
    pred_arg: np.ndarray
    n_act: np.ndarray | None
    act_pred: np.ndarray | None
    act_level: np.ndarray | None
    act_util: np.ndarray | None
    struct_err: np.ndarray
    slot_major: int = 0

    @classmethod
    def empty(cls, n: int, K: int, B: int, admit: bool, slot_major: int = 0) -> "PredictResult":
        return cls(K, B, np.zeros(n, np.int32), np.zeros(n * K, np.int32),
                   np.zeros(n * K, np.uint8), np.full(n * K * B, -1, np.int64),
                   np.zeros(n, np.int32) if admit else None,
                   np.zeros(n * K, np.int16) if admit else None,
                   np.zeros(n * K, np.uint8) if admit else None,
                   np.zeros(n * K, np.float64) if admit else None,
                   np.zeros(n, np.int32), slot_major)

    def session_major(self) -> "PredictResult":
        """The same records in per-session layout ([n][K], args [n][K][B])."""
        if not self.slot_major:
            return self
        n, K, B = len(self.n_pred), self.K, self.B

        def tr(a, width=1):
            if a is None:
                return None
            return np.ascontiguousarray(a.reshape(K * width, n).T).reshape(-1)

        return PredictResult(K, B, self.n_pred, tr(self.pred_pat), tr(self.pred_comp),
                             tr(self.pred_arg, B), self.n_act, tr(self.act_pred),
                             tr(self.act_level), tr(self.act_util), self.struct_err, 0)


def decode_predictions(res: PredictResult, image: PoolImage, arena: TapeArena,
                       created: Sequence[float | None], now: float | None):
    """Kernel records -> reference PredictedInvocation lists."""
    from .prediction import Completeness, PredictedInvocation

    comp_enum = (Completeness.FULL, Completeness.PARTIAL, Completeness.TOOL_ONLY)
    res = res.session_major()
    out = []
    K, B = res.K, res.B
    for s in range(len(res.n_pred)):
        preds = []
        stamp = now if now is not None else created[s]
        for i in range(int(res.n_pred[s])):
            slot = s * K + i
            pid = int(res.pred_pat[slot])
            pat = image.pool.patterns[pid]
            comp = comp_enum[int(res.pred_comp[slot])]
            args: dict[str, Any] = {}
            if pat.mapping is not None:
                for j, b in enumerate(pat.mapping.bindings):
                    ref = int(res.pred_arg[slot * B + j])
                    if ref < 0:
                        continue
                    value = arena.node_object(ref >> 32, ref & 0xFFFFFFFF)
                    if isinstance(b.expr, FormatTemplate):
                        value = b.expr.prefix + b.expr.normalization.apply(leaf_str_of(value)) \
                            + b.expr.suffix
                    args[b.arg_name] = value
            preds.append(PredictedInvocation(tool_type=pat.target, args=args, completeness=comp,
                                             probability=pat.p,
                                             source_pattern=image.pattern_ids[pid],
                                             created_at=stamp))
        out.append(preds)
    return out


def decode_actions(res: PredictResult, preds_per_session):
    from .policy import SpecLevel, SpeculativeAction

    out = []
    res = res.session_major()
    K = res.K
    for s, preds in enumerate(preds_per_session):
        acts = []
        for j in range(int(res.n_act[s])):
            o = s * K + j
            acts.append(SpeculativeAction(prediction=preds[int(res.act_pred[o])],
                                          level=SpecLevel(int(res.act_level[o])),
                                          expected_utility=float(res.act_util[o])))
        out.append(acts)
    return out
