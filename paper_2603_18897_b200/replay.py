"""C2: score_accuracy replay on the device (prediction.py:133-169).

The reference replays a corpus session by session: before every tool call
after a session's first it predicts from the window of preceding events
(LLM steps take window slots), then tallies top-1, top-3 and "hit" -- some
FULL prediction of the call's tool whose ``canonical_arg_hash`` equals the
call's.  Here the corpus is one event stream in HBM (tokens, payload
indices, the calls' argument tapes) and ``paste_replay_score`` runs K4 on
every call's window -- read in place from the stream -- and tallies the
three counts on the device.  Hit checks that need Unicode or container semantics come back
"unsure" and are decided on the host with the reference's hash, so the
report is exact.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Any, Sequence

import numpy as np

from . import _native
from ._native import PredictOut, ReplayDesc, check, ptr
from .mappings import FormatTemplate

INT32_MAX = 2**31 - 1
FMT_NON_ASCII = 0x100  # PASTE_FMT_NON_ASCII
_NORM_CODE = {"none": 0, "trim": 1, "lowercase": 2}


class KeysetTable:
    """Interned argument-name sets.  Two argument dicts can have equal
    canonical JSON only if their NFC key sets are equal; ids are handed out
    only for ASCII string keys (NFC is then the identity and the device's
    key lookup by interned id is exact), everything else is -1 ("host")."""

    def __init__(self) -> None:
        self.ids: dict[frozenset, int] = {}

    def of_names(self, names: Sequence[Any]) -> int:
        if not all(isinstance(k, str) and k.isascii() for k in names):
            return -1
        ks = frozenset(names)
        if len(ks) != len(names):
            return -1  # duplicate names: dict semantics (last wins) stay on the host
        return self.ids.setdefault(ks, len(self.ids))

    def of_args(self, args: Any) -> int:
        if not isinstance(args, dict):
            return -2
        return self.of_names(list(args))


def pool_hit_tables(dp, ksets: KeysetTable):
    """Per-pattern key-set ids, per-binding arg-name key ids and
    FormatTemplate rows, in PoolImage order (packing.py PoolImage.compile)."""
    pat_ks, bind_key, fmt, fbytes = [], [], [], bytearray()
    for pat in dp.pool.patterns:
        binds = pat.mapping.bindings if pat.mapping is not None else ()
        pat_ks.append(ksets.of_names([b.arg_name for b in binds]))
        for b in binds:
            bind_key.append(dp.keys.intern(b.arg_name))
            if isinstance(b.expr, FormatTemplate):
                pre = b.expr.prefix.encode("utf-8", "surrogatepass")
                suf = b.expr.suffix.encode("utf-8", "surrogatepass")
                flag = 0 if (pre + suf).isascii() else FMT_NON_ASCII
                fmt += [len(fbytes), len(pre), len(fbytes) + len(pre), len(suf),
                        _NORM_CODE[b.expr.normalization.value] | flag]
                fbytes += pre + suf
            else:
                fmt += [0, 0, 0, 0, 0]
    return (np.array(pat_ks or [0], np.int32), np.array(bind_key or [0], np.int32),
            np.array(fmt or [0] * 5, np.int32), np.frombuffer(bytes(fbytes) + b"\0", np.uint8))


@dataclass
class ReplayCorpus:
    """A replay corpus as host arrays (the C2 boundary's inputs)."""

    ev_tok: np.ndarray      # i32[E] sig, -1 = LLM step
    ev_evt: np.ndarray      # i32[E] result payload index, -1 for LLM steps
    call_pos: np.ndarray    # i64[C] stream index of each scored call
    call_len: np.ndarray    # i64[C] window length
    call_tool: np.ndarray   # i32[C] tool id
    call_args: np.ndarray   # i32[C] args payload index
    call_keyset: np.ndarray # i32[C]
    nodes: np.ndarray       # NODE_DTYPE
    data: np.ndarray        # u8
    refs: np.ndarray        # i64[P, 2]

    @property
    def n_calls(self) -> int:
        return len(self.call_pos)

    def arrays(self) -> dict[str, np.ndarray]:
        return {k: getattr(self, k) for k in ("ev_tok", "ev_evt", "call_pos", "call_len",
                                              "call_tool", "call_args", "call_keyset", "nodes",
                                              "data", "refs")}

    def nbytes(self) -> int:
        return sum(int(a.nbytes) for a in self.arrays().values())


def corpus_from_traces(traces, dp, window_capacity: int, ksets: KeysetTable):
    """Sessions -> ReplayCorpus (+ the scored call events, for host re-checks)."""
    from .events import EventKind
    from .tape import TapeArena

    arena = TapeArena(dp.keys)
    payloads: list = []  # tape i = payloads[i], encoded in one batch below
    ev_tok, ev_evt, calls, call_len, actual = [], [], [], [], []
    call_args, call_ks = [], []
    g = 0
    for session in traces:
        start = g
        seen_tool = False
        for ev in session.events:
            if ev.kind is EventKind.TOOL_CALL:
                if seen_tool:
                    calls.append(g)
                    call_len.append(min(window_capacity, g - start))
                    actual.append(ev)
                    call_args.append(len(payloads))
                    payloads.append(ev.args)
                    call_ks.append(ksets.of_args(ev.args))
                seen_tool = True
                ev_tok.append(dp.sigs.sig(ev.tool_type, ev.status))
                ev_evt.append(len(payloads))
                payloads.append(ev.result)
            else:
                ev_tok.append(-1)
                ev_evt.append(-1)
            g += 1
    arena.add_many(payloads)
    nodes, data, refs = arena.arrays()
    corpus = ReplayCorpus(
        np.array(ev_tok or [-1], np.int32), np.array(ev_evt or [-1], np.int32),
        np.array(calls, np.int64), np.array(call_len, np.int64),
        np.array([dp.sigs.tool(e.tool_type) for e in actual], np.int32),
        np.array(call_args, np.int32), np.array(call_ks, np.int32), nodes, data, refs)
    return corpus, actual, arena


class ReplayBatch:
    """A device-resident replay: corpus arrays, pool hit tables, outputs."""

    def __init__(self, dp, corpus: ReplayCorpus, window_capacity: int,
                 max_candidates: int | None, ksets: KeysetTable, upload: bool = True):
        import torch

        from .device_ops import to_dev

        self.lib = _native.lib()
        self.dp, self.corpus, self.W = dp, corpus, window_capacity
        self.K, slice_after = dp._k_for(max_candidates)
        self.cand_limit = int(max_candidates) if slice_after else INT32_MAX
        self.B = max(dp.image.max_bindings, 1)
        n = corpus.n_calls
        pat_ks, bind_key, fmt, fbytes = pool_hit_tables(dp, ksets)
        self.tables = {k: to_dev(v) for k, v in dict(pat_ks=pat_ks, bind_key=bind_key, fmt=fmt,
                                                       fbytes=fbytes).items()}
        dev = torch.device("cuda")
        self.dev: dict[str, Any] = {}
        if upload:
            self.dev = {k: to_dev(v) for k, v in corpus.arrays().items()}
        else:  # the caller copies in (e2e timing): allocate only
            self.dev = {k: torch.empty(v.nbytes, dtype=torch.uint8, device=dev)
                        for k, v in corpus.arrays().items()}
        m = max(n, 1)
        self.o = {"n_pred": torch.zeros(m, dtype=torch.int32, device=dev),
                  "pred_pat": torch.zeros(m * self.K, dtype=torch.int32, device=dev),
                  "pred_comp": torch.zeros(m * self.K, dtype=torch.uint8, device=dev),
                  "pred_arg": torch.full((m * self.K * self.B,), -1, dtype=torch.int64, device=dev),
                  "struct_err": torch.zeros(m, dtype=torch.int32, device=dev)}
        self.tallies = torch.zeros(4, dtype=torch.int64, device=dev)
        self.unsure = torch.zeros(m, dtype=torch.uint8, device=dev)
        if window_capacity < 1:
            raise ValueError("window capacity must be >= 1")
        o = self.o
        self.out = PredictOut(self.K, self.B, 1, 0, ptr(o["n_pred"]), ptr(o["pred_pat"]),
                              ptr(o["pred_comp"]), ptr(o["pred_arg"]), 0, 0, 0, 0,
                              ptr(o["struct_err"]))
        self.pool_desc = dp.desc(self.K, window_capacity)
        d, t = self.dev, self.tables
        self.desc = ReplayDesc(n, window_capacity, self.cand_limit, *[ptr(x) for x in (
            d["ev_tok"], d["ev_evt"], d["call_pos"], d["call_len"], d["call_tool"], d["call_args"],
            d["call_keyset"], t["pat_ks"], t["bind_key"], t["fmt"], t["fbytes"], d["nodes"],
            d["data"], d["refs"], self.tallies, self.unsure)])

    def upload_from(self, pinned: dict[str, Any], non_blocking: bool = True) -> int:
        """Copy host (pinned uint8 views) corpus arrays in; returns bytes."""
        total = 0
        for k, v in pinned.items():
            self.dev[k].copy_(v, non_blocking=non_blocking)
            total += v.numel()
        return total

    def launch(self, stream: int | None = None) -> None:
        from .device_ops import stream_handle

        self.tallies.zero_()
        check(self.lib.paste_replay_score(ctypes.byref(self.pool_desc), ctypes.byref(self.desc),
                                          ctypes.byref(self.out), stream_handle() if stream is None else stream), self.lib)

    def launch_fused(self, stream: int | None = None) -> bool:
        """The fused replay (paste_replay_fused: one kernel, no prediction
        records); False when the pool is outside its envelope (no match
        table for this window / K) -- use launch()."""
        from .device_ops import stream_handle

        self.tallies.zero_()
        rc = self.lib.paste_replay_fused(ctypes.byref(self.pool_desc), ctypes.byref(self.desc),
                                         self.K, stream_handle() if stream is None else stream)
        if rc == _native.PASTE_ERR_UNSUPPORTED:
            return False
        check(rc, self.lib)
        return True

    def launch_count(self) -> int:
        return int(self.lib.paste_last_launch_count())

    def host_recheck(self, actual, arena) -> int:
        """Hits among the unsure calls, decided with canonical_arg_hash."""
        from .events import canonical_arg_hash
        from .packing import PredictResult, decode_predictions

        rows = np.flatnonzero(self.unsure.cpu().numpy()[:self.corpus.n_calls])
        if not len(rows):
            return 0
        n, K, B = self.corpus.n_calls, self.K, self.B
        h = {k: v.cpu().numpy() for k, v in self.o.items()}
        res = PredictResult(K, B, h["n_pred"][:n], h["pred_pat"][:n * K], h["pred_comp"][:n * K],
                            h["pred_arg"][:n * K * B], None, None, None, None,
                            h["struct_err"][:n], 1).session_major()
        sub = PredictResult(K, B, res.n_pred[rows], res.pred_pat.reshape(n, K)[rows].reshape(-1),
                            res.pred_comp.reshape(n, K)[rows].reshape(-1),
                            res.pred_arg.reshape(n, K * B)[rows].reshape(-1), None, None, None,
                            None, res.struct_err[rows])
        preds = decode_predictions(sub, self.dp.image, arena, [0.0] * len(rows), 0.0)
        hits = 0
        lim = None if self.cand_limit == INT32_MAX else self.cand_limit
        for r, plist in zip(rows.tolist(), preds):
            ev = actual[r]
            want = canonical_arg_hash(ev.args)
            if any(p.completeness.value == "full" and p.tool_type == ev.tool_type
                   and canonical_arg_hash(p.args) == want for p in plist[:lim]):
                hits += 1
        return hits


def score_replay(traces, pool, window_capacity: int, max_candidates):
    from .device_ops import DevicePool
    from .prediction import AccuracyReport

    if window_capacity < 1:
        raise ValueError("window capacity must be >= 1")
    dp = DevicePool(pool)
    ksets = KeysetTable()
    corpus, actual, arena = corpus_from_traces(traces, dp, window_capacity, ksets)
    scored = corpus.n_calls
    if scored == 0:
        return AccuracyReport(0.0, 0.0, 0.0, 0)
    rb = ReplayBatch(dp, corpus, window_capacity, max_candidates, ksets)
    fused = rb.launch_fused()
    top1, top3, hits, unsure = (int(x) for x in rb.tallies.cpu().numpy())
    if unsure or not fused:  # undecided calls need the prediction records
        rb.launch()
        top1, top3, hits, unsure = (int(x) for x in rb.tallies.cpu().numpy())
        if unsure:
            hits += rb.host_recheck(actual, arena)
    return AccuracyReport(top1 / scored, top3 / scored, hits / scored, scored)
