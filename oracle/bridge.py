"""ctypes bridge to the CPU oracle (TEST INFRASTRUCTURE ONLY).

Imported by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs
to run oracle/paste_oracle.c on the same packed host arrays the device path
consumes.  The product package never imports this module.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_int, c_void_p

import numpy as np

from paper_2603_18897_b200._native import AdmitDesc, PoolDesc, PredictOut, WindowsDesc
from paper_2603_18897_b200.packing import PoolImage, PredictResult, WindowBatch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "libpaste_oracle.so")

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = ctypes.CDLL(LIB)
        _lib.oracle_predict_batch.restype = c_int
        _lib.oracle_predict_batch.argtypes = [POINTER(PoolDesc), c_char_p, POINTER(WindowsDesc),
                                              POINTER(AdmitDesc), POINTER(PredictOut), c_int]
    return _lib


def _p(a: np.ndarray | None) -> int:
    return 0 if a is None else a.ctypes.data


def pool_desc(im: PoolImage) -> tuple[PoolDesc, bytes, list]:
    keep = [im.patterns, im.bindings, im.ctx_sig, im.steps, im.bucket_off, im.bucket_pat,
            im.bucket_scan_all if len(im.bucket_scan_all) else np.zeros(1, np.uint8)]
    desc = PoolDesc(len(im.pool.patterns), im.n_bucket_sigs, im.k, im.relation, im.max_ctx,
                    im.max_bindings, *[_p(a) for a in keep], 0, 0, 0)
    pids = b"".join(pid.encode().ljust(16, b"\0") for pid in im.pattern_ids) or b"\0" * 16
    return desc, pids, keep


def predict(im: PoolImage, batch: WindowBatch, K: int,
            admit: tuple[np.ndarray, np.ndarray, np.ndarray] | None = None,
            new_tok: np.ndarray | None = None, new_ref: np.ndarray | None = None,
            new_evt_base: int = 0, new_byte_base: int = 0,
            threads: int = 1, out_slot_major: int = 0,
            stream_end: np.ndarray | None = None) -> PredictResult:
    """Run the oracle; like the device it mutates the window rings (and the
    event directory) when new_tok / new_ref are given."""
    desc, pids, keep = pool_desc(im)
    nodes, data, refs = batch.arena.arrays() if hasattr(batch.arena, "arrays") else batch.arena
    win = WindowsDesc(batch.n, batch.capacity, batch.slot_major, _p(batch.tok), _p(batch.evt), _p(batch.count),
                      _p(nodes), _p(data), _p(refs), _p(new_tok), _p(new_ref), new_evt_base,
                      new_byte_base, _p(stream_end))
    res = PredictResult.empty(batch.n, K, max(im.max_bindings, 1), admit is not None,
                              out_slot_major)
    if admit is not None:
        adm = AdmitDesc(1, len(admit[0]), *[_p(a) for a in admit])
    else:
        adm = AdmitDesc(0, 0, 0, 0, 0)
    out = PredictOut(K, res.B, out_slot_major, 0, _p(res.n_pred), _p(res.pred_pat), _p(res.pred_comp),
                     _p(res.pred_arg), _p(res.n_act), _p(res.act_pred), _p(res.act_level),
                     _p(res.act_util), _p(res.struct_err))
    rc = lib().oracle_predict_batch(ctypes.byref(desc), pids, ctypes.byref(win),
                                    ctypes.byref(adm), ctypes.byref(out), threads)
    if rc != 0:
        raise RuntimeError(f"oracle_predict_batch failed: {rc}")
    del keep
    return res


def mine_counts(tokens: np.ndarray, n_sigs: int, k: int, relation: int, threads: int = 1):
    """Oracle mining tables (tool_count, support, match, follow) as numpy;
    threads > 1 counts stream-aligned chunks in parallel and sums them."""
    L = lib()
    fn = L.oracle_mine_counts_mt
    fn.restype = c_int
    fn.argtypes = [c_void_p, ctypes.c_int64, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p,
                   c_void_p, c_int]
    T = (n_sigs + 1) // 2
    n_ctx = sum(n_sigs ** q for q in range(1, k + 1))
    tool_count = np.zeros(T, np.uint64)
    support = np.zeros(T * n_ctx, np.uint64)
    match = np.zeros(n_ctx, np.uint64)
    follow = np.zeros(n_ctx * T, np.uint64)
    tok = np.ascontiguousarray(tokens, np.int32)
    rc = fn(_p(tok), len(tok), n_sigs, k, relation, _p(tool_count), _p(support), _p(match),
            _p(follow), threads)
    if rc != 0:
        raise RuntimeError("oracle_mine_counts failed")
    return tool_count, support, match, follow


def select_candidates(tool_count, support, match, follow, n_sigs, k, sigma, tau):
    """Host restatement of the mine() gates over oracle tables:
    [(tool, ctx index, support, match, follow)] with follow/match >= tau."""
    T = (n_sigs + 1) // 2
    n_ctx = len(match)
    out = []
    sup = support.reshape(T, n_ctx)
    fol = follow.reshape(n_ctx, T)
    for t in range(T):
        if tool_count[t] < sigma:
            continue
        for c in np.flatnonzero(sup[t] >= sigma):
            m = int(match[c])
            if m and int(fol[c, t]) / m >= tau:
                out.append((t, int(c), int(sup[t, c]), m, int(fol[c, t])))
    return out


def greedy(p, benefit, duration, cost, ids, slack, budget) -> list[int]:
    """Oracle greedy selection: indices of the chosen jobs, in order."""
    fn = lib().oracle_greedy
    fn.restype = ctypes.c_int64
    fn.argtypes = [ctypes.c_int64] + [c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int64, c_void_p]
    arrs = [np.ascontiguousarray(a, dt) for a, dt in ((p, np.float64), (benefit, np.float64),
                                                      (duration, np.float64), (cost, np.int32),
                                                      (ids, np.int64))]
    out = np.zeros(max(len(arrs[0]), 1), np.int32)
    m = fn(len(arrs[0]), *[_p(a) for a in arrs], slack, budget, _p(out))
    return out[:m].tolist()


def leaf_scan(nodes, data, refs, target_off, target_bytes, node_budget=10_000, target_type=5,
              max_matches=4, threads=1):
    """Oracle candidate_paths over a tape batch: (n_out, first matches, truncated)."""
    from paper_2603_18897_b200._native import LeafScanDesc

    fn = lib().oracle_leaf_scan
    fn.restype = c_int
    fn.argtypes = [POINTER(LeafScanDesc), c_int]
    n = len(refs)
    arrs = dict(nodes=np.ascontiguousarray(nodes), data=np.ascontiguousarray(data),
                refs=np.ascontiguousarray(refs, np.int64), ev=np.arange(n, dtype=np.int32),
                tt=np.full(n, target_type, np.int32), tn=np.zeros(n, np.uint8),
                toff=np.ascontiguousarray(target_off, np.int64),
                tb=np.ascontiguousarray(target_bytes, np.uint8),
                oo=np.arange(n + 1, dtype=np.int64) * max_matches,
                out=np.zeros(n * max_matches, np.int32), n_out=np.zeros(n, np.int64),
                tr=np.zeros(n, np.uint8))
    d = LeafScanDesc(n, node_budget, *[_p(arrs[k]) for k in (
        "nodes", "data", "refs", "ev", "tt", "tn", "toff", "tb", "oo", "out", "n_out", "tr")])
    if fn(ctypes.byref(d), threads) != 0:
        raise RuntimeError("oracle_leaf_scan failed")
    return arrs["n_out"], arrs["out"].reshape(n, max_matches), arrs["tr"]


def score_corpus(im: PoolImage, corpus, keys, window_capacity: int, max_candidates,
                 threads: int = 1, calls: slice | None = None,
                 stream: bool = True) -> tuple[int, int, int, int]:
    """score_accuracy (prediction.py:133-169) over a ReplayCorpus with the C
    oracle's predictions and the Python canonical_arg_hash check.  Returns
    (top1, top3, hits, scored) over ``calls`` (default: all)."""
    from paper_2603_18897_b200.events import canonical_arg_hash
    from paper_2603_18897_b200.packing import WindowBatch, decode_predictions
    from paper_2603_18897_b200.tape import ArrayTapes

    W = window_capacity
    sl = calls or slice(None)
    pos = corpus.call_pos[sl]
    lens = corpus.call_len[sl].astype(np.int64)
    n = len(pos)
    if n == 0:
        return 0, 0, 0, 0
    tapes = ArrayTapes(corpus.nodes, corpus.data, corpus.refs, keys)
    if stream:  # windows read in place (paste_windows stream mode)
        tok, evt = corpus.ev_tok, corpus.ev_evt
        stream_end = np.ascontiguousarray(pos, np.int64)
    else:  # gathered [n][W] rings
        idx = (pos - lens)[:, None] + np.arange(W)[None, :]
        valid = np.arange(W)[None, :] < lens[:, None]
        idx = np.where(valid, idx, 0)
        tok = np.where(valid, corpus.ev_tok[idx], -1).astype(np.int32).reshape(-1)
        evt = np.where(valid, corpus.ev_evt[idx], -1).astype(np.int32).reshape(-1)
        stream_end = None
    if max_candidates is not None and max_candidates > 0:
        K, lim = max_candidates, None
    else:
        K, lim = max(im.max_bucket, 1), max_candidates
    batch = WindowBatch(W, tok, evt, np.ascontiguousarray(lens, np.int64), tapes, [None] * n)
    res = predict(im, batch, K, threads=threads, stream_end=stream_end)
    tool_of = im.patterns["target_tool"]
    act_tool = corpus.call_tool[sl]
    args_pid = corpus.call_args[sl]
    preds = decode_predictions(res, im, tapes, [0.0] * n, 0.0)
    top1 = top3 = hits = 0
    for r, plist in enumerate(preds):
        plist = plist[:lim]
        pats = [int(res.pred_pat[r * K + i]) for i in range(len(plist))]
        tools = [int(tool_of[p]) for p in pats]
        t = int(act_tool[r])
        top1 += bool(tools) and tools[0] == t
        top3 += t in tools[:3]
        cand = [p for p, pt in zip(plist, tools) if pt == t and p.completeness.value == "full"]
        if cand:
            want = canonical_arg_hash(tapes.node_object(int(args_pid[r]), 0))
            hits += any(canonical_arg_hash(p.args) == want for p in cand)
    return top1, top3, hits, n
