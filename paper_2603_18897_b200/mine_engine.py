"""Device mining engine: packing, K2 count / expand / select, Phase II glue.

``mine()`` (mining.py:248-292) becomes:

1. pack every session's tool events into one flagged token stream (tools
   interned in sorted name order, so sig order == the reference's
   (tool_type, status.value) order);
2. K2 on the device: (k+1)-gram histogram -> tool_count / support / match /
   follow tables -> candidate (target, context) pairs that clear sigma and
   whose follow/match bound clears tau (libpaste: paste_mine_*);
3. per candidate, Phase II mapping inference on its occurrences (host, see
   phase2.py) and p = hits / matches;
4. the reference's deterministic output order (_sort_key, mining.py:105-111).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Any, Sequence

import numpy as np

from . import _native
from ._native import MineDesc, check, ptr
from .events import Event, EventSignature, Session, Status, signature_of
from .mappings import MatchedContext, ValueMapping
from .mining import MatchRelation, MiningConfig, PatternTuple, pattern_sort_key
from .packing import SigTable
from . import phase2

SEG_START = np.int32(-2**31)


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# packing
# ---------------------------------------------------------------------------

def pack_streams(streams: Sequence[Sequence[Event]], sigs: SigTable) -> np.ndarray:
    """Flagged token stream: sig ids, bit 31 on each stream's first event."""
    total = sum(len(s) for s in streams)
    tok = np.empty(total, np.int32)
    at = 0
    for st in streams:
        for i, ev in enumerate(st):
            t = sigs.sig(ev.tool_type, ev.status)
            tok[at] = t | SEG_START if i == 0 else t
            at += 1
    return tok


def ctx_offsets(S: int, k: int) -> list[int]:
    off = [0, 0]
    for n in range(1, k + 1):
        off.append(off[-1] + S ** n)
    return off


def decode_context(idx: int, S: int, k: int) -> tuple[int, ...]:
    off = ctx_offsets(S, k)
    n = next(n for n in range(1, k + 1) if off[n] <= idx < off[n + 1])
    v = idx - off[n]
    out = []
    for _ in range(n):
        out.append(v % S)
        v //= S
    return tuple(reversed(out))


def encode_context(ctx: Sequence[int], S: int, k: int) -> int:
    v = 0
    for c in ctx:
        v = v * S + c
    return ctx_offsets(S, k)[len(ctx)] + v


# ---------------------------------------------------------------------------
# device tables
# ---------------------------------------------------------------------------

@dataclass
class MineTables:
    """Device-resident K2 state for one (n_sigs, k, relation) geometry."""

    n_sigs: int
    k: int
    relation: int
    n_bins: int
    n_ctx: int
    hist: Any
    tool_count: Any
    support: Any
    match: Any
    follow: Any

    @classmethod
    def allocate(cls, n_sigs: int, k: int, relation: int) -> "MineTables":
        torch = _torch()
        lib = _native.lib()
        nb, nc = ctypes.c_int64(), ctypes.c_int64()
        check(lib.paste_mine_geometry(n_sigs, k, ctypes.byref(nb), ctypes.byref(nc)), lib)
        T = (n_sigs + 1) // 2
        dev = torch.device("cuda")
        nc_ = nc.value
        # the four u64 tables share one allocation (one memset per expand)
        flat = torch.zeros(T + 2 * T * nc_ + nc_, dtype=torch.int64, device=dev)
        tool_count, support, match, follow = torch.split(flat, [T, T * nc_, nc_, nc_ * T])
        t = cls(n_sigs, k, relation, nb.value, nc_,
                torch.zeros(nb.value, dtype=torch.int32, device=dev),
                tool_count, support, match, follow)
        t._flat = flat
        return t

    def desc(self, tokens=None, n_tokens: int = 0) -> MineDesc:
        return MineDesc(self.n_sigs, self.k, self.relation, 0, ptr(tokens), n_tokens,
                        ptr(self.hist), ptr(self.tool_count), ptr(self.support), ptr(self.match),
                        ptr(self.follow))

    def count(self, tokens) -> None:
        """Accumulate the (k+1)-gram histogram of a device token stream."""
        from .device_ops import stream_handle

        lib = _native.lib()
        d = self.desc(tokens, int(tokens.numel()))
        check(lib.paste_mine_count(ctypes.byref(d), stream_handle()), lib)

    def expand(self) -> None:
        from .device_ops import stream_handle

        lib = _native.lib()
        self._flat.zero_()
        d = self.desc()
        check(lib.paste_mine_expand(ctypes.byref(d), stream_handle()), lib)

    def select_sorted(self, sigma: int, tau: float, cap: int | None = None,
                      done_event=None) -> "MinedTable":
        """Mapping-free patterns in mine()'s output order, selected and sorted
        on the device (paste_mine_select_sorted) and read back as one table.
        ``done_event`` (a torch.cuda.Event) is recorded on the stream right
        after the table's device-to-host copy, i.e. when the result is in
        host memory, before the host wraps it."""
        from .device_ops import stream_handle

        torch = _torch()
        lib = _native.lib()
        st = getattr(self, "_sel", None)
        cap = cap or (st["cap"] if st else 1 << 14)
        while True:
            if st is None or st["cap"] < cap:
                st = {"cap": cap,
                      "n": torch.zeros(1, dtype=torch.int64, device="cuda"),
                      "out": torch.empty(6 * cap, dtype=torch.int64, device="cuda"),
                      "scratch": torch.empty(lib.paste_mine_sort_scratch_bytes(cap),
                                             dtype=torch.uint8, device="cuda"),
                      "n_h": torch.empty(1, dtype=torch.int64, pin_memory=True),
                      "out_h": torch.empty(6 * cap, dtype=torch.int64, pin_memory=True),
                      "last": st["last"] if st else 0}
                self._sel = st
            d = self.desc()
            check(lib.paste_mine_select_sorted(ctypes.byref(d), sigma, float(tau), st["cap"],
                                               ptr(st["n"]), ptr(st["out"]), ptr(st["scratch"]),
                                               stream_handle()), lib)
            # one round trip in the common case: the count and the first
            # `guess` rows (last step's size + slack) come back together
            guess = min(st["cap"], max(st.get("last", 0) * 5 // 4, 1024))
            st["n_h"].copy_(st["n"], non_blocking=True)
            st["out_h"][:6 * guess].copy_(st["out"][:6 * guess], non_blocking=True)
            stream = torch.cuda.current_stream()
            if done_event is not None:
                done_event.record(stream)
            stream.synchronize()
            m = int(st["n_h"][0])
            if m <= st["cap"]:
                if m > guess:
                    st["out_h"][:6 * m].copy_(st["out"][:6 * m], non_blocking=True)
                    if done_event is not None:
                        done_event.record(stream)
                    stream.synchronize()
                st["last"] = m
                return MinedTable(st["out_h"][:6 * m].numpy().reshape(m, 6).copy(), self.n_sigs,
                                  self.k)
            cap = m

    def select(self, sigma: int, tau: float) -> np.ndarray:
        """Candidates [m, 5] = (tool, ctx index, support, match, follow)."""
        from .device_ops import stream_handle

        torch = _torch()
        lib = _native.lib()
        cap = 1 << 16
        while True:
            n_out = torch.zeros(1, dtype=torch.int64, device="cuda")
            out = torch.empty(5 * cap, dtype=torch.int64, device="cuda")
            d = self.desc()
            check(lib.paste_mine_select(ctypes.byref(d), sigma, float(tau), cap, ptr(n_out),
                                        ptr(out), stream_handle()), lib)
            m = int(n_out.item())
            if m <= cap:
                return out[:5 * m].view(m, 5).cpu().numpy()
            cap = m


# ---------------------------------------------------------------------------
# host matching (Phase II occurrences and the match_at utility)
# ---------------------------------------------------------------------------

def match_events(stream: Sequence[Event], sig_stream: Sequence, anchor: int, context: Sequence,
                 k: int, relation: MatchRelation) -> MatchedContext | None:
    """match_at over a precomputed signature stream (mining.py:119-156)."""
    n = len(context)
    if n == 0 or anchor >= len(stream) or sig_stream[anchor] != context[-1]:
        return None
    if relation is MatchRelation.CONTIGUOUS_SUFFIX:
        start = anchor - n + 1
        if start < 0 or any(sig_stream[start + i] != context[i] for i in range(n)):
            return None
        sl = tuple(stream[start:anchor + 1])
        return MatchedContext(events=sl, history=sl)
    lo = max(0, anchor - k + 1)
    picked = [anchor]
    j, pos = n - 2, anchor - 1
    while j >= 0 and pos >= lo:
        if sig_stream[pos] == context[j]:
            picked.append(pos)
            j -= 1
        pos -= 1
    if j >= 0:
        return None
    picked.reverse()
    return MatchedContext(events=tuple(stream[p] for p in picked),
                          history=tuple(stream[picked[0]:anchor + 1]))


def match_at(stream, anchor, context, k, relation):
    sig_stream = [signature_of(e) for e in stream]
    return match_events(stream, sig_stream, anchor, context, k, relation)


def device_occurrences(tok_dev, flat_events: Sequence[Event], sigs: SigTable, cands: list,
                       cfg: MiningConfig) -> list[list]:
    """Phase II occurrence lists for many candidates at once on the device
    (paste_mine_occurrences + the K1 sort for stream order): for every
    (context sig tuple, target tool id, follow count) in ``cands`` the
    (MatchedContext, next event) pairs of _collect_occurrences whose next
    event is the target (mining.py:215-227,277-279), in stream order.  The
    host only wraps the device's positions in the reference's objects."""
    rel = cfg.match_relation is MatchRelation.CONTIGUOUS_SUFFIX
    out = []
    for (cs, _tool, _f), (anc, pk) in zip(cands, occurrence_positions(tok_dev, sigs, cands, cfg)):
        L = len(cs)
        occ = []
        for r in range(len(anc)):
            a = int(anc[r])
            if rel:
                sl = tuple(flat_events[a - L + 1:a + 1])
                m = MatchedContext(events=sl, history=sl)
            else:
                pos = pk[r].tolist()
                m = MatchedContext(events=tuple(flat_events[p] for p in pos),
                                   history=tuple(flat_events[pos[0]:a + 1]))
            occ.append((m, flat_events[a + 1]))
        out.append(occ)
    return out


def occurrence_positions(tok_dev, sigs: SigTable, cands: list, cfg: MiningConfig) -> list:
    """Per candidate (anchors int64[M], matched positions int32[M, len(ctx)])
    in stream order, from one device pass (paste_mine_occurrences) and the K1
    sort (candidate = session, anchor = t_start)."""
    from .device_ops import stream_handle
    from ._native import OccDesc

    torch = _torch()
    lib = _native.lib()
    C = len(cands)
    if C == 0:
        return []
    kmax = max(len(c[0]) for c in cands)
    if tok_dev is None:
        return [(np.zeros(0, np.int64), np.zeros((0, len(c[0])), np.int32)) for c in cands]
    n_tools = (sigs.n_sigs + 1) // 2
    ctx = np.zeros((C, kmax), np.int32)
    ctx_len = np.zeros(C, np.int32)
    follow = np.zeros(C, np.int64)
    keys = np.zeros(C, np.int64)
    for i, (cs, tool, f) in enumerate(cands):
        ctx[i, :len(cs)] = cs
        ctx_len[i] = len(cs)
        follow[i] = f
        keys[i] = cs[-1] * n_tools + tool
    order = np.argsort(keys, kind="stable")
    bucket_off = np.zeros(sigs.n_sigs * n_tools + 1, np.int32)
    np.add.at(bucket_off, keys + 1, 1)
    bucket_off = np.cumsum(bucket_off).astype(np.int32)
    off = np.zeros(C + 1, np.int64)
    off[1:] = np.cumsum(follow)
    total = int(off[-1])
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in dict(
        ctx=ctx.reshape(-1), ctx_len=ctx_len, bucket_off=bucket_off,
        bucket=order.astype(np.int32), off=off).items()}
    cursor = torch.zeros(C, dtype=torch.int64, device="cuda")
    anchor = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    picked = torch.empty(max(total, 1) * kmax, dtype=torch.int32, device="cuda")
    overflow = torch.zeros(1, dtype=torch.int64, device="cuda")
    rel = 0 if cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1
    d = OccDesc(int(tok_dev.numel()), ptr(tok_dev), C, cfg.k, rel, kmax, sigs.n_sigs, n_tools,
                ptr(dev["ctx"]), ptr(dev["ctx_len"]), ptr(dev["bucket_off"]), ptr(dev["bucket"]),
                ptr(dev["off"]), ptr(cursor), ptr(anchor), ptr(picked), ptr(overflow))
    check(lib.paste_mine_occurrences(ctypes.byref(d), stream_handle()), lib)
    # stream order inside every candidate's range: the K1 sort, candidate =
    # session, anchor = t_start (slots are grouped by candidate already)
    slot_cand = torch.repeat_interleave(torch.arange(C, dtype=torch.int32, device="cuda"),
                                        torch.from_numpy(follow).cuda())
    t = anchor[:total].to(torch.float64)
    zeros = torch.zeros(total, dtype=torch.int32, device="cuda")
    srt = order_columnar({"session": slot_cand, "seq": zeros, "t_start": t, "t_end": t,
                          "sig": zeros}, C, float("inf"), with_order=True)
    if int(overflow.item()) or int(cursor.sum().item()) != total:
        raise _native.PasteError("occurrence counts disagree with the follow table")
    perm = srt.order.long()
    anc = anchor[:total][perm].cpu().numpy()
    pk = picked.view(-1, kmax)[:total][perm].cpu().numpy()
    return [(anc[off[i]:off[i + 1]], pk[off[i]:off[i + 1], :len(cands[i][0])])
            for i in range(C)]


def _occurrences(streams, sig_streams, context: tuple, target: str, cfg: MiningConfig):
    """(matched, next) pairs whose next event is ``target``, in stream order."""
    occ = []
    for st, sg in zip(streams, sig_streams):
        for a in range(len(st) - 1):
            if st[a + 1].tool_type != target or sg[a] != context[-1]:
                continue
            m = match_events(st, sg, a, context, cfg.k, cfg.match_relation)
            if m is not None:
                occ.append((m, st[a + 1]))
    return occ


# ---------------------------------------------------------------------------
# public entry points
# ---------------------------------------------------------------------------

def _gather(obj, group) -> list:
    import torch.distributed as dist

    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


def _count_corpus(streams, cfg: MiningConfig, group=None):
    torch = _torch()
    tools = {e.tool_type for st in streams for e in st}
    if group is not None:  # one signature table for every shard
        tools = set().union(*_gather(tools, group))
    sigs = SigTable(sorted(tools))
    relation = 0 if cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1
    tables = MineTables.allocate(max(sigs.n_sigs, 2), cfg.k, relation)
    tok = pack_streams(streams, sigs)
    tok_dev = None
    if len(tok):
        tok_dev = torch.from_numpy(tok).cuda()
        tables.count(tok_dev)
    if group is not None:  # K3: shards are whole sessions, histograms add up
        import torch.distributed as dist

        dist.all_reduce(tables.hist, group=group)
    tables.expand()
    return sigs, tables, tok_dev


def _local_follow(tables: "MineTables", tok_dev, rows: list, S: int, cfg: MiningConfig) -> list:
    """This shard's follow counts of the given candidates (the merged tables
    hold the corpus totals): a count pass over the shard alone."""
    if tok_dev is None:
        return [0] * len(rows)
    local = MineTables.allocate(tables.n_sigs, tables.k, tables.relation)
    local.count(tok_dev)
    local.expand()
    T = (local.n_sigs + 1) // 2
    fol = local.follow.cpu().numpy()
    return [int(fol[cidx * T + tool]) for tool, cidx, *_ in rows]


def _phase2(occ, cfg: MiningConfig, hits: int):
    """Mapping inference for one candidate and its hit count (K7 on device)."""
    from . import phase2_device

    if len(occ) < 2 or not phase2.common_scalar_args(occ):
        return None, hits
    if phase2_device._aliased_histories(occ):
        mapping = phase2.infer_mapping(occ, cfg.validation_fraction)
        if mapping is None:
            return None, hits
        return mapping, sum(1 for m, nxt in occ if phase2.mapping_holds(mapping, m, nxt))
    occs = phase2_device.OccurrenceSet(occ, occ[0][1].tool_type)
    mapping = phase2_device.infer_mapping(occ, cfg.validation_fraction, occs)
    if mapping is None:
        return None, hits
    return mapping, phase2_device.count_mapping_hits(mapping, occs)


def _phase2_corpus(tok_dev, flat, sigs: SigTable, rows: list, idx: list, S: int,
                   cfg: MiningConfig, corpus=None) -> dict:
    """Phase II of every candidate over one corpus tape (phase2_corpus.py):
    occurrence positions from the device pass, the argument test, hypothesis
    scoring and mapping_holds counts on the device."""
    from . import phase2_corpus as pc

    cands = [(decode_context(r[1], S, cfg.k), r[0], r[4]) for r in rows]
    positions = occurrence_positions(tok_dev, sigs, cands, cfg)
    tok_host = tok_dev.cpu().numpy() if tok_dev is not None else np.zeros(0, np.int32)
    ct = None
    out = {}
    for i, r, (anc, pk) in zip(idx, rows, positions):
        first = flat[int(anc[0]) + 1].args if len(anc) else None
        if len(anc) < 2 or not isinstance(first, dict) or not first:
            out[i] = (None, r[4])
            continue
        if ct is None:
            try:
                ct = corpus() if corpus is not None else \
                    pc.CorpusTapes.from_events(flat, tok_host, tok_dev, sigs)
            except TypeError:
                # a payload the tape cannot hold (not JSON-like) somewhere in the
                # corpus: per-candidate occurrence sets, as in the sharded path
                ct = False
        if ct is False:
            occ = device_occurrences(tok_dev, flat, sigs, [cands[idx.index(i)]], cfg)[0]
            out[i] = _phase2(occ, cfg, r[4])
            continue
        co = pc.CorpusOccurrences(ct, anc, pk, sigs.tools[r[0]])
        mapping = pc.infer_mapping(co, cfg.validation_fraction)
        out[i] = (None, r[4]) if mapping is None else (mapping, pc.count_mapping_hits(mapping, co))
    return out


def mine(traces: Sequence[Session], cfg: MiningConfig, group=None) -> list[PatternTuple]:
    """mine() (mining.py:248-292).  With a torch.distributed ``group`` every
    rank passes its shard -- a contiguous range of the sessions, ranks in
    session order -- counts it on its device, and the (k+1)-gram histograms
    are all-reduced; Phase II sees every candidate's occurrences gathered in
    rank (= stream) order, so every rank returns the single-device result."""
    if group is not None:
        if not sum(_gather(len(traces), group)):
            raise ValueError("traces must be non-empty")
    elif not traces:
        raise ValueError("traces must be non-empty")
    streams = [s.tool_events() for s in traces]
    sigs, tables, tok_dev = _count_corpus(streams, cfg, group)
    flat = [e for st in streams for e in st]
    return _select_patterns(tables, sigs, tok_dev, flat, cfg, group)


def _select_patterns(tables: "MineTables", sigs: SigTable, tok_dev, flat: Sequence, cfg,
                     group=None, corpus=None) -> list[PatternTuple]:
    """Selection + Phase II + the reference's order (mining.py:264-292) over a
    counted corpus: ``flat`` maps stream positions to events (a list, or a
    lazy view over tapes); ``corpus`` builds the CorpusTapes on first need."""
    cands = tables.select(cfg.sigma, cfg.tau)
    if group is not None:  # the select kernel compacts with atomics: fix one order for all ranks
        cands = cands[np.lexsort((cands[:, 1], cands[:, 0]))]
    S = tables.n_sigs
    rows = cands.tolist()
    # Phase II occurrences of every candidate that can carry a mapping, from
    # one device pass; under sharding each rank collects its shard (its own
    # follow counts) and the lists are gathered in rank = stream order
    need = [i for i, r in enumerate(rows) if r[4] >= 2]
    phase2_of: dict[int, tuple] = {}
    if need:
        if group is not None:  # this shard's follow counts size the slots
            local = _local_follow(tables, tok_dev, [rows[i] for i in need], S, cfg)
            lists = device_occurrences(
                tok_dev, flat, sigs, [(decode_context(rows[i][1], S, cfg.k), rows[i][0], f)
                                      for i, f in zip(need, local)], cfg)
            for i, occ in zip(need, lists):
                occ = [o for part in _gather(occ, group) for o in part]
                phase2_of[i] = _phase2(occ, cfg, rows[i][4])
        else:
            phase2_of = _phase2_corpus(tok_dev, flat, sigs, [rows[i] for i in need], need, S,
                                       cfg, corpus)
    patterns = []
    for i, (tool, cidx, support, n_match, follow) in enumerate(rows):
        context = tuple(sigs.signature(x) for x in decode_context(cidx, S, cfg.k))
        target = sigs.tools[tool]
        mapping = None
        hits = follow
        if follow >= 2:
            mapping, hits = phase2_of[i]
        p = hits / n_match
        if p >= cfg.tau:
            patterns.append(PatternTuple(context=context, target=target, mapping=mapping, p=p,
                                         support=support))
    patterns.sort(key=pattern_sort_key)
    return patterns


def validate(context, target: str, mapping: ValueMapping | None, traces: Sequence[Session],
             cfg: MiningConfig | None = None) -> float:
    cfg = cfg or MiningConfig()
    if not context:  # match_at never matches an empty context (mining.py:128-130)
        raise ValueError("context has no matches in the given traces")
    streams = [s.tool_events() for s in traces]
    if len(context) > cfg.k and cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE:
        raise ValueError("context has no matches in the given traces")
    tools = sorted({e.tool_type for st in streams for e in st} | {s.tool_type for s in context}
                   | {target})
    sigs = SigTable(tools)
    relation = 0 if cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1
    k = max(cfg.k, len(context))
    tables = MineTables.allocate(max(sigs.n_sigs, 2), k, relation)
    torch = _torch()
    tok = pack_streams(streams, sigs)
    tok_dev = torch.from_numpy(tok).cuda() if len(tok) else None
    if tok_dev is not None:
        tables.count(tok_dev)
    tables.expand()
    cidx = encode_context([sigs.sig_of(s) for s in context], tables.n_sigs, k)
    n_match = int(tables.match[cidx].item())
    if n_match == 0:
        raise ValueError("context has no matches in the given traces")
    follow = int(tables.follow[cidx * ((tables.n_sigs + 1) // 2) + sigs.tool(target)].item())
    if mapping is None:
        return follow / n_match
    ctx_sigs = tuple(sigs.sig_of(s) for s in context)
    occ = device_occurrences(tok_dev, [e for st in streams for e in st], sigs,
                             [(ctx_sigs, sigs.tool(target), follow)], cfg)[0] if follow else []
    if not occ:
        return 0.0
    from . import phase2_device

    if phase2_device._aliased_histories(occ):
        hits = sum(1 for m, nxt in occ if phase2.mapping_holds(mapping, m, nxt))
    else:
        hits = phase2_device.count_mapping_hits(
            mapping, phase2_device.OccurrenceSet(occ, occ[0][1].tool_type))
    return hits / n_match


def frequent_subsequences(windows, sigma: int) -> dict:
    """Distinct-subsequence support over arbitrary windows (mining.py:164-183):
    each window becomes a segment ``window + [probe]`` and its support is
    read from the probe tool's row of the device support table."""
    torch = _torch()
    windows = [tuple(w) for w in windows]
    kmax = max((len(w) for w in windows), default=0)
    if kmax == 0:
        return {}
    if kmax > 6:
        raise _native.PasteUnsupported("windows longer than 6 signatures")
    tools = sorted({s.tool_type for w in windows for s in w})
    probe = "\x00probe"
    sigs = SigTable(tools + [probe])
    tables = MineTables.allocate(sigs.n_sigs, kmax, 0)
    toks = []
    for w in windows:
        seg = [sigs.sig_of(s) for s in w] + [sigs.sig(probe, Status.SUCCESS)]
        seg[0] |= int(SEG_START)
        toks += seg
    tables.count(torch.from_numpy(np.array(toks, np.int32)).cuda())
    tables.expand()
    row = tables.support[sigs.tool(probe) * tables.n_ctx:(sigs.tool(probe) + 1) * tables.n_ctx]
    sup = row.cpu().numpy()
    out = {}
    for cidx in np.flatnonzero(sup >= sigma):
        ctx = decode_context(int(cidx), tables.n_sigs, kmax)
        if any(c == sigs.sig(probe, Status.SUCCESS) or c == sigs.sig(probe, Status.FAIL)
               for c in ctx):
            continue
        out[tuple(sigs.signature(c) for c in ctx)] = int(sup[cidx])
    return out


# ---------------------------------------------------------------------------
# columnar traces (K1 + K2 fused) and sharded mining (K3)
# ---------------------------------------------------------------------------

def ingest_count(tables: MineTables, trace: dict, inactivity_ms: float = 300_000.0,
                 tokens_out=None, staged: bool = True):
    """Fused ingest + count of a device-resident columnar trace into
    ``tables.hist``; returns device counters (n_segments, n_unsorted).
    ``staged`` runs the two-pass count (paste_mine_ingest_count_staged) with
    a staging buffer cached on ``tables``."""
    from .device_ops import stream_handle
    from ._native import ColumnarDesc

    torch = _torch()
    lib = _native.lib()
    counters = getattr(tables, "_counters", None)
    if counters is None:
        counters = tables._counters = torch.zeros(2, dtype=torch.int64, device="cuda")
    else:
        counters.zero_()
    n = int(trace["sig"].numel())
    c = ColumnarDesc(n, ptr(trace["session"]), ptr(trace["seq"]), ptr(trace["t_start"]),
                     ptr(trace["t_end"]), ptr(trace["sig"]), float(inactivity_ms), ptr(tokens_out),
                     ptr(counters), ptr(counters) + 8)
    d = tables.desc()
    if staged and tokens_out is None:
        need = int(lib.paste_mine_stage_bytes(n, tables.n_sigs, tables.k))
        buf = getattr(tables, "_stage", None)
        if buf is None or buf.numel() < need:
            buf = tables._stage = torch.empty(max(need, 16), dtype=torch.uint8, device="cuda")
        check(lib.paste_mine_ingest_count_staged(ctypes.byref(c), ctypes.byref(d), ptr(buf),
                                                 buf.numel(), stream_handle()), lib)
    else:
        check(lib.paste_mine_ingest_count(ctypes.byref(c), ctypes.byref(d), stream_handle()), lib)
    return counters


def patterns_from_candidates(cands: np.ndarray, sigs: SigTable, S: int, cfg: MiningConfig):
    """Mapping-free patterns (columnar traces carry no payloads): p = follow /
    match, the tau gate, and the reference's output order."""
    if len(cands) == 0:
        return []
    cands = np.asarray(cands, np.int64).reshape(-1, 5)
    p = cands[:, 4] / cands[:, 3]  # IEEE division of exact ints == Python's int / int
    cands, p = cands[p >= cfg.tau], p[p >= cfg.tau]
    # decode context indices into (length, digits) without Python loops
    off = np.array(ctx_offsets(S, cfg.k), np.int64)
    cidx = cands[:, 1]
    length = np.searchsorted(off[1:], cidx, side="right")
    local = cidx - off[length]
    digits = np.zeros((len(cands), cfg.k), np.int64)
    for d in range(cfg.k):  # most significant first, left-aligned
        shift = length - 1 - d
        ok = shift >= 0
        digits[ok, d] = (local[ok] // (S ** shift[ok])) % S
    # the reference order (mining.py:105-111): -p, -len, target name, context;
    # sig ids preserve (tool_type, status.value) order (sorted interning)
    keys = [digits[:, d] for d in reversed(range(cfg.k))] + [cands[:, 0], -length, -p]
    order = np.lexsort(keys)
    sig_obj = [sigs.signature(x) for x in range(S)]
    # contexts are non-empty and 0 < tau <= p <= 1 by construction, so the
    # frozen dataclass is filled directly (its __init__ + validation would
    # dominate the host side of a 100M-event mining step)
    new, cls = object.__new__, PatternTuple
    out = []
    lens = length[order].tolist()
    digs = digits[order].tolist()
    tools = cands[order, 0].tolist()
    sups = cands[order, 2].tolist()
    ps = p[order].tolist()
    for n, dg, t, sup, pv in zip(lens, digs, tools, sups, ps):
        obj = new(cls)
        obj.__dict__.update(context=tuple(sig_obj[x] for x in dg[:n]), target=sigs.tools[t],
                            mapping=None, p=pv, support=sup)
        out.append(obj)
    return out


class MinedTable:
    """mine()'s mapping-free output as sorted columns (rows of (tool, context
    index, support, match, follow, p)), the form the device returns and a
    pool image is compiled from.  ``patterns()`` materialises the reference's
    ``list[PatternTuple]`` (same order, same values)."""

    __slots__ = ("rows", "n_sigs", "k")

    def __init__(self, rows: np.ndarray, n_sigs: int, k: int):
        self.rows, self.n_sigs, self.k = rows, n_sigs, k

    def __len__(self) -> int:
        return len(self.rows)

    @property
    def p(self) -> np.ndarray:
        return self.rows[:, 5].view(np.float64)

    def patterns(self, sigs: SigTable) -> list[PatternTuple]:
        if len(self.rows) == 0:
            return []
        import gc

        enabled = gc.isenabled()
        gc.disable()  # thousands of small acyclic objects: skip the gen-0 scans
        try:
            return self._materialize(sigs)
        finally:
            if enabled:
                gc.enable()

    def _materialize(self, sigs: SigTable) -> list[PatternTuple]:
        S, k = self.n_sigs, self.k
        rows = self.rows
        # one context tuple per distinct context index
        uniq, inv = np.unique(rows[:, 1], return_inverse=True)
        off = np.array(ctx_offsets(S, k), np.int64)
        length = np.searchsorted(off[1:], uniq, side="right")
        local = uniq - off[length]
        sig_obj = [sigs.signature(x) for x in range(S)]
        ctxs = []
        for n, v in zip(length.tolist(), local.tolist()):
            dg = []
            for _ in range(n):
                v, r = divmod(v, S)
                dg.append(sig_obj[r])
            dg.reverse()
            ctxs.append(tuple(dg))
        ctx_of = [ctxs[i] for i in inv.tolist()]
        tools = [sigs.tools[t] for t in range(len(sigs.tools))]
        # contexts are non-empty and 0 < tau <= p <= 1 by construction: fill the
        # frozen dataclass directly (its validating __init__ would dominate)
        new, cls = object.__new__, PatternTuple
        out = []
        append = out.append
        for ctx, t, sup, pv in zip(ctx_of, rows[:, 0].tolist(), rows[:, 2].tolist(),
                                   self.p.tolist()):
            obj = new(cls)
            obj.__dict__.update(context=ctx, target=tools[t], mapping=None, p=pv, support=sup)
            append(obj)
        return out


def sharded_tail(tables: "MineTables", group, sigma: int, tau: float) -> "MinedTable":
    """The target-sliced mining tail: every rank expands one
    block of histogram columns and selects the candidates of its tools, so
    the expansion and selection work falls with the rank count.

      * support / follow / tool_count of target t read only column s0 in
        {2t, 2t+1} (the gram's last symbol); match[c] reads only the grams
        whose last symbol is c's last symbol (the anchor).  The histogram is
        transposed to s0-major blocks (paste_mine_transpose_slices) and
        reduce-scattered: rank r receives block r summed over the shards;
      * paste_mine_expand_slice fills the rank's tools' tables and the
        match of the contexts anchored in its block; one all-reduce (sum)
        of the match array (n_ctx u64) completes it;
      * each rank selects + sorts its own candidates on the device; the
        sorted rows (a few thousand) are all-gathered and merged in the
        reference's order (-p, -len, target, context).
    Every rank returns the single-device table."""
    import torch.distributed as dist

    from .device_ops import stream_handle

    torch = _torch()
    lib = _native.lib()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    w = int(lib.paste_mine_slice_cols(tables.n_sigs, world))
    base = tables.n_sigs + 2
    n_win = tables.n_bins // base
    d = tables.desc()
    hist_t = torch.empty(world * w * n_win, dtype=torch.int32, device="cuda")
    check(lib.paste_mine_transpose_slices(ctypes.byref(d), world, ptr(hist_t), stream_handle()), lib)
    if dist.get_backend(group) == "nccl":
        block = torch.empty(w * n_win, dtype=torch.int32, device="cuda")
        dist.reduce_scatter_tensor(block, hist_t, group=group)
    else:  # gloo has no reduce-scatter: sum everything, keep this rank's block
        dist.all_reduce(hist_t, group=group)
        block = hist_t[rank * w * n_win:(rank + 1) * w * n_win].contiguous()
    for t in (tables.tool_count, tables.support, tables.match, tables.follow):
        t.zero_()
    check(lib.paste_mine_expand_slice(ctypes.byref(d), ptr(block), rank * w, w, stream_handle()),
          lib)
    dist.all_reduce(tables.match, group=group)
    mine = tables.select_sorted(sigma, tau)
    return merge_sorted_tables(mine.rows, tables.n_sigs, tables.k, group)


def merge_sorted_tables(rows: np.ndarray, n_sigs: int, k: int, group) -> "MinedTable":
    """All-gather every rank's sorted selection rows (tool, context, support,
    match, follow, p bits) and merge them in mine()'s order (-p, -len,
    target, context): the device sort key (hi = ~bits(p), lo = (k - len,
    tool, context digits)) restated in numpy."""
    import torch.distributed as dist

    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, np.asarray(rows, np.int64), group=group)
    rows = np.concatenate([p for p in parts if len(p)] or [np.zeros((0, 6), np.int64)])
    if len(rows):
        off = np.array(ctx_offsets(n_sigs, k), np.int64)
        length = np.searchsorted(off[1:], rows[:, 1], side="right")
        local = rows[:, 1] - off[length]
        p = rows[:, 5].view(np.float64)
        rows = rows[np.lexsort((local, rows[:, 0], -length, -p))]
    return MinedTable(np.ascontiguousarray(rows), n_sigs, k)


def merge_shard_histograms(hist, counters, group) -> None:
    """K3: sum the per-shard (k+1)-gram histograms (and the ingest counters)
    across ranks.  Windows and matches never cross a session, so with shards
    made of whole sessions the summed histogram is exactly the one of the
    whole corpus; over NCCL this is one in-place all-reduce on the device."""
    import torch.distributed as dist

    dist.all_reduce(hist, group=group)
    dist.all_reduce(counters, group=group)


@dataclass
class OrderedTrace:
    columns: dict          # device columnar mining trace (tool events, session = segment)
    n_segments: int
    reordered_sessions: int
    order: Any = None      # optional: arrival index of every event in sorted order
    tokens: Any = None     # optional: flagged token stream of the output


_ORDER_DTYPES = {"session": "int32", "seq": "int32", "t_start": "float64", "t_end": "float64",
                 "sig": "int32"}


def order_columnar(raw: dict, n_sessions: int, inactivity_ms: float = 300_000.0,
                   with_order: bool = False, with_tokens: bool = False) -> OrderedTrace:
    """K1 general path (paste_ingest_order): ingest_trace's grouping by
    session id, stable (t_start, seq) sort, reorder tally and inactivity
    split (events.py:196-252) over a device-resident columnar trace in
    arrival order.  ``raw['sig']`` is -1 for LLM steps (they take part in
    the sort and the gap split, and are dropped from the output like
    Session.tool_events drops them); session ids are first-appearance
    indices in [0, n_sessions).  One host sync (the result counts)."""
    from .device_ops import stream_handle
    from ._native import OrderDesc

    torch = _torch()
    lib = _native.lib()
    for k, dt in _ORDER_DTYPES.items():
        if str(raw[k].dtype) != "torch." + dt or not raw[k].is_cuda:
            raise ValueError(f"column {k!r} must be a CUDA {dt} tensor")
    n = int(raw["sig"].numel())
    dev = raw["sig"].device
    out = {k: torch.empty(n, dtype=getattr(torch, dt), device=dev)
           for k, dt in _ORDER_DTYPES.items()}
    res = torch.zeros(4, dtype=torch.int64, device=dev)
    order = torch.empty(n, dtype=torch.int32, device=dev) if with_order else None
    tok = torch.empty(n, dtype=torch.int32, device=dev) if with_tokens else None
    need = int(lib.paste_ingest_order_scratch_bytes(n, int(n_sessions)))
    scratch = torch.empty(max(need, 16), dtype=torch.uint8, device=dev)
    base = ptr(res)
    cols = [raw[k].contiguous() for k in _ORDER_DTYPES]  # alive until the sync below
    d = OrderDesc(n, int(n_sessions), 0, *[ptr(c) for c in cols],
                  float(inactivity_ms), *[ptr(out[k]) for k in _ORDER_DTYPES], ptr(order),
                  ptr(tok), base, base + 8, base + 16, base + 24)
    check(lib.paste_ingest_order(ctypes.byref(d), ptr(scratch), need, stream_handle()), lib)
    n_out, n_seg, reord, status = (int(x) for x in res.tolist())
    if status & _native.PASTE_ORDER_BAD_SESSION:
        raise ValueError(f"session ids outside [0, {n_sessions})")
    if status & _native.PASTE_ORDER_NAN_T:
        raise _native.PasteUnsupported("NaN t_start: Python's sort order for it is undefined "
                                       "(use the host ingest_trace)")
    return OrderedTrace({k: v[:n_out] for k, v in out.items()}, n_seg, reord, order,
                        tok[:n_out] if with_tokens else None)


def mine_columnar(trace: dict, sigs: SigTable, cfg: MiningConfig,
                  inactivity_ms: float = 300_000.0, group=None,
                  tail: str = "allreduce") -> list[PatternTuple]:
    """mine() over a columnar trace shard on this device.  With a
    torch.distributed ``group`` every rank counts its shard (whole sessions)
    and the (k+1)-gram histograms are summed with one NCCL all-reduce before
    expansion -- windows and matches never cross a session, so the merged
    histogram equals the single-device one.  ``tail="sliced"`` runs the
    target-sliced tail instead (sharded_tail: reduce-scatter + per-block
    expansion and selection)."""
    relation = 0 if cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1
    tables = MineTables.allocate(max(sigs.n_sigs, 2), cfg.k, relation)
    counters = ingest_count(tables, trace, inactivity_ms)
    if int(counters[1].item()):
        # not grouped by session / sorted by (t_start, seq): the K1 general
        # path orders it on the device (ingest_trace's stable sort and gap
        # split), then the count runs again over the ordered segments
        n_sessions = int(trace["session"].max().item()) + 1
        ordered = order_columnar(trace, n_sessions, inactivity_ms)
        tables.hist.zero_()
        counters = ingest_count(tables, ordered.columns, float("inf"))
    if group is not None and tail == "sliced":  # target-sliced tail (sharded_tail)
        import torch.distributed as dist

        dist.all_reduce(counters, group=group)
        return sharded_tail(tables, group, cfg.sigma, cfg.tau).patterns(sigs)
    if group is not None:
        merge_shard_histograms(tables.hist, counters, group)
    tables.expand()
    return tables.select_sorted(cfg.sigma, cfg.tau).patterns(sigs)
