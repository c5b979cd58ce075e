"""Columnar ingest of JSONL traces for mining at scale.

``ingest_columnar(text)`` turns a JSONL trace (the reference's trace format,
events.py:165-184) into the columnar trace the device count pass consumes:
tool events of every inactivity segment, in ``ingest_trace`` order
(events.py:196-252), with the session column holding the segment index.  The
native parser (csrc/ingest.cpp, OpenMP over lines) handles the common exact
subset; other input (escaped ids, coerced types, NaN start times, ...) is
ingested by the host ``ingest_trace`` with the reference semantics, so the
result is the same either way.  ``mine_jsonl`` mines it on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Any

import numpy as np

from . import _native
from ._native import IngestDesc, PASTE_ERR_UNSUPPORTED, check
from .events import DEFAULT_INACTIVITY_THRESHOLD_MS, IngestError, Status, ingest_trace
from .packing import SigTable


@dataclass
class ColumnarTrace:
    columns: dict[str, np.ndarray]   # session (segment index), seq, t_start, t_end, sig
    sigs: SigTable                   # tools in sorted name order
    n_segments: int
    reordered_sessions: int
    errors: list[IngestError] = field(default_factory=list)
    native: bool = True              # False: the host ingest decided

    @property
    def n_events(self) -> int:
        return len(self.columns["sig"])


def _host(text: str, inactivity_ms: float) -> ColumnarTrace:
    res = ingest_trace(text, inactivity_ms)
    streams = [s.tool_events() for s in res.sessions]
    sigs = SigTable(sorted({e.tool_type for st in streams for e in st}))
    n = sum(len(st) for st in streams)
    cols = {"session": np.empty(n, np.int32), "seq": np.empty(n, np.int32),
            "t_start": np.empty(n, np.float64), "t_end": np.empty(n, np.float64),
            "sig": np.empty(n, np.int32)}
    at = 0
    for seg, st in enumerate(streams):
        for e in st:
            cols["session"][at] = seg
            cols["seq"][at] = e.seq
            cols["t_start"][at] = e.t_start
            cols["t_end"][at] = e.t_end
            cols["sig"][at] = sigs.sig(e.tool_type, e.status)
            at += 1
    return ColumnarTrace(cols, sigs, len(res.sessions), res.reordered_sessions, res.errors,
                         native=False)


_REQUIRED_FIELDS = ("session_id", "seq", "kind", "tool", "status", "t_start_ms", "t_end_ms")


def _error_message(code: int, seq: int) -> str:
    """The reference's IngestError text for a native error code
    (events.py:59-63 Event.__post_init__, :142-145 _parse_record)."""
    if code & _native.PASTE_INGEST_MISSING:
        missing = [f for i, f in enumerate(_REQUIRED_FIELDS) if code >> i & 1]
        return f"missing fields: {', '.join(missing)}"
    if code & _native.PASTE_INGEST_T_ORDER:
        return f"event seq={seq}: t_start > t_end"
    return f"event seq={seq}: tool_call with empty tool_type"


def ingest_columnar(source: str | bytes,
                    inactivity_ms: float = DEFAULT_INACTIVITY_THRESHOLD_MS) -> ColumnarTrace:
    text = source.decode("utf-8") if isinstance(source, bytes) else source  # UTF-8 as the reference
    raw = text.encode("utf-8", "surrogatepass")
    lib = _native.load_library()
    cap = max(raw.count(b"\n") + 1, 1)
    cols = {"session": np.empty(cap, np.int32), "seq": np.empty(cap, np.int32),
            "t_start": np.empty(cap, np.float64), "t_end": np.empty(cap, np.float64),
            "sig": np.empty(cap, np.int32)}
    err = np.empty(cap, np.int32)
    code = np.empty(cap, np.int32)
    eseq = np.empty(cap, np.int64)
    names = ctypes.create_string_buffer(len(raw) + 1)
    d = IngestDesc(cap, *[c.ctypes.data for c in cols.values()], err.ctypes.data, cap,
                   ctypes.addressof(names), len(raw) + 1)
    d.error_codes, d.error_seq = code.ctypes.data, eseq.ctypes.data
    rc = lib.paste_ingest_jsonl(raw, len(raw), float(inactivity_ms), ctypes.byref(d))
    if rc == PASTE_ERR_UNSUPPORTED:
        return _host(text, inactivity_ms)
    check(rc, lib)
    tools = names.raw[:d.tool_names_len].split(b"\0")[:d.n_tools]
    sigs = SigTable([t.decode("utf-8", "surrogatepass") for t in tools])
    n = d.n_events
    errors = [IngestError(int(line), _error_message(int(c), int(q)))
              for line, c, q in zip(err[:d.n_errors], code[:d.n_errors], eseq[:d.n_errors])]
    return ColumnarTrace({k: v[:n] for k, v in cols.items()}, sigs, d.n_segments,
                         d.reordered_sessions, errors)


@dataclass
class RawTrace:
    """paste_jsonl_parse output: valid records in FILE order (the input of the
    device K1 path) and, optionally, their payload tapes."""
    columns: dict[str, np.ndarray]   # session (first-appearance id), seq, t_start, t_end, sig
    n_sessions: int
    sigs: SigTable
    errors: list[IngestError]
    tapes: tuple | None = None       # (nodes, data, refs): tape 2r = result, 2r + 1 = args
    keys: Any = None                 # KeyTable of the tapes


_as_utf8 = ctypes.pythonapi.PyUnicode_AsUTF8AndSize
_as_utf8.restype = ctypes.c_void_p
_as_utf8.argtypes = [ctypes.py_object, ctypes.POINTER(ctypes.c_ssize_t)]


def _utf8_view(text: str):
    """The UTF-8 bytes of `text` without a copy when CPython can lend them (an
    ASCII str's own buffer; otherwise its cached UTF-8 form), else encoded."""
    n = ctypes.c_ssize_t()
    try:
        p = _as_utf8(text, ctypes.byref(n))
    except UnicodeEncodeError:  # lone surrogates: the reference's text never has them
        p = None
    if not p:
        raw = text.encode("utf-8", "surrogatepass")
        return raw, len(raw)
    return ctypes.cast(p, ctypes.c_char_p), n.value


def parse_jsonl_raw(source: str | bytes, payloads: bool = True) -> RawTrace | None:
    """Native parallel parse (paste_jsonl_parse) of a JSONL trace; None when
    the input is outside the parser's exact subset (use the host ingest)."""
    from ._native import JsonlOut, JsonlSizes
    from .tape import NODE_DTYPE, KeyTable

    text = source.decode("utf-8") if isinstance(source, bytes) else source
    raw, n_raw = _utf8_view(text)
    lib = _native.load_library()
    h = ctypes.c_void_p()
    rc = lib.paste_jsonl_parse(raw, n_raw, 1 if payloads else 0, ctypes.byref(h))
    if rc == PASTE_ERR_UNSUPPORTED:
        return None
    check(rc, lib)
    try:
        z = JsonlSizes()
        check(lib.paste_jsonl_sizes_of(h, ctypes.byref(z)), lib)
        n = z.n_rows
        cols = {"session": np.empty(n, np.int32), "seq": np.empty(n, np.int32),
                "t_start": np.empty(n, np.float64), "t_end": np.empty(n, np.float64),
                "sig": np.empty(n, np.int32)}
        err = [np.empty(z.n_errors, np.int32), np.empty(z.n_errors, np.int32),
               np.empty(z.n_errors, np.int64)]
        tools = ctypes.create_string_buffer(max(z.tool_names_len, 1))
        nodes = np.empty(z.n_nodes, NODE_DTYPE)
        data = np.empty(max(z.n_bytes, 1), np.uint8)
        refs = np.empty((2 * n if payloads else 0, 2), np.int64)
        knames = ctypes.create_string_buffer(max(z.key_names_len, 1))
        o = JsonlOut(*[c.ctypes.data for c in cols.values()], *[e.ctypes.data for e in err],
                     ctypes.addressof(tools), nodes.ctypes.data, data.ctypes.data,
                     refs.ctypes.data, ctypes.addressof(knames))
        check(lib.paste_jsonl_copy(h, ctypes.byref(o)), lib)
    finally:
        lib.paste_jsonl_destroy(h)
    names = tools.raw[:z.tool_names_len].split(b"\0")[:z.n_tools]
    sigs = SigTable([t.decode("utf-8", "surrogatepass") for t in names])
    errors = [IngestError(int(line), _error_message(int(c), int(q))) for line, c, q in zip(*err)]
    tr = RawTrace(cols, int(z.n_sessions), sigs, errors)
    if payloads:
        keys = KeyTable()
        for k in knames.raw[:z.key_names_len].split(b"\0")[:z.n_keys]:
            keys.intern(k.decode("utf-8", "surrogatepass"))
        tr.tapes, tr.keys = (nodes, data, refs), keys
    return tr


def mine_jsonl(source: str | bytes, cfg: Any = None,
               inactivity_ms: float = DEFAULT_INACTIVITY_THRESHOLD_MS, group=None):
    """mine(ingest_trace(source).sessions, cfg) with the trace never
    materialised as Python sessions: native parallel parse of the records
    and their payload tapes (paste_jsonl_parse), then on the device the K1
    grouping / stable sort / gap split (paste_ingest_order), the count,
    selection and Phase II over the corpus tapes (mappings included).
    Input outside the native parser's exact subset goes through the host
    ingest_trace and the device mine() of its sessions: same result."""
    import torch

    from . import phase2_corpus as pc
    from .mine_engine import MineTables, _select_patterns, mine, order_columnar
    from .mining import MatchRelation, MiningConfig

    cfg = cfg or MiningConfig()
    tr = parse_jsonl_raw(source, payloads=group is None)
    if tr is None or group is not None:
        text = source.decode("utf-8") if isinstance(source, bytes) else source
        if group is not None:  # sharded: every rank mines its sessions, merged on device
            res = ingest_trace(text, inactivity_ms)
            return mine(res.sessions, cfg, group)
        return mine(ingest_trace(text, inactivity_ms).sessions, cfg)
    sig_raw = tr.columns["sig"]
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in tr.columns.items()}
    ordered = order_columnar(dev, tr.n_sessions, inactivity_ms, with_order=True,
                             with_tokens=True)
    if ordered.n_segments == 0:
        raise ValueError("traces must be non-empty")
    rel = 0 if cfg.match_relation is MatchRelation.ANCHORED_SUBSEQUENCE else 1
    tables = MineTables.allocate(max(tr.sigs.n_sigs, 2), cfg.k, rel)
    tok_dev = ordered.tokens
    if tok_dev.numel():
        tables.count(tok_dev)
    tables.expand()
    order = ordered.order.cpu().numpy()
    rows = order[sig_raw[order] >= 0]          # arrival row of every tool event, stream order
    tok_host = tok_dev.cpu().numpy()
    cols = {k: tr.columns[k][rows] for k in ("seq", "t_start", "t_end")}
    res_tape, args_tape = 2 * rows.astype(np.int64), 2 * rows.astype(np.int64) + 1
    events = pc.TapeEvents(tr.tapes, tr.keys, tr.sigs, tok_host, res_tape, args_tape, cols)

    def corpus():
        nodes, data, refs = tr.tapes
        return pc.CorpusTapes(nodes, data, refs, tr.keys, tok_host, tok_dev if tok_dev.numel()
                              else None, tr.sigs, events, res_tape, args_tape)

    return _select_patterns(tables, tr.sigs, tok_dev if tok_dev.numel() else None, events, cfg,
                            corpus=corpus)
