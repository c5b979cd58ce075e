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


def mine_jsonl(source: str | bytes, cfg: Any = None,
               inactivity_ms: float = DEFAULT_INACTIVITY_THRESHOLD_MS, group=None):
    """mine(ingest_trace(source).sessions, cfg) through the columnar path:
    native ingest, then the device count / expand / select."""
    import torch

    from .mine_engine import mine_columnar
    from .mining import MiningConfig

    tr = ingest_columnar(source, inactivity_ms)
    if tr.n_events == 0:
        raise ValueError("traces must be non-empty")
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in tr.columns.items()}
    # segments are already split: the count pass only follows the segment ids
    return mine_columnar(dev, tr.sigs, cfg or MiningConfig(), inactivity_ms=float("inf"),
                         group=group)
